#!/usr/bin/env python
"""bench.py -- PCG+POD-2G converged solves/s (fp64) on B200.

Workload (BASELINE.json configs[1], "c2"): 2D Q4 plane-stress cantilever on a
256x128 grid (66,048 dofs, 1.18M nonzeros), lognormal KL modulus, POD basis
k=20 from 50 GPU-solved snapshots, a batch of 64 seeded instances sharing the
CSR pattern, each solved by PCG + POD-2G to relative residual 1e-8 from
x0 = Phi A_c^{-1} Phi^T b.  One STEP = one batch: value upload/relayout,
per-instance setup (A_c = Phi^T K Phi + LDL^T), x0, and the PCG loop.  The
basis is the offline stage's product, uploaded once and shared by every batch
(the reference shares it by shared_ptr across instances, pod.hpp:261-263).

  python bench.py [--gpus N --steps K --warmup W --config cN --impl ours|reference]

N > 1: one process per GPU.  Under torchrun (WORLD_SIZE set) WORLD_SIZE must
equal --gpus; without it bench.py launches torchrun itself (127.0.0.1).  The
default config is c2 at N = 1 (BASELINE.json configs[1], a 1-GPU config) and
c4 at N > 1 (configs[3], the sharded hex8 batch): BASELINE's instance total
(64 for c4, 256 for c3) is split across the ranks (strong scaling), no
data-path collective; max-over-ranks time.
--impl reference: the unmodified reference (oracle/_ref, compiled from
/root/reference by oracle/Makefile) on the host cores, rank 0 only; its
inputs come from the CPU-only generator library (libpod2g_gen.so), so that
arm never loads the CUDA library.
--dry-run: no GPU work; ranks (gloo) agree on the sharding and rank 0 prints
the line's n_gpus / config (the CPU test of the multi-GPU plumbing).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG+POD-2G converged solves/sec (fp64)"
UNIT = "solves/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="c1..c5 (default: c2 at --gpus 1, c4 at --gpus > 1)")
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--c5-snapshots", type=int, default=48,
                    help="c5 offline stage: snapshot solves behind the k = 40 basis")
    ap.add_argument("--c5-cpu-iters", type=int, default=2,
                    help="c5 CPU baseline: reference PCG iterations timed (1 core)")
    ap.add_argument("--instances", type=int, default=0,
                    help="solve only the first N instances of this rank's shard (what a rank of a "
                         "larger job holds; threshold calibration, not a BASELINE workload)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-instances", type=int, default=0,
                    help="instances in the CPU sample (default: one per host core, <= batch)")
    a = ap.parse_args()
    if a.gpus < 1:
        ap.error("--gpus must be >= 1")
    if a.config is None:
        a.config = "c2" if a.gpus == 1 else "c4"
    return a


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args):
    """--gpus N outside torchrun: launch N ranks with torchrun on this node
    (rendezvous on 127.0.0.1); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[5:9]):
                if "Active" in v and "Not" not in v:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# FP64 tensor-core (DMMA m8n8k4) peak measured on this pool's B200s with
# tools/dmma_lab.cu (profiles/r02_dmma_peak.txt): 128 flop / clk / SM.
FP64_TENSOR_TFLOPS = 37.0


def class_table(prof, peak, n, k, B):
    """Per kernel class: event-bracketed ms, algorithmic bytes and the HBM
    fraction; the two projections (DMMA kernels) also carry their tensor-core
    work (k padded to the m-block / k-step the kernels run) against the measured
    FP64 tensor peak -- the restriction at k = 30 is tensor-bound (7 flop/B
    against a machine balance of 5.7)."""
    out = {}
    for name, (ms, by) in prof.items():
        e = {"ms": ms, "bytes": by}
        if ms > 0 and by > 0:
            e["hbm_frac"] = by / (ms * 1e-3) / 1e9 / peak
        if ms > 0 and B > 1 and name in ("restrict", "prolong"):
            kp = (k + 7) // 8 * 8 if name == "restrict" else (k + 3) // 4 * 4
            fl = 2.0 * n * kp * ((B + 31) // 32 * 32)
            e["tensor_tflops"] = fl / (ms * 1e-3) / 1e12
            e["tensor_frac"] = e["tensor_tflops"] / FP64_TENSOR_TFLOPS
        out[name] = e
    return out


def ncu_traffic(config, kclass):
    """dram bytes per iteration of kernel class `kclass` on `config`, from the
    committed ncu --set full capture of THAT config (profiles/ncu_traffic.json,
    written by tools/ncu_classes.py), or None when that config has none."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d[config]["per_iteration_dram_bytes"].get(kclass)
    except Exception:
        return None


def cpu_reference_run(prob, values, F, instances, jobs):
    """The unmodified reference (oracle/_ref): fresh Pod2gPreconditioner +
    reduced_solve x0 + pcg_solve per instance, parallel_for over `jobs`
    threads (bench.hpp:290-330).  Returns (seconds, iters)."""
    from oracle.bindings import Reference
    R = Reference()
    t = time.perf_counter()
    u, it, conv, failed = R.pcg_pod2g_batch(prob.rp.astype(np.int64), prob.ci.astype(np.int64),
                                            values[:instances], F[:instances], prob.phi, 1,
                                            prob.cfg.tol, 100000, jobs)
    dt = time.perf_counter() - t
    if np.any(failed) or not np.all(conv):
        raise RuntimeError("reference CPU arm: an instance failed")
    return dt, it


# Large configs: one reference solve takes minutes per core (c3 ~160 s, c4 ~100 s), so
# a step times a bounded PREFIX of every solve instead -- per instance the setup
# (reduced_solve x0 + Pod2gPreconditioner: A_c, LU; max_iter = 0) and the first
# REF_PREFIX PCG iterations, all instances in parallel -- and extrapolates with
# the reference's own natural-order mean iteration count on that config, measured
# with full solves on the GPU box in round 1 (profiles/r01_configs/bench_cN.json).
REF_PREFIX = 10
REF_ITERS = {"c3": 668.8, "c4": 139.3}


def cpu_reference_prefix(prob, values, F, instances, jobs, nref):
    """(extrapolated seconds for `instances` full solves in parallel, setup s, s/iteration):
    per instance, its measured setup (x0 + A_c + LU) plus nref x its measured seconds per
    PCG iteration over the first REF_PREFIX iterations; the batch takes the slowest."""
    from oracle.bindings import Reference
    R = Reference()
    it, su, lo = R.pcg_pod2g_batch_timed(prob.rp.astype(np.int64), prob.ci.astype(np.int64),
                                         values[:instances], F[:instances], prob.phi,
                                         prob.cfg.tol, REF_PREFIX, jobs)
    t_it = lo / np.maximum(it, 1)
    est = float(np.max(su + nref * t_it))
    return est, float(np.mean(su)), float(np.mean(t_it))


def pin_limit():
    """largest value batch to pin (the pinned copy doubles its host footprint)"""
    try:
        import psutil
        return int(min(64 << 30, 0.35 * psutil.virtual_memory().available))
    except Exception:
        return 16 << 30


def workload_name(cfg):
    """the config's workload label, shared by both arms"""
    if cfg.dim == 2:
        return f"{cfg.name}: Q4 plane-stress {cfg.nx}x{cfg.ny} cantilever"
    return f"{cfg.name}: hex8 {cfg.nx}^3 elasticity"


def dry_run(args, cfg, PR, ws, rank):
    """The multi-GPU plumbing without a GPU: gloo ranks, sharding, gathers."""
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
    from paper_2207_02543_b200 import dist as D
    B, seeds, strong = PR.shard(cfg, ws, rank)
    counts = D.gather_counts(np.array([B]))
    first = D.gather_counts(np.array([int(seeds[0]) if B else -1]))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": ws,
                          "dry_run": True, "scaling": "strong" if strong else "weak",
                          "config": {"workload": workload_name(cfg),
                                     "instances_total": int(counts.sum()),
                                     "instances_per_rank": counts.tolist(),
                                     "first_seed_per_rank": first.tolist(),
                                     "parallelism": f"instance-sharded x{ws}"}}), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return spawn_ranks(args)
    ws, rank, local = dist_env()
    if "WORLD_SIZE" in os.environ and ws != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}")
    if args.impl == "reference" and rank != 0:
        return 0  # the reference arm runs on rank 0 alone

    from paper_2207_02543_b200 import problems as PR
    cfg = PR.CONFIGS[args.config]
    cores = os.cpu_count() or 1

    if args.impl == "reference":
        return reference_arm(args, cfg, PR, cores, args.gpus)
    if args.dry_run:
        return dry_run(args, cfg, PR, ws, rank)
    if cfg.name == "c5":
        return c5_arm(args, cfg, ws, rank, local)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    from paper_2207_02543_b200 import _lib as L
    from paper_2207_02543_b200 import dist as D
    from paper_2207_02543_b200.solver import BatchSolver

    # ---- inputs (outside the timed region): basis, this rank's instances
    t0 = time.perf_counter()
    prob = PR.build_problem(cfg, device=local)
    B, seeds, strong = PR.shard(cfg, ws, rank)
    if args.instances and args.instances < B:
        B, seeds = args.instances, seeds[:args.instances]
    values = prob.values(seeds)                 # [B][nnz] natural order (host)
    n, nnz = prob.mesh.n, prob.mesh.nnz
    F = np.ascontiguousarray(np.broadcast_to(prob.f, (B, n)))
    gen_s = time.perf_counter() - t0

    dev = torch.device("cuda", local)
    vals_d = torch.from_numpy(values).to(dev)
    b_d = torch.from_numpy(F).to(dev)
    x_d = torch.empty_like(b_d)
    s = BatchSolver(local)
    s.set_pattern(prob.rp, prob.ci, prob.mesh.block_size, batch_hint=B)
    stream = torch.cuda.ExternalStream(s.stream(), device=dev)

    s.set_basis(prob.phi)  # the offline basis, shared by every batch (pod.hpp:261-263)

    def step_device():
        s.set_values_device(vals_d.data_ptr(), B)
        st = s.setup()
        it, conv, status, _ = s.solve_device(b_d.data_ptr(), x_d.data_ptr(), None, L.X0_REDUCED,
                                             cfg.tol, 100000)
        return st, it, conv, status

    def barrier():
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step_device()
    barrier()
    l0 = s.launch_counts()[1]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    iters_all = []
    ok = True
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            st, it, conv, status = step_device()
            ok &= bool(np.all(conv)) and bool(np.all(status == 0)) and bool(np.all(st == 0))
            iters_all.append(it.copy())
        ev1.record(stream)
        barrier()
    launches = s.launch_counts()[1] - l0
    ms = D.max_over_ranks(ev0.elapsed_time(ev1), dev)
    total_solves = int(D.gather_counts(np.array([B]), dev).sum()) * args.steps
    value = total_solves / (ms / 1e3)
    iters = np.concatenate(iters_all)

    # ---- roofline: per-kernel-class time of the loop body, same state
    prof = s.profile_iteration(5)
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_bytes) = dom
    peak, peak_src = hbm_peak()
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    iter_ms = sum(v[0] for v in prof.values())
    iter_bytes = sum(v[1] for v in prof.values())
    per_iter, _ = s.launch_counts()
    # the captured WHILE loop itself, every instance active (tol = 0, fixed
    # length): in the graph, consecutive kernels start without the ~4 us of
    # launch latency an event-bracketed kernel class pays per launch, so this
    # is the iteration time the solve really runs at
    LOOP_ITERS = 100
    s.solve_device(b_d.data_ptr(), x_d.data_ptr(), None, L.X0_REDUCED, 0.0, LOOP_ITERS)
    loop_iter_ms = s.last_solve_ms()[1] / LOOP_ITERS

    # ---- e2e through the C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        pin = values.nbytes < pin_limit()  # very large batches: pageable host memory
        vals_h = torch.from_numpy(values)
        b_h = torch.from_numpy(F)
        x_h = torch.empty_like(b_h)
        if pin:
            vals_h, b_h, x_h = vals_h.pin_memory(), b_h.pin_memory(), x_h.pin_memory()
        import ctypes as C
        lib = L.lib()
        Dp = L.D
        it_h = np.zeros(B, dtype=np.int64)
        cv_h = np.zeros(B, dtype=np.int32)
        st_h = np.zeros(B, dtype=np.int32)

        def step_e2e(prefetch_next=False):
            # consumes the copy started during the previous solve, if any
            rc = lib.p2g_set_values(s._h, B, C.cast(vals_h.data_ptr(), Dp))
            assert rc == 0, rc
            if prefetch_next:  # next batch's values cross the link while this one solves
                rc = lib.p2g_prefetch_values(s._h, B, C.cast(vals_h.data_ptr(), Dp))
                assert rc == 0, rc
            s.setup()
            rc = lib.p2g_solve(s._h, C.cast(b_h.data_ptr(), Dp), None, L.X0_REDUCED, cfg.tol,
                               100000, C.cast(x_h.data_ptr(), Dp), it_h.ctypes.data_as(L.I64),
                               cv_h.ctypes.data_as(L.I32), st_h.ctypes.data_as(L.I32), None, 0)
            assert rc == 0, rc
            return float(x_h[0, 0])  # device->host read of the result

        # steady state of the pipeline: the warm-up step starts the upload of the
        # first timed step's values, and EVERY timed step uploads one batch of
        # values (the next step's; 604 MB on c2, ~11 ms over the host link, done
        # long before its 125 ms solve ends), so K timed steps contain K uploads
        step_e2e(prefetch_next=pin)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            step_e2e(prefetch_next=pin)
        e1.record(stream)
        barrier()
        ems = D.max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": total_solves / (ems / 1e3), "unit": UNIT, "pinned": pin,
               "pipelined": bool(pin),
               "h2d_bytes_per_step": int(values.nbytes + F.nbytes),
               "d2h_bytes_per_step": int(F.nbytes + 3 * 4 * B)}

    # ---- CPU baseline: the reference itself on host cores, bounded sample
    cpu = None
    natural_iters = REF_ITERS.get(cfg.name)  # the reference's natural-order SGS count
    if rank == 0 and ws == 1 and not args.no_cpu:
        ninst = args.cpu_instances or min(B, cores)
        try:
            if cfg.name in REF_ITERS:
                est, t0s, t_it = cpu_reference_prefix(prob, values, F, ninst, cores,
                                                      REF_ITERS[cfg.name])
                cpu = {"value": ninst / est, "unit": UNIT, "cores": cores, "kind": "reference",
                       "extrapolated": True,
                       "sample": f"{ninst} of the {B} {cfg.name} instances in parallel, "
                                 f"natural-order SGS, x0=reduced_solve: setup {t0s:.2f} s + "
                                 f"first {REF_PREFIX} PCG iterations ({t_it:.3f} s each) timed, "
                                 f"extrapolated to the reference's {REF_ITERS[cfg.name]} mean "
                                 f"iterations (round-1 full solves on this box type)"}
            else:
                dt, cit = cpu_reference_run(prob, values, F, ninst, cores)
                natural_iters = float(np.mean(cit))
                cpu = {"value": ninst / dt, "unit": UNIT, "cores": cores, "kind": "reference",
                       "sample": f"{ninst} of the {B} {cfg.name} instances, natural-order SGS "
                                 f"(reference default), x0=reduced_solve, tol {cfg.tol:g}; "
                                 f"mean iterations {float(np.mean(cit)):.1f}; {dt:.2f} s wall"}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded KL lognormal modulus; generator in include/pod2g_gen.h)",
            "config": {"workload": workload_name(cfg),
                       "n_dofs": n, "nnz": nnz, "pod_rank": int(prob.phi.shape[1]),
                       "instances_per_gpu": B, "instances_total": total_solves // args.steps,
                       "tol": cfg.tol, "x0": "reduced_solve",
                       "smoother": "multicolour symmetric GS (%d node colour classes, D1)"
                                   % (len(s.permutation()[1]) - 1),
                       "l2": "inputs larger than L2 (values %.0f MB per GPU)" % (values.nbytes / 1e6),
                       "parallelism": f"instance-sharded x{ws}",
                       "iterations_mean": float(np.mean(iters)),
                       "iterations_natural_order_reference": natural_iters,
                       "iterations_max": int(np.max(iters)),
                       "all_converged": ok, "input_generation_s": round(gen_s, 2)},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                         "traffic": ncu_traffic(cfg.name, dom_name),
                         "algorithmic_bytes_per_iteration": iter_bytes,
                         "iteration_ms": iter_ms,
                         "iteration_frac": iter_bytes / (iter_ms * 1e-3) / 1e9 / peak,
                         "loop_iteration_ms": loop_iter_ms,
                         "loop_iteration_frac": iter_bytes / (loop_iter_ms * 1e-3) / 1e9 / peak,
                         "loop_note": f"captured WHILE loop, {LOOP_ITERS} iterations, all instances "
                                      "active (tol 0); iteration_ms is the sum of the event-bracketed "
                                      "class times",
                         "classes": class_table(prof, peak, n, int(prob.phi.shape[1]), B)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "launches_per_iteration": int(per_iter),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    s.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def c5_arm(args, cfg, ws, rank, local):
    """Config c5 (BASELINE.json configs[4]): ONE 12.4 M-dof hex8 system,
    row-partitioned over the N GPUs (p2g_part_*: N = 1 one partition; N > 1
    one partition per rank over NCCL, halo exchange + all-reduces).  A step =
    one solve of the query instance: A_c + LDL^T setup, x0 = reduced_solve,
    PCG to 1e-8.  value = solves/s (timed on the partition stream, max over
    ranks); e2e = the same through host buffers (the rank's values uploaded
    from pinned memory every step, b in, x out)."""
    import torch
    import torch.distributed as dist
    from paper_2207_02543_b200 import c5 as C5
    from paper_2207_02543_b200 import dist as D
    from paper_2207_02543_b200.partition import PartitionedSolver
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
        box = [PartitionedSolver.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, 0)
        uid = box[0]

    def log(*a):
        if rank == 0:
            print(*a, file=sys.stderr, flush=True)

    t0 = time.perf_counter()
    case = C5.prepare(cfg.name, ws, [rank] if ws > 1 else None, uid,
                      n_snapshots=args.c5_snapshots, snap_batch=8, log=log, device=local)
    case.query_values()
    gen_s = time.perf_counter() - t0
    P = case.P
    stream = torch.cuda.ExternalStream(P.stream(), device=dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    its = []
    for _ in range(args.warmup):
        xs, it, conv, status, _ = case.solve()
    barrier()
    l0 = P.launch_counts()[1]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ok = True
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            xs, it, conv, status, _ = case.solve()
            ok &= bool(np.all(conv)) and bool(np.all(status == 0))
            its.append(int(it[0]))
        ev1.record(stream)
        barrier()
    per_iter, l1, loop_mode = P.launch_counts()
    ms = D.max_over_ranks(ev0.elapsed_time(ev1), dev)
    value = args.steps / (ms / 1e3)

    prof = P.profile_iteration(3)
    peak, peak_src = hbm_peak()
    dom_name, (dom_ms, dom_bytes) = max(prof.items(), key=lambda kv: kv[1][0])
    iter_ms = sum(v[0] for v in prof.values())
    iter_bytes = sum(v[1] for v in prof.values())

    # e2e: this rank's values from pinned host memory every step (+ b in, x out)
    e2e = None
    if not args.no_e2e:
        r = case.hosted[0]
        hv = torch.from_numpy(case.host_values(r)).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            P.set_values(r, hv.numpy())  # the basis stays (same batch size)
            xs, it, conv, status, _ = case.solve()
            ok &= bool(np.all(conv)) and bool(np.all(status == 0))
        e1.record(stream)
        barrier()
        ems = D.max_over_ranks(e0.elapsed_time(e1), dev)
        n_own = len(case.bvec[r])
        e2e = {"value": args.steps / (ems / 1e3), "unit": UNIT, "pinned": True,
               "h2d_bytes_per_step": int(hv.numel() * 8 + n_own * 8),
               "d2h_bytes_per_step": int(n_own * 8 + 16),
               "note": "per rank; values re-uploaded every step, basis kept (shared_ptr)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            cpu = c5_cpu_baseline(case, max(its), args.c5_cpu_iters)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank == 0:
        n, nnz = case.mesh.n, case.mesh.nnz
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded KL lognormal modulus; generator in include/pod2g_gen.h)",
            "config": {"workload": workload_name(cfg), "n_dofs": n, "nnz": nnz,
                       "pod_rank": int(case.k), "instances": 1, "tol": cfg.tol,
                       "x0": "reduced_solve", "smoother": "multicolour symmetric GS (mesh "
                       "parity node colouring, D1)",
                       "l2": "inputs larger than L2 (values %.1f GB)" % (8.0 * nnz / 1e9),
                       "parallelism": f"row-partitioned x{ws}" + (" (NCCL)" if ws > 1 else ""),
                       "iterations": its[-1], "loop": {1: "conditional-WHILE graph",
                                                       2: "captured 8-iteration chunks",
                                                       0: "eager"}[loop_mode],
                       "offline": f"{case.n_snapshots} snapshot solves, POD k={case.k}, "
                                  f"{case.offline_s:.0f} s",
                       "all_converged": ok, "input_generation_s": round(gen_s, 1)},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved":
                         dom_bytes / (dom_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": dom_bytes / (dom_ms * 1e-3) / 1e9 / peak,
                         "peak_source": peak_src, "traffic": ncu_traffic(cfg.name, dom_name),
                         "algorithmic_bytes_per_iteration": iter_bytes,
                         "iteration_ms": iter_ms,
                         "iteration_frac": iter_bytes / (iter_ms * 1e-3) / 1e9 / peak,
                         "classes": class_table(prof, peak, 0, 0, 1),
                         "note": "rank 0's partition"},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(l1 - l0), "launches_per_iteration": int(per_iter),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    case.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def c5_cpu_baseline(case, iters_gpu, n_prefix):
    """The unmodified reference (oracle/_ref) on the c5 system, ONE core (the
    reference has no intra-solve parallelism): Pod2gPreconditioner
    construction (A_c = Phi^T K Phi, k SpMVs + k^2 dots, and DenseLu) plus the
    first `n_prefix` PCG iterations (krylov.hpp:243-297, SolveReport
    wall_time_s for the loop).  Extrapolated to a whole solve as 2 x setup
    (reduced_solve builds A_c again) + iters_gpu x seconds per iteration."""
    from oracle.bindings import Reference
    R = Reference()
    mesh = case.mesh
    rp, ci = mesh.pattern()
    v = mesh.assemble(case.E, 0)[0]
    phi = case.phi_own[0]
    f = mesh.rhs()
    t = time.perf_counter()
    res = R.pcg_pod2g(rp.view(np.int64), ci.view(np.int64), v, f, phi, np.zeros(mesh.n), 0.0,
                      n_prefix)
    call = time.perf_counter() - t
    if res.status != 0:
        raise RuntimeError(f"reference pcg_solve status {res.status}")
    t_iter = res.wall_s / max(res.iters, 1)
    setup = call - res.wall_s
    total = 2.0 * setup + iters_gpu * t_iter
    return {"value": 1.0 / total, "unit": UNIT, "cores": 1, "kind": "reference",
            "extrapolated": True,
            "sample": f"c5 query system, 1 core: Pod2gPreconditioner construction {setup:.1f} s "
                      f"(A_c + LU, incl. CSR copy-in) and the first {res.iters} PCG iterations "
                      f"({t_iter:.2f} s each, natural-order SGS); solve = 2 x setup + "
                      f"{iters_gpu} iterations = {total:.0f} s (extrapolated)"}


def reference_arm(args, cfg, PR, cores, ws):
    """--impl reference: the reference CPU path on this box's host cores."""
    mesh = PR.Mesh.for_config(cfg)
    rp, ci = mesh.pattern()
    f = mesh.rhs()
    prob = _basis_for_reference(cfg, PR, mesh, rp, ci, f, cores)
    ninst = args.cpu_instances or min(cfg.batch, cores)
    seeds = PR.query_seeds(cfg, ninst)
    values = mesh.assemble(mesh.kl_field(seeds, cfg.kl_terms)[0])
    F = np.ascontiguousarray(np.broadcast_to(f, (ninst, mesh.n)))
    times, prefix = [], cfg.name in REF_ITERS
    for i in range(args.warmup + args.steps):
        if prefix:  # bounded sample, extrapolated (see REF_ITERS)
            dt, t0s, t_it = cpu_reference_prefix(prob, values, F, ninst, cores, REF_ITERS[cfg.name])
        else:
            dt, it = cpu_reference_run(prob, values, F, ninst, cores)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = ninst * args.steps / tot
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": workload_name(cfg), "n_dofs": mesh.n, "nnz": mesh.nnz,
                   "pod_rank": int(prob.phi.shape[1]), "instances_per_step": ninst,
                   "tol": cfg.tol, "x0": "reduced_solve",
                   "smoother": "natural-order symmetric GS (reference default)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "extrapolated": prefix,
                         "sample": f"{ninst} {cfg.name} instances per step, one per host core "
                                   f"(parallel_for), natural-order SGS, x0=reduced_solve"
                                   + (f"; per step setup + first {REF_PREFIX} PCG iterations "
                                      f"timed, extrapolated to {REF_ITERS.get(cfg.name)} "
                                      f"iterations" if prefix else "")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _basis_for_reference(cfg, PR, mesh, rp, ci, f, jobs):
    """The reference arm's offline basis, made by the reference itself:
    Jacobi-PCG snapshots with generate_snapshots' tolerance ladder and
    compute_pod(RankTarget{k}) (oracle/_ref ref_offline_basis).  Only the
    input generator (mesh, KL field) is ours."""
    from oracle.bindings import Reference
    R = Reference()
    if cfg.name in REF_ITERS:
        # 10^6-dof systems: Jacobi-PCG snapshots would take ~hours on the host;
        # the reference's pcg_solve + Pod2gPreconditioner over the smooth
        # degree <= 3 displacement modes instead, 2 snapshots per core (>= k + 2)
        from paper_2207_02543_b200 import c5 as C5
        nsnap = max(cfg.k + 2, min(cfg.n_snapshots, 2 * jobs))
        S = C5.smooth_space(mesh, np.arange(mesh.n, dtype=np.int64))
        boot = np.ascontiguousarray(S @ np.linalg.inv(np.linalg.cholesky(S.T @ S).T))
        vals = mesh.assemble(mesh.kl_field(PR.snapshot_seeds(cfg, nsnap), cfg.kl_terms)[0])
        F = np.ascontiguousarray(np.broadcast_to(f, (len(vals), mesh.n)))
        phi = R.offline_basis_pod2g(rp.view(np.int64), ci.view(np.int64), vals, F, cfg.k, boot,
                                    PR.SNAP_TOL, jobs)
        return PR.Problem(cfg, mesh, rp, ci, f, phi, np.zeros(0), np.zeros(0))
    vals = mesh.assemble(mesh.kl_field(PR.snapshot_seeds(cfg), cfg.kl_terms)[0])
    F = np.ascontiguousarray(np.broadcast_to(f, (len(vals), mesh.n)))
    phi = R.offline_basis(rp.astype(np.int64), ci.astype(np.int64), vals, F, cfg.k,
                          PR.SNAP_TOL, jobs)
    return PR.Problem(cfg, mesh, rp, ci, f, phi, np.zeros(0), np.zeros(0))


if __name__ == "__main__":
    sys.exit(main())
