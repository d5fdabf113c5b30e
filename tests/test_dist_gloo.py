"""World-size-2 gloo test of the instance-sharded multi-GPU path's host logic
(bench.py under torchrun): disjoint shards, full coverage, max-over-ranks."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_02543_b200 import dist as D
    from paper_2207_02543_b200 import problems as PR
    out = {}
    for name in ("c4", "c3"):
        cfg = PR.CONFIGS[name]
        n, seeds, strong = PR.shard(cfg, world, rank)
        counts = D.gather_counts(np.array([n]))
        allseeds = D.gather_counts(seeds.astype(np.int64)) if not strong or len(set(counts)) == 1 else None
        out[name] = (counts.tolist(), None if allseeds is None else allseeds.tolist(), strong)
    out["max"] = D.max_over_ranks(10.0 + rank)
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_sharding_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2207_02543_b200 import problems as PR
    counts, seeds, strong = out["c4"]
    assert counts == [32, 32] and strong
    assert seeds == PR.query_seeds(PR.CONFIGS["c4"]).astype(np.int64).tolist()
    counts, seeds, strong = out["c3"]
    assert counts == [128, 128] and strong
    assert seeds == PR.query_seeds(PR.CONFIGS["c3"]).astype(np.int64).tolist()
    assert out["max"] == 11.0


def test_bench_gpus_two_dry_run_spawns_two_ranks():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself; the
    N > 1 default config is c4 with BASELINE's 64 instances split 32 + 32."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--dry-run"], capture_output=True, text=True, timeout=300, env=env,
                       cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("c4")
    assert d["config"]["instances_total"] == 64 and d["config"]["instances_per_rank"] == [32, 32]


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4",
                        "--dry-run"], capture_output=True, text=True, timeout=120, env=env,
                       cwd=root)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
