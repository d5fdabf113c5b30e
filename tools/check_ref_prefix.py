"""Check the bounded CPU reference sample of the large configs against full
reference solves of the same instances: python tools/check_ref_prefix.py c4"""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402

cfg = PR.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
import os  # noqa: E402
cores = os.cpu_count()
prob = PR.build_problem(cfg, device=0)
seeds = PR.query_seeds(cfg, cores)
values = prob.values(seeds)
F = np.ascontiguousarray(np.broadcast_to(prob.f, (cores, prob.mesh.n)))
est, su, ti = bench.cpu_reference_prefix(prob, values, F, cores, cores, bench.REF_ITERS[cfg.name])
t = time.perf_counter()
dt, it = bench.cpu_reference_run(prob, values, F, cores, cores)
print(f"{cfg.name}: {cores} instances on {cores} cores; prefix estimate {est:.1f} s (setup {su:.1f} s, "
      f"{ti:.3f} s/iteration, {bench.REF_ITERS[cfg.name]} iterations); full solves {dt:.1f} s "
      f"(iterations mean {np.mean(it):.1f} max {np.max(it)}); ratio {dt / est:.3f}")
