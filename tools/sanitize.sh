#!/bin/bash
# compute-sanitizer passes over the kernel parity tests (one GPU):
#   racecheck  -- shared-memory hazards (colour-phase neighbour lists, DSMEM
#                 cluster partials, k-split sums, mbarrier stages)
#   synccheck  -- barrier / cluster-sync misuse
#   memcheck   -- out-of-bounds / misaligned device accesses
# Summaries under gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
T="tests/test_gpu_parity.py tests/test_gpu_config_shapes.py"
K="precond_apply or gs_sweep or spmv or c4_shape_preconditioner or pcg_3d or tma or two_instance or single_instance"
for tool in racecheck synccheck memcheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest $T -m gpu -q -x -k "$K" -p no:cacheprovider \
    > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize/$tool.log | tail -3
done
