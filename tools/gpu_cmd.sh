timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
echo "== staged"; timeout 300 python tools/ncu_iter.py c2 5 | grep -E "gs_|spmv|resid|total"
echo "== blocked"; P2G_NO_STAGE=1 timeout 300 python tools/ncu_iter.py c2 5 | grep -E "gs_|spmv|resid|total"
