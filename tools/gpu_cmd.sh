echo "== b1h bwd"; timeout 600 python tools/profile_b1.py 3,128 | grep -E "dim|gs_"
echo "== b1 bwd"; P2G_NO_B1H_BWD=1 timeout 600 python tools/profile_b1.py 3,128 | grep -E "dim|gs_"
timeout 900 python -m pytest tests -m gpu -x -q -k "single_instance or hex8 or partition or 3d" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
