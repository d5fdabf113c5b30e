timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/ncu_iter.py c2 5 | grep -E "backward|total"
timeout 600 python tools/ncu_iter.py c4 3 | grep -E "backward|total"
