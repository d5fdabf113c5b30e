timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu.log | head -5
timeout 300 python tools/probe_setup.py c2
P2G_AC_CUDACORE=1 timeout 300 python tools/probe_setup.py c2 | tail -1
