timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/ncu_iter.py c2 5 | grep -E "resid|coarse|prolong|total"
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 | python -c "
import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'])"
