mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log; grep -E "FAIL|Error|assert" gpurun_out/pytest_gpu.log | head -8
for e in 0 1; do
  if [ $e = 1 ]; then export P2G_NO_FUSED_SCALARS=1; fi
  timeout 600 python bench.py --no-cpu --steps 5 | python -c "
import json,sys; d=json.load(sys.stdin); print('nofuse' if $e else 'fused', d['value'], d['e2e']['value'], d['ms_per_step'], d['launches_per_iteration'], d['config']['iterations_max'])"
done
