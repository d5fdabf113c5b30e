mkdir -p gpurun_out/configs
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/configs/bench_c2.json 2> gpurun_out/configs/bench_c2.err; echo c2=$?
CONFIGS=c3 NO_C5=1 bash tools/run_configs.sh
python - <<'PY'
import json
for c in ['c2','c3']:
    d=json.load(open(f'gpurun_out/configs/bench_{c}.json')); print(c, d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['iteration_frac'], d['clocks'])
PY
