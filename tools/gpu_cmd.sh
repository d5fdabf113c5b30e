mkdir -p gpurun_out/configs
timeout 600 python bench.py > gpurun_out/configs/bench_c2.json 2> gpurun_out/configs/bench_c2.err; echo c2=$?
CONFIGS=c4 NO_C5=1 bash tools/run_configs.sh
python - <<'PY'
import json
for c in ['c2','c4']:
    d=json.load(open(f'gpurun_out/configs/bench_{c}.json')); print(c, d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['iteration_frac'], d['clocks'])
PY
