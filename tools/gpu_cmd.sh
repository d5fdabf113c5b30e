mkdir -p gpurun_out/configs
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/configs/bench_c4.json 2> gpurun_out/configs/bench_c4.err; echo c4=$?
python -c "
import json; d=json.load(open('gpurun_out/configs/bench_c4.json')); print(d['value'], d['e2e'])"
