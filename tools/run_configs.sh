#!/bin/bash
# Bench every BASELINE.json config once on one GPU (documentation numbers);
# logs under gpurun_out/configs/.
mkdir -p gpurun_out/configs
for c in ${CONFIGS:-c1 c2 c4 c3}; do
  timeout 1500 python bench.py --config $c --steps ${STEPS:-2} --warmup 3 > gpurun_out/configs/bench_$c.json 2> gpurun_out/configs/bench_$c.err
  echo "$c rc=$?"
done
if [ -z "$NO_C5" ]; then
  timeout 2400 python tools/run_c5.py > gpurun_out/configs/c5.log 2>&1
  echo "c5 rc=$?"
fi
