#!/bin/bash
# Bench every BASELINE.json config once on one GPU (documentation numbers);
# lines under gpurun_out/configs/.
mkdir -p gpurun_out/configs
for c in ${CONFIGS:-c1 c2 c4 c3 c5}; do
  timeout 2400 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 > gpurun_out/configs/bench_$c.json 2> gpurun_out/configs/bench_$c.err
  echo "$c rc=$?"
done
