#!/bin/bash
# Round profile pass: for each config, one ncu --set full capture of ONE PCG
# iteration (eager, NVTX range "profile" of tools/ncu_iter.py; c5's shapes via
# the 128^3 single-instance cube of tools/ncu_b1.py), exported as raw CSV.
# Summarise here with: python tools/ncu_classes.py full <csv.gz> --traffic <cfg>
mkdir -p gpurun_out/prof
for cfg in ${CONFIGS:-c2 c4 c3}; do
  P2G_PROFILE_EAGER=1 timeout 1500 ncu -f --set full --import-source on --clock-control none \
    --cache-control all --nvtx --nvtx-include "profile/" -o /tmp/iter_$cfg \
    python tools/ncu_iter.py $cfg 1 > gpurun_out/prof/ncu_$cfg.log 2>&1; echo "$cfg ncu=$?"
  ncu -i /tmp/iter_$cfg.ncu-rep --page raw --csv | gzip > gpurun_out/prof/iter_${cfg}_raw.csv.gz
done
if [ -z "$NO_B1" ]; then
  P2G_PROFILE_EAGER=1 timeout 1500 ncu -f --set full --import-source on --clock-control none \
    --cache-control all --nvtx --nvtx-include "profile/" -o /tmp/iter_b1 \
    python tools/ncu_b1.py 160 40 1 > gpurun_out/prof/ncu_b1.log 2>&1; echo "b1 ncu=$?"
  ncu -i /tmp/iter_b1.ncu-rep --page raw --csv | gzip > gpurun_out/prof/iter_b1_raw.csv.gz

fi

# launch list of the default bench command (eager loop: every kernel visible)
[ -z "$NO_LAUNCHES" ] && P2G_EAGER_LOOP=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/prof/ncu_launch.log 2>&1; echo launches=$?
[ -z "$NO_LAUNCHES" ] && gzip -f gpurun_out/prof/launches_c2.csv
