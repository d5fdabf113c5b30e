#!/bin/bash
# Round profile pass (c2): bench line, ncu launch list of the bench command
# (eager loop so every solve kernel is visible), one --set full capture of a
# PCG iteration.  Outputs under gpurun_out/prof/; summarised into profiles/ by
# tools/ncu_classes.py.
mkdir -p gpurun_out/prof
timeout 900 python bench.py > gpurun_out/prof/bench_c2.json 2> gpurun_out/prof/bench.err; echo bench=$?
P2G_EAGER_LOOP=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/prof/ncu_launch.log 2>&1; echo launches=$?
NO_SOLVE=1 timeout 1500 ncu --set full --import-source on --clock-control none -o gpurun_out/prof/iter \
  python tools/ncu_iter.py c2 2 > gpurun_out/prof/ncu_full.log 2>&1; echo full=$?
gzip -f gpurun_out/prof/launches.csv
