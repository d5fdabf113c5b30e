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
# graph-level profiling keeps the 3-iteration solve to one result; the last 15
# launches are the eager profiled iteration (tools/ncu_classes.py full)
timeout 1500 ncu -f --set full --import-source on --clock-control none --graph-profiling graph \
  --launch-skip 31 --launch-count 15 -o /tmp/iter python tools/ncu_iter.py c2 1 \
  > gpurun_out/prof/ncu_full.log 2>&1; echo full=$?
ncu -i /tmp/iter.ncu-rep --page raw --csv | gzip > gpurun_out/prof/iter_raw.csv.gz
python tools/ncu_sass.py /tmp/iter.ncu-rep k_gs_backward_blk 30 > gpurun_out/prof/sass_bwd.txt 2>&1
gzip -f gpurun_out/prof/launches.csv
