mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 1500 ncu -f --set full --import-source on --clock-control none --graph-profiling graph --launch-skip 31 --launch-count 15 -o /tmp/iter python tools/ncu_iter.py c2 1 > gpurun_out/prof/ncu_full.log 2>&1; echo full=$?; tail -2 gpurun_out/prof/ncu_full.log
ls -la /tmp/iter.ncu-rep
ncu -i /tmp/iter.ncu-rep --page raw --csv | gzip > gpurun_out/prof/iter_raw.csv.gz
python tools/ncu_sass.py /tmp/iter.ncu-rep k_gs_backward_blk 30 > gpurun_out/prof/sass_bwd.txt 2>&1
S=$(stat -c %s /tmp/iter.ncu-rep); if [ $S -lt 40000000 ]; then cp /tmp/iter.ncu-rep gpurun_out/prof/; fi
