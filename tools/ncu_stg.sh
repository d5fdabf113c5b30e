#!/bin/bash
# ncu --set full of the staged backward phases of one c2 iteration (eager
# profile, NVTX range "profile"): SASS stall summary + DRAM bytes per launch.
mkdir -p gpurun_out/stg
P2G_PROFILE_EAGER=1 timeout 900 ncu -f --set full --import-source on --clock-control none --cache-control all \
  --nvtx --nvtx-include "profile/" --kernel-name regex:k_gs_backward_stg -o /tmp/stg \
  python tools/ncu_iter.py c2 1 > gpurun_out/stg/ncu.log 2>&1; echo ncu=$?
python tools/ncu_sass.py /tmp/stg.ncu-rep k_gs_backward_stg 30 > gpurun_out/stg/sass_gs_backward_stg.txt 2>&1
ncu -i /tmp/stg.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__shared_mem_per_block_dynamic']
idx=[h.index(w) for w in want if w in h]
print([h[i] for i in idx]); print([rows[1][i] for i in idx])
for r in rows[2:]:
    print([r[i][:60] for i in idx])
" > gpurun_out/stg/raw_gs_backward_stg.txt 2>&1
