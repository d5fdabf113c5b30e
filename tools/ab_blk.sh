#!/bin/bash
# A/B of the node-blocked row kernels vs the row kernels (per-class eager timings)
for cfg in "$@"; do
  echo "== $cfg node-blocked"; timeout 600 python tools/ncu_iter.py $cfg 5
  echo "== $cfg row kernels"; P2G_NO_NODEBLK=1 timeout 600 python tools/ncu_iter.py $cfg 5
done
