#!/bin/bash
# per-class eager timings of tuning variants: tools/ab_variants.sh CFG NAME...
cfg=$1; shift
echo "== $cfg default"; timeout 600 python tools/ncu_iter.py $cfg 5 | grep -E "gs_|spmv|resid|total"
for v in "$@"; do
  echo "== $cfg $v"; P2G_LIB_PATH=tools/variants/$v.so timeout 600 python tools/ncu_iter.py $cfg 5 | grep -E "gs_|spmv|resid|total"
done
