./tools/ab_variants.sh c2 ru8 ru6 ru2 2>&1 | grep -E "==|resid|total"
