./tools/ab_variants.sh c2 f5 f6 f8 2>&1 | grep -E "==|forward|total"
