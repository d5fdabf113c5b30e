./tools/ab_variants.sh c2 xp5 2>&1
