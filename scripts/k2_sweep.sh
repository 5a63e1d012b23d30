#!/usr/bin/env bash
# slab-staged K2 schedule sweep (env knobs read at plan creation)
for cfg in "c4 0 496" "c5 0 90" "c5 135 90"; do
  for T in 6 8 12 16; do
    for TU in 16 32; do
      echo "T=$T TU=$TU $(TG_K2_STATS=1 TG_K2_T=$T TG_K2_TU=$TU timeout 300 python scripts/k2_one.py $cfg 2>&1 | grep -v 'slabs [0-9]' | tr '\n' ' ')"
    done
  done
done
