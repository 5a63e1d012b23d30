#!/usr/bin/env bash
# quad-volume K2 launched per block of views: c4 (all 496) and c5 (180 views)
for B in 8 16 32 64 65535; do
  echo "QBLK=$B $(TG_K2_QBLK=$B python scripts/k2_one.py c4 0 496 0 2>&1 | tail -1) | $(TG_K2_QBLK=$B python scripts/k2_one.py c5 0 180 0 2>&1 | tail -1)"
done
echo "slab $(python scripts/k2_one.py c4 0 496 1 2>&1 | tail -1) | $(python scripts/k2_one.py c5 0 180 1 2>&1 | tail -1)"
