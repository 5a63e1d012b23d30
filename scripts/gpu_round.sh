#!/usr/bin/env bash
# One gpurun pass: GPU parity tests, smoke, bench (both arms), ncu launch list
# and one full-set capture of K1.  Usage (from the repo root, on the box):
#   bash scripts/gpu_round.sh TAG [tests|bench|ncu ...]
# Outputs land in gpurun_out/TAG_*.
set -u
TAG=${1:-run}; shift || true
WHAT=${*:-tests bench ncu}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
for w in $WHAT; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest.log 2>&1
      echo "pytest rc=$?" >> $OUT/${TAG}_pytest.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1
      echo "smoke rc=$?" >> $OUT/${TAG}_smoke.log ;;
    bench)
      timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
      timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err ;;
    quick)
      timeout 600 python bench.py --no-cpu-baseline --steps 5 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $OUT/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --fp-steps 1 \
        --no-cpu-baseline > $OUT/${TAG}_ncu_bench.log 2>&1
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cone_bp_kernel \
        -s 3 -c 1 -o $OUT/${TAG}_k1 -f python bench.py --steps 3 --warmup 3 --fp-steps 1 \
        --no-cpu-baseline > $OUT/${TAG}_ncu_k1.log 2>&1 ;;
    ncuk3)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter_kernel \
        -c 1 -o $OUT/${TAG}_k3 -f python bench.py --steps 3 --warmup 3 --fp-steps 1 \
        --no-cpu-baseline --c5-iters 0 > $OUT/${TAG}_ncu_k3.log 2>&1 ;;
    ncufp)
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cone_fp_kernel \
        -c 1 -o $OUT/${TAG}_k2 -f python bench.py --steps 3 --warmup 3 --fp-steps 1 \
        --no-cpu-baseline > $OUT/${TAG}_ncu_k2.log 2>&1 ;;
  esac
done
ls -la $OUT
