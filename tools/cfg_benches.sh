#!/bin/bash
# Bench lines + ncu launch lists for cfg1..cfg3 (the non-headline BASELINE configs), one GPU.
#   bash tools/cfg_benches.sh [prefix]   -> gpurun_out/<prefix>_bench_cfgN_n1.json, _launches_cfgN.csv
set -u
P=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
for c in cfg1 cfg2 cfg3; do
  case $c in cfg3) CC="--cpu-cells 8 --cpu-repeats 3";; *) CC="--cpu-cells 1 --cpu-repeats 3";; esac
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 $CC > $OUT/${P}_bench_${c}_n1.json 2> $OUT/${P}_bench_${c}.err
  echo "$c rc=$?" >> $OUT/${P}_cfg_benches.log
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${P}_launches_${c}.csv $CMD > /dev/null 2>&1
  echo "$c ncu rc=$?" >> $OUT/${P}_cfg_benches.log
done
