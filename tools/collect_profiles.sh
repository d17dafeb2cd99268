#!/bin/bash
# Copy a tools/round_run.sh session's outputs from gpurun_out/ into profiles/ under a round
# prefix: bash tools/collect_profiles.sh r2
set -eu
R=${1:?round prefix, e.g. r2}
IN=gpurun_out
OUT=profiles
cp $IN/bench.json $OUT/${R}_bench_cfg4_n1.json
cp $IN/bench_ref.json $OUT/${R}_bench_reference_n1.json
[ -s $IN/bench_fp32.json ] && cp $IN/bench_fp32.json $OUT/${R}_bench_cfg4_estep_fp32_n1.json
[ -f $IN/gen_time.txt ] && cp $IN/gen_time.txt $OUT/${R}_generate_time.txt
[ -f $IN/indexed_time.txt ] && cp $IN/indexed_time.txt $OUT/${R}_indexed_time.txt
cp $IN/launches.csv $OUT/${R}_ncu_launches_cfg4.csv
python tools/ncu_summary.py $IN/prof_round.ncu-rep > $OUT/${R}_ncu_full_cfg4_bench.txt
python tools/ncu_traffic.py $IN/prof_round.ncu-rep $OUT/ncu_traffic_cfg4.json > /dev/null
for f in fit_latency.txt metrics_time.txt; do [ -f $IN/$f ] && cp $IN/$f $OUT/${R}_${f/metrics_time/cell_metrics_time}; done
[ -f $IN/sweep.md ] && cp $IN/sweep.md $OUT/${R}_sweep_k_bins.md && cp $IN/sweep.json $OUT/${R}_sweep_k_bins.json
echo "collected into $OUT/ with prefix $R"
