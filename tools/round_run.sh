#!/bin/bash
# One GPU-box session producing the round's evidence into gpurun_out/ (copied to profiles/):
#   smoke, bench (+ reference arm), ncu launch list + full capture of the bench's top
#   kernels, single-fit latency, cell-metrics timing and the K x bins sweep.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt
timeout 600 python __graft_entry__.py > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# the FP32 E-step option (not the reference precision; informative only)
timeout 600 python bench.py --estep-fp32 --no-e2e --no-indexed --no-weighted --no-cpu > $OUT/bench_fp32.json 2> $OUT/bench_fp32.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > $OUT/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
# full capture of the two top kernels on the SAME bench command (first launch of each)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"em_kernel|cells_bitmap|cells_sort|cells_dense|ix_downsweep" -c 4 -o $OUT/prof_round $CMD > $OUT/ncu_full.log 2>&1
if [ "${ROUND_EXTRA:-1}" = "1" ]; then
  timeout 300 python tools/prof_fit.py > $OUT/fit_latency.txt 2>&1
  timeout 300 python tools/prof_metrics.py > $OUT/metrics_time.txt 2>&1
  timeout 300 python tools/prof_metrics.py --d 2 --bins 64 --cells 65536 --per 5000 >> $OUT/metrics_time.txt 2>&1
  timeout 1200 python tools/sweep.py --json $OUT/sweep.json > $OUT/sweep.md 2>&1
  timeout 300 python tools/prof_generate.py > $OUT/gen_time.txt 2>&1
  timeout 300 python tools/prof_indexed.py > $OUT/indexed_time.txt 2>&1
  timeout 300 python tools/prof_indexed.py --sorted >> $OUT/indexed_time.txt 2>&1
fi
echo done
