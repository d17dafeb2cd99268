#!/bin/bash
# One GPU-box session producing the round's evidence into gpurun_out/ (copied to profiles/).
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt
timeout 600 python __graft_entry__.py > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > $OUT/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
# full capture of the two top kernels on the SAME bench command (first launch of each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"em_kernel|cells_bitmap|cells_sort|cells_dense" -c 2 -o $OUT/prof_round $CMD > $OUT/ncu_full.log 2>&1
echo done
