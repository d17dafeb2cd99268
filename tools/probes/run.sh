#!/bin/bash
# Micro-probes behind DESIGN.md's FP64-pipe decisions; run on the GPU box:
#   gpurun -- bash tools/probes/run.sh   -> gpurun_out/fp64_probes.txt
set -eu
mkdir -p gpurun_out /tmp/probes
for p in pipe_probe dmma_probe; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probes/$p tools/probes/$p.cu
  echo "== $p" >> gpurun_out/fp64_probes.txt
  timeout 120 /tmp/probes/$p >> gpurun_out/fp64_probes.txt
done
