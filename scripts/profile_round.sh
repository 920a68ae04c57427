#!/usr/bin/env bash
# Evidence for profiles/ (run on the GPU box from the repo root; one GPU):
#   1. bench.py at N=1 (the number, without a profiler)
#   2. ncu launch list of the same command (per-launch gpu__time_duration, cold/serialised)
#   3. ncu --set full of the 9 tcgen05 GEMM launches of one step (gate, 6 expert GEMMs, gate dW, gate dX)
# Usage: scripts/profile_round.sh <tag>   (outputs gpurun_out/<tag>_*)
set -u
tag=${1:-r01}
mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err || exit 1
timeout -s KILL 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${tag}_ncu_launches.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -c 9 \
  -o gpurun_out/${tag}_gemms python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/${tag}_ncu_full.log 2>&1
echo done
