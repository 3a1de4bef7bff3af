#!/usr/bin/env bash
# Profile one bench config on the GPU box (run under gpurun, ONE GPU):
#   tools/profile.sh <config> <tag> [extra bench args]
# Writes gpurun_out/launches_<config>_<tag>.csv (per-launch times of every
# kernel, the B200_PROFILING.md launch-list pass) and
# gpurun_out/full_<config>_<tag>.ncu-rep (ncu --set full of ONE replay-kernel
# launch, source-correlated).  Numbers printed under ncu are never bench values.
set -u
cfg=$1; tag=$2; shift 2
mkdir -p gpurun_out
export RS_BENCH_PREWARM_S=0
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${cfg}_${tag}.csv \
    python bench.py --config "$cfg" --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > gpurun_out/launches_${cfg}_${tag}.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"replay_(fast|pair)_kernel" -s ${SKIP:-3} -c 1 \
    -o gpurun_out/full_${cfg}_${tag} -f \
    python bench.py --config "$cfg" --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > gpurun_out/full_${cfg}_${tag}.log 2>&1
echo "full capture rc=$?"
