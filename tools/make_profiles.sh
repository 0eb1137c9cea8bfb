#!/usr/bin/env bash
# Regenerates the committed round-2 measurement artifacts (run on a B200,
# e.g. through gpurun; outputs land in gpurun_out/, copy the ones to keep
# into profiles/):
#   bench line            -> profiles/r02_bench_final.json
#   ncu launch list       -> profiles/r02_launches_c4_final.csv (+ _summary.txt)
#   ncu --set full, one warm C4 solve (65 kernels, the bench's roofline
#   traffic source)       -> profiles/ncu_c4_kernels.json, profiles/r02_ncu_c4_final.txt
#   C5 on one GPU         -> profiles/r02_bench_c5_1gpu.json
set -euo pipefail
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-paper-config \
    > gpurun_out/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
# the second of two timed C4 solves (tools/c4_once.py runs them with the
# per-stage timers, i.e. serially): skip the first solve's 66 launches
ncu --set full --clock-control none -s 66 -c 65 -o /tmp/c4full \
    python tools/c4_once.py c4 2 > gpurun_out/c4full.log 2>&1
python tools/ncu_summary.py /tmp/c4full.ncu-rep gpurun_out/ncu_c4_kernels.json \
    > gpurun_out/ncu_c4.txt
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-paper-config \
    > gpurun_out/c5.json 2> gpurun_out/c5.err
