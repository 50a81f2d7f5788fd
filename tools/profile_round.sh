#!/bin/bash
# Round evidence: ncu --set full of every kernel, the launch list, and a bench line.
set -x
mkdir -p gpurun_out
bash tools/ncu_all.sh ${1:-r1_v13} > gpurun_out/ncu_all_stdout.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-b512 > gpurun_out/ncu_bench.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
