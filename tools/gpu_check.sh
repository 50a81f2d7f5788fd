#!/bin/bash
# One gpurun call: GPU parity tests, smoke, a bench line (N=1), the
# multi-GPU plumbing on this box (2 ranks sharing the GPU: one process with a
# host thread per rank, and torchrun), optionally the ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "$1" = "multi" ] || [ "$2" = "multi" ]; then
  timeout 900 python bench.py --gpus 2 --share-devices --steps 3 --warmup 1 --no-cpu > gpurun_out/bench_g2_thread.json 2> gpurun_out/bench_g2_thread.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --share-devices --steps 3 --warmup 1 --no-cpu > gpurun_out/bench_g2_torchrun.json 2> gpurun_out/bench_g2_torchrun.err
fi
if [ "$1" = "ncu" ] || [ "$2" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-b512 > gpurun_out/ncu_bench.log 2>&1
fi
tail -c 3000 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -3; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
for f in gpurun_out/bench_g2_*.json; do echo "== $f"; cat $f; tail -3 ${f%.json}.err; done
