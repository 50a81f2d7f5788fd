#!/bin/bash
# ncu --set full of the first launch of every extractor kernel (256-frame batch, B8, 4K).
mkdir -p gpurun_out
TAG=${1:-all}
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-id ::regex:'^(k_|void k_)':1 \
  -o gpurun_out/${TAG} -f python bench.py --batch 256 --max-batch 256 --steps 1 --warmup 0 --no-cpu --no-e2e --no-b512 \
  > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}.log
tail -3 gpurun_out/${TAG}.log
