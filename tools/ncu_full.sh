#!/bin/bash
# ncu --set full captures of the hot kernels (one launch each) on a 256-frame batch.
#   bash tools/ncu_full.sh TAG "kernel|regex" COUNT [extra bench args]
mkdir -p gpurun_out
TAG=${1:-cap}
REGEX=${2:-"k_blur|k_detect"}
COUNT=${3:-2}
shift 3
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:${REGEX}" -c ${COUNT} \
  -o gpurun_out/${TAG} -f python bench.py --batch 256 --max-batch 256 --steps 1 --warmup 0 --no-cpu --no-e2e "$@" \
  > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}.log
tail -3 gpurun_out/${TAG}.log
