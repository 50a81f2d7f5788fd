#!/bin/bash
# ncu --set full (with source) of the first launch of each kernel matching REGEX
# on a 256-frame VGA batch, plus the per-instruction SASS page and the summary.
#   bash tools/prof_kernels.sh TAG "k_detect_walk|k_sample" [extra bench args]
mkdir -p gpurun_out
TAG=${1:-prof}
REGEX=${2:-"k_detect_walk|k_blur|k_sample|k_describe"}
shift 2
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-id ::regex:"^(void )?(${REGEX})":1 \
  -o gpurun_out/${TAG} -f python bench.py --batch 256 --max-batch 256 --steps 1 --warmup 0 --no-cpu --no-e2e --no-b512 "$@" \
  > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}.log
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}_summary.json 2>&1
python tools/sass_mix.py gpurun_out/${TAG}_sass.csv > gpurun_out/${TAG}_mix.txt 2>&1
tail -3 gpurun_out/${TAG}.log
