#!/bin/bash
# Usage: build variants/libcdvz_gpu_<name>.so (e.g. with -D macros), then on the GPU box
#   bash tools/ab_variants.sh name1 name2 ...
# A/B of prebuilt library variants: bench value and stage times per variant.
cp paper_1705_09776_b200/libcdvz_gpu.so /tmp/lib_orig.so
for v in "$@"; do
  cp variants/libcdvz_gpu_$v.so paper_1705_09776_b200/libcdvz_gpu.so
  for rep in 1 2; do
    python bench.py --no-cpu --no-e2e --no-b512 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readline());print('$v', round(d['value']), {k: round(x,3) for k,x in d['stage_ms_per_step_unoverlapped'].items()})"
  done
done
cp /tmp/lib_orig.so paper_1705_09776_b200/libcdvz_gpu.so
