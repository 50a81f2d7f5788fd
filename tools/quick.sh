#!/bin/bash
# Quick GPU iteration: parity tests, one bench line (no CPU arm), optional ncu of named kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"] if d.get("e2e") else None, "frac", d["roofline"]["frac"], "fp64", d["roofline"]["fp64"]["frac"])
print("stages", d.get("stage_ms_per_step_unoverlapped"), "b512", d.get("secondary"))
PY
if [ -n "$1" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"$1" --launch-count ${2:-2} \
    -o gpurun_out/quick -f python bench.py --batch 256 --max-batch 256 --steps 1 --warmup 0 --no-cpu --no-e2e --no-b512 > gpurun_out/ncu.log 2>&1
  echo "ncu rc=$?"; python tools/ncu_summary.py gpurun_out/quick.ncu-rep 2>&1 | tail -40
fi
