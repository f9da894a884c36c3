#!/bin/bash
# Build-time variants of the stage-4 kernel (CTA size / CTAs per SM): parity subset + c2 bench stage times each.
mkdir -p gpurun_out
for v in "$@"; do
  rm -f build/k_newton.o
  make cuda EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "=== $v"
  python -m pytest tests/test_gpu_parity.py -q -k "newton or eval" 2>&1 | grep -E "passed|failed|Error|assert" | head -12
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline'].get('stages_ms_per_step'))"
done
