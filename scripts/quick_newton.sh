# parity subset + stage-4 timings (under gpurun)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "candidate_groups or newton or eval" 2>&1 | grep -E "passed|failed|^FAILED|Error|assert" | head -20
python scripts/newton_bands.py 2>&1 | grep -v -i "exception\|traceback\|__del__\|attributeerror" | tail -11
for c in c2 c5; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline'].get('stages_ms_per_step'))"
done
