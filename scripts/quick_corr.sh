python -m pytest tests/test_gpu_parity.py -q -k "corr_coeffs or eval_corr_parity or paper" 2>&1 | grep -E "passed|failed|^FAILED|Error|assert" | head -20
python -m pytest tests/test_gpu_fullsize.py -q -k "c5 or c3" 2>&1 | grep -E "passed|failed|^FAILED|Error|assert" | head -20
for c in c3 c5 paper; do
python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['config']['workload'][:10], d['value'], d['ms_per_step'], d['roofline'].get('stages_ms_per_step'))"
done
