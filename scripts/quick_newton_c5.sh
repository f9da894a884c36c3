timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "newton" 2>&1 | tail -1
for c in c5 c2; do BENCH_ALLOW_SHORT=1 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['stages_ms_per_step']['newton_refine'])"; done
