# usage (under gpurun): bash scripts/quick.sh "<pytest -k expr>"   -> targeted GPU tests + the default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$1" > gpurun_out/quick_pytest.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|Error" gpurun_out/quick_pytest.log | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/quick_bench.log 2>&1; echo bench_exit=$?
tail -1 gpurun_out/quick_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'ms',d['ms_per_step']); print(r['kernel'],r['bound'],r['frac'],r['stages_ms_per_step'])"
