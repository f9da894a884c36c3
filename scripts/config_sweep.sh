# Bench every preset once (under gpurun): gpurun_out/<tag>_<config>_bench.json
TAG=${1:-sweep}
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3 c3u c4 c5 c2b c2m paper}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_${c}_bench.json 2> gpurun_out/${TAG}_${c}_bench.err
  echo "$c exit=$?"; tail -1 gpurun_out/${TAG}_${c}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('stages_ms_per_step'))" 2>/dev/null
done
