# ncu launch lists (gpu__time_duration, cold-cache, serialised) of one bench step per preset (under gpurun), each
# after the same command has exited 0 without ncu: gpurun_out/<tag>_<config>_launches.csv
TAG=${1:-cl}
mkdir -p gpurun_out
for c in ${CONFIGS:-c3 c3u c5 paper}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  BENCH_ALLOW_SHORT=1 $CMD > /dev/null 2>&1 && \
  BENCH_ALLOW_SHORT=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/${TAG}_${c}_launches.csv $CMD > /dev/null 2>&1
  echo "$c exit=$?"
done
