# usage (under gpurun): bash scripts/prof.sh <tag> <kernel-regex> [skip] [count]
mkdir -p gpurun_out
TAG=$1; KRE=$2; SKIP=${3:-2}; CNT=${4:-2}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
BENCH_ALLOW_SHORT=1 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; echo launches_exit=$?
BENCH_ALLOW_SHORT=1 $CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s $SKIP -c $CNT -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo full_exit=$?
ls -la gpurun_out/
