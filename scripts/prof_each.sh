# usage (under gpurun): bash scripts/prof_each.sh <tag> [kernel ...]
# one ncu --set full capture (with source) per kernel name, each after the bench command has exited 0 alone
mkdir -p gpurun_out
TAG=$1; shift
KS=${@:-k_sh_rings k_sh_legendre k_corr k_so3_search k_newton_refine}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
BENCH_ALLOW_SHORT=1 $CMD > gpurun_out/${TAG}_plain.log 2>&1; echo plain_exit=$?
for K in $KS; do
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s ${SKIP:-2} -c 1 -o gpurun_out/${TAG}_$K $CMD > gpurun_out/${TAG}_$K.log 2>&1; echo $K exit=$?
done
ls gpurun_out/
