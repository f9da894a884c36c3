# Full evidence run (under gpurun): GPU tests, the default bench line, the ncu launch list of the same bench
# command, one ncu --set full capture per hot kernel (c2 sub-batch / full-batch launches), clocks.
# Outputs in gpurun_out/<tag>_*; summarise here with: python scripts/summarize_profile.py <tag>
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > gpurun_out/${TAG}_gpu.txt
nproc > gpurun_out/${TAG}_nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/${TAG}_nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_exit=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_exit=$?
tail -c 1500 gpurun_out/${TAG}_bench.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; echo launches_exit=$?
# one --set full capture per kernel: skip the reference-analysis launch and warm-up launches
for K in k_sh_rings_tc k_sh_legendre_pers k_corr_tc k_so3_grid k_newton_refine; do
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s 3 -c 1 -o gpurun_out/${TAG}_full_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1; echo full_$K=$?
done
# warm-cache DRAM traffic of the same launches (--cache-control none: what the pipeline really moves; the --set full
# captures above flush the caches before every kernel)
for K in k_sh_rings_tc k_sh_legendre_pers k_corr_tc k_so3_grid k_newton_refine; do
  ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k "regex:$K" -s 3 -c 1 --csv $CMD 2>/dev/null | grep -E "dram__|gpu__time" > gpurun_out/${TAG}_warm_$K.csv; echo warm_$K=$?
done
