# one ncu --set full capture of the main kernel of each f-row / non-c2 preset (under gpurun), each after the same
# bench command has exited 0 without ncu: gpurun_out/<tag>_<config>_<kernel>.ncu-rep
TAG=${1:-rows}
mkdir -p gpurun_out
run() {  # config kernel-regex
  CMD="python bench.py --config $1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  BENCH_ALLOW_SHORT=1 $CMD > /dev/null 2>&1 && \
  BENCH_ALLOW_SHORT=1 ncu --set full --clock-control none --import-source on -k "regex:$2" -s 2 -c 1 \
      -o gpurun_out/${TAG}_$1_$2 $CMD > gpurun_out/${TAG}_$1_$2.log 2>&1
  echo "$1 $2 exit=$?"
}
run c3u k_ups_left
run c3 k_plane_fft
run c5 k_sh_rings_tc
run c5 k_corr_tiled
run paper k_sh_rings
