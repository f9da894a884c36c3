# time stage 1 at the paper point with alternative builds of libmatcha.so (build/variants/*.so), then the tree's own
for v in build/variants/*.so; do
  cp paper_2603_15285_b200/libmatcha.so /tmp/libmatcha_orig.so
  cp "$v" paper_2603_15285_b200/libmatcha.so
  echo "== $v"; TS_N=200 TS_L=100 TS_B=100 python scripts/time_sh.py 0 2>&1 | grep dbg
  cp /tmp/libmatcha_orig.so paper_2603_15285_b200/libmatcha.so
done
echo "== tree"; TS_N=200 TS_L=100 TS_B=100 python scripts/time_sh.py 0 2>&1 | grep dbg
