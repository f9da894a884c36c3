# c2 bench stage times with alternative builds of libmatcha.so (build/variants/*.so), then the tree's own
for v in build/variants/*.so; do
  cp paper_2603_15285_b200/libmatcha.so /tmp/libmatcha_orig.so
  cp "$v" paper_2603_15285_b200/libmatcha.so
  echo "== $v"
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['stages_ms_per_step'])"
  cp /tmp/libmatcha_orig.so paper_2603_15285_b200/libmatcha.so
done
echo "== tree"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['stages_ms_per_step'])"
