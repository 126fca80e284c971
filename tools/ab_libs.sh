# A/B of variant builds (tools/build_variant.sh) on one workload: LIBS="a b ..." names
run() { env "$@" python bench.py --workload ${WL:-cfg4} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
for rep in 1 2; do
  run SNB_X=base
  for l in $LIBS; do run SNB_LIB=$PWD/paper_2305_02510_b200/libsnmat_$l.so; done
done
