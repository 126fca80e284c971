# A/B of the cfg3 sweep across library builds: LIBS="path1 path2 ..." (SNB_LIB
# values); prints sweep ms / HBM fraction / steps/s per run, two rounds.
run() { env "$@" python bench.py --workload ${WL:-cfg3} --steps ${K:-50} --warmup 5 --no-cpu --no-e2e --no-per-config 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
for rep in 1 2; do
  run SNB_X=current
  for l in $LIBS; do run SNB_LIB=$l; done
done
