# A/B of environment knobs on one workload: VARS="A=1 B=2 ..." (each one run), WL, K
run() { env "$@" python bench.py --workload ${WL:-cfg4} --steps ${K:-50} --warmup 5 --no-cpu --no-e2e --no-per-config 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', r['kernel'], round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
for rep in 1 2; do
  run SNB_X=base
  for v in $VARS; do run $v; done
done
