# A/B: TMA-staged sweep item granularity on cfg3 / cfg5
run() { env "$@" python bench.py --workload ${WL:-cfg3} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
for w in 10 14 20 30 45; do run SNB_DENSE_KERNEL=tma SNB_TMA_WAVES=$w; done
for w in 10 20 40; do WL=cfg5 run SNB_DENSE_KERNEL=tma SNB_TMA_WAVES=$w; done
