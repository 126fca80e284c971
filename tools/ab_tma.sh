# A/B: streaming LDG sweep vs TMA-staged sweep on cfg3 / cfg5
run() { env "$@" python bench.py --workload ${WL:-cfg3} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
run SNB_DENSE_KERNEL=stream
run SNB_DENSE_KERNEL=tma
run SNB_DENSE_KERNEL=tma SNB_TMA_WAVES=4
run SNB_DENSE_KERNEL=tma SNB_TMA_WAVES=10
WL=cfg5 run SNB_DENSE_KERNEL=stream
WL=cfg5 run SNB_DENSE_KERNEL=tma
SNB_DENSE_KERNEL=tma timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "dense_f32 or generated or stdp_n1024 or profile" 2>&1 | tail -2
