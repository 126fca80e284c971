# A/B of dense-sweep launch plans on one box (env knobs read by engine.cpp plan_launches)
run() { env "$@" python bench.py --workload ${WL:-cfg3} --steps 50 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],3))"; }
for rep in 1 2; do
run SNB_SWEEP_WAVES=4
run SNB_SWEEP_WAVES=4 SNB_SWEEP_ALIGN=32
run SNB_SWEEP_RPC=896
run SNB_SWEEP_RPC=512
run SNB_SWEEP_RPC=256
run SNB_SWEEP_RPC=1024
run SNB_SWEEP_RPC=2048
run SNB_SWEEP_TILES=64 SNB_SWEEP_RPC=896
run SNB_SWEEP_TILES=64 SNB_SWEEP_RPC=512
run SNB_SWEEP_TILES=16 SNB_SWEEP_RPC=896
done
