# A/B of the one-weight list order on cfg4: joint per-warp bank schedule (default)
# vs the per-list bank-sorted deal (SNB_SPARSE_BANK_JOINT=0) vs pre order (SNB_SPARSE_BANK_ORDER=0)
run() { env "$@" python bench.py --workload ${WL:-cfg4} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
for rep in 1 2; do run SNB_X=1; run SNB_SPARSE_BANK_JOINT=0; run SNB_SPARSE_BANK_ORDER=0; done
