# A/B of the sparse kernels on cfg4 (256k neurons, 1%, delays 1..16)
run() { env "$@" python bench.py --workload ${WL:-cfg4} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(r['bytes_per_launch']/1e9,3), round(d['value'],1))"; }
run SNB_SPARSE_SUB=4
run SNB_SPARSE_SUB=2
run SNB_SPARSE_SUB=1
