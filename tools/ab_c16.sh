# A/B of k_sparse_count16 build variants (UL) x lanes per post on cfg4, against the 32-bit count kernel
run() { env "$@" timeout 300 python bench.py --workload ${WL:-cfg4} --steps 60 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*'.replace('$PWD/',''), r['kernel'], round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
run SNB_SPARSE_COUNT16=0
run SNB_SPARSE_COUNT16=1
for lib in ${LIBS:-paper_2305_02510_b200/libsnmat_c16*.so}; do for s in ${SUBS:-8 16}; do run SNB_LIB=$PWD/$lib SNB_SPARSE_SUB=$s; done; done
