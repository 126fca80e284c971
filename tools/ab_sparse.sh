# A/B of sparse build variants (UL chunk loads per batch, min CTAs/SM) on cfg4: build
# paper_2305_02510_b200/libsnmat_ul<N>.so with -DSNB_SPARSE_COUNT_UL=<N> (or -DSNB_SPARSE_UL for k_sparse_pull)
run() { env "$@" python bench.py --workload ${WL:-cfg4} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['value'],1))"; }
run SNB_SPARSE_SUB=4
for lib in paper_2305_02510_b200/libsnmat_ul*.so; do run SNB_LIB=$PWD/$lib SNB_SPARSE_SUB=4; run SNB_LIB=$PWD/$lib SNB_SPARSE_SUB=8; done
