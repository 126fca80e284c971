# A/B of the persistent step loop grid on cfg2 (1k dense, delays 1..8)
run() { env "$@" python bench.py --workload ${WL:-cfg2} --steps 1000 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step']*1e3,2), 'us/step', round(d['value'],1))"; }
for c in 16 32 64 128 256; do run SNB_PERSIST_CTAS=$c; done
