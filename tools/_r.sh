for wl in cfg5 cfg3; do python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu --no-e2e --no-per-config 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl', d['value'], d['ms_per_step'], d['fixed_per_step'])"; done
python -m pytest tests -m gpu -q -x -k "partition or determinism or repeated" 2>&1 | tail -1
