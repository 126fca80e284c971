import json, sys, time
sys.path.insert(0, '.')
from oracle import bridge as B
t0 = time.time()
r = B.ref_bench_run(32000, 1.0, 0, 100, 1, 3, True, 0)
r.pop('steps'); r.pop('neurons')
r['wall_s'] = time.time() - t0
print(json.dumps(r))
