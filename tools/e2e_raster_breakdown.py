"""Where the e2e time of sn_simulate_raster goes (cfg4 / cfg3, 100 steps):
host wall of the call vs the device time of its graph replays, repeated.
  python tools/e2e_raster_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02510_b200 as sn  # noqa: E402

K = 100
for wl, n, p, stdp, dmax in (("cfg4", 256000, 0.01, False, 16), ("cfg3", 32000, 1.0, True, 1)):
    eng = sn.MatEngine(stream_io=True)
    eng.generate_erdos_renyi(n, p, 0, stdp=stdp, delay_max=dmax)
    if stdp:
        d = sn.StdpConfig.defaults()
        eng.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
    eng.setup()
    eng.add_stimulus(*sn.netgen.scenario_stimulus(n, 6 * K + 10, 0).to_arrays())
    eng.simulate(5)
    eng.raster()
    eng.clear_raster()
    import numpy as np
    cap = K * n
    bufs = (np.empty(cap, np.int32), np.empty(cap, np.int32))
    for rep in range(6):
        out = bufs if rep >= 3 else None   # fresh arrays (page faults in the decode) vs reused ones
        t0 = time.perf_counter()
        eng.simulate_raster(K, out=out)
        t1 = time.perf_counter()
        st = eng.stats()
        print(f"{wl} rep {rep} out={'reused' if out else 'fresh'}: simulate_raster wall {1e3 * (t1 - t0):.2f} ms, "
              f"device {st['last_simulate_ms']:.2f} ms", flush=True)
    eng.close()
