"""Where the end-to-end (stream_io) time goes: host wall of sn_simulate vs
its device time, and the raster decode/copy (cfg3 and cfg4, 100 steps).
  python tools/e2e_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02510_b200 as sn  # noqa: E402

K = 100
for wl, n, p, stdp, dmax in (("cfg3", 32000, 1.0, True, 1), ("cfg4", 256000, 0.01, False, 16)):
    for graphs in (True, False):
        eng = sn.MatEngine(stream_io=True, use_graphs=graphs)
        eng.generate_erdos_renyi(n, p, 0, stdp=stdp, delay_max=dmax)
        if stdp:
            d = sn.StdpConfig.defaults()
            eng.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
        eng.setup()
        eng.add_stimulus(*sn.netgen.scenario_stimulus(n, 3 * K + 10, 0).to_arrays())
        eng.simulate(5)
        eng.clear_raster()
        for rep in range(2):
            t0 = time.perf_counter()
            eng.simulate(K)
            t1 = time.perf_counter()
            s, q = eng.raster()
            t2 = time.perf_counter()
            st = eng.stats()
            print(f"{wl} graphs={graphs} rep {rep}: simulate wall {1e3 * (t1 - t0):.2f} ms, device "
                  f"{st['last_simulate_ms']:.2f} ms, raster {1e3 * (t2 - t1):.2f} ms for {len(s)} events", flush=True)
            eng.clear_raster()
        eng.close()
