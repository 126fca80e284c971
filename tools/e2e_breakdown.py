"""Where the end-to-end (stream_io) time of cfg3 goes: host wall of
sn_simulate vs its device time, and the raster decode/copy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02510_b200 as sn  # noqa: E402

n, K = 32000, 100
for graphs in (True, False):
    eng = sn.MatEngine(stream_io=True, use_graphs=graphs)
    eng.generate_erdos_renyi(n, 1.0, 0, stdp=True)
    d = sn.StdpConfig.defaults()
    eng.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
    eng.setup()
    eng.add_stimulus(*sn.netgen.scenario_stimulus(n, K + 10, 0).to_arrays())
    eng.simulate(5)
    eng.clear_raster()
    t0 = time.perf_counter()
    eng.simulate(K)
    t1 = time.perf_counter()
    s, q = eng.raster()
    t2 = time.perf_counter()
    st = eng.stats()
    print(f"graphs={graphs} simulate wall {1e3 * (t1 - t0):.1f} ms, device {st['last_simulate_ms']:.1f} ms, "
          f"raster {1e3 * (t2 - t1):.1f} ms for {len(s)} events")
    eng.close()
