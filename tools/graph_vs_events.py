"""Device time per step of cfg3 with (a) per-kernel CUDA events and host
launches (profile mode) vs (b) per-step CUDA graph replay without events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02510_b200 as sn  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32000
for profile in (True, False, True, False):
    eng = sn.MatEngine(profile=profile, use_graphs=True)
    eng.generate_erdos_renyi(n, 1.0, 0, stdp=True)
    d = sn.StdpConfig.defaults()
    eng.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
    eng.setup()
    eng.add_stimulus(*sn.netgen.scenario_stimulus(n, 120, 0).to_arrays())
    eng.simulate(5)
    eng.reset_stats()
    eng.simulate(100)
    st = eng.stats()
    print(f"profile={profile} ms/step={st['last_simulate_ms'] / 100:.4f} "
          f"sweep_avg={st['sweep_ms'] / max(1, st['sweep_launches']):.4f}")
    eng.close()
