"""Per-step fixed cost of a partitioned cfg4 run, emulated on one GPU: G
engines (ranks of a G-way post partition of ER(256000, 0.01), delays 1..16)
driven through the host exchange (sn_step_local -> spike words -> sn_step_finish),
so every rank's k_neuron, k_hist and sweep run as they would on its own GPU
(no kernel waits on another).  Run under ncu --metrics gpu__time_duration.sum to
get the per-kernel durations; tools/partition_cost_summary.py reduces the csv.
  python tools/partition_cost.py [G] [steps] [cfg4|cfg5]
cfg5: ER(96000, p=1) all plastic, STDP defaults, dense column blocks."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_02510_b200.engine import MatEngine, partition_range  # noqa: E402
from paper_2305_02510_b200.netgen import scenario_stimulus  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 14
wl = sys.argv[3] if len(sys.argv) > 3 else "cfg4"
n, p = (256000, 0.01) if wl == "cfg4" else (96000, 1.0)
engines = []
for r in range(G):
    if wl == "cfg4":
        e = MatEngine(storage=2, rank=r, world=G)
        e.generate_erdos_renyi(n, p, 0, delay_max=16)
    else:
        from paper_2305_02510_b200.model import StdpConfig
        d = StdpConfig.defaults()
        e = MatEngine(storage=1, rank=r, world=G)
        e.generate_erdos_renyi(n, p, 0, stdp=True)
        e.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
    e.setup()
    e.add_stimulus(*scenario_stimulus(n, T, 0).to_arrays())
    engines.append(e)
wpr = (max(partition_range(n, 0, G)[1], 1) + 31) // 32
for t in range(T):
    for e in engines:
        e.step_local()
    words = [e.spike_words(wpr * G)[r * wpr:(r + 1) * wpr].copy() for r, e in enumerate(engines)]
    for r, e in enumerate(engines):
        for q in range(G):
            if q != r:
                e.put_spike_words(q * wpr, words[q])
    for e in engines:
        e.step_finish()
spikes = sum(len(e.raster()[0]) for e in engines)
print(f"G={G} T={T} spikes={spikes} kernels={[e.stats()['sweep_kernel'] for e in engines][:1]}")
for e in engines:
    e.close()
