"""Debug: sparse STDP with delays vs the oracle at several horizons."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from oracle import bridge as B
from paper_2305_02510_b200.engine import MatEngine
from paper_2305_02510_b200.model import StdpConfig
from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays, scenario_stimulus

def run(storage, dmax, steps, precision, n=2048):
    p, seed = 0.02, 23
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    rs = RandomStream(seed, 5)
    k = np.arange(m, dtype=np.uint64)
    w = 0.2 + 0.6 * rs.unit_np(k)
    delay = (1 + rs.below_np(k + np.uint64(m), dmax)).astype(np.int32)
    plastic = (rs.unit_np(k + np.uint64(2 * m)) < 0.8).astype(np.uint8)
    arrays = {"threshold": np.full(n, 3.0), "leak": np.full(n, 0.5), "reset": np.zeros(n),
              "refractory": np.ones(n, np.int32), "axonal": np.zeros(n, np.int32), "pre": pre, "post": post,
              "weight": w, "delay": delay, "stdp": plastic}
    d = StdpConfig.defaults()
    sd = (d.window, np.array(d.a_plus), np.array(d.a_minus), d.w_min, d.w_max)
    stim = scenario_stimulus(n, steps, seed, count=400, period=1, amplitude=3.5).to_arrays()
    o = B.run_oracle(arrays, steps, stim, sd, f32_weights=(precision == "f32"))
    eng = MatEngine(storage=storage, precision=precision)
    eng.add_neurons(arrays["threshold"], arrays["leak"], arrays["reset"], arrays["refractory"], arrays["axonal"])
    eng.add_synapses(pre, post, w, delay, plastic)
    eng.set_stdp(*sd)
    eng.setup()
    eng.add_stimulus(*stim)
    eng.simulate(steps)
    s, q = eng.raster()
    wt = eng.synapse_weights()
    kern = eng.stats()["sweep_kernel"]
    eng.close()
    ras = np.array_equal(s, o["steps"]) and np.array_equal(q, o["neurons"])
    bad = np.nonzero(wt != o["weights"])[0]
    perm = np.array_equal(np.sort(wt), np.sort(o["weights"]))
    info = ""
    if len(bad):
        b = bad[0]
        info = f"first bad s={b} pre={pre[b]} post={post[b]} d={delay[b]} pl={plastic[b]} got={wt[b]} want={o['weights'][b]}; bad by delay {np.bincount(delay[bad], minlength=dmax+1)[1:]}, plastic {plastic[bad].mean():.2f}"
    print(f"storage={storage} dmax={dmax} T={steps} {precision} kernel={kern} raster_eq={ras} bad={len(bad)}/{m} perm={perm} {info}", flush=True)

for prec in ("f64", "f32"):
    for steps in (5, 20, 40, 100, 300):
        run(2, 4, steps, prec)
run(2, 3, 300, "f32"); run(2, 2, 300, "f32"); run(1, 4, 300, "f32"); run(2, 4, 300, "f32", n=4096)
