"""Small runs of each hot kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): python tools/sanitize_cases.py <case>; exits non-zero
if the raster differs from the oracle.  Cases: dense_tma, dense_tma_delay,
cluster, tiny, count16, sparse_pull, p2p."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import bridge as B  # noqa: E402
from paper_2305_02510_b200.engine import MatEngine, p2p_connect_local  # noqa: E402
from paper_2305_02510_b200.model import StdpConfig  # noqa: E402
from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays, scenario_stimulus  # noqa: E402


def problem(n, p, seed, steps, dmax=1, plastic=0.0, one_weight=False):
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    rs = RandomStream(seed, 9)
    k = np.arange(m, dtype=np.uint64)
    arrays = {"threshold": np.full(n, 1.5), "leak": np.full(n, 0.3), "reset": np.zeros(n),
              "refractory": np.ones(n, np.int32), "axonal": np.zeros(n, np.int32), "pre": pre, "post": post,
              "weight": np.ones(m) if one_weight else -0.3 + 1.2 * rs.unit_np(k),
              "delay": (1 + rs.below_np(k + np.uint64(m), dmax)).astype(np.int32),
              "stdp": (rs.unit_np(k + np.uint64(2 * m)) < plastic).astype(np.uint8)}
    d = StdpConfig.defaults()
    sd = (d.window, np.array(d.a_plus), np.array(d.a_minus), d.w_min, d.w_max) if plastic > 0 else None
    stim = scenario_stimulus(n, steps, seed, count=max(4, n // 40), period=2, amplitude=2.5).to_arrays()
    return arrays, stim, sd


def engine(arrays, sd, rank=0, world=1, **opts):
    e = MatEngine(rank=rank, world=world, **opts)
    e.add_neurons(arrays["threshold"], arrays["leak"], arrays["reset"], arrays["refractory"], arrays["axonal"])
    e.add_synapses(arrays["pre"], arrays["post"], arrays["weight"], arrays["delay"], arrays["stdp"])
    if sd is not None:
        e.set_stdp(*sd)
    e.setup()
    return e


CASES = {  # name: (problem args, engine options, expected sweep kernel)
    "dense_tma": (dict(n=2048, p=1.0, seed=1, steps=8, plastic=1.0), dict(storage=1, persistent=False), 2),
    "dense_tma_delay": (dict(n=2048, p=0.5, seed=2, steps=8, dmax=3, plastic=1.0), dict(storage=1, persistent=False), 2),
    "cluster": (dict(n=600, p=0.5, seed=3, steps=20, dmax=8, one_weight=True), dict(storage=1), 14),
    "tiny": (dict(n=200, p=0.1, seed=4, steps=30, dmax=3, plastic=0.7), dict(storage=0), 9),
    "count16": (dict(n=20000, p=0.002, seed=5, steps=12, dmax=8, one_weight=True), dict(storage=2), 15),
    "sparse_pull": (dict(n=5000, p=0.01, seed=6, steps=10, dmax=2, plastic=0.6), dict(storage=2), 5),
}


def main(name):
    if name == "p2p":
        arrays, stim, sd = problem(300, 0.06, 7, 20, dmax=3, plastic=0.7)
        o = B.run_oracle(arrays, 20, stim, sd)
        es = [engine(arrays, sd, rank=r, world=2, storage=1, precision="f64") for r in range(2)]
        for e in es:
            e.add_stimulus(*stim)
        p2p_connect_local(es)
        for _ in range(20):
            for e in es:
                e.step_local()
            for e in es:
                e.step_finish()
        s = np.concatenate([e.raster()[0] for e in es])
        q = np.concatenate([e.raster()[1] for e in es])
        order = np.lexsort((q, s))
        s, q = s[order], q[order]
        kernel = es[0].stats()["sweep_kernel"]
        for e in es:
            e.close()
    else:
        pa, opts, want = CASES[name]
        steps = pa["steps"]
        arrays, stim, sd = problem(**pa)
        o = B.run_oracle(arrays, steps, stim, sd)
        e = engine(arrays, sd, **opts)
        e.add_stimulus(*stim)
        e.simulate(steps)
        s, q = e.raster()
        kernel = e.stats()["sweep_kernel"]
        e.close()
        assert kernel == want, (name, kernel, want)
    ok = np.array_equal(s, o["steps"]) and np.array_equal(q, o["neurons"])
    print(f"{name}: kernel {kernel}, {len(s)} spikes, raster {'==' if ok else '!='} oracle")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main(sys.argv[1])
