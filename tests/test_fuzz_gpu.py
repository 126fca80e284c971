"""Randomised cross-check of every engine plan against the C oracles: random
nets (delays, axonal delays, refractory periods, infinite leaks, plastic
subsets, STDP windows past 64 steps), random stimulus and random engine
options (storage, precision, exact order, graphs, persistent loop, stream
I/O, simulate() chunking, MAT or agent-based mode).  Rasters must be
identical; fp64 + exact order (or the one-CTA loop) bit-exact; fp64 weights
bit-exact in every plan; fp32 weights bit-exact against the reference
algorithm with fp32 storage (oracle f32 model) and within the accumulated
storage rounding of the fp64 reference."""
from __future__ import annotations

import os

import numpy as np
import pytest

import cases as CS
from support import close_rel, fp32_weight_floor, random_net, random_stim

pytestmark = pytest.mark.gpu


def _stdp(rng):
    from paper_2305_02510_b200.model import StdpConfig
    w = int(rng.choice([1, 3, 20, 40, 70]))
    return StdpConfig(window=w, a_plus=list(0.03 * rng.random(w)), a_minus=list(0.03 * rng.random(w)),
                      w_min=float(rng.choice([0.0, -1.0])), w_max=float(rng.choice([1.0, 3.0])))


@pytest.mark.parametrize("seed", range(int(os.environ.get("SNB_FUZZ_CASES", "240"))))
def test_random_plans_match_oracle(seed):
    from oracle import bridge as B
    from paper_2305_02510_b200.engine import MatEngine
    rng = np.random.default_rng(9000 + seed)
    abm = seed % 4 == 3
    net = random_net(9000 + seed, min_neurons=2, max_neurons=int(rng.choice([12, 40, 90])),
                     edge_prob=float(rng.choice([0.05, 0.2, 0.5])), max_delay=int(rng.choice([1, 3, 9])),
                     max_axonal=int(rng.choice([0, 2])), max_refractory=int(rng.choice([0, 3])))
    n = net.neuron_count()
    stdp = None
    if not abm and rng.random() < 0.5:
        stdp = _stdp(rng)
        for s in net.synapses:
            s.stdp_enabled = bool(rng.random() < 0.7)
    steps = int(rng.choice([30, 120]))
    stim = random_stim(9000 + seed, n, steps, int(rng.integers(5, 4 * n + 6)))
    c = CS.Case(f"fuzz_{seed}", net, steps, stim, stdp=stdp, record=bool(rng.random() < 0.3))
    a = c.arrays()
    fire_p = None
    if abm and rng.random() < 0.7:
        fire_p = np.where(rng.random(n) < 0.5, rng.choice([0.0, 0.3, 0.5, 0.9], n), 1.0)
    run_seed = int(rng.integers(0, 1 << 40))
    if abm:
        o = B.run_abm_oracle(a, steps, c.stim_arrays(), seed=run_seed, fire_p=fire_p, record_membrane=c.record)
    else:
        o = B.run_oracle(a, steps, c.stim_arrays(), c.stdp_tuple(), c.record)
    opts = dict(storage=int(rng.integers(0, 3)), precision=str(rng.choice(["f32", "f64"])),
                exact_order=bool(rng.random() < 0.5), use_graphs=bool(rng.random() < 0.7),
                persistent=bool(rng.random() < 0.7), stream_io=bool(rng.random() < 0.3))
    chunks = [steps] if rng.random() < 0.5 else [1, steps // 3, steps - 1 - steps // 3]
    eng = MatEngine(record_membrane=c.record, mode="abm" if abm else "mat", **opts)
    try:
        eng.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
        if len(a["pre"]):
            eng.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], None if abm else a["stdp"])
        if stdp is not None:
            eng.set_stdp(stdp.window, stdp.a_plus, stdp.a_minus, stdp.w_min, stdp.w_max)
        if abm:
            eng.set_seed(run_seed)
            if fire_p is not None:
                eng.set_fire_probability(fire_p)
        eng.setup()
        st = c.stim_arrays()
        if len(st[0]):
            eng.add_stimulus(*st)
        for k in chunks:
            eng.simulate(k)
        s, q = eng.raster()
        mem = eng.membrane()
        w = eng.synapse_weights() if len(a["pre"]) else None
        tr = eng.membrane_trace() if c.record else None
        kernel = eng.stats()["sweep_kernel"]
    finally:
        eng.close()
    tag = (seed, opts, chunks, abm, kernel)
    assert np.array_equal(s, o["steps"]) and np.array_equal(q, o["neurons"]), tag
    exact = opts["precision"] == "f64" and (opts["exact_order"] or kernel == 9)
    if exact:
        assert np.array_equal(mem, o["membrane"]), tag
        if w is not None and stdp is not None:
            assert np.array_equal(w, o["weights"]), tag
        if tr is not None:
            assert np.array_equal(tr, o["membrane_trace"]), tag
    elif opts["precision"] == "f64":
        assert close_rel(mem, o["membrane"]), tag
        if w is not None and stdp is not None:
            assert np.array_equal(w, o["weights"]), tag  # the per-synapse update is elementwise
    elif abm:
        assert close_rel(mem, o["membrane"]), tag   # integer weights: fp32 storage is exact
    else:
        # fp32 weight storage, fp64 STDP arithmetic: the engine's weights are the
        # reference algorithm's with every stored weight rounded to float once
        # (oracle f32 model, bit-exact); vs the fp64 reference they are within
        # the accumulated storage rounding
        o32 = B.run_oracle(a, steps, c.stim_arrays(), c.stdp_tuple(), c.record, f32_weights=True)
        assert close_rel(mem, o32["membrane"]), tag
        if w is not None and stdp is not None:
            assert np.array_equal(w, o32["weights"]), tag
            assert close_rel(w, o["weights"], abs_floor=fp32_weight_floor(steps, a["weight"], stdp.w_min,
                                                                           stdp.w_max)), tag


@pytest.mark.parametrize("seed", range(int(os.environ.get("SNB_FUZZ_MEDIUM", "12"))))
def test_random_medium_plans_match_oracle(seed):
    """Medium nets (2k-20k neurons: several dense row chunks / TMA items,
    several sparse pre blocks) with random weights, delays, plasticity and
    options against the C oracle (rasters identical, fp64 weights exact)."""
    from oracle import bridge as B
    from paper_2305_02510_b200.engine import MatEngine
    from paper_2305_02510_b200.model import StdpConfig
    from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays, scenario_stimulus
    rng = np.random.default_rng(7700 + seed)
    n = int(rng.choice([2048, 5000, 12000, 20000]))
    p = float({2048: 0.05, 5000: 0.01, 12000: 0.003, 20000: 0.002}[n])
    pre, post = erdos_renyi_arrays(n, p, 7700 + seed)
    m = len(pre)
    rs = RandomStream(7700 + seed, 5)
    k = np.arange(m, dtype=np.uint64)
    dmax = int(rng.choice([1, 4, 20, 40]))
    delay = (1 + rs.below_np(k, dmax)).astype(np.int32)
    kind = str(rng.choice(["one", "three", "float"]))
    w = (np.ones(m) if kind == "one" else np.array([1.0, 2.0, -1.0])[rs.below_np(k + np.uint64(m), 3)]
         if kind == "three" else 0.2 + rs.unit_np(k + np.uint64(2 * m)))
    stdp = None
    plastic = np.zeros(m, np.uint8)
    if rng.random() < 0.4 and dmax <= 20:
        stdp = StdpConfig.defaults()
        plastic = (rs.unit_np(k + np.uint64(3 * m)) < 0.5).astype(np.uint8)
    thr = np.full(n, 1.0 if kind != "float" else 1.3)
    arrays = {"threshold": thr, "leak": np.full(n, 0.25), "reset": np.zeros(n), "refractory": np.full(n, 1, np.int32),
              "axonal": np.zeros(n, np.int32), "pre": pre, "post": post, "weight": w, "delay": delay, "stdp": plastic}
    steps = 30
    stim = scenario_stimulus(n, steps, 7700 + seed, count=max(3, n // 50), period=3, amplitude=2.0).to_arrays()
    sd = None if stdp is None else (stdp.window, np.array(stdp.a_plus), np.array(stdp.a_minus), stdp.w_min, stdp.w_max)
    o = B.run_oracle(arrays, steps, stim, sd)
    opts = dict(storage=int(rng.integers(1, 3)), precision="f64", exact_order=bool(rng.random() < 0.3),
                use_graphs=bool(rng.random() < 0.7), persistent=bool(rng.random() < 0.5),
                stream_io=bool(rng.random() < 0.3))
    eng = MatEngine(**opts)
    try:
        eng.add_neurons(thr, arrays["leak"], arrays["reset"], arrays["refractory"], arrays["axonal"])
        eng.add_synapses(pre, post, w, delay, plastic)
        if stdp is not None:
            eng.set_stdp(*sd)
        eng.setup()
        eng.add_stimulus(*stim)
        eng.simulate(steps)
        s, q = eng.raster()
        mem = eng.membrane()
        wt = eng.synapse_weights()
        kernel = eng.stats()["sweep_kernel"]
    finally:
        eng.close()
    tag = (seed, n, dmax, kind, stdp is not None, opts, kernel)
    assert len(o["steps"]) > 0, tag
    assert np.array_equal(s, o["steps"]) and np.array_equal(q, o["neurons"]), tag
    assert close_rel(mem, o["membrane"]), tag
    if stdp is not None:
        assert np.array_equal(wt, o["weights"]), tag
