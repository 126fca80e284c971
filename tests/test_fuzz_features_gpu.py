"""Randomised cross-check of the round-2 features against the reference:
delays beyond 64 steps (relay chains), STDP windows beyond 512 steps (history
in global memory), plasticity switched on and off (sn_set_plasticity), and
per-step driving (sn_step with mat_run's ext rows) interleaved with
simulate() calls -- on random nets, storages and precisions.  Checkers: the
reference's own mat_step / apply_stdp loop with apply_stdp skipped on the
same steps (oracle/ref_shim.cpp, delays lowered by the reference's
lower_delays), or the pinned C oracle for unmasked runs; fp64 weights
bit-exact, fp32 weights bit-exact against the fp32 storage model."""
from __future__ import annotations

import os

import numpy as np
import pytest

import cases as CS
from support import close_rel, random_net, random_stim

pytestmark = pytest.mark.gpu


def _ext_rows(n, steps, stim):
    st, nid, amp = stim
    rows = [None] * steps
    for i in np.argsort(st, kind="stable"):
        t = int(st[i])
        if rows[t] is None:
            rows[t] = np.zeros(n)
        rows[t][nid[i]] += amp[i]
    return rows


@pytest.mark.parametrize("seed", range(int(os.environ.get("SNB_FUZZ_FEATURES", "48"))))
def test_random_feature_plans(seed):
    from oracle import bridge as B
    from paper_2305_02510_b200.engine import MatEngine
    from paper_2305_02510_b200.model import StdpConfig
    rng = np.random.default_rng(31000 + seed)
    kind = ("long_delay", "long_window", "plasticity", "steps")[seed % 4]
    max_delay = int(rng.choice([30, 90, 150])) if kind == "long_delay" else int(rng.choice([1, 4]))
    net = random_net(31000 + seed, min_neurons=8, max_neurons=int(rng.choice([20, 45])),
                     edge_prob=float(rng.choice([0.15, 0.35])), max_delay=max_delay, max_axonal=2)
    n = net.neuron_count()
    if kind == "long_window":
        w = int(rng.choice([520, 600]))
        steps = 620
    else:
        w = int(rng.choice([5, 20, 70]))
        steps = int(rng.choice([120, 220])) if kind == "long_delay" else 90
    stdp = StdpConfig(window=w, a_plus=list(0.02 * 0.999 ** np.arange(w)), a_minus=list(0.025 * 0.999 ** np.arange(w)),
                      w_min=float(rng.choice([-1.0, 0.0])), w_max=float(rng.choice([2.0, 3.0])))
    for s in net.synapses:
        s.stdp_enabled = bool(rng.random() < 0.7)
    stim = random_stim(31000 + seed, n, steps, int(rng.integers(3 * n, 8 * n)))
    c = CS.Case(f"feat_{seed}", net, steps, stim, stdp=stdp)
    a = c.arrays()
    sd = c.stdp_tuple()
    mask = np.ones(steps, np.uint8)
    if kind == "plasticity":
        for lo in rng.choice(steps - 10, 3, replace=False):
            mask[lo:lo + int(rng.integers(3, 12))] = 0
    precision = str(rng.choice(["f64", "f32"]))
    storage = int(rng.integers(0, 3))
    lowered = max_delay > 1 or bool(a["axonal"].any())
    if kind == "plasticity":
        if not B.ref_available():
            pytest.skip("oracle/_ref not built")
        o = B.run_ref_mat_masked(a, steps, c.stim_arrays(), sd, mask, lower=lowered)   # fp64 reference
    else:
        o = B.run_oracle(a, steps, c.stim_arrays(), sd, f32_weights=precision == "f32")
    e = MatEngine(storage=storage, precision=precision)
    try:
        e.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
        e.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], a["stdp"])
        e.set_stdp(*sd)
        e.setup()
        if kind == "steps":   # per-step driving interleaved with simulate() over the same schedule
            rows = _ext_rows(n, steps, c.stim_arrays())
            e.add_stimulus(*c.stim_arrays())
            t = 0
            while t < steps:
                if rng.random() < 0.5:
                    e.step(rows[t])
                    t += 1
                else:
                    k = int(min(steps - t, rng.integers(1, 25)))
                    e.simulate(k)
                    t += k
        else:
            e.add_stimulus(*c.stim_arrays())
            t = 0
            while t < steps:   # segments of equal plasticity
                on = bool(mask[t])
                k = 1
                while t + k < steps and bool(mask[t + k]) == on:
                    k += 1
                e.set_plasticity(on)
                e.simulate(k)
                t += k
        s_, q_ = e.raster()
        wt = e.synapse_weights()
        mem = e.membrane()
    finally:
        e.close()
    tag = (seed, kind, storage, precision, n, max_delay, w)
    assert np.array_equal(s_, o["steps"]) and np.array_equal(q_, o["neurons"]), tag
    if precision == "f64" or kind != "plasticity":   # fp64, or fp32 against the fp32 storage model
        assert np.array_equal(wt, o["weights"]), tag
        assert close_rel(mem, o["membrane"]), tag
    else:   # fp32 against the fp64 reference: the storage drift bound
        from support import fp32_weight_floor
        assert close_rel(wt, o["weights"], abs_floor=fp32_weight_floor(steps, a["weight"], sd[3], sd[4])), tag
