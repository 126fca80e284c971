"""Pins the plain-C oracle (oracle/mat_oracle.c) to the reference:
(1) against the committed golden fixtures produced by the reference's own
compiled code (tests/golden/make_golden.py), and (2) live against
oracle/_ref/libspikeforge_ref.so when it is present.  CPU only."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import cases as CS
from oracle import bridge as B

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(fname):
    return np.load(os.path.join(GOLD, fname))


def digest(steps, neurons):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(steps, np.int32).tobytes())
    h.update(np.ascontiguousarray(neurons, np.int32).tobytes())
    return h.hexdigest()


SUITES = [
    ("kat.npz", CS.kat_cases),
    ("rand_unit.npz", CS.random_unit_cases),
    ("rand_delay.npz", CS.random_delay_cases),
    ("rand_stdp.npz", CS.random_stdp_cases),
    ("crit1.npz", CS.crit1_cases),
    ("crit7.npz", CS.crit7_cases),
]


@pytest.mark.parametrize("fname,factory", SUITES, ids=[s[0] for s in SUITES])
def test_oracle_matches_reference_goldens(fname, factory):
    g = _gold(fname)
    n_checked = 0
    for c in factory():
        o = B.run_oracle(c.arrays(), c.steps, c.stim_arrays(), c.stdp_tuple(), c.record)
        assert np.array_equal(o["steps"], g[f"{c.name}/steps"]), c.name
        assert np.array_equal(o["neurons"], g[f"{c.name}/neurons"]), c.name
        # bit-exact state: integer nets trivially, float STDP nets because the
        # restatement keeps the reference's fp64 operation order
        assert np.array_equal(o["membrane"], g[f"{c.name}/membrane"]), c.name
        gw = g[f"{c.name}/weights"]
        if gw.size:
            assert np.array_equal(o["weights"], gw), c.name
        if c.record:
            assert np.array_equal(o["membrane_trace"], g[f"{c.name}/trace"]), c.name
        n_checked += 1
    assert n_checked > 0


def test_kat_literal_values():
    """The literal expectations of the reference tests, straight from the goldens."""
    g = _gold("kat.npz")

    def pairs(name):
        return list(zip(g[f"{name}/steps"].tolist(), g[f"{name}/neurons"].tolist()))

    assert pairs("chain_thr05") == [(0, 0), (1, 1)]            # test_mat_engine.cpp:61-75
    assert pairs("refractory3") == [(0, 0), (4, 0)]            # test_mat_engine.cpp:85-96
    assert pairs("chain_raster") == [(0, 0), (1, 1)]           # test_mat_engine.cpp:98-102
    assert g["membrane_trace/trace"][0].tolist() == [0.75, 0.0]  # test_mat_engine.cpp:109-116
    assert pairs("self_loop") == [(t, 0) for t in range(6)]    # test_oracle.cpp:20-26
    assert pairs("threshold_equal") == []
    assert pairs("threshold_above") == [(0, 0)]
    assert pairs("delay3") == [(0, 0), (3, 1)]
    assert pairs("axonal2") == [(0, 0), (3, 1)]
    assert pairs("refractory_resume") == [(0, 0), (3, 0)]
    assert pairs("refractory_hold") == [(0, 0)]
    assert pairs("leak_decay") == []
    assert pairs("leak_decay_fires") == [(2, 0)]
    assert pairs("infinite_leak") == []
    assert pairs("negative_weight") == [(0, 0), (0, 1)]
    assert pairs("horizon_drop") == [(0, 0)]
    assert pairs("lowered_delay3_thr05") == [(0, 0), (3, 1)]
    assert pairs("subthreshold_proxy") == [(0, 0)]
    assert g["stdp_pre_then_post/weights"].tolist() == [0.5 + 0.1]       # test_stdp.cpp:46-57
    assert g["stdp_post_then_pre/weights"].tolist() == [0.5 - 0.2]       # :59-71
    assert g["stdp_simultaneous/weights"].tolist() == [0.5]              # :73-80
    assert g["stdp_quiet/weights"].tolist() == [0.5]                     # :82-89
    assert g["stdp_clip_max/weights"].tolist() == [1.0]                  # :91-101
    assert g["stdp_clip_min/weights"].tolist() == [0.0]                  # :102-111
    assert g["stdp_window_accumulates/weights"].tolist() == [0.25 + 0.125 + 0.0625]
    assert g["stdp_only_enabled/weights"].tolist() == [0.5 + 0.1, 0.5]   # :129-149
    a_plus = [0.01 * np.exp(-k / 5.0) for k in range(1, 21)]
    for k in (1, 3, 5):                                                  # acceptance crit 5
        assert g[f"crit5_pair_k{k}/weights"].tolist() == [0.5 + a_plus[k - 1], 0.25]


def test_scale_goldens_cfg1_and_stdp():
    with open(os.path.join(GOLD, "scale.json")) as f:
        sc = json.load(f)
    assert sc["er100_025_counts"] == {"0": 2536, "1": 2527, "42": 2483}   # test_netgen.cpp:65-69
    assert sc["cfg1_seed0"]["spikes"] == 96917
    assert sc["n1000_p1_seed0"]["spikes"] == 999003
    assert sc["cfg2_seed0"]["spikes"] == 998057
    assert sc["stdp_n1024_seed0"]["spikes"] == 101379
    from golden_scale import scenario_problem
    for tag in ("cfg1_seed0", "cfg1_seed1", "cfg1_seed42"):
        arrays, stim, stdp, steps = scenario_problem(sc[tag])
        o = B.run_oracle(arrays, steps, stim, stdp)
        assert len(o["steps"]) == sc[tag]["spikes"]
        assert digest(o["steps"], o["neurons"]) == sc[tag]["digest"]


@pytest.mark.slow
def test_scale_goldens_large():
    with open(os.path.join(GOLD, "scale.json")) as f:
        sc = json.load(f)
    from golden_scale import scenario_problem
    for tag in ("n1000_p1_seed0", "stdp_n1024_seed0"):
        arrays, stim, stdp, steps = scenario_problem(sc[tag])
        o = B.run_oracle(arrays, steps, stim, stdp)
        assert digest(o["steps"], o["neurons"]) == sc[tag]["digest"], tag
        if tag.startswith("stdp"):
            ref = np.load(os.path.join(GOLD, "stdp_n1024.npz"))
            assert np.array_equal(o["weights"], ref["weights"])


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_random():
    """Fresh seeds outside the golden set, against the reference library."""
    from support import random_net, random_stim, stdp_tuple
    from paper_2305_02510_b200.model import StdpConfig
    sd = stdp_tuple(StdpConfig.defaults())
    for seed in range(1000, 1012):
        net = random_net(seed, max_neurons=30, edge_prob=0.4, max_delay=4, max_axonal=1)
        a = net.to_arrays()
        a["stdp"][:] = seed % 2
        st = random_stim(seed, net.neuron_count(), 150, 80).to_arrays()
        stdp = sd if seed % 2 else None
        r = B.run_ref_mat(a, 150, st, stdp, lower=True)
        o = B.run_oracle(a, 150, st, stdp)
        assert np.array_equal(r["steps"], o["steps"]) and np.array_equal(r["neurons"], o["neurons"])
        # float membranes on delayed nets: the lowered net sums proxy inputs
        # after direct ones (lowering.cpp:36-57), so only the order differs
        assert np.allclose(r["membrane"], o["membrane"], rtol=1e-12, atol=1e-12)
        if stdp is not None and "weights" in r:
            assert np.array_equal(r["weights"], o["weights"])
        t = B.run_ref_oracle(a, 150, st)
        if stdp is None:
            assert np.array_equal(t["steps"], o["steps"]) and np.array_equal(t["neurons"], o["neurons"])


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_oracle_long_window_matches_reference():
    """window 70 (> 64 history bits), delays up to 6: weights bit-exact vs the
    reference MAT path (lower_delays + mat_run)."""
    from support import random_net, random_stim
    w = 70
    sd = (w, np.array([0.02 * 0.97 ** k for k in range(w)]), np.array([0.025 * 0.96 ** k for k in range(w)]),
          0.0, 1.0)
    for seed in (400, 401, 402):
        net = random_net(seed, max_neurons=30, edge_prob=0.3, max_delay=4, max_axonal=2)
        a = net.to_arrays()
        a["stdp"][:] = 1
        st = random_stim(seed, net.neuron_count(), 150, 120).to_arrays()
        r = B.run_ref_mat(a, 150, st, sd, lower=True)
        o = B.run_oracle(a, 150, st, sd)
        assert np.array_equal(r["steps"], o["steps"]) and np.array_equal(r["neurons"], o["neurons"])
        assert np.array_equal(r["weights"], o["weights"])


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_shim_loop_equals_mat_run():
    """ref_shim's spelled-out mat_run loop == the reference's mat_run."""
    from support import random_net, random_stim
    for seed in range(10):
        net = random_net(seed)
        a = net.to_arrays()
        st = random_stim(seed, net.neuron_count(), 100, 30).to_arrays()
        for storage in (1, 2):
            r = B.run_ref_mat(a, 100, st, storage=storage)
            q = B.run_ref_mat_raster(a, 100, st, storage=storage)
            assert np.array_equal(r["steps"], q["steps"]) and np.array_equal(r["neurons"], q["neurons"])


# ---------------------------------------------------------------------------
# agent-based mode: oracle/abm_oracle.c vs the reference's abm_run
def test_abm_oracle_matches_reference_goldens():
    """abm.npz: the reference's abm_run (stochastic behaviours registered in
    its own registry) on every case of cases.abm_cases(); the C restatement
    must reproduce rasters, final membranes and traces bit for bit."""
    g = _gold("abm.npz")
    for c in CS.abm_cases():
        o = B.run_abm_oracle(c.arrays(), c.steps, c.stim_arrays(), seed=c.seed, fire_p=c.fire_p,
                             record_membrane=c.record)
        assert np.array_equal(o["steps"], g[f"{c.name}/steps"]), c.name
        assert np.array_equal(o["neurons"], g[f"{c.name}/neurons"]), c.name
        assert np.array_equal(o["membrane"], g[f"{c.name}/membrane"]), c.name
        if c.record:
            assert np.array_equal(o["membrane_trace"], g[f"{c.name}/trace"]), c.name


def test_abm_kat_literal_values():
    """The literal expectations of test_abm_engine.cpp, from the goldens."""
    g = _gold("abm.npz")

    def pairs(name):
        return list(zip(g[f"{name}/steps"].tolist(), g[f"{name}/neurons"].tolist()))

    assert pairs("abm_chain") == [(0, 0), (1, 1)]                      # :38-42
    assert pairs("abm_delay3") == [(0, 0), (3, 1)]                     # :44-48
    assert pairs("abm_axonal2") == [(0, 0), (3, 1)]                    # :50-55
    assert pairs("abm_same_step") == [(0, 0), (1, 1)]                  # :57-63
    assert pairs("abm_two_phase") == [(0, 0), (0, 1), (0, 3), (0, 4)]  # :65-73
    assert pairs("abm_p0_never") == [(0, 0)]                           # :113-120
    a, b = pairs("abm_seeded_9"), pairs("abm_seeded_10")               # :122-141
    assert a != b
    fires = sum(1 for _, j in a if j == 1)
    assert 20 < fires < 80


def test_abm_float_order_differs_from_mat():
    """On float nets the agent step sums leak(v) + (pending + ext) while MAT
    sums ((leak(v) + w...) + ext): the two modes are distinguishable, so the
    ABM parity tests do check the ABM order."""
    c = [c for c in CS.abm_cases() if c.name == "abm_float_1"][0]
    a = c.arrays()
    abm = B.run_abm_oracle(a, c.steps, c.stim_arrays(), record_membrane=True)
    mat = B.run_oracle(a, c.steps, c.stim_arrays(), None, True)
    assert not np.array_equal(abm["membrane_trace"], mat["membrane_trace"])
    assert np.allclose(abm["membrane_trace"], mat["membrane_trace"], rtol=0, atol=1e-9)


def test_abm_scale_golden():
    """ER(1000, 0.1), delays 1..8, half the neurons stochastic_lif, 500 steps."""
    with open(os.path.join(GOLD, "scale.json")) as f:
        sc = json.load(f)["abm_er1000_stoch"]
    from golden_scale import abm_scale_problem
    arrays, stim, fp, steps, seed = abm_scale_problem(sc)
    o = B.run_abm_oracle(arrays, steps, stim, seed=seed, fire_p=fp)
    assert len(o["steps"]) == sc["spikes"]
    assert digest(o["steps"], o["neurons"]) == sc["digest"]
    assert float(np.sum(o["membrane"])) == sc["membrane_sum"]


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_abm_oracle_matches_live_reference_random():
    """Fresh seeds and probabilities outside the golden set."""
    from support import random_net, random_stim
    for seed in range(2000, 2010):
        net = random_net(seed, max_neurons=40, edge_prob=0.3, max_delay=6, max_axonal=3)
        n = net.neuron_count()
        fp = CS._fire_mix(n, seed, choices=(0.1, 0.33, 0.5, 0.9), frac=0.6)
        st = random_stim(seed, n, 160, 120).to_arrays()
        o = B.run_abm_oracle(net.to_arrays(), 160, st, seed=seed, fire_p=fp, record_membrane=True)
        r = B.run_ref_abm_full(net.to_arrays(), 160, st, seed=seed, fire_p=fp, record_membrane=True)
        assert np.array_equal(o["steps"], r["steps"]) and np.array_equal(o["neurons"], r["neurons"])
        assert np.array_equal(o["membrane_trace"], r["membrane_trace"])


def test_fp32_storage_model_against_fp64_and_numpy():
    """The oracle's fp32 weight-storage model (mat_oracle_run_f32w, the bit-exact
    target of fp32 engines): with the fp64 run's spike train, its weights equal
    an independent numpy replay of apply_stdp (mat_engine.cpp:210-250) with one
    float rounding per update, and stay within the rigorous drift bound
    (T + 1) 2^-24 max|w| of the fp64 reference weights."""
    from paper_2305_02510_b200.model import StdpConfig
    from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays, scenario_stimulus
    from support import fp32_weight_floor
    n, p, seed, steps = 300, 0.05, 5, 120
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    rs = RandomStream(seed, 3)
    k = np.arange(m, dtype=np.uint64)
    w = 0.1 + 0.8 * rs.unit_np(k)
    plastic = (rs.unit_np(k + np.uint64(m)) < 0.7).astype(np.uint8)
    arrays = {"threshold": np.full(n, 2.0), "leak": np.full(n, 0.5), "reset": np.zeros(n),
              "refractory": np.ones(n, np.int32), "axonal": np.zeros(n, np.int32), "pre": pre, "post": post,
              "weight": w, "delay": np.ones(m, np.int32), "stdp": plastic}
    d = StdpConfig.defaults()
    sd = (d.window, np.array(d.a_plus), np.array(d.a_minus), d.w_min, d.w_max)
    stim = scenario_stimulus(n, steps, seed, count=40, period=1, amplitude=3.0).to_arrays()
    o = B.run_oracle(arrays, steps, stim, sd)
    o32 = B.run_oracle(arrays, steps, stim, sd, f32_weights=True)
    assert len(o["steps"]) > 2000
    assert np.array_equal(o32["steps"], o["steps"]) and np.array_equal(o32["neurons"], o["neurons"])
    S = np.zeros((steps, n), bool)
    S[o["steps"], o["neurons"]] = True
    ap, am = np.array(d.a_plus), np.array(d.a_minus)
    w32 = w.astype(np.float32)
    for t in range(steps):
        pot = np.zeros(n)
        dep = np.zeros(n)
        for kk in range(1, min(d.window, t) + 1):
            pot += ap[kk - 1] * S[t - kk]
            dep += am[kk - 1] * S[t - kk]
        dw = np.where(S[t][post], pot[pre], 0.0)
        dw = np.where(S[t][pre], dw - dep[post], dw)
        upd = np.clip((w32.astype(np.float64) + dw).astype(np.float32), np.float32(d.w_min), np.float32(d.w_max))
        w32 = np.where(plastic == 1, upd, w32)
    assert np.array_equal(o32["weights"], w32.astype(np.float64))
    floor = fp32_weight_floor(steps, w, d.w_min, d.w_max)
    assert np.all(np.abs(o32["weights"] - o["weights"]) <= floor)
    assert not np.array_equal(o32["weights"], o["weights"])   # the rounding is visible
