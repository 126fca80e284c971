"""Per-step API (sn_step = mat_step, mat_engine.cpp:168-208 / mat_engine.hpp:92-94)
and the plasticity switch (sn_set_plasticity: mat_step with or without
apply_stdp, mat_engine.hpp:92-98), against the engine's own simulate() and the
reference's public API driven step by step (oracle/ref_shim.cpp mat_loop)."""
from __future__ import annotations

import numpy as np
import pytest

from support import close_rel

pytestmark = pytest.mark.gpu


def _problem(n=200, p=0.08, seed=41, steps=60, dmax=4, wlo=-0.3, whi=1.2):
    from paper_2305_02510_b200.model import StdpConfig
    from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays, scenario_stimulus
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    rs = RandomStream(seed, 9)
    k = np.arange(m, dtype=np.uint64)
    arrays = {"threshold": np.full(n, 1.5), "leak": np.full(n, 0.3), "reset": np.zeros(n),
              "refractory": np.ones(n, np.int32), "axonal": np.zeros(n, np.int32), "pre": pre, "post": post,
              "weight": wlo + (whi - wlo) * rs.unit_np(k),
              "delay": (1 + rs.below_np(k + np.uint64(m), dmax)).astype(np.int32),
              "stdp": (rs.unit_np(k + np.uint64(2 * m)) < 0.7).astype(np.uint8)}
    d = StdpConfig.defaults()
    sd = (d.window, np.array(d.a_plus), np.array(d.a_minus), d.w_min, d.w_max)
    stim = scenario_stimulus(n, steps, seed, count=12, period=2, amplitude=2.5).to_arrays()
    return arrays, stim, sd, steps


def _engine(arrays, sd, storage, precision="f64"):
    from paper_2305_02510_b200.engine import MatEngine
    e = MatEngine(storage=storage, precision=precision)
    e.add_neurons(arrays["threshold"], arrays["leak"], arrays["reset"], arrays["refractory"], arrays["axonal"])
    e.add_synapses(arrays["pre"], arrays["post"], arrays["weight"], arrays["delay"], arrays["stdp"])
    if sd is not None:
        e.set_stdp(*sd)
    e.setup()
    return e


def _ext_rows(n, steps, stim):
    """mat_run's per-step ext (mat_engine.cpp:256-275): stable by step, each
    neuron's amplitudes summed from 0.0 in list order; None for steps without
    stimulus (mat_run passes an empty span)."""
    st, nid, amp = stim
    rows = [None] * steps
    for i in np.argsort(st, kind="stable"):
        t = int(st[i])
        if rows[t] is None:
            rows[t] = np.zeros(n)
        rows[t][nid[i]] += amp[i]
    return rows


@pytest.mark.parametrize("storage", [0, 1, 2])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_step_equals_simulate(storage, precision):
    """step(ext_t) for t = 0..T-1 with mat_run's ext rows reproduces
    simulate(T) over the same schedule: each step's spike list is that row of
    the raster, and final weights and membranes are identical."""
    arrays, stim, sd, steps = _problem()
    n = len(arrays["threshold"])
    a = _engine(arrays, sd, storage, precision)
    a.add_stimulus(*stim)
    a.simulate(steps)
    s_ref, q_ref = a.raster()
    w_ref, m_ref = a.synapse_weights(), a.membrane()
    a.close()
    b = _engine(arrays, sd, storage, precision)
    total = 0
    for t, ext in enumerate(_ext_rows(n, steps, stim)):
        spikes = b.step(ext)
        assert np.array_equal(spikes, q_ref[s_ref == t]), t
        total += len(spikes)
    assert total == len(s_ref) > 500
    s2, q2 = b.raster()   # the per-step calls also accumulate the raster
    assert np.array_equal(s2, s_ref) and np.array_equal(q2, q_ref)
    assert np.array_equal(b.synapse_weights(), w_ref)
    assert np.array_equal(b.membrane(), m_ref)
    b.close()


def test_step_ext_length_and_schedule():
    """mat_step's ext contract: n amplitudes or none ("mat_step: ext must have
    one amplitude per neuron", mat_engine.cpp:170-171); the schedule added with
    add_stimulus is not consulted by step() but is by a later simulate()."""
    arrays, stim, sd, steps = _problem(steps=10)
    n = len(arrays["threshold"])
    e = _engine(arrays, None, 1)
    with pytest.raises(ValueError, match="mat_step: ext must have one amplitude per neuron"):
        e.step(np.zeros(n - 1))
    e.add_stimulus(np.array([0, 1], np.int32), np.array([5, 6], np.int32), np.array([9.0, 9.0]))
    assert len(e.step(None)) == 0            # step 0: schedule ignored, nothing fires
    x = np.zeros(n)
    x[[3, 7]] = 9.0
    assert list(e.step(x)) == [3, 7]         # step 1: exactly ext
    e.simulate(1)                            # step 2 via the schedule: no entry for step 2
    s, q = e.raster()
    assert list(zip(s.tolist(), q.tolist()))[:2] == [(1, 3), (1, 7)]
    e.close()


@pytest.mark.parametrize("storage", [0, 1, 2])
@pytest.mark.parametrize("dmax", [1, 3])
def test_plasticity_switch_matches_reference(storage, dmax):
    """Plasticity off for steps 0-9 and 30-39, on otherwise, against the
    reference's own mat_step loop with apply_stdp skipped on the same steps
    (lower_delays first for delayed nets, the reference MAT path for delays).
    Initial weights outside [w_min, w_max] are clamped by the first
    apply_stdp, which here is step 10: raster and fp64 weights identical."""
    from oracle import bridge as B
    if not B.ref_available():
        pytest.skip("oracle/_ref not built")
    arrays, stim, sd, steps = _problem(n=150, dmax=dmax, wlo=-0.5, whi=1.5)
    mask = np.ones(steps, np.uint8)
    mask[0:10] = 0
    mask[30:40] = 0
    o = B.run_ref_mat_masked(arrays, steps, stim, sd, mask, lower=dmax > 1)
    on = B.run_ref_mat(arrays, steps, stim, sd, lower=dmax > 1)
    assert not np.array_equal(o["weights"], on["weights"])   # the switch matters for this net
    w0 = arrays["weight"][arrays["stdp"] == 1]
    assert (w0 < 0).any() and (w0 > 1).any()
    e = _engine(arrays, sd, storage, "f64")
    e.add_stimulus(*stim)
    t = 0
    for lo, hi, on_ in ((0, 10, False), (10, 30, True), (30, 40, False), (40, steps, True)):
        e.set_plasticity(on_)
        e.simulate(hi - lo)
        if hi == 10:   # nothing plastic has run yet: initial weights untouched, outside the bounds too
            assert np.array_equal(e.synapse_weights(), arrays["weight"])
        t = hi
    s, q = e.raster()
    assert np.array_equal(s, o["steps"]) and np.array_equal(q, o["neurons"])
    assert np.array_equal(e.synapse_weights(), o["weights"])
    assert close_rel(e.membrane(), o["membrane"])
    e.close()


def test_new_entry_points_error_contract():
    """Error behaviour of the round-2 entry points: wrong ext length
    (mat_step's message), plasticity toggles on a net without STDP (no-op),
    the weight census on sparse storage and delay relays on a partitioned
    engine (SN_ERR_UNSUPPORTED), and a 1-rank communicator after the first
    step (SN_ERR_LOGIC)."""
    import paper_2305_02510_b200 as sn
    arrays, stim, sd, steps = _problem(n=64, steps=10)
    e = _engine(arrays, None, 2)
    e.set_plasticity(False)
    e.set_plasticity(True)                        # no STDP configured: nothing to apply
    with pytest.raises(ValueError, match="mat_step: ext must have one amplitude per neuron"):
        e.step(np.zeros(65))
    with pytest.raises(NotImplementedError, match="dense weight storage"):
        e.weight_value_counts([1.0])
    e.close()
    from paper_2305_02510_b200.engine import MatEngine
    e = MatEngine(storage=1, precision="f64", persistent=False)
    e.add_neurons(arrays["threshold"], arrays["leak"], arrays["reset"], arrays["refractory"], arrays["axonal"])
    e.add_synapses(arrays["pre"], arrays["post"], arrays["weight"], arrays["delay"], arrays["stdp"])
    e.setup()
    e.simulate(1)
    with pytest.raises(RuntimeError, match="before its first step"):
        e.comm_init(sn.comm_unique_id(), 0, 1)
    e.close()
    e = _engine(arrays, None, 0)                  # the one-CTA whole-call loop cannot join a communicator
    with pytest.raises(RuntimeError, match="whole simulate calls in one kernel"):
        e.comm_init(sn.comm_unique_id(), 0, 1)
    e.close()
    a = dict(arrays, delay=np.full(len(arrays["pre"]), 90, np.int32))
    e = MatEngine(storage=1, rank=0, world=2)
    e.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
    e.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], a["stdp"])
    with pytest.raises(NotImplementedError, match="single-partition engines only"):
        e.setup()
    e.close()


@pytest.mark.parametrize("opts", [dict(storage=2, stream_io=True), dict(storage=1, stream_io=True, persistent=False),
                                  dict(storage=1, stream_io=False, persistent=False), dict(storage=0, stream_io=True),
                                  dict(storage=2, stream_io=True, use_graphs=False)],
                         ids=["sparse_io", "dense_io", "dense_noio", "tiny_io", "sparse_io_nograph"])
def test_simulate_raster_equals_simulate_then_raster(opts):
    """sn_simulate_raster (the events of exactly the call's steps, expanded
    chunk by chunk while later chunks run when stream_io is on) equals
    simulate + raster on the same engine configuration, across calls."""
    from paper_2305_02510_b200.engine import MatEngine
    arrays, stim, sd, steps = _problem(n=300, steps=90)

    def make():
        e = MatEngine(precision="f64", **opts)
        e.add_neurons(arrays["threshold"], arrays["leak"], arrays["reset"], arrays["refractory"], arrays["axonal"])
        e.add_synapses(arrays["pre"], arrays["post"], arrays["weight"], arrays["delay"], arrays["stdp"])
        e.set_stdp(*sd)
        e.setup()
        e.add_stimulus(*stim)
        return e

    a = make()
    a.simulate(37)
    a.simulate(steps - 37)
    s_ref, q_ref = a.raster()
    a.close()
    b = make()
    s1, q1 = b.simulate_raster(37)
    s2, q2 = b.simulate_raster(steps - 37)
    s_all, q_all = b.raster()
    b.close()
    assert len(s_ref) > 500
    assert np.array_equal(np.concatenate([s1, s2]), s_ref) and np.array_equal(np.concatenate([q1, q2]), q_ref)
    assert np.all(s1 < 37) and np.all(s2 >= 37)
    assert np.array_equal(s_all, s_ref) and np.array_equal(q_all, q_ref)
    # caller-owned output arrays, reused across calls (views of them come back)
    c = make()
    bufs = (np.full(300 * 60, -1, np.int32), np.full(300 * 60, -1, np.int32))
    s1, q1 = c.simulate_raster(37, out=bufs)
    s1, q1 = s1.copy(), q1.copy()
    s2, q2 = c.simulate_raster(steps - 37, out=bufs)
    c.close()
    assert np.shares_memory(s2, bufs[0]) and np.shares_memory(q2, bufs[1])
    assert np.array_equal(np.concatenate([s1, s2]), s_ref) and np.array_equal(np.concatenate([q1, q2]), q_ref)
    d = make()
    with pytest.raises(ValueError, match="int32"):
        d.simulate_raster(3, out=(np.zeros(900, np.int64), np.zeros(900, np.int64)))
    d.close()


def test_empty_network_runs_like_the_reference():
    """mat_run / abm_run accept a network with no neurons (no minimum size in
    mat_init, mat_engine.cpp:109-166): T empty steps, an empty raster; a
    stimulus entry is then out of range with the reference's message."""
    import paper_2305_02510_b200 as sn
    from oracle import bridge as B
    net = sn.NetworkDef()
    r = sn.mat_run(net, sn.SimulationConfig(steps=7))
    assert len(r.raster.events) == 0 and r.raster.step_count == 7 and r.raster.neuron_count == 0
    if B.ref_available():
        ref = B.run_ref_mat({"threshold": np.zeros(0), "leak": np.zeros(0), "reset": np.zeros(0),
                             "refractory": np.zeros(0, np.int32), "pre": [], "post": [], "weight": []}, 7)
        assert len(ref["steps"]) == 0
    from paper_2305_02510_b200.engine import MatEngine
    for mode in ("mat", "abm"):
        e = MatEngine(mode=mode, record_membrane=True)
        e.setup()
        e.simulate(3)
        assert len(e.step(None)) == 0
        s, q = e.raster()
        assert len(s) == 0 and len(e.membrane()) == 0 and e.membrane_trace().shape == (4, 0)
        assert e.stats()["spike_count"] == 0 and e.stats()["steps_done"] == 4
        with pytest.raises(ValueError, match="out of range"):
            e.add_stimulus(np.array([0], np.int32), np.array([0], np.int32), np.array([1.0]))
        e.close()
    with pytest.raises(ValueError, match=r"stimulus\[0\]: neuron id 0 out of range \(0 neurons\)"):
        sn.mat_run(net, sn.SimulationConfig(steps=3),
                   sn.StimulusSchedule([sn.StimulusEntry(0, 0, 1.0)]))


def test_cluster_loop_simulate_raster_in_launch_chunks():
    """The cluster loop (cfg2's plan) under sn_simulate_raster with stream_io
    runs a long call as 4 launches and expands each launch's rows while the
    next runs; the events equal simulate + raster of an engine without
    stream_io, across calls of different lengths."""
    from paper_2305_02510_b200.engine import MatEngine
    from paper_2305_02510_b200.netgen import scenario_stimulus

    def make(io):
        e = MatEngine(storage=1, stream_io=io)
        e.generate_erdos_renyi(1000, 1.0, 0, delay_max=8, delay_by_synapse_index=True)
        e.setup()
        e.add_stimulus(*scenario_stimulus(1000, 1300, 0).to_arrays())
        return e

    a = make(False)
    for k in (700, 300, 257):
        a.simulate(k)
    s_ref, q_ref = a.raster()
    assert a.stats()["sweep_kernel"] == 14
    a.close()
    b = make(True)
    parts = [b.simulate_raster(k) for k in (700, 300, 257)]
    assert b.stats()["sweep_kernel"] == 14
    b.close()
    s = np.concatenate([p[0] for p in parts])
    q = np.concatenate([p[1] for p in parts])
    assert len(s_ref) > 100000
    assert np.array_equal(s, s_ref) and np.array_equal(q, q_ref)
