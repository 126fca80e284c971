"""GPU parity of the agent-based mode (sn_options.mode = SN_MODE_ABM) against
the reference's abm_run (tests/golden/abm.npz, made by the reference's own
compiled code) and the C restatement oracle/abm_oracle.c.

Bar: rasters identical in every configuration; with fp64 weights and
exact_order (the abm_run default) membranes and traces bit-exact; with fp32
weights and the parallel sum, integer nets stay bit-exact and float nets are
within 1e-9 absolute (fp64 weights) or 1e-6 relative (fp32 weights) of the reference."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import cases as CS

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CONFIGS = {
    "auto_f64_exact": dict(storage=0, precision="f64", exact_order=True),       # k_tiny for small nets
    "dense_f64_exact": dict(storage=1, precision="f64", exact_order=True),
    "sparse_f64_exact": dict(storage=2, precision="f64", exact_order=True),
    "dense_f64": dict(storage=1, precision="f64", exact_order=False),
    "sparse_f64": dict(storage=2, precision="f64", exact_order=False),
    "dense_f32_stream": dict(storage=1, precision="f32", exact_order=False, stream_io=True),
    "auto_f32_stream": dict(storage=0, precision="f32", exact_order=False, stream_io=True),
}


def run_abm_engine(c, chunks=None, **cfg):
    from paper_2305_02510_b200.engine import MatEngine
    a = c.arrays()
    eng = MatEngine(record_membrane=c.record, mode="abm", **cfg)
    try:
        eng.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
        if len(a["pre"]):
            eng.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], None)
        eng.set_seed(c.seed)
        if c.fire_p is not None:
            eng.set_fire_probability(c.fire_p)
        eng.setup()
        st = c.stim_arrays()
        if len(st[0]):
            eng.add_stimulus(*st)
        for k in (chunks or [c.steps]):
            eng.simulate(k)
        steps, neurons = eng.raster()
        out = {"steps": steps, "neurons": neurons, "membrane": eng.membrane(), "stats": eng.stats()}
        if c.record:
            out["trace"] = eng.membrane_trace()
        return out
    finally:
        eng.close()


def _is_float(c):
    a = c.arrays()
    vals = [a["weight"], a["threshold"], a["reset"], c.stim_arrays()[2]]
    lk = a["leak"][np.isfinite(a["leak"])]
    return any(np.any(v != np.round(v)) for v in vals + [lk])


@pytest.mark.parametrize("cfg_name", list(CONFIGS))
def test_abm_engine_matches_reference_goldens(cfg_name):
    cfg = CONFIGS[cfg_name]
    g = np.load(os.path.join(GOLD, "abm.npz"))
    exact = cfg["precision"] == "f64" and cfg["exact_order"]
    kernels = set()
    for c in CS.abm_cases():
        r = run_abm_engine(c, **cfg)
        kernels.add(r["stats"]["sweep_kernel"])
        assert np.array_equal(r["steps"], g[f"{c.name}/steps"]), (c.name, cfg_name)
        assert np.array_equal(r["neurons"], g[f"{c.name}/neurons"]), (c.name, cfg_name)
        gm = g[f"{c.name}/membrane"]
        if exact or not _is_float(c):
            assert np.array_equal(r["membrane"], gm), (c.name, cfg_name)
            if c.record:
                assert np.array_equal(r["trace"], g[f"{c.name}/trace"]), (c.name, cfg_name)
        else:
            tol = dict(rtol=0, atol=1e-9) if cfg["precision"] == "f64" else dict(rtol=1e-6, atol=1e-6)
            assert np.allclose(r["membrane"], gm, **tol), (c.name, cfg_name)
    if cfg_name.startswith("auto"):
        assert 9 in kernels, "no case took the shared-memory k_tiny path"


def test_abm_chunked_calls_continue_the_agent_streams():
    """simulate(a); simulate(b) == simulate(a + b): the per-(agent, step)
    draws are keyed by the global step."""
    g = np.load(os.path.join(GOLD, "abm.npz"))
    for c in [c for c in CS.abm_cases() if c.name.startswith(("abm_stoch_", "abm_float_"))]:
        for storage in (0, 1, 2):
            r = run_abm_engine(c, chunks=[1, 17, c.steps - 18], storage=storage, precision="f64",
                               exact_order=True)
            assert np.array_equal(r["steps"], g[f"{c.name}/steps"]), (c.name, storage)
            assert np.array_equal(r["trace"], g[f"{c.name}/trace"]), (c.name, storage)


def _digest(steps, neurons):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(steps, np.int32).tobytes())
    h.update(np.ascontiguousarray(neurons, np.int32).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("storage", [1, 2])
@pytest.mark.parametrize("exact", [True, False])
def test_abm_scale_stochastic_er1000(storage, exact):
    """ER(1000, 0.1), delays 1..8, half the agents stochastic_lif, 500 steps:
    the reference abm_run raster (368,519 spikes) bit for bit."""
    from paper_2305_02510_b200.engine import MatEngine
    from golden_scale import abm_scale_problem
    with open(os.path.join(GOLD, "scale.json")) as f:
        e = json.load(f)["abm_er1000_stoch"]
    a, stim, fp, steps, seed = abm_scale_problem(e)
    eng = MatEngine(mode="abm", storage=storage, precision="f64", exact_order=exact)
    eng.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
    eng.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], None)
    eng.set_seed(seed)
    eng.set_fire_probability(fp)
    eng.setup()
    eng.add_stimulus(*stim)
    eng.simulate(steps)
    s, n = eng.raster()
    mem = eng.membrane()
    eng.close()
    assert len(s) == e["spikes"]
    assert _digest(s, n) == e["digest"]
    assert float(np.sum(mem)) == e["membrane_sum"]


@pytest.mark.parametrize("storage", [1, 2])
def test_cfg2_through_abm_mode(storage):
    """BASELINE cfg2's golden came from the reference's abm_run: the ABM mode
    on the on-device generated network reproduces it (998,057 spikes)."""
    from paper_2305_02510_b200.engine import MatEngine
    from paper_2305_02510_b200.netgen import scenario_stimulus
    with open(os.path.join(GOLD, "scale.json")) as f:
        e = json.load(f)["cfg2_seed0"]
    eng = MatEngine(mode="abm", storage=storage, precision="f32", exact_order=False)
    eng.generate_erdos_renyi(1000, 1.0, 0, delay_max=8, delay_by_synapse_index=True)
    eng.setup()
    eng.add_stimulus(*scenario_stimulus(1000, 1000, 0).to_arrays())
    eng.simulate(1000)
    s, n = eng.raster()
    eng.close()
    assert len(s) == e["spikes"] == 998057
    assert _digest(s, n) == e["digest"]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("storage", [1, 2])
def test_abm_partitions_emulated_on_one_gpu(world, storage):
    """Post partitions with the host-driven spike-word exchange: stochastic
    draws are keyed by the global agent id, so the merged raster equals the
    single engine's (and the reference's)."""
    from paper_2305_02510_b200.engine import MatEngine, partition_range
    g = np.load(os.path.join(GOLD, "abm.npz"))
    for c in [c for c in CS.abm_cases() if c.name.startswith(("abm_stoch_4", "abm_float_"))]:
        a = c.arrays()
        n = len(a["threshold"])
        engines = []
        for r in range(world):
            e = MatEngine(mode="abm", storage=storage, precision="f64", exact_order=True, rank=r, world=world)
            e.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
            if len(a["pre"]):
                e.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], None)
            e.set_seed(c.seed)
            if c.fire_p is not None:
                e.set_fire_probability(c.fire_p)
            e.setup()
            e.add_stimulus(*c.stim_arrays())
            engines.append(e)
        words_per = max(partition_range(n, 0, world)[1], 32) // 32
        for _ in range(c.steps):
            for e in engines:
                e.step_local()
            slices = [e.spike_words(words_per * world)[r * words_per:(r + 1) * words_per].copy()
                      for r, e in enumerate(engines)]
            for r, e in enumerate(engines):
                for q in range(world):
                    if q != r:
                        e.put_spike_words(q * words_per, slices[q])
            for e in engines:
                e.step_finish()
        steps = np.concatenate([e.raster()[0] for e in engines])
        neurons = np.concatenate([e.raster()[1] for e in engines])
        mem = np.concatenate([e.membrane() for e in engines])
        order = np.lexsort((neurons, steps))
        assert np.array_equal(steps[order], g[f"{c.name}/steps"]), c.name
        assert np.array_equal(neurons[order], g[f"{c.name}/neurons"]), c.name
        assert np.array_equal(mem, g[f"{c.name}/membrane"]), c.name
        for e in engines:
            e.close()


def test_abm_run_api_end_to_end():
    import paper_2305_02510_b200 as sn
    from support import kick, two_neuron_chain
    r = sn.abm_run(two_neuron_chain(2.0, 3), sn.SimulationConfig(steps=8), kick())
    assert r.raster.pairs() == [(0, 0), (3, 1)]               # test_abm_engine.cpp:44-48
    net = two_neuron_chain(2.0)
    net.neurons[1].behavior = "stochastic_lif"
    stim = sn.StimulusSchedule([sn.StimulusEntry(t, 0, 2.0) for t in range(100)])
    a = sn.abm_run(net, sn.SimulationConfig(steps=100, seed=9), stim)
    b = sn.abm_run(net, sn.SimulationConfig(steps=100, seed=9), stim)
    c = sn.abm_run(net, sn.SimulationConfig(steps=100, seed=10), stim)
    assert a.raster.pairs() == b.raster.pairs() != c.raster.pairs()   # :122-141
    g = np.load(os.path.join(GOLD, "abm.npz"))
    assert a.raster.pairs() == list(zip(g["abm_seeded_9/steps"].tolist(), g["abm_seeded_9/neurons"].tolist()))


def test_mode_errors():
    from paper_2305_02510_b200.engine import MatEngine
    from paper_2305_02510_b200.model import StdpConfig
    # MAT mode refuses stochastic neurons at setup (mat_engine.cpp:116-119)
    eng = MatEngine()
    eng.add_neurons([1.0, 1.0], [0.0, 0.0], [0.0, 0.0], [0, 0])
    eng.set_fire_probability([1.0, 0.5])
    with pytest.raises(ValueError, match='supports "lif" only; neuron 1'):
        eng.setup()
    eng.close()
    # fire probabilities are validated like StochasticLifBehavior's constructor
    eng = MatEngine(mode="abm")
    eng.add_neurons([1.0], [0.0], [0.0], [0])
    with pytest.raises(ValueError, match=r"fire probability must be in \[0, 1\]"):
        eng.set_fire_probability([1.5])
    with pytest.raises(ValueError, match="outside the 1 neurons"):
        eng.set_fire_probability([0.5, 0.5])
    # the agent-based engine has no plasticity
    d = StdpConfig.defaults()
    eng.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
    with pytest.raises(RuntimeError, match="no plasticity"):
        eng.setup()
    eng.close()
