"""Reference-side drop-in proof: the reference's own pybind11 module
spikeforge._core (proj/python/src/bindings.cpp, compiled unmodified by
`make -C oracle pyref`) with its Python mat_run rerouted to the B200 engine
through integration/pybind/spikeforge_gpu.cpp -- the binding a spikeforge
maintainer would add.  The reference's own smoke tests
(proj/python/tests/test_smoke.py, copied into oracle/_ref/py at build time)
run against it, plus a differential of the CPU mat_run and mat_run_gpu on
random nets built with the reference's own types."""
from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PY = os.path.join(ROOT, "oracle", "_ref", "py")
needs_pyref = pytest.mark.skipif(not os.path.exists(os.path.join(REF_PY, "test_smoke_reference.py")),
                                 reason="oracle/_ref/py not built (make -C oracle pyref)")


def _modules():
    if REF_PY not in sys.path:
        sys.path.insert(0, REF_PY)
    import spikeforge as sf
    import spikeforge_gpu as g
    return sf, g


@needs_pyref
def test_reference_smoke_suite_on_the_gpu_binding(monkeypatch):
    sf, g = _modules()
    cpu_mat_run = sf.mat_run
    monkeypatch.setattr(sf, "mat_run", g.mat_run_gpu)
    spec = importlib.util.spec_from_file_location("test_smoke_reference", os.path.join(REF_PY, "test_smoke_reference.py"))
    smoke = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(smoke)
    tests = [n for n in dir(smoke) if n.startswith("test_")]
    assert {"test_chain_spikes_propagate", "test_backends_agree_on_random_net",
            "test_delay_lowering_preserves_dynamics"} <= set(tests)
    for name in tests:   # the mat cases run on the GPU; the file-format ones are unaffected
        getattr(smoke, name)()
    assert sf.mat_run is g.mat_run_gpu and cpu_mat_run is not g.mat_run_gpu


@needs_pyref
def test_reference_types_differential_cpu_vs_gpu():
    """Random float nets with STDP, refractory periods and infinite leaks,
    built with the reference's own classes: spikeforge.mat_run (CPU) and
    mat_run_gpu give identical rasters; membrane traces within fp32 weight
    storage rounding; reference error messages pass through unchanged."""
    sf, g = _modules()
    rng = np.random.default_rng(17)
    for seed in range(6):
        n = int(rng.integers(20, 120))
        net = sf.erdos_renyi(n, float(rng.choice([0.1, 0.3])), seed=seed)
        for i, q in enumerate(net.neurons):
            q.threshold = 1.0 + float(rng.integers(0, 3))
            q.leak = float("inf") if rng.random() < 0.1 else float(rng.integers(0, 2)) * 0.5
            q.refractory = int(rng.integers(0, 3))
        syn = list(net.synapses)
        for s in syn:
            s.weight = float(rng.choice([0.5, 1.0, 1.5, 2.0, -1.0]))
            s.stdp_enabled = bool(rng.random() < 0.5)
        net.synapses = syn
        cfg = sf.SimulationConfig()
        cfg.steps = 120
        cfg.record_membrane = True
        cfg.stdp = sf.StdpConfig.defaults()
        stim = sf.StimulusSchedule()
        stim.entries = [sf.StimulusEntry(int(t), int(j), 2.5) for t, j in
                        zip(rng.integers(0, 120, 4 * n), rng.integers(0, n, 4 * n))]
        a = sf.mat_run(net, cfg, stim)
        b = g.mat_run_gpu(net, cfg, stim)
        assert len(a.raster.events) > 50, seed
        assert sf.raster_equal(a.raster, b.raster), seed
        ta, tb = np.array(a.membrane_trace), np.array(b.membrane_trace)
        assert ta.shape == tb.shape == (120, n)
        assert np.allclose(tb, ta, rtol=1e-5, atol=1e-5), seed
    bad = sf.StimulusSchedule()
    bad.entries = [sf.StimulusEntry(200, 0, 1.0)]
    cfg = sf.SimulationConfig()
    cfg.steps = 10
    net = sf.erdos_renyi(5, 0.5, seed=1)
    with pytest.raises(ValueError) as e_cpu:
        sf.mat_run(net, cfg, bad)
    with pytest.raises(ValueError) as e_gpu:
        g.mat_run_gpu(net, cfg, bad)
    assert str(e_cpu.value) == str(e_gpu.value)
