"""Agent-based (ABM) mode on the GPU engine: ``abm_run`` and the behaviour
registry, mirroring spikeforge's (reference proj/src/abm_engine.cpp:20-243,
Python bindings proj/python/src/bindings.cpp:157-186).

A behaviour the GPU can run is a stochastic LIF rule with a fire probability
``p``: above threshold the neuron fires iff the first unit draw of
``RandomStream(seed, 0x61626d2d6167656e, id, step)`` is below ``p``
(StochasticLifBehavior, abm_engine.cpp:28-39).  ``"lif"`` is ``p = 1`` (the
draw is always below 1, so the rule is the deterministic one,
abm_engine.cpp:22-26), ``"stochastic_lif"`` is ``p = 0.5`` (abm_engine.cpp:41),
and ``register_stochastic_lif(name, p)`` adds a named rule exactly as the
reference binding does (bindings.cpp:180-186).  Arbitrary C++ behaviour
subclasses have no GPU form; the Python API of the reference cannot create
them either.

Numerics follow AbmWorld::step: the synaptic input is summed from 0.0 in
ascending pre order (channels sorted by (pre, post), abm_engine.cpp:95-103),
the step's stimulus is added to it, and only then the leaked membrane:
``u = leak(v) + (pending + ext)``.  With ``exact_order=True`` and fp64
weights this is bit-exact; otherwise it is the fixed-order parallel sum.
"""
from __future__ import annotations

import threading
from typing import Dict, List, Optional

import numpy as np

from .engine import MatEngine
from .model import (NetworkDef, RunResult, SimulationConfig, SpikeRaster, StimulusSchedule,
                    validate_network, validate_stimulus)

_lock = threading.Lock()
_registry: Dict[str, float] = {"lif": 1.0, "stochastic_lif": 0.5}  # abm_engine.cpp:39-42


def _check_probability(p: float) -> float:
    p = float(p)
    if not (0.0 <= p <= 1.0):  # abm_engine.cpp:30-32
        raise ValueError("stochastic lif: fire probability must be in [0, 1]")
    return p


def register_stochastic_lif(name: str, fire_probability: float) -> None:
    """Register a named above-threshold-fires-with-probability-p rule
    (bindings.cpp:180-186; names are claimed once, abm_engine.cpp:49-55)."""
    p = _check_probability(fire_probability)
    with _lock:
        if name in _registry:
            raise ValueError(f'register_behavior: "{name}" is already registered')
        _registry[name] = p


def behavior_names() -> List[str]:
    """Registered behaviour names, sorted (BehaviorRegistry::names, abm_engine.cpp:63-70)."""
    with _lock:
        return sorted(_registry)


def find_behavior(name: str) -> Optional[float]:
    """Fire probability of a registered behaviour, or None."""
    with _lock:
        return _registry.get(name)


def fire_probabilities(net: NetworkDef) -> Optional[np.ndarray]:
    """Per-neuron fire probability of `net` (None when every neuron is "lif");
    unregistered names fail like the AbmWorld constructor (abm_engine.cpp:86-91)."""
    names = net.to_arrays().get("behavior")
    if names is None:
        return None
    out = np.ones(len(names), np.float64)
    for i, b in enumerate(names):
        p = find_behavior(b)
        if p is None:
            raise ValueError(f'abm world: neuron {i} uses unregistered behavior "{b}"')
        out[i] = p
    return None if np.all(out == 1.0) else out


def _world_checks(net: NetworkDef) -> Optional[np.ndarray]:
    """The AbmWorld constructor's checks (abm_engine.cpp:78-92), in order."""
    violations = validate_network(net)
    if violations:  # AbmWorld reports the first violation only (abm_engine.cpp:14-17)
        raise ValueError("abm world: " + violations[0])
    return fire_probabilities(net)


def abm_engine(net: NetworkDef, cfg: SimulationConfig, *, device: int = 0, storage: int = 0,
               precision: str = "f64", exact_order: bool = True, stream_io: bool = False,
               use_graphs: bool = True, rank: int = 0, world: int = 1) -> MatEngine:
    """An ABM-mode engine for `net` (AbmWorld construction, abm_engine.cpp:78-144)."""
    fp = _world_checks(net)
    a = net.to_arrays()
    eng = MatEngine(device=device, storage=int(storage), precision=precision,
                    exact_order=exact_order, record_membrane=cfg.record_membrane,
                    stream_io=stream_io, use_graphs=use_graphs, rank=rank, world=world, mode="abm")
    try:
        eng.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
        if a["pre"].shape[0]:
            eng.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], None)
        eng.set_seed(cfg.seed)
        if fp is not None:
            eng.set_fire_probability(fp)
        eng.setup()
    except Exception:
        eng.close()
        raise
    return eng


def abm_run(net: NetworkDef, cfg: SimulationConfig, stim: Optional[StimulusSchedule] = None, *,
            device: int = 0, storage: int = 0, precision: str = "f64", exact_order: bool = True,
            stream_io: bool = False, use_graphs: bool = True) -> RunResult:
    """T invocations of the two-phase agent step (abm_run, abm_engine.cpp:218-243):
    delays run natively, no plasticity (cfg.stdp is ignored as in the reference)."""
    if stim is None:
        stim = StimulusSchedule()
    if cfg.steps < 1:
        raise ValueError("abm_run: steps must be >= 1")
    _world_checks(net)  # (checked before any device work; abm_engine repeats it cheaply)
    n = net.neuron_count()
    bad = validate_stimulus(stim, n, cfg.steps)
    if bad:
        raise ValueError("abm_run: " + bad[0])
    eng = abm_engine(net, cfg, device=device, storage=storage, precision=precision,
                     exact_order=exact_order, stream_io=stream_io, use_graphs=use_graphs)
    try:
        if stim.entries:
            eng.add_stimulus(*stim.to_arrays())
        eng.simulate(cfg.steps)
        st, nr = eng.raster()
        result = RunResult(raster=SpikeRaster(neuron_count=n, step_count=cfg.steps,
                                              steps_array=st, neurons_array=nr))
        if cfg.record_membrane:
            result.membrane_trace = eng.membrane_trace().tolist()
        return result
    finally:
        eng.close()
