"""Reference-facing entry points of the MAT path.

* ``mat_run(net, cfg, stim, storage)`` mirrors spikeforge's ``mat_run``
  (proj/src/mat_engine.cpp:252-287; Python binding bindings.cpp:150-156):
  same argument meaning, same error types and messages, same RunResult.
  Unlike the reference it accepts synaptic and axonal delays natively (the
  reference requires ``lower_delays`` first, mat_engine.cpp:114-131); the
  spike timing is that of ``mat_run(lower_delays(net))`` (lowering.cpp:22-59).
* ``NeuromorphicModel`` carries the north-star model API of SuperNeuro's MAT
  mode: ``create_neuron`` / ``create_synapse`` / ``add_spike`` / ``setup`` /
  ``simulate``.
"""
from __future__ import annotations

import math
from typing import List, Optional

import numpy as np

from . import _capi
from .engine import MatEngine
from .model import (NetworkDef, RunResult, SimulationConfig, SpikeRaster, StdpConfig,
                    StimulusEntry, StimulusSchedule, WeightStorage, throw_first,
                    validate_network, validate_stdp, validate_stimulus)


def _engine_for(net: NetworkDef, cfg: SimulationConfig, storage, device, precision,
                exact_order, stream_io, use_graphs):
    a = net.to_arrays()
    n = a["threshold"].shape[0]
    # mat_init's check order (mat_engine.cpp:112-132): network, behaviors, stdp
    if a.get("behavior") is not None:
        throw_first("mat_init", validate_network(net))
        for i, b in enumerate(a["behavior"]):
            if b != "lif":
                raise ValueError('mat_init: homogeneous backend supports "lif" only; '
                                 f'neuron {i} has behavior "{b}"')
    if cfg.stdp is not None:
        throw_first("mat_init", validate_stdp(cfg.stdp))
    eng = MatEngine(device=device, storage=int(storage), precision=precision,
                    exact_order=exact_order, record_membrane=cfg.record_membrane,
                    stream_io=stream_io, use_graphs=use_graphs)
    eng.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
    if a["pre"].shape[0]:
        eng.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], a["stdp"])
    if cfg.stdp is not None:
        s = cfg.stdp
        eng.set_stdp(s.window, s.a_plus, s.a_minus, s.w_min, s.w_max)
    eng.setup()
    return eng, n


def _raster_from(eng: MatEngine, n: int, steps: int) -> SpikeRaster:
    st, nr = eng.raster()
    return SpikeRaster(neuron_count=n, step_count=steps, steps_array=st, neurons_array=nr)


def mat_run(net: NetworkDef, cfg: SimulationConfig, stim: Optional[StimulusSchedule] = None,
            storage: WeightStorage = WeightStorage.Auto, *, device: int = 0,
            precision: str = "f32", exact_order: bool = False, stream_io: bool = False,
            use_graphs: bool = True, return_engine: bool = False):
    """T steps of the MAT step (+ STDP when cfg.stdp), collecting the raster."""
    if stim is None:
        stim = StimulusSchedule()
    if cfg.steps < 1:
        raise ValueError("mat_run: steps must be >= 1")
    eng, n = _engine_for(net, cfg, storage, device, precision, exact_order, stream_io, use_graphs)
    throw_first("mat_run", validate_stimulus(stim, n, cfg.steps))
    if stim.entries:
        eng.add_stimulus(*stim.to_arrays())
    eng.simulate(cfg.steps)
    result = RunResult(raster=_raster_from(eng, n, cfg.steps))
    if cfg.record_membrane:
        result.membrane_trace = eng.membrane_trace().tolist()
    if return_engine:
        return result, eng
    eng.close()
    return result


class NeuromorphicModel:
    """SuperNeuro MAT-mode model API (north star): build neuron by neuron and
    synapse by synapse, then ``setup()`` and ``simulate(T)``.

    Argument meaning follows spikeforge's NeuronParams / SynapseDef /
    StimulusEntry / StdpConfig (model.hpp:20-78).  ``simulate`` continues from
    the current step on repeated calls; spikes are reported as a RunResult.
    """

    def __init__(self, device: int = 0, storage: WeightStorage = WeightStorage.Auto,
                 precision: str = "f32", exact_order: bool = False):
        self._neurons: List[tuple] = []
        self._syn: List[tuple] = []
        self._spikes: List[tuple] = []
        self._device = device
        self._storage = storage
        self._precision = precision
        self._exact = exact_order
        self._engine: Optional[MatEngine] = None
        self._stdp: Optional[StdpConfig] = None
        self._record = False
        self._t = 0
        self._pushed_spikes = 0

    @property
    def num_neurons(self) -> int:
        return len(self._neurons)

    def create_neuron(self, threshold: float = 1.0, leak: float = 0.0, reset_state: float = 0.0,
                      refractory_period: int = 0, axonal_delay: int = 0) -> int:
        if self._engine is not None:
            raise RuntimeError("create_neuron: the network is fixed after setup()")
        self._neurons.append((float(threshold), float(leak), float(reset_state),
                              int(refractory_period), int(axonal_delay)))
        return len(self._neurons) - 1

    def create_synapse(self, pre_id: int, post_id: int, weight: float = 1.0, delay: int = 1,
                       enable_stdp: bool = False) -> int:
        if self._engine is not None:
            raise RuntimeError("create_synapse: the network is fixed after setup()")
        self._syn.append((int(pre_id), int(post_id), float(weight), int(delay), bool(enable_stdp)))
        return len(self._syn) - 1

    def add_spike(self, time: int, neuron_id: int, value: float = 1.0) -> None:
        self._spikes.append((int(time), int(neuron_id), float(value)))

    def setup(self, stdp: Optional[StdpConfig] = None, record_membrane: bool = False) -> None:
        net = NetworkDef()
        arr = np.array(self._neurons, dtype=np.float64).reshape(-1, 5)
        syn = np.array(self._syn, dtype=np.float64).reshape(-1, 5)
        net = NetworkDef.from_arrays(
            threshold=arr[:, 0], leak=arr[:, 1], reset=arr[:, 2], refractory=arr[:, 3].astype(np.int32),
            axonal_delay=arr[:, 4].astype(np.int32), pre=syn[:, 0].astype(np.int32),
            post=syn[:, 1].astype(np.int32), weight=syn[:, 2], delay=syn[:, 3].astype(np.int32),
            stdp=syn[:, 4].astype(np.uint8))
        self._stdp = stdp
        self._record = record_membrane
        cfg = SimulationConfig(steps=1, stdp=stdp, record_membrane=record_membrane)
        self._engine, _ = _engine_for(net, cfg, self._storage, self._device, self._precision,
                                      self._exact, False, True)

    def simulate(self, time_steps: int) -> RunResult:
        if self._engine is None:
            raise RuntimeError("simulate: call setup() first")
        if time_steps < 1:
            raise ValueError("mat_run: steps must be >= 1")
        new = self._spikes[self._pushed_spikes:]
        if new:
            st = np.array([s[0] for s in new], np.int32)
            nr = np.array([s[1] for s in new], np.int32)
            am = np.array([s[2] for s in new], np.float64)
            self._engine.add_stimulus(st, nr, am)
            self._pushed_spikes = len(self._spikes)
        self._engine.clear_raster()
        self._engine.simulate(time_steps)
        self._t += time_steps
        res = RunResult(raster=_raster_from(self._engine, self.num_neurons, time_steps))
        if self._record:
            res.membrane_trace = self._engine.membrane_trace()[-time_steps:].tolist()
        return res

    def membrane(self) -> np.ndarray:
        return self._engine.membrane()

    def weights(self) -> np.ndarray:
        """Current weight of every synapse, in create_synapse order."""
        return self._engine.synapse_weights()

    def close(self):
        if self._engine is not None:
            self._engine.close()
            self._engine = None
