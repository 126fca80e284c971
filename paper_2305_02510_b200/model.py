"""Model types of the MAT path, mirroring spikeforge's (reference
proj/include/spikeforge/model.hpp:20-138, exposed to Python by
proj/python/src/bindings.cpp:36-131) so code written against
``spikeforge`` runs unchanged against this package.

Large networks can skip the per-object lists: ``NetworkDef.from_arrays``
keeps structure-of-arrays numpy buffers that go straight through the C ABI.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

INFINITE_LEAK = math.inf  # kInfiniteLeak (model.hpp:16)


def is_infinite_leak(leak: float) -> bool:
    return math.isinf(leak)


class WeightStorage(enum.IntEnum):
    """WeightStorage (mat_engine.hpp:16): Auto / Dense / Sparse."""

    Auto = 0
    Dense = 1
    Sparse = 2


@dataclass
class NeuronParams:  # model.hpp:20-29
    threshold: float = 1.0
    leak: float = 0.0
    reset: float = 0.0
    refractory: int = 0
    axonal_delay: int = 0
    behavior: str = "lif"


@dataclass
class SynapseDef:  # model.hpp:31-39
    pre: int = 0
    post: int = 0
    weight: float = 1.0
    delay: int = 1
    stdp_enabled: bool = False

    def __init__(self, pre: int = 0, post: int = 0, weight: float = 1.0, delay: int = 1,
                 stdp: bool = False, stdp_enabled: Optional[bool] = None):
        self.pre = pre
        self.post = post
        self.weight = weight
        self.delay = delay
        self.stdp_enabled = bool(stdp if stdp_enabled is None else stdp_enabled)


class NetworkDef:  # model.hpp:43-51
    """neurons + synapses (+ metadata); optionally array-backed."""

    def __init__(self):
        self.neurons: List[NeuronParams] = []
        self.synapses: List[SynapseDef] = []
        self.metadata: Dict[str, str] = {}
        self._arrays: Optional[dict] = None

    @classmethod
    def from_arrays(cls, threshold, leak, reset, refractory, pre, post, weight,
                    delay=None, stdp=None, axonal_delay=None) -> "NetworkDef":
        net = cls()
        n = len(threshold)
        m = len(pre)
        net._arrays = {
            "threshold": np.ascontiguousarray(threshold, dtype=np.float64),
            "leak": np.ascontiguousarray(leak, dtype=np.float64),
            "reset": np.ascontiguousarray(reset, dtype=np.float64),
            "refractory": np.ascontiguousarray(refractory, dtype=np.int32),
            "axonal": np.ascontiguousarray(np.zeros(n) if axonal_delay is None else axonal_delay, dtype=np.int32),
            "pre": np.ascontiguousarray(pre, dtype=np.int32),
            "post": np.ascontiguousarray(post, dtype=np.int32),
            "weight": np.ascontiguousarray(weight, dtype=np.float64),
            "delay": np.ascontiguousarray(np.ones(m) if delay is None else delay, dtype=np.int32),
            "stdp": np.ascontiguousarray(np.zeros(m) if stdp is None else stdp, dtype=np.uint8),
            "behavior": None,
        }
        return net

    def neuron_count(self) -> int:
        if self._arrays is not None and not self.neurons:
            return int(self._arrays["threshold"].shape[0])
        return len(self.neurons)

    def synapse_count(self) -> int:
        if self._arrays is not None and not self.synapses:
            return int(self._arrays["pre"].shape[0])
        return len(self.synapses)

    def to_arrays(self) -> dict:
        """Structure-of-arrays view used by the C ABI (and by tests' oracles)."""
        if self._arrays is not None and not self.neurons and not self.synapses:
            return self._arrays
        nn = self.neurons
        ss = self.synapses
        return {
            "threshold": np.array([q.threshold for q in nn], dtype=np.float64),
            "leak": np.array([q.leak for q in nn], dtype=np.float64),
            "reset": np.array([q.reset for q in nn], dtype=np.float64),
            "refractory": np.array([q.refractory for q in nn], dtype=np.int32),
            "axonal": np.array([q.axonal_delay for q in nn], dtype=np.int32),
            "pre": np.array([s.pre for s in ss], dtype=np.int32),
            "post": np.array([s.post for s in ss], dtype=np.int32),
            "weight": np.array([s.weight for s in ss], dtype=np.float64),
            "delay": np.array([s.delay for s in ss], dtype=np.int32),
            "stdp": np.array([1 if s.stdp_enabled else 0 for s in ss], dtype=np.uint8),
            "behavior": [q.behavior for q in nn],
        }

    def __eq__(self, other) -> bool:
        if not isinstance(other, NetworkDef):
            return NotImplemented
        a, b = self.to_arrays(), other.to_arrays()
        for k in a:
            if k == "behavior":
                continue
            if not np.array_equal(a[k], b[k]):
                return False
        return self.metadata == other.metadata


@dataclass
class StimulusEntry:  # model.hpp:53-59
    step: int = 0
    neuron: int = 0
    amplitude: float = 0.0


@dataclass
class StimulusSchedule:  # model.hpp:61-65
    entries: List[StimulusEntry] = field(default_factory=list)

    def to_arrays(self):
        return (np.array([e.step for e in self.entries], dtype=np.int32),
                np.array([e.neuron for e in self.entries], dtype=np.int32),
                np.array([e.amplitude for e in self.entries], dtype=np.float64))


@dataclass
class StdpConfig:  # model.hpp:67-78
    window: int = 20
    a_plus: List[float] = field(default_factory=list)
    a_minus: List[float] = field(default_factory=list)
    w_min: float = 0.0
    w_max: float = 1.0

    @staticmethod
    def defaults() -> "StdpConfig":
        """StdpConfig::defaults() (model.cpp:10-22)."""
        w = 20
        return StdpConfig(
            window=w,
            a_plus=[0.01 * math.exp(-k / 5.0) for k in range(1, w + 1)],
            a_minus=[0.012 * math.exp(-k / 5.0) for k in range(1, w + 1)],
            w_min=0.0,
            w_max=1.0,
        )


@dataclass
class SimulationConfig:  # model.hpp:80-85
    steps: int = 1
    seed: int = 0
    stdp: Optional[StdpConfig] = None
    record_membrane: bool = False


@dataclass(order=True, frozen=True)
class SpikeEvent:  # model.hpp:87-92
    step: int = 0
    neuron: int = 0


class SpikeRaster:  # model.hpp:96-100
    """(step, neuron) events, ascending.  Built from the engine's int32 arrays;
    the SpikeEvent objects are materialised on first access of ``events``."""

    def __init__(self, events=None, neuron_count: int = 0, step_count: int = 0,
                 steps_array: Optional[np.ndarray] = None,
                 neurons_array: Optional[np.ndarray] = None):
        self._events = list(events) if events is not None else None
        self.neuron_count = neuron_count
        self.step_count = step_count
        if steps_array is None and self._events is not None:
            steps_array = np.array([e.step for e in self._events], dtype=np.int32)
            neurons_array = np.array([e.neuron for e in self._events], dtype=np.int32)
        self.steps_array = steps_array if steps_array is not None else np.zeros(0, np.int32)
        self.neurons_array = neurons_array if neurons_array is not None else np.zeros(0, np.int32)

    @property
    def events(self) -> List[SpikeEvent]:
        if self._events is None:
            self._events = [SpikeEvent(int(s), int(n)) for s, n in
                            zip(self.steps_array.tolist(), self.neurons_array.tolist())]
        return self._events

    @events.setter
    def events(self, ev):
        self._events = list(ev)
        self.steps_array = np.array([e.step for e in self._events], dtype=np.int32)
        self.neurons_array = np.array([e.neuron for e in self._events], dtype=np.int32)

    def __len__(self) -> int:
        return int(self.steps_array.shape[0])

    def pairs(self):
        return list(zip(self.steps_array.tolist(), self.neurons_array.tolist()))


@dataclass
class RunResult:  # model.hpp:102-105
    raster: SpikeRaster = field(default_factory=SpikeRaster)
    membrane_trace: List[List[float]] = field(default_factory=list)


def leak_toward(v: float, leak: float, reset: float) -> float:
    """leak_toward (model.hpp:127-138)."""
    d = v - reset
    if d > 0.0:
        stepped = d - leak
        return reset + (stepped if stepped > 0.0 else 0.0)
    if d < 0.0:
        stepped = d + leak
        return reset + (stepped if stepped < 0.0 else 0.0)
    return v


def _fmt_double(v: float) -> str:
    """std::ostream << double with default precision 6 (model.cpp:26-30)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    s = "%.6g" % v
    return s


def validate_network(net: NetworkDef) -> List[str]:
    """validate_network (model.cpp:34-84): one message per violation."""
    a = net.to_arrays()
    n = a["threshold"].shape[0]
    out: List[str] = []
    beh = a.get("behavior")
    for i in range(n):
        who = f"neurons[{i}]"
        if not math.isfinite(a["threshold"][i]):
            out.append(f"{who}: threshold must be finite")
        lk = float(a["leak"][i])
        if math.isnan(lk) or lk < 0.0:
            out.append(f"{who}: leak must be >= 0 or infinite (got {_fmt_double(lk)})")
        if not math.isfinite(a["reset"][i]):
            out.append(f"{who}: reset must be finite")
        if a["refractory"][i] < 0:
            out.append(f"{who}: refractory_period must be >= 0 (got {int(a['refractory'][i])})")
        if a["axonal"][i] < 0:
            out.append(f"{who}: axonal_delay must be >= 0 (got {int(a['axonal'][i])})")
        if beh is not None and beh[i] == "":
            out.append(f"{who}: behavior tag must be non-empty")
    seen = set()
    for s in range(a["pre"].shape[0]):
        who = f"synapses[{s}]"
        pre, post = int(a["pre"][s]), int(a["post"][s])
        pre_ok = 0 <= pre < n
        post_ok = 0 <= post < n
        if not pre_ok:
            out.append(f"{who}: pre id {pre} out of range ({n} neurons)")
        if not post_ok:
            out.append(f"{who}: post id {post} out of range ({n} neurons)")
        if not math.isfinite(a["weight"][s]):
            out.append(f"{who}: weight must be finite")
        if a["delay"][s] < 1:
            out.append(f"{who}: delay must be >= 1 (got {int(a['delay'][s])})")
        if pre_ok and post_ok:
            key = (pre, post)
            if key in seen:
                out.append(f"{who}: duplicate synapse ({pre}, {post})")
            seen.add(key)
    return out


def validate_stimulus(stim: StimulusSchedule, neuron_count: int, steps: int) -> List[str]:
    """validate_stimulus (model.cpp:86-102)."""
    out = []
    for i, e in enumerate(stim.entries):
        who = f"stimulus[{i}]"
        if e.step < 0 or e.step >= steps:
            out.append(f"{who}: step {e.step} outside [0, {steps})")
        if e.neuron < 0 or e.neuron >= neuron_count:
            out.append(f"{who}: neuron id {e.neuron} out of range ({neuron_count} neurons)")
        if not math.isfinite(e.amplitude):
            out.append(f"{who}: amplitude must be finite")
    return out


def validate_stdp(cfg: StdpConfig) -> List[str]:
    """validate_stdp (model.cpp:104-117)."""
    out = []
    if cfg.window < 1:
        out.append("stdp: window must be >= 1")
    if len(cfg.a_plus) != cfg.window:
        out.append("stdp: a_plus must have exactly `window` entries")
    if len(cfg.a_minus) != cfg.window:
        out.append("stdp: a_minus must have exactly `window` entries")
    for a in cfg.a_plus:
        if not (a >= 0.0):
            out.append("stdp: a_plus entries must be >= 0")
            break
    for a in cfg.a_minus:
        if not (a >= 0.0):
            out.append("stdp: a_minus entries must be >= 0")
            break
    if not (cfg.w_min <= cfg.w_max):
        out.append("stdp: w_min must be <= w_max")
    return out


def throw_first(where: str, violations: List[str]) -> None:
    """throw_first (mat_engine.cpp:15-21) as ValueError."""
    if not violations:
        return
    msg = f"{where}: {violations[0]}"
    if len(violations) > 1:
        msg += f" (+{len(violations) - 1} more)"
    raise ValueError(msg)


def raster_equal(a: SpikeRaster, b: SpikeRaster, restrict_to=None) -> bool:
    """raster_equal (model.cpp:119-139)."""
    if restrict_to is None:
        return (np.array_equal(a.steps_array, b.steps_array)
                and np.array_equal(a.neurons_array, b.neurons_array))
    keep = np.array(sorted(set(restrict_to)), dtype=np.int64)
    ka = np.isin(a.neurons_array, keep)
    kb = np.isin(b.neurons_array, keep)
    return (np.array_equal(a.steps_array[ka], b.steps_array[kb])
            and np.array_equal(a.neurons_array[ka], b.neurons_array[kb]))


def restrict_raster(r: SpikeRaster, neuron_limit: int) -> SpikeRaster:
    """restrict_raster (model.cpp:141-151)."""
    keep = r.neurons_array < neuron_limit
    return SpikeRaster(neuron_count=neuron_limit, step_count=r.step_count,
                       steps_array=r.steps_array[keep], neurons_array=r.neurons_array[keep])
