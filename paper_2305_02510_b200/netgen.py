"""Seeded network + stimulus generation, bit-identical to the reference's
counter-based RNG (proj/include/spikeforge/rng.hpp:8-60) and generators
(proj/src/netgen.cpp:19-86).  Host-side numpy; the large configurations use
the on-device generator behind ``sn_generate_erdos_renyi`` instead.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

from .model import (NetworkDef, NeuronParams, SimulationConfig, StimulusEntry,
                    StimulusSchedule, SynapseDef)

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
EDGE_STREAM = 1      # kEdgeStream (netgen.cpp:15)
INPUT_STREAM = 2     # kInputStream (netgen.cpp:16)
DELAY_STREAM = 0x64656C6179  # "delay": acceptance_main.cpp:98 pattern


def mix64(z: int) -> int:
    """splitmix64 finalizer (rng.hpp:8-12)."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


class RandomStream:
    """RandomStream (rng.hpp:14-45): draw i = mix64(key + i * phi)."""

    def __init__(self, seed: int, stream: int, sub0: int = 0, sub1: int = 0):
        k = mix64((seed + GOLDEN) & M64)
        k = mix64(k ^ (stream & M64))
        k = mix64(k ^ (sub0 & M64))
        self.key = mix64(k ^ (sub1 & M64))

    def u64_at(self, index: int) -> int:
        return mix64((self.key + (index & M64) * GOLDEN) & M64)

    def unit_at(self, index: int) -> float:
        return (self.u64_at(index) >> 11) * (2.0 ** -53)

    def below_at(self, index: int, n: int) -> int:
        return (self.u64_at(index) * n) >> 64

    # vectorized forms (uint64 arrays of indices)
    def u64_np(self, index: np.ndarray) -> np.ndarray:
        idx = np.asarray(index, dtype=np.uint64)
        with np.errstate(over="ignore"):
            return _mix64_np(np.uint64(self.key) + idx * np.uint64(GOLDEN))

    def unit_np(self, index: np.ndarray) -> np.ndarray:
        return (self.u64_np(index) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def below_np(self, index: np.ndarray, n: int) -> np.ndarray:
        """floor(u * n / 2^64) for n < 2^32, via 32-bit halves."""
        assert 0 < n < (1 << 32)
        u = self.u64_np(index)
        nn = np.uint64(n)
        with np.errstate(over="ignore"):
            hi = (u >> np.uint64(32)) * nn
            lo = (u & np.uint64(0xFFFFFFFF)) * nn
            return (hi + (lo >> np.uint64(32))) >> np.uint64(32)


class SequentialRng:
    """SequentialRng (rng.hpp:47-60)."""

    def __init__(self, stream: RandomStream):
        self.stream = stream
        self.index = 0

    def next_u64(self) -> int:
        v = self.stream.u64_at(self.index)
        self.index += 1
        return v

    def next_unit(self) -> float:
        v = self.stream.unit_at(self.index)
        self.index += 1
        return v

    def next_below(self, n: int) -> int:
        v = self.stream.below_at(self.index, n)
        self.index += 1
        return v


def erdos_renyi_arrays(n: int, p: float, seed: int):
    """(pre, post) int32 arrays of erdos_renyi(n, p, seed) in list order
    (netgen.cpp:36-51: i ascending, j ascending, i != j, unit_at(i*n+j) < p)."""
    if n < 1:
        raise ValueError("erdos_renyi: n must be >= 1")
    if not (0.0 <= p <= 1.0):
        raise ValueError("erdos_renyi: p must be in [0, 1]")
    if p <= 0.0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    rs = RandomStream(seed, EDGE_STREAM)
    pres, posts = [], []
    j = np.arange(n, dtype=np.uint64)
    rows_per = max(1, (1 << 22) // n)
    for i0 in range(0, n, rows_per):
        i1 = min(n, i0 + rows_per)
        ii = np.arange(i0, i1, dtype=np.uint64)[:, None]
        pair = ii * np.uint64(n) + j[None, :]
        keep = rs.unit_np(pair) < p if p < 1.0 else np.ones(pair.shape, bool)
        keep[np.arange(i1 - i0), np.arange(i0, i1)] = False
        r, c = np.nonzero(keep)
        pres.append((r + i0).astype(np.int32))
        posts.append(c.astype(np.int32))
    return np.concatenate(pres), np.concatenate(posts)


def erdos_renyi(n: int, p: float, seed: int) -> NetworkDef:
    """erdos_renyi (netgen.cpp:19-54): thr 1, leak 0, reset 0, refr 0, w 1, delay 1."""
    pre, post = erdos_renyi_arrays(n, p, seed)
    return NetworkDef.from_arrays(
        threshold=np.ones(n), leak=np.zeros(n), reset=np.zeros(n),
        refractory=np.zeros(n, np.int32), pre=pre, post=post, weight=np.ones(len(pre)))


def delays_by_index(seed: int, keys: np.ndarray, delay_max: int,
                    stream: int = DELAY_STREAM) -> np.ndarray:
    """1 + RandomStream(seed, stream).below_at(key, delay_max) (acceptance_main.cpp:98-100)."""
    return (1 + RandomStream(seed, stream).below_np(keys, delay_max)).astype(np.int32)


@dataclass
class BenchScenario:  # netgen.hpp:11-20
    neuron_count: int = 100
    connection_probability: float = 0.25
    steps: int = 1000
    input_neuron_count: int = 3
    input_period: int = 10
    amplitude: float = 2.0
    seed: int = 0


@dataclass
class ScenarioBundle:  # netgen.hpp:22-27
    net: NetworkDef = None
    cfg: SimulationConfig = None
    stim: StimulusSchedule = None
    input_neurons: List[int] = field(default_factory=list)


def scenario_inputs(neuron_count: int, count: int, seed: int) -> List[int]:
    """build_scenario's input picks (netgen.cpp:71-81), ascending."""
    picks = RandomStream(seed, INPUT_STREAM)
    chosen: List[int] = []
    draw = 0
    while len(chosen) < count:
        cand = picks.below_at(draw, neuron_count)
        draw += 1
        if cand not in chosen:
            chosen.append(cand)
    return sorted(chosen)


def scenario_stimulus(neuron_count: int, steps: int, seed: int, count: int = 3,
                      period: int = 10, amplitude: float = 2.0) -> StimulusSchedule:
    inputs = scenario_inputs(neuron_count, count, seed)
    stim = StimulusSchedule()
    for t in range(0, steps, period):
        for j in inputs:
            stim.entries.append(StimulusEntry(t, j, amplitude))
    return stim


def build_scenario(s: BenchScenario) -> ScenarioBundle:
    """build_scenario (netgen.cpp:56-86)."""
    if s.neuron_count < s.input_neuron_count:
        raise ValueError(f"build_scenario: need at least {s.input_neuron_count} neurons, got {s.neuron_count}")
    if s.input_neuron_count < 0:
        raise ValueError("build_scenario: input_neuron_count must be >= 0")
    if s.steps < 1:
        raise ValueError("build_scenario: steps must be >= 1")
    if s.input_period < 1:
        raise ValueError("build_scenario: input_period must be >= 1")
    b = ScenarioBundle()
    b.net = erdos_renyi(s.neuron_count, s.connection_probability, s.seed)
    b.cfg = SimulationConfig(steps=s.steps, seed=s.seed)
    b.input_neurons = scenario_inputs(s.neuron_count, s.input_neuron_count, s.seed)
    b.stim = StimulusSchedule()
    for t in range(0, s.steps, s.input_period):
        for j in b.input_neurons:
            b.stim.entries.append(StimulusEntry(t, j, s.amplitude))
    return b
