"""Test fixtures mirroring the reference's proj/tests/support.hpp:16-104
(two_neuron_chain, kick, random_net, random_stim) bit-for-bit, plus small
helpers shared by the CPU and GPU suites."""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2305_02510_b200.model import (INFINITE_LEAK, NetworkDef, NeuronParams,  # noqa: E402
                                         StdpConfig, StimulusEntry, StimulusSchedule, SynapseDef)
from paper_2305_02510_b200.netgen import RandomStream, SequentialRng  # noqa: E402

NET_TAG = 0x746573746E6574   # support.hpp:41
STIM_TAG = 0x74657374737469  # support.hpp:84


def two_neuron_chain(weight=1.0, delay=1, threshold=1.0) -> NetworkDef:
    net = NetworkDef()
    net.neurons = [NeuronParams(threshold=threshold), NeuronParams(threshold=threshold)]
    net.synapses = [SynapseDef(0, 1, weight, delay, False)]
    return net


def kick(neuron=0, step=0, amplitude=2.0) -> StimulusSchedule:
    return StimulusSchedule([StimulusEntry(step, neuron, amplitude)])


def random_net(seed, min_neurons=2, max_neurons=20, edge_prob=0.3, max_delay=1, max_axonal=0,
               max_refractory=3, infinite_leaks=True) -> NetworkDef:
    """support.hpp:39-80: integer-valued random LIF net, self-loops allowed."""
    rng = SequentialRng(RandomStream(seed, NET_TAG))
    net = NetworkDef()
    n = min_neurons + rng.next_below(max_neurons - min_neurons + 1)
    for _ in range(n):
        p = NeuronParams()
        p.threshold = 1.0 + float(rng.next_below(3))
        p.leak = float(rng.next_below(3))
        if infinite_leaks and rng.next_below(8) == 0:
            p.leak = INFINITE_LEAK
        p.reset = float(rng.next_below(3)) - 1.0
        p.refractory = int(rng.next_below(max_refractory + 1))
        p.axonal_delay = int(rng.next_below(max_axonal + 1))
        net.neurons.append(p)
    weights = [-2.0, -1.0, 1.0, 2.0, 3.0]
    for i in range(n):
        for j in range(n):
            if rng.next_unit() < edge_prob:
                w = weights[rng.next_below(5)]
                d = 1 + int(rng.next_below(max_delay))
                net.synapses.append(SynapseDef(i, j, w, d, False))
    return net


def random_stim(seed, neurons, steps, entry_count) -> StimulusSchedule:
    """support.hpp:83-95."""
    rng = SequentialRng(RandomStream(seed, STIM_TAG))
    stim = StimulusSchedule()
    for _ in range(entry_count):
        step = int(rng.next_below(steps))
        neuron = int(rng.next_below(neurons))
        amp = 1.0 + float(rng.next_below(4))
        stim.entries.append(StimulusEntry(step, neuron, amp))
    return stim


def stdp_tuple(cfg: StdpConfig):
    return (cfg.window, np.array(cfg.a_plus, float), np.array(cfg.a_minus, float), cfg.w_min, cfg.w_max)


def single_tap(window, k, a_plus_k, a_minus_k=0.0) -> StdpConfig:
    """test_stdp.cpp:16-27."""
    ap = [0.0] * window
    am = [0.0] * window
    ap[k - 1] = a_plus_k
    am[k - 1] = a_minus_k
    return StdpConfig(window=window, a_plus=ap, a_minus=am, w_min=0.0, w_max=1.0)


def float_stdp_net(n, seed, p=1.0, w_lo=0.1, w_hi=0.9, thr=0.5):
    """Dense float-weight plastic net (weights uniform in [w_lo, w_hi])."""
    rs = RandomStream(seed, 0x666C6F6174)
    from paper_2305_02510_b200.netgen import erdos_renyi_arrays
    pre, post = erdos_renyi_arrays(n, p, seed)
    w = w_lo + (w_hi - w_lo) * rs.unit_np(np.arange(len(pre), dtype=np.uint64))
    return NetworkDef.from_arrays(threshold=np.full(n, thr), leak=np.zeros(n), reset=np.zeros(n),
                                  refractory=np.zeros(n, np.int32), pre=pre, post=post, weight=w,
                                  stdp=np.ones(len(pre), np.uint8))


def stim_arrays(stim: StimulusSchedule):
    return stim.to_arrays()


def fp32_weight_floor(steps, *weights) -> float:
    """Rigorous bound on how far an fp32-stored weight can drift from the
    reference's fp64 weight over `steps` STDP updates when every update is
    computed in fp64 and rounded to float once: each rounding adds at most
    half an ulp <= 2^-24 |w| and the clamp is 1-Lipschitz, so after the
    initial rounding and T updates |w32 - w64| <= (T + 1) 2^-24 max|w|."""
    m = max(float(np.max(np.abs(np.asarray(w, float)))) if np.size(w) else 0.0 for w in weights)
    return (steps + 1) * 2.0 ** -24 * m


def close_rel(a, b, rel=1e-5, abs_floor=1e-6):
    """|a-b| <= rel*|b| + abs_floor elementwise (north star: 1e-5 relative,
    absolute floor near 0 where weights clip to w_min)."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return np.all(np.abs(a - b) <= rel * np.abs(b) + abs_floor)
