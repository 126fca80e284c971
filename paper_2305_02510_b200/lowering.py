"""Delay lowering, mirroring spikeforge (proj/src/lowering.cpp:22-86,
lowering.hpp:10-40) so code that lowers before calling mat_run keeps
working.  The engine itself never needs it: delays and axonal delays are
simulated natively with exactly this timing, without proxy neurons."""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

from .model import NetworkDef, NeuronParams, SynapseDef, validate_network


@dataclass(frozen=True)
class ProxyInfo:  # lowering.hpp:10-18
    pre: int = 0
    post: int = 0
    position: int = 0


@dataclass
class LoweredNetwork:  # lowering.hpp:20-31
    net: NetworkDef = None
    original_count: int = 0
    proxy_map: List[ProxyInfo] = field(default_factory=list)

    def proxy_id_base(self) -> int:
        return self.original_count


def _proxy_params() -> NeuronParams:  # lowering.cpp:9-18
    return NeuronParams(threshold=0.0, leak=math.inf, reset=0.0, refractory=0, axonal_delay=0,
                        behavior="lif")


def _lists(net: NetworkDef) -> NetworkDef:
    """Object-list view of an (optionally array-backed) network."""
    if net.neurons or net.synapses or net._arrays is None:
        return net
    a = net.to_arrays()
    out = NetworkDef()
    out.metadata = dict(net.metadata)
    out.neurons = [NeuronParams(float(a["threshold"][i]), float(a["leak"][i]), float(a["reset"][i]),
                                int(a["refractory"][i]), int(a["axonal"][i]))
                   for i in range(len(a["threshold"]))]
    out.synapses = [SynapseDef(int(a["pre"][s]), int(a["post"][s]), float(a["weight"][s]), int(a["delay"][s]),
                               bool(a["stdp"][s])) for s in range(len(a["pre"]))]
    return out


def lower_delays(net: NetworkDef) -> LoweredNetwork:
    """lower_delays (lowering.cpp:22-59): each synapse of effective delay d > 1
    becomes a chain of d-1 threshold-0, infinite-leak proxies; the weight and
    the stdp flag ride the last hop."""
    bad = validate_network(net)
    if bad:
        raise ValueError(f"lower_delays: invalid network: {bad[0]}")
    src = _lists(net)
    out = LoweredNetwork(net=NetworkDef(), original_count=len(src.neurons))
    out.net.metadata = dict(src.metadata)
    for p in src.neurons:
        out.net.neurons.append(NeuronParams(p.threshold, p.leak, p.reset, p.refractory, 0, p.behavior))
    for syn in src.synapses:
        d = syn.delay + src.neurons[syn.pre].axonal_delay
        if d == 1:
            out.net.synapses.append(SynapseDef(syn.pre, syn.post, syn.weight, 1, syn.stdp_enabled))
            continue
        hop = syn.pre
        for k in range(1, d):
            pid = len(out.net.neurons)
            out.net.neurons.append(_proxy_params())
            out.proxy_map.append(ProxyInfo(syn.pre, syn.post, k))
            out.net.synapses.append(SynapseDef(hop, pid, 1.0, 1, False))
            hop = pid
        out.net.synapses.append(SynapseDef(hop, syn.post, syn.weight, 1, syn.stdp_enabled))
    return out


def proxy_count(net: NetworkDef) -> int:
    """proxy_count (lowering.cpp:78-86)."""
    bad = validate_network(net)
    if bad:
        raise ValueError(f"proxy_count: invalid network: {bad[0]}")
    a = net.to_arrays()
    return int(sum(int(a["delay"][s]) + int(a["axonal"][a["pre"][s]]) - 1 for s in range(len(a["pre"]))))


def annotate_proxy_metadata(lowered: LoweredNetwork) -> NetworkDef:
    """annotate_proxy_metadata (lowering.cpp:61-76)."""
    net = NetworkDef()
    net.neurons = list(lowered.net.neurons)
    net.synapses = list(lowered.net.synapses)
    net.metadata = dict(lowered.net.metadata)
    net.metadata["original_count"] = str(lowered.original_count)
    net.metadata["proxy_map"] = "[" + ",".join(f"[{p.pre},{p.post},{p.position}]" for p in lowered.proxy_map) + "]"
    return net
