"""lower_delays mirror (proj/src/lowering.cpp) against the reference's own
lowering tests (test_lowering.cpp) and, on the GPU, native delays vs the
lowered network through the same engine."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2305_02510_b200.lowering import (ProxyInfo, annotate_proxy_metadata, lower_delays,
                                            proxy_count)
from paper_2305_02510_b200.model import NetworkDef, NeuronParams, SynapseDef, validate_network
from support import random_net, two_neuron_chain


def test_delay3_chain_structure():  # test_lowering.cpp:15-40
    low = lower_delays(two_neuron_chain(1.0, 3))
    assert low.original_count == 2 and low.net.neuron_count() == 4
    assert low.proxy_map == [ProxyInfo(0, 1, 1), ProxyInfo(0, 1, 2)]
    for p in low.net.neurons[2:]:
        assert p.threshold == 0.0 and math.isinf(p.leak) and p.reset == 0.0 and p.refractory == 0
    assert [s.delay for s in low.net.synapses] == [1, 1, 1]
    assert [s.weight for s in low.net.synapses] == [1.0, 1.0, 1.0]
    assert validate_network(low.net) == []


def test_weight_and_stdp_on_last_hop_axonal_fold_and_counts():  # :50-110
    low = lower_delays(two_neuron_chain(5.0, 2))
    assert [s.weight for s in low.net.synapses] == [1.0, 5.0]
    net = two_neuron_chain(0.5, 3)
    net.synapses[0].stdp_enabled = True
    assert [s.stdp_enabled for s in lower_delays(net).net.synapses] == [False, False, True]
    net = NetworkDef()
    net.neurons = [NeuronParams(axonal_delay=2), NeuronParams(), NeuronParams()]
    net.synapses = [SynapseDef(0, 1, 1.0, 1), SynapseDef(0, 2, 1.0, 2)]
    low = lower_delays(net)
    assert len(low.proxy_map) == 5 and proxy_count(net) == 5
    assert all(p.axonal_delay == 0 for p in low.net.neurons)
    once = lower_delays(random_net(11, max_neurons=12, edge_prob=0.4, max_delay=5, max_axonal=2))
    twice = lower_delays(once.net)
    assert twice.proxy_map == [] and twice.net == once.net
    ann = annotate_proxy_metadata(lower_delays(two_neuron_chain(1.0, 3)))
    assert ann.metadata["original_count"] == "2" and ann.metadata["proxy_map"] == "[[0,1,1],[0,1,2]]"


@pytest.mark.gpu
def test_native_delays_equal_lowered_run():
    import paper_2305_02510_b200 as sn
    from support import random_stim
    for seed in range(300, 310):
        net = random_net(seed, max_neurons=15, edge_prob=0.35, max_delay=5, max_axonal=2)
        stim = random_stim(seed, net.neuron_count(), 120, 50)
        cfg = sn.SimulationConfig(steps=120)
        native = sn.mat_run(net, cfg, stim).raster
        low = lower_delays(net)
        lowered = sn.restrict_raster(sn.mat_run(low.net, cfg, stim).raster, low.original_count)
        assert sn.raster_equal(native, lowered), seed
