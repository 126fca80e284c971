"""Wire formats: the Python mirror of io.cpp is byte-identical
to the reference's own serializers (oracle/_ref built with io.cpp) and parses
what they write; committed fixtures cover the box without the reference."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from oracle import bridge as B
from paper_2305_02510_b200 import io as fio
from paper_2305_02510_b200.model import StdpConfig, StimulusEntry, StimulusSchedule
from support import random_net, random_stim, two_neuron_chain

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
needs_ref_io = pytest.mark.skipif(not B.ref_has_io(), reason="oracle/_ref built without io.cpp")


@needs_ref_io
def test_serialize_network_byte_identical():
    for seed in range(40):
        net = random_net(seed, max_neurons=12, max_delay=5, max_axonal=2)
        for i, s in enumerate(net.synapses):
            s.stdp_enabled = (i % 3 == 0)
            s.weight = s.weight * (0.37 if i % 2 else 1.0)
        mine = fio.serialize_network(net)
        assert mine == B.ref_serialize_network(net.to_arrays()), seed
        # the reference parses ours and writes the same bytes back
        assert B.ref_roundtrip_network(mine) == mine


@needs_ref_io
def test_raster_stimulus_stdp_byte_identical():
    rng = np.random.default_rng(3)
    for k in range(20):
        ev = sorted({(int(rng.integers(0, 300)), int(rng.integers(0, 50))) for _ in range(int(rng.integers(0, 200)))})
        steps = np.array([e[0] for e in ev], np.int32)
        neurons = np.array([e[1] for e in ev], np.int32)
        from paper_2305_02510_b200.model import SpikeRaster
        r = SpikeRaster(steps_array=steps, neurons_array=neurons)
        assert fio.write_raster(r) == B.ref_write_raster(steps, neurons)
    for seed in range(10):
        stim = random_stim(seed, 20, 100, 30)
        stim.entries.append(StimulusEntry(5, 1, 0.1))
        stim.entries.append(StimulusEntry(7, 2, 1e-7))
        stim.entries.append(StimulusEntry(9, 3, 12345.678))
        assert fio.write_stimulus(stim) == B.ref_write_stimulus(stim.to_arrays())
    d = StdpConfig.defaults()
    assert fio.serialize_stdp(d) == B.ref_serialize_stdp((d.window, np.array(d.a_plus), np.array(d.a_minus),
                                                          d.w_min, d.w_max))


def test_round_trips_and_errors():
    for seed in range(30):   # acceptance criterion 8 pattern (acceptance_main.cpp:440-480)
        net = random_net(seed, max_neurons=12, max_delay=5, max_axonal=2)
        net.metadata["case"] = str(seed)
        if net.synapses:
            net.synapses[0].stdp_enabled = True
        back = fio.parse_network(fio.serialize_network(net))
        assert back == net
    stim = random_stim(1, 10, 50, 20)
    assert fio.parse_stimulus(fio.write_stimulus(stim)) == stim
    d = StdpConfig.defaults()
    assert fio.parse_stdp(fio.serialize_stdp(d)) == d
    with pytest.raises(fio.FormatError, match="unsupported version"):
        fio.parse_network('{"version": 2, "neurons": [], "synapses": []}')
    with pytest.raises(fio.FormatError, match="strictly increasing"):
        fio.parse_raster("step,neuron_id\n1,2\n1,2\n")
    with pytest.raises(fio.FormatError, match="out of range"):
        fio.parse_network('{"version": 1, "neurons": [], "synapses": [{"pre": 0, "post": 1, "weight": 1, "delay": 1}]}')
    net = two_neuron_chain()
    net.neurons[0].leak = math.inf
    assert '"leak": "inf"' in fio.serialize_network(net)
    assert math.isinf(fio.parse_network(fio.serialize_network(net)).neurons[0].leak)


def test_committed_fixture_bytes():
    """Reference-written files (tests/golden/io_*) parse and re-serialise identically."""
    with open(os.path.join(GOLD, "io_network.json")) as f:
        text = f.read()
    assert fio.serialize_network(fio.parse_network(text)) == text
    with open(os.path.join(GOLD, "io_raster.csv")) as f:
        rt = f.read()
    assert fio.write_raster(fio.parse_raster(rt)) == rt


def test_shortest_matches_std_to_chars():
    """io.cpp:17-21 renders numbers with std::to_chars(double): shortest
    round-trip digits, fixed or scientific, whichever is shorter (fixed on a
    tie).  tests/golden/to_chars.txt holds 4,000+ values rendered by libstdc++
    (generator: tests/golden/to_chars_gen.cpp)."""
    with open(os.path.join(GOLD, "to_chars.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip()]
    assert len(rows) > 4000
    bad = [(h, ref, fio._shortest(float.fromhex(h))) for h, ref in rows if fio._shortest(float.fromhex(h)) != ref]
    assert not bad, bad[:5]
    for v, s in ((1e-4, "1e-04"), (2e-4, "2e-04"), (1e5, "1e+05"), (1e6, "1e+06"), (1e15, "1e+15"),
                 (0.001, "0.001"), (2.0, "2"), (123456.0, "123456")):
        assert fio._shortest(v) == s


@needs_ref_io
def test_stimulus_small_and_large_amplitudes_byte_identical():
    amps = [1e-4, 2e-4, 1e5, 1e6, 1e15, 0.001, 2.0, -3.5e-9, 531527556293501632.0]
    stim = StimulusSchedule([StimulusEntry(i, i % 3, a) for i, a in enumerate(amps)])
    assert fio.write_stimulus(stim) == B.ref_write_stimulus(stim.to_arrays())
