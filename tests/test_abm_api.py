"""Host-side behaviour of the agent-based API (no GPU): the behaviour
registry and the error contract of abm_run, each against the reference's
wording (proj/src/abm_engine.cpp, proj/python/src/bindings.cpp:157-186)."""
from __future__ import annotations

import pytest

import paper_2305_02510_b200 as sn
from support import kick, two_neuron_chain


def test_builtin_behaviors_are_registered():
    names = sn.behavior_names()                 # test_abm_engine.cpp:17-23
    assert "lif" in names and "stochastic_lif" in names
    assert names == sorted(names)


def test_register_stochastic_lif_contract():
    sn.register_stochastic_lif("api_test_p03", 0.3)
    assert "api_test_p03" in sn.behavior_names()
    with pytest.raises(ValueError, match='"api_test_p03" is already registered'):
        sn.register_stochastic_lif("api_test_p03", 0.4)       # test_abm_engine.cpp:25-29
    with pytest.raises(ValueError, match="already registered"):
        sn.register_stochastic_lif("lif", 1.0)
    for bad in (-0.1, 1.5):                                    # test_abm_engine.cpp:143-146
        with pytest.raises(ValueError, match=r"fire probability must be in \[0, 1\]"):
            sn.register_stochastic_lif(f"api_bad_{bad}", bad)


def test_abm_run_errors_in_reference_order():
    cfg = sn.SimulationConfig(steps=5)
    with pytest.raises(ValueError, match="abm_run: steps must be >= 1"):
        sn.abm_run(two_neuron_chain(), sn.SimulationConfig(steps=0))
    net = two_neuron_chain()
    net.neurons[0].behavior = "martian"                        # test_abm_engine.cpp:31-36
    with pytest.raises(ValueError, match='abm world: neuron 0 uses unregistered behavior "martian"'):
        sn.abm_run(net, cfg)
    net = two_neuron_chain()
    net.synapses[0].post = 9
    net.synapses[0].delay = 0
    # only the first violation, no "(+N more)" suffix (abm_engine.cpp:14-17)
    with pytest.raises(ValueError) as e:
        sn.abm_run(net, cfg)
    assert str(e.value) == "abm world: synapses[0]: post id 9 out of range (2 neurons)"
    with pytest.raises(ValueError, match=r"abm_run: stimulus\[0\]: step 7 outside \[0, 5\)"):
        sn.abm_run(two_neuron_chain(), cfg, kick(0, 7))


def test_mat_run_rejects_stochastic_behaviours():
    net = two_neuron_chain()
    net.neurons[1].behavior = "stochastic_lif"
    with pytest.raises(ValueError, match='supports "lif" only; neuron 1 has behavior "stochastic_lif"'):
        sn.mat_run(net, sn.SimulationConfig(steps=3))
