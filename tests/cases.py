"""Named parity cases, each restating a reference test or known-answer case
(file:line cited).  Shared by tests/golden/make_golden.py (which records the
reference's outputs) and by the CPU/GPU parity suites."""
from __future__ import annotations

import numpy as np

from support import (kick, random_net, random_stim, single_tap, two_neuron_chain)
from paper_2305_02510_b200.model import (INFINITE_LEAK, NetworkDef, NeuronParams, StdpConfig,
                                         StimulusEntry, StimulusSchedule, SynapseDef)
from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays


class Case:
    def __init__(self, name, net, steps, stim=None, stdp=None, record=False, lower=False,
                 cite="", seed=0, fire_p=None):
        self.seed = seed        # SimulationConfig::seed (agent-based cases)
        self.fire_p = fire_p    # per-neuron fire probability (agent-based cases), None = all lif
        self.name = name
        self.net = net
        self.steps = steps
        self.stim = stim if stim is not None else StimulusSchedule()
        self.stdp = stdp
        self.record = record
        self.lower = lower      # the reference MAT path needs lower_delays first
        self.cite = cite

    def arrays(self):
        return self.net.to_arrays()

    def stim_arrays(self):
        return self.stim.to_arrays()

    def stdp_tuple(self):
        if self.stdp is None:
            return None
        s = self.stdp
        return (s.window, np.array(s.a_plus, float), np.array(s.a_minus, float), s.w_min, s.w_max)


def _one(thr=1.0, leak=0.0, refr=0):
    net = NetworkDef()
    net.neurons = [NeuronParams(threshold=thr, leak=leak, refractory=refr)]
    return net


def _sched(entries):
    return StimulusSchedule([StimulusEntry(*e) for e in entries])


def _stdp_pair(weight):
    net = two_neuron_chain(weight)
    net.synapses[0].stdp_enabled = True
    return net


def kat_cases():
    c = []
    # test_mat_engine.cpp
    c.append(Case("chain_thr05", two_neuron_chain(1.0, 1, 0.5), 3, _sched([(0, 0, 1.0)]),
                  cite="test_mat_engine.cpp:61-75"))
    c.append(Case("zero_weights_silent", NetworkDef.from_arrays(np.ones(4), np.zeros(4), np.zeros(4),
                                                                np.zeros(4, np.int32), [], [], []), 20,
                  cite="test_mat_engine.cpp:77-83"))
    c.append(Case("refractory3", _one(refr=3), 5, _sched([(t, 0, 2.0) for t in range(5)]),
                  cite="test_mat_engine.cpp:85-96"))
    c.append(Case("chain_raster", two_neuron_chain(2.0), 5, kick(), cite="test_mat_engine.cpp:98-102"))
    c.append(Case("membrane_trace", two_neuron_chain(0.5), 4, kick(0, 0, 0.75), record=True,
                  cite="test_mat_engine.cpp:109-116"))
    # test_oracle.cpp
    net = _one()
    net.synapses = [SynapseDef(0, 0, 2.0, 1, False)]
    c.append(Case("self_loop", net, 6, kick(), cite="test_oracle.cpp:20-26"))
    c.append(Case("no_stimulus", two_neuron_chain(), 10, cite="test_oracle.cpp:28-31"))
    c.append(Case("threshold_equal", _one(thr=2.0), 3, kick(0, 0, 2.0), cite="test_oracle.cpp:33-45"))
    c.append(Case("threshold_above", _one(thr=2.0), 3, kick(0, 0, 2.5), cite="test_oracle.cpp:33-45"))
    c.append(Case("delay3", two_neuron_chain(2.0, 3), 8, kick(), lower=True, cite="test_oracle.cpp:47-51"))
    net = two_neuron_chain(2.0, 1)
    net.neurons[0].axonal_delay = 2
    c.append(Case("axonal2", net, 8, kick(), lower=True, cite="test_oracle.cpp:53-58"))
    c.append(Case("refractory_resume", _one(refr=2), 6, _sched([(t, 0, 2.0) for t in range(6)]),
                  cite="test_oracle.cpp:60-69"))
    c.append(Case("refractory_hold", _one(refr=3), 6, _sched([(0, 0, 2.0), (1, 0, 0.6), (4, 0, 0.6)]),
                  cite="test_oracle.cpp:71-81"))
    c.append(Case("leak_decay", _one(leak=0.25), 4, _sched([(0, 0, 0.75), (1, 0, 0.5)]),
                  cite="test_oracle.cpp:83-97"))
    c.append(Case("leak_decay_fires", _one(leak=0.25), 4, _sched([(0, 0, 0.75), (1, 0, 0.5), (2, 0, 0.3)]),
                  cite="test_oracle.cpp:83-97"))
    c.append(Case("infinite_leak", _one(leak=INFINITE_LEAK), 3, _sched([(0, 0, 0.9), (1, 0, 0.9)]),
                  cite="test_oracle.cpp:99-107"))
    net = NetworkDef()
    net.neurons = [NeuronParams() for _ in range(3)]
    net.synapses = [SynapseDef(0, 2, 2.0, 1, False), SynapseDef(1, 2, -1.5, 1, False)]
    c.append(Case("negative_weight", net, 4, _sched([(0, 0, 2.0), (0, 1, 2.0)]), cite="test_oracle.cpp:109-119"))
    c.append(Case("horizon_drop", two_neuron_chain(2.0, 5), 3, kick(), lower=True, cite="test_oracle.cpp:121-125"))
    # test_lowering.cpp
    c.append(Case("lowered_delay3_thr05", two_neuron_chain(1.0, 3, 0.5), 6, kick(0, 0, 1.0), lower=True,
                  cite="test_lowering.cpp:115-123"))
    c.append(Case("subthreshold_proxy", two_neuron_chain(0.4, 3), 8, kick(), lower=True,
                  cite="test_lowering.cpp:125-132"))
    # test_stdp.cpp (ext per step -> stimulus entries)
    c.append(Case("stdp_pre_then_post", _stdp_pair(0.5), 3, _sched([(0, 0, 2.0), (2, 1, 2.0)]),
                  stdp=single_tap(4, 2, 0.1), cite="test_stdp.cpp:46-57"))
    c.append(Case("stdp_post_then_pre", _stdp_pair(0.5), 4, _sched([(0, 1, 2.0), (3, 0, 2.0)]),
                  stdp=single_tap(5, 3, 0.0, 0.2), cite="test_stdp.cpp:59-71"))
    c.append(Case("stdp_simultaneous", _stdp_pair(0.5), 1, _sched([(0, 0, 2.0), (0, 1, 2.0)]),
                  stdp=single_tap(4, 1, 0.25, 0.25), cite="test_stdp.cpp:73-80"))
    c.append(Case("stdp_quiet", _stdp_pair(0.5), 10, stdp=single_tap(4, 2, 0.1, 0.1), cite="test_stdp.cpp:82-89"))
    c.append(Case("stdp_clip_max", _stdp_pair(0.95), 3, _sched([(0, 0, 2.0), (2, 1, 2.0)]),
                  stdp=single_tap(4, 2, 0.1), cite="test_stdp.cpp:91-101"))
    c.append(Case("stdp_clip_min", _stdp_pair(0.05), 3, _sched([(0, 1, 2.0), (2, 0, 2.0)]),
                  stdp=single_tap(4, 2, 0.0, 0.3), cite="test_stdp.cpp:102-111"))
    cfg = single_tap(4, 1, 0.125)
    cfg.a_plus[1] = 0.0625
    c.append(Case("stdp_window_accumulates", _stdp_pair(0.25), 3,
                  _sched([(0, 0, 2.0), (1, 0, 2.0), (2, 1, 2.0)]), stdp=cfg, cite="test_stdp.cpp:114-127"))
    net = NetworkDef()
    net.neurons = [NeuronParams() for _ in range(3)]
    net.synapses = [SynapseDef(0, 1, 0.5, 1, True), SynapseDef(0, 2, 0.5, 1, False)]
    c.append(Case("stdp_only_enabled", net, 3, _sched([(0, 0, 2.0), (2, 1, 2.0), (2, 2, 2.0)]),
                  stdp=single_tap(4, 2, 0.1), cite="test_stdp.cpp:129-149"))
    # acceptance_main.cpp:212-249 criterion 5 single pairs
    for k in (1, 3, 5):
        net = NetworkDef()
        net.neurons = [NeuronParams(threshold=2.0, leak=INFINITE_LEAK) for _ in range(3)]
        net.synapses = [SynapseDef(0, 1, 0.5, 1, True), SynapseDef(2, 1, 0.25, 1, True)]
        entries = [(0, 0, 3.0), (k, 1, 3.0)]
        c.append(Case(f"crit5_pair_k{k}", net, k + 1, _sched(entries), stdp=StdpConfig.defaults(),
                      cite="acceptance_main.cpp:212-249"))
    return c


def random_unit_cases():
    """test_mat_engine.cpp:130-143: seeds 100..139, 200 steps, 60 entries."""
    out = []
    for seed in range(100, 140):
        net = random_net(seed)
        out.append(Case(f"rand_unit_{seed}", net, 200, random_stim(seed, net.neuron_count(), 200, 60)))
    return out


def random_delay_cases():
    """test_lowering.cpp:134-146: seeds 300..329, delays 1..5, axonal 0..2, 120 steps."""
    out = []
    for seed in range(300, 330):
        net = random_net(seed, max_neurons=15, edge_prob=0.35, max_delay=5, max_axonal=2)
        out.append(Case(f"rand_delay_{seed}", net, 120, random_stim(seed, net.neuron_count(), 120, 50),
                        lower=True))
    return out


def random_stdp_cases():
    """test_stdp.cpp:151-175 / 213-222 style: all synapses plastic, defaults."""
    out = []
    for seed in range(0, 20):
        net = random_net(seed)
        for s in net.synapses:
            s.stdp_enabled = True
        out.append(Case(f"rand_stdp_{seed}", net, 200, random_stim(seed, net.neuron_count(), 200, 80),
                        stdp=StdpConfig.defaults()))
    for seed in range(300, 315):
        net = random_net(seed, max_neurons=15, edge_prob=0.35, max_delay=5, max_axonal=2)
        for s in net.synapses:
            s.stdp_enabled = True
        out.append(Case(f"rand_stdp_delay_{seed}", net, 120, random_stim(seed, net.neuron_count(), 120, 50),
                        stdp=StdpConfig.defaults(), lower=True))
    return out


def periodic_drive(n, steps, inputs, period, amplitude, seed):
    """acceptance_main.cpp:70-86 (stream 0x6472697665)."""
    picks = RandomStream(seed, 0x6472697665)
    chosen = []
    draw = 0
    while len(chosen) < inputs:
        cand = picks.below_at(draw, n)
        draw += 1
        if cand not in chosen:
            chosen.append(cand)
    chosen.sort()
    return _sched([(t, j, amplitude) for t in range(0, steps, period) for j in chosen])


def crit1_cases():
    """acceptance_main.cpp:90-123: 24 delayed ER configs, 500 steps."""
    out = []
    for n in (10, 50, 100):
        for p in (0.25, 1.0):
            for net_seed in (11, 23):
                for sim_seed in (0, 1):
                    pre, post = erdos_renyi_arrays(n, p, net_seed)
                    d = 1 + RandomStream(net_seed, 0x64656C6179).below_np(np.arange(len(pre), dtype=np.uint64), 5)
                    net = NetworkDef.from_arrays(np.ones(n), np.zeros(n), np.zeros(n), np.zeros(n, np.int32),
                                                 pre, post, np.ones(len(pre)), delay=d.astype(np.int32))
                    out.append(Case(f"crit1_n{n}_p{p}_ns{net_seed}_ss{sim_seed}", net, 500,
                                    periodic_drive(n, 500, 3, 10, 2.0, sim_seed), lower=True))
    return out


def crit7_cases():
    """acceptance_main.cpp:409-436: ER(20, 0.6) with refractory 0..4, 400 steps."""
    out = []
    for seed in range(25):
        pre, post = erdos_renyi_arrays(20, 0.6, seed)
        refr = RandomStream(seed, 0x72656672).below_np(np.arange(20, dtype=np.uint64), 5).astype(np.int32)
        net = NetworkDef.from_arrays(np.ones(20), np.zeros(20), np.zeros(20), refr, pre, post, np.ones(len(pre)))
        out.append(Case(f"crit7_seed{seed}", net, 400, periodic_drive(20, 400, 3, 5, 2.0, seed)))
    return out


# ---------------------------------------------------------------------------
# Agent-based (abm_run) cases: each restates a test of
# proj/tests/test_abm_engine.cpp, plus float-weight nets (where the ABM
# summation order, leak(v) + (pending + ext), differs from MAT's) and
# heterogeneous stochastic behaviours.
def _fire_mix(n, seed, choices=(0.0, 0.25, 0.5, 0.8, 1.0), frac=0.5):
    rng = np.random.default_rng(seed)
    fp = np.where(rng.random(n) < frac, rng.choice(np.array(choices), n), 1.0)
    return fp.astype(np.float64)


def float_abm_net(n, p, seed, max_delay=4, max_axonal=1):
    """Float weights/thresholds/leaks so the summation order is observable."""
    rs = RandomStream(seed, 0x61626D666C74)
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    k = np.arange(m, dtype=np.uint64)
    w = -0.15 + 0.75 * rs.unit_np(k)
    d = (1 + rs.below_np(k + np.uint64(m), max_delay)).astype(np.int32)
    kn = np.arange(n, dtype=np.uint64) + np.uint64(3 * m)
    thr = 0.6 + 0.5 * rs.unit_np(kn)
    leak = 0.01 + 0.1 * rs.unit_np(kn + np.uint64(n))
    reset = -0.1 + 0.2 * rs.unit_np(kn + np.uint64(2 * n))
    refr = rs.below_np(kn + np.uint64(3 * n), 3).astype(np.int32)
    ax = rs.below_np(kn + np.uint64(4 * n), max_axonal + 1).astype(np.int32)
    return NetworkDef.from_arrays(threshold=thr, leak=leak, reset=reset, refractory=refr, pre=pre,
                                  post=post, weight=w, delay=d, axonal_delay=ax)


def float_stim(n, steps, count, seed):
    rs = RandomStream(seed, 0x61626D7374)
    k = np.arange(count, dtype=np.uint64)
    st = rs.below_np(k, steps).astype(np.int32)
    nr = rs.below_np(k + np.uint64(count), n).astype(np.int32)
    am = 0.2 + 1.3 * rs.unit_np(k + np.uint64(2 * count))
    return _sched([(int(a), int(b), float(c)) for a, b, c in zip(st, nr, am)])


def abm_cases():
    out = []
    c = "test_abm_engine.cpp"
    out.append(Case("abm_chain", two_neuron_chain(2.0), 5, kick(), cite=f"{c}:38-42"))
    out.append(Case("abm_delay3", two_neuron_chain(2.0, 3), 8, kick(), cite=f"{c}:44-48"))
    net = two_neuron_chain(2.0, 1)
    net.neurons[0].axonal_delay = 2
    out.append(Case("abm_axonal2", net, 8, kick(), cite=f"{c}:50-55"))
    out.append(Case("abm_same_step", two_neuron_chain(5.0), 3, kick(), cite=f"{c}:57-63"))
    net = NetworkDef()
    net.neurons = [NeuronParams() for _ in range(5)]
    out.append(Case("abm_two_phase", net, 1, _sched([(0, j, 2.0) for j in (0, 1, 3, 4)]),
                    cite=f"{c}:65-73"))
    for seed in range(500, 540, 3):
        net = random_net(seed)
        out.append(Case(f"abm_rand_{seed}", net, 150, random_stim(seed, net.neuron_count(), 150, 50),
                        cite=f"{c}:75-85"))
    for seed in range(600, 630, 3):
        net = random_net(seed, max_neurons=15, edge_prob=0.35, max_delay=5, max_axonal=2)
        out.append(Case(f"abm_delay_{seed}", net, 120, random_stim(seed, net.neuron_count(), 120, 50),
                        cite=f"{c}:87-98"))
    net = random_net(900)
    fp = np.ones(net.neuron_count())
    fp[::2] = 1.0  # "always_fires_when_above" = StochasticLif(1.0): identical to lif
    out.append(Case("abm_p1_degenerate", net, 100, random_stim(900, net.neuron_count(), 100, 40),
                    fire_p=fp, cite=f"{c}:100-111"))
    out.append(Case("abm_p0_never", two_neuron_chain(5.0), 10, kick(), fire_p=np.array([1.0, 0.0]),
                    cite=f"{c}:113-120"))
    drive = _sched([(t, 0, 2.0) for t in range(100)])
    for seed in (9, 10):
        out.append(Case(f"abm_seeded_{seed}", two_neuron_chain(2.0), 100, drive, seed=seed,
                        fire_p=np.array([1.0, 0.5]), cite=f"{c}:122-141"))
    for seed in range(40, 46):
        net = random_net(seed, max_neurons=30, edge_prob=0.3, max_delay=4, max_axonal=2)
        out.append(Case(f"abm_stoch_{seed}", net, 200, random_stim(seed, net.neuron_count(), 200, 150),
                        seed=seed * 1000 + 7, fire_p=_fire_mix(net.neuron_count(), seed),
                        record=True, cite="heterogeneous stochastic behaviours"))
    for seed, n, p in ((1, 40, 0.3), (2, 64, 0.2), (3, 100, 0.1), (4, 33, 1.0)):
        net = float_abm_net(n, p, seed)
        out.append(Case(f"abm_float_{seed}", net, 200, float_stim(n, 200, 6 * n, seed), seed=seed,
                        fire_p=_fire_mix(n, seed + 100, frac=0.3), record=True,
                        cite="float nets: leak(v) + (pending + ext) order"))
    return out
