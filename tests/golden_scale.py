"""Rebuilds the scale-golden problems (scenario nets of tests/golden/scale.json)
from their parameters: build_scenario (netgen.cpp:56-86), optional delays
keyed by synapse index (acceptance_main.cpp:98-100) and all-plastic STDP."""
from __future__ import annotations

import numpy as np

from paper_2305_02510_b200.model import StdpConfig
from paper_2305_02510_b200.netgen import (DELAY_STREAM, RandomStream, erdos_renyi_arrays,
                                          scenario_stimulus)


def scenario_problem(entry: dict):
    n, p, seed, steps = entry["n"], entry.get("p", 1.0), entry.get("seed", 0), entry["steps"]
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    arrays = {"threshold": np.ones(n), "leak": np.zeros(n), "reset": np.zeros(n),
              "refractory": np.zeros(n, np.int32), "axonal": np.zeros(n, np.int32),
              "pre": pre, "post": post, "weight": np.ones(m),
              "delay": np.ones(m, np.int32), "stdp": np.zeros(m, np.uint8)}
    dmax = entry.get("delay_max", 1)
    if dmax > 1:
        arrays["delay"] = (1 + RandomStream(seed, DELAY_STREAM).below_np(
            np.arange(m, dtype=np.uint64), dmax)).astype(np.int32)
    stdp = None
    if "weight_sum" in entry:
        arrays["stdp"][:] = 1
        d = StdpConfig.defaults()
        stdp = (d.window, np.array(d.a_plus), np.array(d.a_minus), d.w_min, d.w_max)
    stim = scenario_stimulus(n, steps, seed).to_arrays()
    return arrays, stim, stdp, steps


def abm_scale_problem(entry: dict):
    """scale.json "abm_er1000_stoch" (tests/golden/make_golden.py abm_scale_case):
    ER(n, p, net_seed) with synapse-index keyed delays, every other neuron
    "stochastic_lif" (p = 0.5), paper stimulus, run seed `run_seed`."""
    arrays, stim, _, steps = scenario_problem({"n": entry["n"], "p": entry["p"], "seed": entry["net_seed"],
                                               "steps": entry["steps"], "delay_max": entry["delay_max"]})
    fp = np.ones(entry["n"])
    fp[1::2] = 0.5
    return arrays, stim, fp, steps, entry["run_seed"]
