"""Regenerates tests/golden/*.npz / scale.json from the REFERENCE's own code
(oracle/_ref/libspikeforge_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src).  Run in the build container (the reference tree
does not exist on the GPU box):

    python tests/golden/make_golden.py

Each case records the reference MAT path's raster, final membrane, final
synapse weights (list order) and, when asked, the membrane trace.  Delayed
cases use the reference MAT path for delays: lower_delays -> mat_run ->
restrict_raster (spikeforge_main.cpp:44-64).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import bridge as B  # noqa: E402
import cases as CS  # noqa: E402
from paper_2305_02510_b200.model import StdpConfig  # noqa: E402
from paper_2305_02510_b200.netgen import (DELAY_STREAM, RandomStream, erdos_renyi_arrays,  # noqa: E402
                                          scenario_stimulus)


def raster_digest(steps, neurons) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(steps, np.int32).tobytes())
    h.update(np.ascontiguousarray(neurons, np.int32).tobytes())
    return h.hexdigest()


def run_case(c):
    return B.run_ref_mat(c.arrays(), c.steps, c.stim_arrays(), c.stdp_tuple(), c.record, lower=c.lower)


def dump_suite(fname, cases):
    out = {}
    for c in cases:
        r = run_case(c)
        out[f"{c.name}/steps"] = r["steps"]
        out[f"{c.name}/neurons"] = r["neurons"]
        out[f"{c.name}/membrane"] = r["membrane"]
        out[f"{c.name}/weights"] = r.get("weights", np.zeros(0))
        if "membrane_trace" in r:
            out[f"{c.name}/trace"] = r["membrane_trace"]
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(f"{fname}: {len(cases)} cases")


def dump_abm_suite(fname, cases):
    """abm_run of the reference (stochastic behaviours registered through its
    own registry): raster, final membrane and, when asked, the trace."""
    out = {}
    for c in cases:
        r = B.run_ref_abm_full(c.arrays(), c.steps, c.stim_arrays(), seed=c.seed, fire_p=c.fire_p,
                               record_membrane=c.record)
        out[f"{c.name}/steps"] = r["steps"]
        out[f"{c.name}/neurons"] = r["neurons"]
        out[f"{c.name}/membrane"] = r["membrane"]
        if "membrane_trace" in r:
            out[f"{c.name}/trace"] = r["membrane_trace"]
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(f"{fname}: {len(cases)} cases")


def abm_scale_case():
    """ER(1000, 0.1, seed 3), delays 1..8 (synapse-index keyed), every other
    neuron "stochastic_lif", paper stimulus, 500 steps, run seed 77."""
    n, steps = 1000, 500
    arrays, stim = scenario(n, 0.1, 3, steps, 8)
    fp = np.ones(n)
    fp[1::2] = 0.5
    return arrays, stim, fp, steps, 77


def main_abm():
    B.build(ref=True)
    dump_abm_suite("abm.npz", CS.abm_cases())
    path = os.path.join(HERE, "scale.json")
    with open(path) as f:
        scale = json.load(f)
    arrays, stim, fp, steps, seed = abm_scale_case()
    t0 = time.time()
    r = B.run_ref_abm_full(arrays, steps, stim, seed=seed, fire_p=fp)
    scale["abm_er1000_stoch"] = {"n": 1000, "p": 0.1, "net_seed": 3, "delay_max": 8, "steps": steps,
                                 "run_seed": seed, "spikes": int(len(r["steps"])),
                                 "digest": raster_digest(r["steps"], r["neurons"]),
                                 "membrane_sum": float(np.sum(r["membrane"])), "ref_path": "abm_run",
                                 "ref_seconds": round(time.time() - t0, 3)}
    print("abm scale", scale["abm_er1000_stoch"])
    with open(path, "w") as f:
        json.dump(scale, f, indent=1)


def scenario(n, p, seed, steps, delay_max=1):
    pre, post = erdos_renyi_arrays(n, p, seed)
    arrays = {"threshold": np.ones(n), "leak": np.zeros(n), "reset": np.zeros(n),
              "refractory": np.zeros(n, np.int32), "axonal": np.zeros(n, np.int32),
              "pre": pre, "post": post, "weight": np.ones(len(pre)),
              "delay": np.ones(len(pre), np.int32), "stdp": np.zeros(len(pre), np.uint8)}
    if delay_max > 1:
        arrays["delay"] = (1 + RandomStream(seed, DELAY_STREAM).below_np(
            np.arange(len(pre), dtype=np.uint64), delay_max)).astype(np.int32)
    return arrays, scenario_stimulus(n, steps, seed).to_arrays()


def main():
    B.build(ref=True)
    dump_suite("kat.npz", CS.kat_cases())
    dump_suite("rand_unit.npz", CS.random_unit_cases())
    dump_suite("rand_delay.npz", CS.random_delay_cases())
    dump_suite("rand_stdp.npz", CS.random_stdp_cases())
    dump_suite("crit1.npz", CS.crit1_cases())
    dump_suite("crit7.npz", CS.crit7_cases())

    scale = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/libspikeforge_ref.so"}
    # netgen goldens (test_netgen.cpp:65-69, 124-134)
    scale["er100_025_counts"] = {str(s): int(len(B.ref_erdos_renyi(100, 0.25, s)[0])) for s in (0, 1, 42)}
    # scenario rasters (paper protocol, BASELINE cfg1 and the N=1000 p=1 row)
    for tag, (n, p, seed, steps, dmax) in {
        "cfg1_seed0": (100, 0.05, 0, 1000, 1),
        "cfg1_seed1": (100, 0.05, 1, 1000, 1),
        "cfg1_seed42": (100, 0.05, 42, 1000, 1),
        "n1000_p1_seed0": (1000, 1.0, 0, 1000, 1),
    }.items():
        arrays, stim = scenario(n, p, seed, steps, dmax)
        t0 = time.time()
        r = B.run_ref_mat_raster(arrays, steps, stim)
        scale[tag] = {"n": n, "p": p, "seed": seed, "steps": steps, "spikes": int(len(r["steps"])),
                      "digest": raster_digest(r["steps"], r["neurons"]), "ref_path": "mat_run",
                      "ref_seconds": round(time.time() - t0, 3)}
        print(tag, scale[tag])
    # cfg2: 1k all-to-all, delays 1..8 keyed by synapse index (acceptance_main.cpp:98-100)
    arrays, stim = scenario(1000, 1.0, 0, 1000, 8)
    t0 = time.time()
    r = B.run_ref_abm(arrays, 1000, stim)
    scale["cfg2_seed0"] = {"n": 1000, "p": 1.0, "seed": 0, "steps": 1000, "delay_max": 8,
                           "spikes": int(len(r["steps"])), "digest": raster_digest(r["steps"], r["neurons"]),
                           "ref_path": "abm_run (== oracle_run == mat_run(lower_delays))",
                           "ref_seconds": round(time.time() - t0, 3)}
    print("cfg2", scale["cfg2_seed0"])
    # dense STDP, defaults, N=1024, T=100
    n = 1024
    arrays, stim = scenario(n, 1.0, 0, 100)
    arrays["stdp"][:] = 1
    d = StdpConfig.defaults()
    sd = (d.window, np.array(d.a_plus), np.array(d.a_minus), d.w_min, d.w_max)
    t0 = time.time()
    r = B.run_ref_mat(arrays, 100, stim, sd)
    w = r["weights"]
    scale["stdp_n1024_seed0"] = {"n": n, "steps": 100, "spikes": int(len(r["steps"])),
                                 "digest": raster_digest(r["steps"], r["neurons"]),
                                 "weight_sum": float(np.sum(w)), "weight_min": float(w.min()),
                                 "weight_max": float(w.max()),
                                 "membrane_sum": float(np.sum(r["membrane"])),
                                 "ref_seconds": round(time.time() - t0, 3)}
    np.savez_compressed(os.path.join(HERE, "stdp_n1024.npz"), weights=w.astype(np.float64),
                        membrane=r["membrane"])
    print("stdp", scale["stdp_n1024_seed0"])
    with open(os.path.join(HERE, "scale.json"), "w") as f:
        json.dump(scale, f, indent=1)


def cfg4_entry(steps: int) -> dict:
    """BASELINE cfg4 at full size, truncated T: build_scenario(256000, 0.01,
    seed 0) with delays 1 + below_at(i*n + j, 16) on the "delay" stream (the
    engine's sn_generate_erdos_renyi pair-keyed delays), run by the
    reference's native-delay path abm_run (abm_engine.cpp:208-243; equal to
    mat_run(lower_delays) and oracle_run on every small golden).  Needs ~45 GB
    of host RAM and ~15 min: generated on the GPU box's host
    (python tests/golden/make_golden.py --cfg4 OUT.json), merged into
    scale.json by --merge-cfg4 OUT.json."""
    n, p, seed, dmax = 256000, 0.01, 0, 16
    t0 = time.time()
    r = B.ref_scenario_abm_raster(n, p, seed, steps, dmax, False)
    return {"n": n, "p": p, "seed": seed, "steps": steps, "delay_max": dmax, "delay_key": "pair",
            "synapses": r["synapses"], "spikes": int(len(r["steps"])),
            "digest": raster_digest(r["steps"], r["neurons"]),
            "per_step": np.bincount(r["steps"], minlength=steps).astype(int).tolist(),
            "ref_path": "abm_run (reference, oracle/_ref)", "ref_build_s": round(r["build_s"], 1),
            "ref_run_s": round(r["run_s"], 1), "ref_peak_rss_gb": round(r["peak_rss_gb"], 1),
            "ref_seconds": round(time.time() - t0, 1)}


def cfg3_entry(steps: int) -> dict:
    """BASELINE cfg3 at full size, truncated T: the reference's own mat_run
    on build_scenario(32000, 1.0, seed 0), all synapses plastic,
    StdpConfig::defaults(), Auto storage (CSR).  ~70 GB of host RAM, ~4 min
    plus ~4 s per step: generated on the GPU box's host
    (python tests/golden/make_golden.py --cfg3 OUT.json)."""
    t0 = time.time()
    r = B.ref_scenario_stdp_raster(32000, 1.0, 0, steps)
    return {"n": 32000, "p": 1.0, "seed": 0, "steps": steps, "stdp": "defaults", "synapses": r["synapses"],
            "spikes": int(len(r["steps"])), "digest": raster_digest(r["steps"], r["neurons"]),
            "per_step": np.bincount(r["steps"], minlength=steps).astype(int).tolist(),
            "ref_path": "mat_run (reference, oracle/_ref, Auto storage)", "ref_seconds": round(time.time() - t0, 1),
            "ref_peak_rss_gb": round(r["peak_rss_gb"], 1)}


if __name__ == "__main__":
    if "--cfg3" in sys.argv:     # full-size cfg3 golden (run on a host with >= 96 GB RAM)
        out = sys.argv[sys.argv.index("--cfg3") + 1]
        e = cfg3_entry(int(os.environ.get("CFG3_STEPS", "6")))
        with open(out, "w") as f:
            json.dump(e, f, indent=1)
        print(json.dumps(e))
        sys.exit(0)
    if "--merge-cfg3" in sys.argv:
        with open(sys.argv[sys.argv.index("--merge-cfg3") + 1]) as f:
            e = json.load(f)
        path = os.path.join(HERE, "scale.json")
        with open(path) as f:
            scale = json.load(f)
        scale[f"cfg3_seed0_T{e['steps']}"] = e
        with open(path, "w") as f:
            json.dump(scale, f, indent=1)
        sys.exit(0)
    if "--cfg4" in sys.argv:     # full-size cfg4 golden (run on a host with >= 64 GB RAM)
        out = sys.argv[sys.argv.index("--cfg4") + 1]
        steps = int(os.environ.get("CFG4_STEPS", "24"))
        B.build(ref=False)
        e = cfg4_entry(steps)
        with open(out, "w") as f:
            json.dump(e, f, indent=1)
        print(json.dumps({k: v for k, v in e.items() if k != "per_step"}))
        sys.exit(0)
    if "--merge-cfg4" in sys.argv:
        with open(sys.argv[sys.argv.index("--merge-cfg4") + 1]) as f:
            e = json.load(f)
        path = os.path.join(HERE, "scale.json")
        with open(path) as f:
            scale = json.load(f)
        scale[f"cfg4_seed0_T{e['steps']}"] = e
        with open(path, "w") as f:
            json.dump(scale, f, indent=1)
        sys.exit(0)
    if "--abm" in sys.argv:   # agent-based fixtures only (abm.npz + scale.json abm entries)
        main_abm()
    else:
        main()
        main_abm()
