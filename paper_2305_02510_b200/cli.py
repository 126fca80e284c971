"""Command line front end mirroring the reference CLI for the MAT path
(proj/tools/spikeforge_main.cpp): ``run``, ``gen``, ``compare`` and ``bench``
with GPU backends.  Exit codes as the reference: 0 ok, 1 diverged, 2 error
(spikeforge_main.cpp:26-27, 319-328).

  python -m paper_2305_02510_b200 run --network net.json --stimulus stim.csv \\
         --steps 1000 [--backend gpu|gpu-sparse|gpu-exact|gpu-abm] [--stdp stdp.json] [--out raster.csv]

Backends: ``gpu`` (Auto storage, fp32 weights), ``gpu-dense`` / ``gpu-sparse``
(forced storage), ``gpu-exact`` (fp64 weights + ascending-pre order: bit-exact
with the reference mat path on float nets).  ``mat`` is accepted as an alias of
``gpu``.  ``gpu-abm`` (alias ``abm``) runs the agent-based mode (abm_run
semantics: heterogeneous/stochastic behaviours, the run seed, no plasticity;
fp64 + ascending order, bit-exact with the reference abm backend) and
``gpu-abm-fast`` the same with fp32 weights and the parallel sum.
Delays need no lowering on any backend.  ``compare --against FILE``
checks a run against a raster CSV produced by the reference CLI.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from typing import List, Optional

import numpy as np

from . import io as fio
from .abm import abm_run
from .api import mat_run
from .model import SimulationConfig, SpikeRaster, StimulusSchedule, WeightStorage
from .netgen import BenchScenario, build_scenario, erdos_renyi

EXIT_DIVERGED = 1
EXIT_ERROR = 2

BACKENDS = {
    "gpu": dict(storage=WeightStorage.Auto),
    "mat": dict(storage=WeightStorage.Auto),
    "gpu-dense": dict(storage=WeightStorage.Dense),
    "gpu-sparse": dict(storage=WeightStorage.Sparse),
    "gpu-exact": dict(storage=WeightStorage.Auto, precision="f64", exact_order=True),
    "gpu-abm": dict(storage=WeightStorage.Auto, precision="f64", exact_order=True, abm=True),
    "abm": dict(storage=WeightStorage.Auto, precision="f64", exact_order=True, abm=True),
    "gpu-abm-fast": dict(storage=WeightStorage.Auto, precision="f32", exact_order=False, abm=True),
}


def run_backend(backend: str, net, cfg, stim, device: int = 0):
    if backend not in BACKENDS:
        raise ValueError(f'unknown backend "{backend}"')
    opts = dict(BACKENDS[backend])
    storage = opts.pop("storage")
    t0 = time.perf_counter()
    if opts.pop("abm", False):
        res = abm_run(net, cfg, stim, device=device, storage=int(storage), **opts)
    else:
        res = mat_run(net, cfg, stim, storage, device=device, **opts)
    return res.raster, time.perf_counter() - t0


def cmd_run(a) -> int:
    net = fio.parse_network(fio.read_file(a.network))
    stim = fio.parse_stimulus(fio.read_file(a.stimulus)) if a.stimulus else StimulusSchedule()
    cfg = SimulationConfig(steps=a.steps, seed=a.seed)
    if a.stdp:
        cfg.stdp = fio.parse_stdp(fio.read_file(a.stdp))
    raster, wall = run_backend(a.backend, net, cfg, stim, a.device)
    csv = fio.write_raster(raster)
    report = sys.stderr if not a.out else sys.stdout
    if a.out:
        fio.write_file(a.out, csv)
    else:
        sys.stdout.write(csv)
    report.write(f"backend={a.backend} neurons={net.neuron_count()} steps={cfg.steps} "
                 f"spikes={len(raster)} wall_seconds={wall:.6g}\n")
    return 0


def cmd_gen(a) -> int:
    if a.stimulus_out:
        b = build_scenario(BenchScenario(neuron_count=a.neurons, connection_probability=a.prob,
                                         steps=a.steps, input_neuron_count=a.inputs,
                                         input_period=a.period, amplitude=a.amplitude, seed=a.seed))
        fio.write_file(a.out, fio.serialize_network(b.net))
        fio.write_file(a.stimulus_out, fio.write_stimulus(b.stim))
    else:
        fio.write_file(a.out, fio.serialize_network(erdos_renyi(a.neurons, a.prob, a.seed)))
    return 0


def first_divergence(x: SpikeRaster, y: SpikeRaster):
    xs = list(zip(x.steps_array.tolist(), x.neurons_array.tolist()))
    ys = list(zip(y.steps_array.tolist(), y.neurons_array.tolist()))
    for p, q in zip(xs, ys):
        if p != q:
            return min(p, q)
    if len(xs) != len(ys):
        return (xs if len(xs) > len(ys) else ys)[min(len(xs), len(ys))]
    return None


def cmd_compare(a) -> int:
    net = fio.parse_network(fio.read_file(a.network))
    stim = fio.parse_stimulus(fio.read_file(a.stimulus)) if a.stimulus else StimulusSchedule()
    cfg = SimulationConfig(steps=a.steps, seed=a.seed)
    rasters = []
    names = [b for b in a.backends.split(",") if b]
    for b in names:
        rasters.append((b, run_backend(b, net, cfg, stim, a.device)[0]))
    if a.against:
        rasters.append((os.path.basename(a.against), fio.parse_raster(fio.read_file(a.against))))
    base_name, base = rasters[0]
    for name, r in rasters[1:]:
        d = first_divergence(base, r)
        if d is not None:
            sys.stdout.write(f"divergence: step {d[0]} neuron {d[1]} ({base_name} vs {name})\n")
            return EXIT_DIVERGED
    sys.stdout.write("identical\n")
    return 0


def cmd_bench(a) -> int:
    """Reference bench methodology (bench.cpp:24-97): scenario built outside
    the clock, the step loop timed (device time of sn_simulate)."""
    from .engine import MatEngine
    rows: List[fio.BenchRow] = []
    sizes = [int(s) for s in a.sizes.split(",")]
    probs = [float(p) for p in a.probs.split(",")]
    for backend in a.backends.split(","):
        opts = dict(BACKENDS[backend])
        storage = int(opts.pop("storage"))
        mode = "abm" if opts.pop("abm", False) else "mat"
        for n in sizes:
            for p in probs:
                eng = MatEngine(device=a.device, storage=storage, mode=mode, **opts)
                eng.generate_erdos_renyi(n, p, a.seed)
                if mode == "abm":
                    eng.set_seed(a.seed)
                eng.setup()
                from .netgen import scenario_stimulus
                eng.add_stimulus(*scenario_stimulus(n, a.steps, a.seed, amplitude=a.amplitude).to_arrays())
                eng.simulate(a.steps)
                st = eng.stats()
                rows.append(fio.BenchRow(backend, n, p, a.steps, st["last_simulate_ms"] / 1e3,
                                         int(st["spike_count"]), a.seed))
                eng.close()
    text = fio.write_bench(rows)
    if a.out:
        fio.write_file(a.out, text)
    else:
        sys.stdout.write(text)
    return 0


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2305_02510_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="Simulate a network and write its spike raster")
    r.add_argument("--network", required=True)
    r.add_argument("--steps", type=int, default=1000)
    r.add_argument("--backend", default="gpu")
    r.add_argument("--stimulus", default="")
    r.add_argument("--seed", type=int, default=int(os.environ.get("SPIKEFORGE_SEED", "0")))
    r.add_argument("--out", default="")
    r.add_argument("--stdp", default="")
    r.add_argument("--device", type=int, default=0)
    g = sub.add_parser("gen", help="Generate a random network (and stimulus)")
    g.add_argument("--neurons", type=int, default=100)
    g.add_argument("--prob", type=float, default=0.25)
    g.add_argument("--seed", type=int, default=int(os.environ.get("SPIKEFORGE_SEED", "0")))
    g.add_argument("--out", required=True)
    g.add_argument("--stimulus-out", default="")
    g.add_argument("--steps", type=int, default=1000)
    g.add_argument("--inputs", type=int, default=3)
    g.add_argument("--period", type=int, default=10)
    g.add_argument("--amplitude", type=float, default=2.0)
    c = sub.add_parser("compare", help="Differential run across backends")
    c.add_argument("--network", required=True)
    c.add_argument("--steps", type=int, default=1000)
    c.add_argument("--stimulus", default="")
    c.add_argument("--seed", type=int, default=int(os.environ.get("SPIKEFORGE_SEED", "0")))
    c.add_argument("--backends", default="gpu,gpu-exact")
    c.add_argument("--against", default="", help="raster CSV from another implementation")
    c.add_argument("--device", type=int, default=0)
    b = sub.add_parser("bench", help="Benchmark sweep over network sizes")
    b.add_argument("--sizes", default="100,1000")
    b.add_argument("--probs", default="0.25,0.5,0.75,1.0")
    b.add_argument("--steps", type=int, default=1000)
    b.add_argument("--backends", default="gpu")
    b.add_argument("--seed", type=int, default=int(os.environ.get("SPIKEFORGE_SEED", "0")))
    b.add_argument("--amplitude", type=float, default=2.0)
    b.add_argument("--out", default="")
    b.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "gen": cmd_gen, "compare": cmd_compare, "bench": cmd_bench}[a.cmd](a)
    except Exception as e:  # spikeforge_main.cpp:319-328
        sys.stderr.write(f"error: {e}\n")
        return EXIT_ERROR
