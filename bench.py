#!/usr/bin/env python
"""Benchmark of the MAT-mode step on B200.

Metric (BASELINE.json): simulated timesteps/s (+ synaptic events/s) vs the
HBM roofline, with the reference CPU path timed beside it.

Default workload = BASELINE cfg3: ER(32,000, p=1) with every synapse plastic,
StdpConfig::defaults(), paper stimulus (3 inputs every 10 steps, amplitude 2),
fp32 weights (4.1 GB, larger than L2).  One bench "step" = one simulated
timestep (LIF update + fused STDP/propagation sweep over all 1.024e9
weights).  --workload selects the other BASELINE configs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) each rank owns a contiguous post partition; the spike
bitmask is all-gathered with NCCL once per step inside the engine.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated timesteps/sec and synaptic events/sec vs HBM roofline; CPU ref"
UNIT = "timesteps/s"

WORKLOADS = {
    # name: (n, p, stdp, delay_max, by_syn_index, horizon T, description)
    "cfg1": (100, 0.05, False, 1, False, 1000, "ER(100, p=0.05), delay 1, no STDP, paper stimulus"),
    "cfg2": (1000, 1.0, False, 8, True, 1000, "ER(1000, p=1), delays 1..8 (synapse-index keyed), no STDP"),
    "cfg3": (32000, 1.0, True, 1, False, 100, "ER(32000, p=1) all synapses plastic, STDP defaults, fp32 weights"),
    "cfg4": (256000, 0.01, False, 16, False, 1000, "ER(256000, p=0.01) CSC, delays 1..16 (pair keyed), no STDP"),
    "cfg5": (96000, 1.0, True, 1, False, 100, "ER(96000, p=1) all plastic, STDP defaults, fp32 weights"),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML polled
    every 2 ms from a thread (the timed regions are 0.1-1 s), nvidia-smi as a
    fallback."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []
        self.stop_flag = threading.Event()

    def _nvml_loop(self, nv, h):
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, [k for k, b in bits.items() if rs & b]))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.nvml = nv
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Start of the timed region: only samples from here on count (the
        sampler itself is started before the warm-up, so NVML's start-up and
        an idle gap do not fall on the first timed launch)."""
        self.mark_at = len(self.samples)

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            m = getattr(self, "mark_at", 0)
            # a region shorter than the 2 ms poll keeps the sample taken just before it
            samples = self.samples[m:] or self.samples[max(0, m - 1):m]
            sm = [s for s, _ in samples]
            reasons = sorted({r for _, rs in samples for r in rs})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_engine(sn, wl, device, rank, world, stream_io=False, profile=False):
    n, p, stdp, dmax, by_syn, T, _ = WORKLOADS[wl]
    eng = sn.MatEngine(device=device, rank=rank, world=world, stream_io=stream_io, profile=profile,
                       use_graphs=True)
    eng.generate_erdos_renyi(n, p, 0, delay_max=dmax, delay_by_synapse_index=by_syn, stdp=stdp)
    if stdp:
        d = sn.StdpConfig.defaults()
        eng.set_stdp(d.window, d.a_plus, d.a_minus, d.w_min, d.w_max)
    return eng


def connect(sn, eng, rank, world, transport):
    """Join the per-step spike exchange of a partitioned run: one in-place
    ncclAllGather (nccl) or stores fused into the neuron kernel (p2p)."""
    if world == 1:
        return
    from paper_2305_02510_b200 import distributed as D
    if transport == "p2p":
        eng.p2p_open(D.exchange_p2p_handles(eng.p2p_handles()), world)
    else:
        eng.comm_init(D.broadcast_uid(sn.comm_unique_id() if rank == 0 else None), rank, world)


def add_protocol_stimulus(sn, eng, n, horizon):
    st = sn.netgen.scenario_stimulus(n, horizon, 0)
    arr = st.to_arrays()
    eng.add_stimulus(*arr)
    return arr


def run_ours(args):
    import paper_2305_02510_b200 as sn
    rank, world, local = dist_env()
    device = local
    torch_dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        torch_dist = dist
    wl = args.workload
    n, p, stdp, dmax, by_syn, T, desc = WORKLOADS[wl]
    K, W = args.steps, args.warmup
    horizon = W + K

    eng = build_engine(sn, wl, device, rank, world, profile=True)
    eng.setup()
    connect(sn, eng, rank, world, args.transport)
    stim = add_protocol_stimulus(sn, eng, n, horizon)
    clocks = ClockSampler(device)
    clocks.start()
    eng.simulate(W)                       # warm-up
    eng.synchronize()
    eng.reset_stats()
    if torch_dist:
        torch_dist.barrier()
    clocks.mark()
    t0 = time.perf_counter()
    eng.simulate(K)                       # timed: device events inside the engine
    eng.synchronize()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    st = eng.stats()
    ms = st["last_simulate_ms"]
    if torch_dist:
        import torch
        t = torch.tensor([ms], dtype=torch.float64)
        torch_dist.all_reduce(t, op=torch_dist.ReduceOp.MAX)
        ms = float(t.item())
        sp = torch.tensor([st["spike_count"]], dtype=torch.float64)
        torch_dist.all_reduce(sp)
        spikes_total = float(sp.item())
    else:
        spikes_total = float(st["spike_count"])
    steps_s, nspk = eng.raster()
    timed_spikes = int(np.count_nonzero(steps_s >= W))
    if torch_dist:
        import torch
        ts = torch.tensor([timed_spikes], dtype=torch.float64)
        torch_dist.all_reduce(ts)
        timed_spikes = int(ts.item())
    value = K / (ms / 1e3)
    # synaptic events: a spike at t is delivered along all out-synapses
    avg_out = (n - 1) if p >= 1.0 else p * (n - 1)
    syn_events = timed_spikes * avg_out
    # one sweep per step; the engine times a sample of the timed region's sweeps
    # (every 8th step's kernels carry CUDA event nodes), the persistent kernel
    # covers all K steps in one launch
    kname = sn._capi.Stats.KERNEL_NAMES.get(st["sweep_kernel"], "?")
    persistent = kname in ("k_persistent_dense", "k_persistent_cols", "k_tiny")
    sweep_avg_ms = st["sweep_ms"] / (K if persistent else max(1, st["sweep_launches"]))
    bytes_per_sweep = st["sweep_bytes_total"] / K
    peak, peak_src = load_peaks()
    achieved = bytes_per_sweep / (sweep_avg_ms / 1e3) / 1e9 if sweep_avg_ms > 0 else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                tj = json.load(f)
            traffic = tj.get(wl)
        except Exception:
            traffic = None
    launches = st["kernel_launches"]
    eng.close()

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        eng2 = build_engine(sn, wl, device, rank, world, stream_io=True)
        eng2.setup()
        connect(sn, eng2, rank, world, args.transport)
        add_protocol_stimulus(sn, eng2, n, horizon)
        eng2.simulate(W)                  # warm-up, including one raster fetch
        eng2.raster()
        eng2.clear_raster()
        if torch_dist:
            torch_dist.barrier()
        t0 = time.perf_counter()
        eng2.simulate(K)                  # H2D of the call's stimulus rows, kernels store each step's spike words to pinned host memory
        s2, n2 = eng2.raster()            # host decode of the raster
        wall2 = time.perf_counter() - t0
        if torch_dist:
            import torch
            t = torch.tensor([wall2], dtype=torch.float64)
            torch_dist.all_reduce(t, op=torch_dist.ReduceOp.MAX)
            wall2 = float(t.item())
        st2 = eng2.stats()   # bytes the engine actually moved in the timed call
        h2d = st2["h2d_bytes_last"] / K
        d2h = st2["d2h_bytes_last"] / K
        eng2.close()
        e2e = {"value": K / wall2, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h * world}

    if rank != 0:
        if torch_dist:
            torch_dist.destroy_process_group()
        return
    cpu = None if args.no_cpu else cpu_baseline(wl, args)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "fp32 weights, fp64 membrane/traces" if stdp else "fp32 weights, fp64 membrane",
        "data": "synthetic (on-device erdos_renyi, bit-identical to netgen.cpp; paper stimulus)",
        "config": {"workload": f"{wl}: {desc}", "n": n, "p": p, "stdp": stdp, "delay_max": dmax,
                   "storage": ("shared-memory in-lists" if kname == "k_tiny"
                               else "dense" if st["dense"] else "sparse"),
                   "parallelism": (f"post-partition x{world} ({args.transport} spike exchange)"
                                   if world > 1 else "single GPU"),
                   "l2": "inputs larger than L2" if n * n * p * 4 > 126e6 else "working set L2-resident"},
        "syn_events_per_s": syn_events / (ms / 1e3),
        "spikes_timed": timed_spikes,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": kname,
                     "kernel_ctas": st["sweep_ctas"],
                     "bytes_per_launch": bytes_per_sweep, "avg_launch_ms": sweep_avg_ms,
                     "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "host_wall_s": wall,
    }
    print(json.dumps(out))
    if torch_dist:
        torch_dist.destroy_process_group()


def cpu_sample_plan(wl):
    """Bounded sample of the reference CPU path (10-30 s) and the factor that
    scales its per-step time to the full workload (synapse-count ratio)."""
    n, p, stdp, dmax, by_syn, T, _ = WORKLOADS[wl]
    if wl == "cfg3":
        ns, steps = 8192, 5
    elif wl == "cfg5":
        ns, steps = 8192, 5
    elif wl == "cfg4":
        ns, steps = 20000, 20
    elif wl == "cfg2":
        ns, steps = 1000, 200
    else:
        ns, steps = n, T
    factor = (n * (n - 1) * p) / (ns * (ns - 1) * p) if ns != n else 1.0
    return ns, steps, factor


def cpu_baseline(wl, args):
    """Reference C++ (oracle/_ref, -O3 -DNDEBUG, single thread) timed on the
    host like bench.cpp:24-50; falls back to the C restatement if absent."""
    from oracle import bridge as B
    n, p, stdp, dmax, by_syn, T, _ = WORKLOADS[wl]
    ns, steps, factor = cpu_sample_plan(wl)
    try:
        if not B.ref_available():
            raise FileNotFoundError
        if dmax > 1:
            # reference MAT path for delays = lower_delays + mat_run; time abm_run
            # (the reference's native-delay path, faster than lowered mat)
            from paper_2305_02510_b200.netgen import erdos_renyi_arrays, DELAY_STREAM, RandomStream, scenario_stimulus
            pre, post = erdos_renyi_arrays(ns, p, 0)
            keys = np.arange(len(pre), dtype=np.uint64) if by_syn else (pre.astype(np.uint64) * np.uint64(ns) + post.astype(np.uint64))
            d = (1 + RandomStream(0, DELAY_STREAM).below_np(keys, dmax)).astype(np.int32)
            arrays = {"threshold": np.ones(ns), "leak": np.zeros(ns), "reset": np.zeros(ns),
                      "refractory": np.zeros(ns, np.int32), "axonal": np.zeros(ns, np.int32), "pre": pre,
                      "post": post, "weight": np.ones(len(pre)), "delay": d, "stdp": np.zeros(len(pre), np.uint8)}
            t0 = time.perf_counter()
            B.run_ref_abm(arrays, steps, scenario_stimulus(ns, steps, 0).to_arrays())
            secs = time.perf_counter() - t0
            kind, path = "reference", "abm_run (native delays; incl. AbmWorld build)"
        else:
            r = B.ref_bench_scenario(ns, p, 0, steps, stdp, 0)
            secs = r["seconds"]
            kind, path = "reference", "mat_step" + ("+apply_stdp" if stdp else "") + " (mat_init untimed)"
    except (FileNotFoundError, OSError):
        from paper_2305_02510_b200.netgen import erdos_renyi_arrays, scenario_stimulus
        pre, post = erdos_renyi_arrays(ns, p, 0)
        arrays = {"threshold": np.ones(ns), "leak": np.zeros(ns), "reset": np.zeros(ns),
                  "refractory": np.zeros(ns, np.int32), "axonal": np.zeros(ns, np.int32), "pre": pre,
                  "post": post, "weight": np.ones(len(pre)), "delay": np.ones(len(pre), np.int32),
                  "stdp": np.full(len(pre), 1 if stdp else 0, np.uint8)}
        d = None
        if stdp:
            from paper_2305_02510_b200.model import StdpConfig
            c = StdpConfig.defaults()
            d = (c.window, np.array(c.a_plus), np.array(c.a_minus), c.w_min, c.w_max)
        t0 = time.perf_counter()
        B.run_oracle(arrays, steps, scenario_stimulus(ns, steps, 0).to_arrays(), d)
        secs = time.perf_counter() - t0
        kind, path = "port", "oracle/mat_oracle.c"
    per_step = secs / steps * factor
    return {"value": 1.0 / per_step, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{path} on ER({ns}, p={p}) for {steps} steps = {secs:.2f} s; per-step time scaled by the "
                      f"synapse-count ratio x{factor:.2f} to {wl} (n={n})",
            "cpu": cpu_model()}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cpus)"
    except Exception:
        pass
    return f"{os.cpu_count()} logical cpus"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl = args.workload
    n, p, stdp, dmax, by_syn, T, desc = WORKLOADS[wl]
    K, W = args.steps, args.warmup
    cpu = cpu_baseline(wl, args)
    value = cpu["value"]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
           "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "fp64", "data": "synthetic (reference erdos_renyi + build_scenario)",
           "config": {"workload": f"{wl}: {desc}", "n": n, "p": p, "stdp": stdp, "delay_max": dmax},
           "impl": "reference",
           "cpu_baseline": cpu,
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default="cfg3")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="per-step spike exchange when N > 1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the timing contract wants >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
