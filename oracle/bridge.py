"""TEST INFRASTRUCTURE ONLY -- ctypes bridge to the two CPU checkers:

* ``oracle/libmat_oracle.so``          plain-C restatement (mat_oracle.c)
* ``oracle/_ref/libspikeforge_ref.so`` the reference's own C++ (ref_shim.cpp)

Imported by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) only.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmat_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspikeforge_ref.so")
REF_SRC = "/root/reference/proj"


class Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("threshold", C.POINTER(C.c_double)),
        ("leak", C.POINTER(C.c_double)),
        ("reset", C.POINTER(C.c_double)),
        ("refractory", C.POINTER(C.c_int32)),
        ("axonal", C.POINTER(C.c_int32)),
        ("m", C.c_int64),
        ("pre", C.POINTER(C.c_int32)),
        ("post", C.POINTER(C.c_int32)),
        ("weight", C.POINTER(C.c_double)),
        ("delay", C.POINTER(C.c_int32)),
        ("stdp", C.POINTER(C.c_uint8)),
        ("k", C.c_int64),
        ("st_step", C.POINTER(C.c_int32)),
        ("st_neuron", C.POINTER(C.c_int32)),
        ("st_amp", C.POINTER(C.c_double)),
        ("steps", C.c_int32),
        ("stdp_on", C.c_int32),
        ("window", C.c_int32),
        ("a_plus", C.POINTER(C.c_double)),
        ("a_minus", C.POINTER(C.c_double)),
        ("w_min", C.c_double),
        ("w_max", C.c_double),
        ("record_membrane", C.c_int32),
        ("seed", C.c_uint64),
        ("fire_p", C.POINTER(C.c_double)),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("error", C.c_char * 1024),
        ("n_events", C.c_int64),
        ("ev_step", C.POINTER(C.c_int32)),
        ("ev_neuron", C.POINTER(C.c_int32)),
        ("n", C.c_int32),
        ("membrane", C.POINTER(C.c_double)),
        ("m", C.c_int64),
        ("weights", C.POINTER(C.c_double)),
        ("membrane_trace", C.POINTER(C.c_double)),
        ("spike_count", C.c_int64),
        ("seconds", C.c_double),
    ]


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle [ref]); ref only where the sources exist."""
    targets = ["all"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        lib.mat_oracle_run.argtypes = [C.POINTER(Problem), C.POINTER(Result)]
        lib.mat_oracle_run.restype = C.c_int
        lib.abm_oracle_run.argtypes = [C.POINTER(Problem), C.POINTER(Result)]
        lib.abm_oracle_run.restype = C.c_int
        lib.orc_result_free.argtypes = [C.POINTER(Result)]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " (build with make -C oracle ref where /root/reference exists)")
        lib = C.CDLL(REF_SO)
        P, R = C.POINTER(Problem), C.POINTER(Result)
        lib.ref_mat_run.argtypes = [P, C.c_int, C.c_int, R]
        lib.ref_mat_run_raster.argtypes = [P, C.c_int, R]
        lib.ref_oracle_run.argtypes = [P, R]
        lib.ref_abm_run.argtypes = [P, R]
        lib.ref_abm_run_full.argtypes = [P, R]
        lib.ref_validate.argtypes = [P, C.c_char_p, C.c_int]
        lib.ref_mat_init_error.argtypes = [P, C.c_char_p, C.c_int]
        lib.ref_erdos_renyi.argtypes = [C.c_int, C.c_double, C.c_uint64, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.c_int64]
        lib.ref_erdos_renyi.restype = C.c_int64
        lib.ref_scenario_inputs.argtypes = [C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_int,
                                            C.POINTER(C.c_int32)]
        lib.ref_stdp_defaults.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
        lib.ref_leak_toward.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.ref_leak_toward.restype = C.c_double
        lib.ref_mix64.argtypes = [C.c_uint64]
        lib.ref_mix64.restype = C.c_uint64
        lib.ref_stream_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        lib.ref_stream_u64.restype = C.c_uint64
        lib.ref_stream_unit.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        lib.ref_stream_unit.restype = C.c_double
        lib.ref_stream_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]
        lib.ref_stream_below.restype = C.c_uint64
        lib.ref_bench_scenario.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int, R]
        lib.orc_result_free.argtypes = [R]
        _ref = lib
    return _ref


class _Keep:
    """Holds the numpy buffers a Problem points into."""


def make_problem(arrays: dict, steps: int, stim=None, stdp=None, record_membrane=False,
                 seed: int = 0, fire_p=None):
    """arrays: NetworkDef.to_arrays() layout; stim: (step, neuron, amp) arrays;
    stdp: (window, a_plus, a_minus, w_min, w_max) or None."""
    keep = _Keep()
    p = Problem()

    def arr(name, a, dtype, ctype):
        a = np.ascontiguousarray(a, dtype=dtype)
        setattr(keep, name, a)
        return a.ctypes.data_as(C.POINTER(ctype))

    n = len(arrays["threshold"])
    p.n = n
    p.threshold = arr("thr", arrays["threshold"], np.float64, C.c_double)
    p.leak = arr("leak", arrays["leak"], np.float64, C.c_double)
    p.reset = arr("reset", arrays["reset"], np.float64, C.c_double)
    p.refractory = arr("refr", arrays["refractory"], np.int32, C.c_int32)
    p.axonal = arr("ax", arrays.get("axonal", np.zeros(n)), np.int32, C.c_int32)
    m = len(arrays["pre"])
    p.m = m
    p.pre = arr("pre", arrays["pre"], np.int32, C.c_int32)
    p.post = arr("post", arrays["post"], np.int32, C.c_int32)
    p.weight = arr("w", arrays["weight"], np.float64, C.c_double)
    p.delay = arr("d", arrays.get("delay", np.ones(m)), np.int32, C.c_int32)
    p.stdp = arr("s", arrays.get("stdp", np.zeros(m)), np.uint8, C.c_uint8)
    if stim is None:
        stim = (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    p.k = len(stim[0])
    p.st_step = arr("sts", stim[0], np.int32, C.c_int32)
    p.st_neuron = arr("stn", stim[1], np.int32, C.c_int32)
    p.st_amp = arr("sta", stim[2], np.float64, C.c_double)
    p.steps = steps
    if stdp is not None:
        window, ap, am, wmin, wmax = stdp
        p.stdp_on = 1
        p.window = window
        p.a_plus = arr("ap", ap, np.float64, C.c_double)
        p.a_minus = arr("am", am, np.float64, C.c_double)
        p.w_min = wmin
        p.w_max = wmax
    p.record_membrane = 1 if record_membrane else 0
    p.seed = int(seed) & ((1 << 64) - 1)
    if fire_p is not None:
        p.fire_p = arr("fp", fire_p, np.float64, C.c_double)
    return p, keep


def _collect(lib, r: Result, steps: int, with_state: bool = True) -> dict:
    if r.status != 0:
        msg = r.error.decode()
        lib.orc_result_free(C.byref(r))
        kind = {1: ValueError, 2: RuntimeError}.get(r.status, RuntimeError)
        raise kind(msg)
    ne = r.n_events
    out = {
        "steps": np.ctypeslib.as_array(r.ev_step, (ne,)).copy() if ne else np.zeros(0, np.int32),
        "neurons": np.ctypeslib.as_array(r.ev_neuron, (ne,)).copy() if ne else np.zeros(0, np.int32),
        "spike_count": r.spike_count,
        "seconds": r.seconds,
    }
    if with_state and r.membrane:
        out["membrane"] = np.ctypeslib.as_array(r.membrane, (r.n,)).copy()
    if with_state and r.weights and r.m:
        out["weights"] = np.ctypeslib.as_array(r.weights, (r.m,)).copy()
    if with_state and r.membrane_trace:
        out["membrane_trace"] = np.ctypeslib.as_array(r.membrane_trace, (steps * r.n,)).copy().reshape(steps, r.n)
    lib.orc_result_free(C.byref(r))
    return out


def run_oracle(arrays, steps, stim=None, stdp=None, record_membrane=False, f32_weights=False) -> dict:
    """mat_oracle.c: the plain-C restatement.  f32_weights: the fp32 weight
    storage model (every stored weight rounded to float once; all arithmetic
    fp64) -- the engine's default precision must reproduce its weights bit
    for bit."""
    lib = oracle_lib()
    p, keep = make_problem(arrays, steps, stim, stdp, record_membrane)
    r = Result()
    (lib.mat_oracle_run_f32w if f32_weights else lib.mat_oracle_run)(C.byref(p), C.byref(r))
    return _collect(lib, r, steps)


def run_ref_mat(arrays, steps, stim=None, stdp=None, record_membrane=False, storage=0,
                lower=False) -> dict:
    """The reference's mat_init/mat_step/apply_stdp loop (lower=True: lower_delays first)."""
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim, stdp, record_membrane)
    r = Result()
    lib.ref_mat_run(C.byref(p), storage, 1 if lower else 0, C.byref(r))
    return _collect(lib, r, steps)


def run_ref_mat_masked(arrays, steps, stim, stdp, plastic_steps, storage=0, lower=False) -> dict:
    """The reference's mat_step loop with apply_stdp only on steps whose
    plastic_steps byte is non-zero (oracle/ref_shim.cpp mat_loop)."""
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim, stdp)
    mask = np.ascontiguousarray(plastic_steps, np.uint8)
    assert len(mask) == steps
    r = Result()
    lib.ref_mat_run_masked.argtypes = [C.POINTER(Problem), C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(Result)]
    lib.ref_mat_run_masked(C.byref(p), storage, 1 if lower else 0, mask.ctypes.data_as(C.POINTER(C.c_uint8)),
                           C.byref(r))
    return _collect(lib, r, steps)


def run_ref_mat_raster(arrays, steps, stim=None, stdp=None, storage=0) -> dict:
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim, stdp)
    r = Result()
    lib.ref_mat_run_raster(C.byref(p), storage, C.byref(r))
    return _collect(lib, r, steps, with_state=False)


def run_ref_oracle(arrays, steps, stim=None) -> dict:
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim)
    r = Result()
    lib.ref_oracle_run(C.byref(p), C.byref(r))
    return _collect(lib, r, steps, with_state=False)


def run_ref_abm(arrays, steps, stim=None) -> dict:
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim)
    r = Result()
    lib.ref_abm_run(C.byref(p), C.byref(r))
    return _collect(lib, r, steps, with_state=False)


def run_abm_oracle(arrays, steps, stim=None, seed=0, fire_p=None, record_membrane=False) -> dict:
    """abm_oracle.c: the plain-C restatement of abm_run."""
    lib = oracle_lib()
    p, keep = make_problem(arrays, steps, stim, None, record_membrane, seed, fire_p)
    r = Result()
    lib.abm_oracle_run(C.byref(p), C.byref(r))
    return _collect(lib, r, steps)


def run_ref_abm_full(arrays, steps, stim=None, seed=0, fire_p=None, record_membrane=False) -> dict:
    """The reference's abm_run with stochastic behaviours and the run seed."""
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim, None, record_membrane, seed, fire_p)
    r = Result()
    lib.ref_abm_run_full(C.byref(p), C.byref(r))
    return _collect(lib, r, steps)


def ref_validate(arrays, steps, stim=None, stdp=None):
    lib = ref_lib()
    p, keep = make_problem(arrays, steps, stim, stdp)
    buf = C.create_string_buffer(1 << 16)
    cnt = lib.ref_validate(C.byref(p), buf, len(buf))
    txt = buf.value.decode()
    return txt.split("\n") if cnt else []


def ref_erdos_renyi(n, p, seed):
    lib = ref_lib()
    cap = n * n
    pre = np.empty(cap, np.int32)
    post = np.empty(cap, np.int32)
    m = lib.ref_erdos_renyi(n, p, seed, pre.ctypes.data_as(C.POINTER(C.c_int32)),
                            post.ctypes.data_as(C.POINTER(C.c_int32)), cap)
    return pre[:m].copy(), post[:m].copy()


def ref_has_io() -> bool:
    return ref_available() and hasattr(ref_lib(), "ref_write_raster")


def _ref_str(fn, *args) -> str:
    lib = ref_lib()
    f = getattr(lib, fn)
    f.restype = C.c_void_p
    ptr = f(*args)
    try:
        return C.string_at(ptr).decode()
    finally:
        lib.ref_free_str.argtypes = [C.c_void_p]
        lib.ref_free_str(ptr)


def ref_serialize_network(arrays) -> str:
    p, keep = make_problem(arrays, 1)
    ref_lib().ref_serialize_network.argtypes = [C.POINTER(Problem)]
    return _ref_str("ref_serialize_network", C.byref(p))


def ref_write_raster(steps, neurons) -> str:
    s = np.ascontiguousarray(steps, np.int32)
    n = np.ascontiguousarray(neurons, np.int32)
    ref_lib().ref_write_raster.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int64]
    return _ref_str("ref_write_raster", s.ctypes.data_as(C.POINTER(C.c_int32)),
                    n.ctypes.data_as(C.POINTER(C.c_int32)), len(s))


def ref_write_stimulus(stim) -> str:
    arrays = {"threshold": np.ones(1), "leak": np.zeros(1), "reset": np.zeros(1),
              "refractory": np.zeros(1, np.int32), "pre": [], "post": [], "weight": []}
    p, keep = make_problem(arrays, 1, stim)
    ref_lib().ref_write_stimulus.argtypes = [C.POINTER(Problem)]
    return _ref_str("ref_write_stimulus", C.byref(p))


def ref_serialize_stdp(stdp) -> str:
    arrays = {"threshold": np.ones(1), "leak": np.zeros(1), "reset": np.zeros(1),
              "refractory": np.zeros(1, np.int32), "pre": [], "post": [], "weight": []}
    p, keep = make_problem(arrays, 1, None, stdp)
    ref_lib().ref_serialize_stdp.argtypes = [C.POINTER(Problem)]
    return _ref_str("ref_serialize_stdp", C.byref(p))


def ref_roundtrip_network(text: str) -> str:
    ref_lib().ref_roundtrip_network.argtypes = [C.c_char_p]
    return _ref_str("ref_roundtrip_network", text.encode())


def ref_bench_run(n, p, seed, horizon, warmup, steps, stdp_on, storage=0, delay_max=1, by_index=False,
                  delay_stream=0) -> dict:
    """Reference CPU path at the given size (oracle/ref_shim.cpp ref_bench_run):
    setup untimed, `warmup` untimed steps, `steps` timed steps (mat_step +
    apply_stdp, or AbmWorld::step for delayed nets)."""
    lib = ref_lib()
    info = np.zeros(6)
    step_s = np.zeros(max(1, steps))
    r = Result()
    dp = C.POINTER(C.c_double)
    lib.ref_bench_run.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_uint64, dp, dp, C.POINTER(Result)]
    lib.ref_bench_run(n, p, seed, horizon, warmup, steps, 1 if stdp_on else 0, storage, delay_max,
                      1 if by_index else 0, delay_stream, info.ctypes.data_as(dp), step_s.ctypes.data_as(dp),
                      C.byref(r))
    out = _collect(lib, r, steps, with_state=False)
    out.update({"setup_s": float(info[0]), "warmup_s": float(info[1]), "timed_s": float(info[2]),
                "storage": {1: "dense", 0: "csr", -1: "abm"}[int(info[3])], "synapses": int(info[4]),
                "peak_rss_gb": float(info[5]), "step_s": step_s[:steps].tolist()})
    return out


def ref_scenario_abm_raster(n, p, seed, steps, delay_max=1, by_index=False, delay_stream=0x64656C6179) -> dict:
    """Raster of the reference's abm_run on a generated scenario (ref_shim.cpp
    ref_scenario_abm_raster); also synapse count, build / run seconds, RSS."""
    lib = ref_lib()
    info = np.zeros(4)
    r = Result()
    dp = C.POINTER(C.c_double)
    lib.ref_scenario_abm_raster.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                            C.c_uint64, dp, C.POINTER(Result)]
    lib.ref_scenario_abm_raster(n, p, seed, steps, delay_max, 1 if by_index else 0, delay_stream,
                                info.ctypes.data_as(dp), C.byref(r))
    out = _collect(lib, r, steps, with_state=False)
    out.update({"synapses": int(info[0]), "build_s": float(info[1]), "run_s": float(info[2]),
                "peak_rss_gb": float(info[3])})
    return out


def ref_scenario_stdp_raster(n, p, seed, steps) -> dict:
    """Raster of the reference's mat_run on the all-plastic STDP scenario
    (ref_shim.cpp ref_scenario_stdp_raster); also synapses, seconds, RSS."""
    lib = ref_lib()
    info = np.zeros(3)
    r = Result()
    dp = C.POINTER(C.c_double)
    lib.ref_scenario_stdp_raster.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, dp, C.POINTER(Result)]
    lib.ref_scenario_stdp_raster(n, p, seed, steps, info.ctypes.data_as(dp), C.byref(r))
    out = _collect(lib, r, steps, with_state=False)
    out.update({"synapses": int(info[0]), "seconds": float(info[1]), "peak_rss_gb": float(info[2])})
    return out


def ref_bench_scenario(n, p, seed, steps, stdp_on, storage=0) -> dict:
    """Reference CPU path timed like bench.cpp:24-50 (mat_init outside the clock)."""
    lib = ref_lib()
    r = Result()
    lib.ref_bench_scenario(n, p, seed, steps, 1 if stdp_on else 0, storage, C.byref(r))
    return _collect(lib, r, steps, with_state=False)
