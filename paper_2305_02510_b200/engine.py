"""Thin object wrapper over the C ABI engine handle (include/superneuro_mat.h).

Everything numeric runs in libsnmat.so on the GPU; this class only moves
numpy buffers across the boundary.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _capi
from ._capi import check, lib, ptr


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


class MatEngine:
    """One engine = one MatState-equivalent on one GPU (or one post partition)."""

    def __init__(self, device: int = 0, storage: int = _capi.SN_STORAGE_AUTO,
                 precision: str = "f32", exact_order: bool = False,
                 record_membrane: bool = False, stream_io: bool = False,
                 use_graphs: bool = True, rank: int = 0, world: int = 1,
                 profile: bool = False, persistent: bool = True, mode: str = "mat"):
        o = _capi.Options()
        check(lib.sn_options_init(C.byref(o)))
        o.device = device
        o.storage = int(storage)
        o.precision = _capi.SN_WEIGHTS_F64 if precision == "f64" else _capi.SN_WEIGHTS_F32
        o.exact_order = 1 if exact_order else 0
        o.record_membrane = 1 if record_membrane else 0
        o.stream_io = 1 if stream_io else 0
        o.use_graphs = 1 if use_graphs else 0
        o.rank = rank
        o.world = world
        o.profile = 1 if profile else 0
        o.persistent = 0 if persistent else -1
        if mode not in ("mat", "abm"):
            raise ValueError(f'unknown engine mode "{mode}" (expected "mat" or "abm")')
        o.mode = _capi.SN_MODE_ABM if mode == "abm" else _capi.SN_MODE_MAT
        h = C.c_void_p()
        check(lib.sn_engine_create(C.byref(o), C.byref(h)))
        self._h = h
        self.options = o
        self.n_synapses = 0

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.sn_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- building ----
    def add_neurons(self, threshold, leak, reset, refractory, axonal_delay=None) -> int:
        thr = _c(threshold, np.float64)
        lk = _c(leak, np.float64)
        rs = _c(reset, np.float64)
        rf = _c(refractory, np.int32)
        ax = _c(axonal_delay, np.int32)
        first = C.c_int64()
        check(lib.sn_add_neurons(self._h, len(thr), ptr(thr, C.c_double), ptr(lk, C.c_double),
                                 ptr(rs, C.c_double), ptr(rf, C.c_int32), ptr(ax, C.c_int32),
                                 C.byref(first)))
        return first.value

    def add_synapses(self, pre, post, weight, delay=None, stdp=None):
        p = _c(pre, np.int32)
        q = _c(post, np.int32)
        w = _c(weight, np.float64)
        d = _c(delay, np.int32)
        s = _c(stdp, np.uint8)
        check(lib.sn_add_synapses(self._h, len(p), ptr(p, C.c_int32), ptr(q, C.c_int32),
                                  ptr(w, C.c_double), ptr(d, C.c_int32), ptr(s, C.c_uint8)))
        self.n_synapses += len(p)

    def add_stimulus(self, step, neuron, amplitude):
        st = _c(step, np.int32)
        nr = _c(neuron, np.int32)
        am = _c(amplitude, np.float64)
        check(lib.sn_add_stimulus(self._h, len(st), ptr(st, C.c_int32), ptr(nr, C.c_int32),
                                  ptr(am, C.c_double)))

    def clear_stimulus(self):
        check(lib.sn_clear_stimulus(self._h))

    def set_stdp(self, window, a_plus, a_minus, w_min, w_max):
        ap = _c(a_plus, np.float64)
        am = _c(a_minus, np.float64)
        if window >= 1 and (len(ap) != window or len(am) != window):
            raise ValueError("mat_init: stdp: a_plus must have exactly `window` entries"
                             if len(ap) != window else
                             "mat_init: stdp: a_minus must have exactly `window` entries")
        check(lib.sn_set_stdp(self._h, int(window), ptr(ap, C.c_double), ptr(am, C.c_double),
                              float(w_min), float(w_max)))

    def generate_erdos_renyi(self, n, p, seed, weight=1.0, delay_max=1,
                             delay_stream=0x64656C6179, delay_by_synapse_index=False,
                             stdp=False):
        check(lib.sn_generate_erdos_renyi(self._h, int(n), float(p), int(seed) & ((1 << 64) - 1),
                                          float(weight), int(delay_max), int(delay_stream),
                                          1 if delay_by_synapse_index else 0, 1 if stdp else 0))

    # ---- agent-based mode ----
    def set_seed(self, seed: int):
        check(lib.sn_set_seed(self._h, int(seed) & ((1 << 64) - 1)))

    def set_fire_probability(self, fire_probability, first: int = 0):
        fp = _c(fire_probability, np.float64)
        check(lib.sn_set_fire_probability(self._h, int(first), len(fp), ptr(fp, C.c_double)))

    def setup(self):
        check(lib.sn_setup(self._h))

    def simulate(self, steps: int):
        check(lib.sn_simulate(self._h, int(steps)))

    def synchronize(self):
        check(lib.sn_synchronize(self._h))

    def simulate_raster(self, steps: int, out=None):
        """simulate(steps) and that call's raster as (steps, neurons) int32
        arrays; with stream_io the host expands finished chunks while later
        ones run (sn_simulate_raster).  out=(s, q): caller-owned int32 buffers
        of steps * n_local entries each, reused across calls (the returned
        arrays are views of them)."""
        cap = int(steps) * max(1, self.stats()["n_local"])
        if out is None:
            s = np.empty(cap, np.int32)
            q = np.empty(cap, np.int32)
        else:
            s, q = out
            if s.dtype != np.int32 or q.dtype != np.int32 or not (s.flags.c_contiguous and q.flags.c_contiguous):
                raise ValueError("simulate_raster: out must be two C-contiguous int32 arrays")
            cap = min(len(s), len(q))
        cnt = C.c_int64()
        check(lib.sn_simulate_raster(self._h, int(steps), ptr(s, C.c_int32), ptr(q, C.c_int32), cap, C.byref(cnt)))
        return s[:cnt.value], q[:cnt.value]

    def step(self, ext=None) -> np.ndarray:
        """mat_step (mat_engine.cpp:168-208): one step with external input
        exactly `ext` (n amplitudes, or None), then apply_stdp when plasticity
        is on; returns the step's spiking ids ascending."""
        e = None if ext is None else _c(ext, np.float64)
        n = 0 if e is None else len(e)
        cnt = C.c_int64()
        cap = max(1, self.stats()["n_local"])
        out = np.empty(cap, np.int32)
        check(lib.sn_step(self._h, ptr(e, C.c_double) if e is not None else None, n,
                          ptr(out, C.c_int32), cap, C.byref(cnt)))
        return out[:cnt.value].copy()

    def set_plasticity(self, enabled: bool):
        """Whether following steps run apply_stdp after mat_step."""
        check(lib.sn_set_plasticity(self._h, 1 if enabled else 0))

    # ---- results ----
    def raster(self):
        n = C.c_int64()
        check(lib.sn_raster_size(self._h, C.byref(n)))
        steps = np.empty(n.value, np.int32)
        neurons = np.empty(n.value, np.int32)
        check(lib.sn_get_raster(self._h, ptr(steps, C.c_int32), ptr(neurons, C.c_int32), n.value))
        return steps, neurons

    def clear_raster(self):
        check(lib.sn_clear_raster(self._h))

    def stats(self) -> dict:
        s = _capi.Stats()
        check(lib.sn_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        check(lib.sn_reset_stats(self._h))

    def membrane(self) -> np.ndarray:
        nl = self.stats()["n_local"]
        out = np.empty(nl, np.float64)
        check(lib.sn_get_membrane(self._h, ptr(out, C.c_double), nl))
        return out

    def membrane_trace(self) -> np.ndarray:
        rows = C.c_int64()
        check(lib.sn_membrane_trace_rows(self._h, C.byref(rows)))
        nl = self.stats()["n_local"]
        out = np.empty((rows.value, nl), np.float64)
        check(lib.sn_get_membrane_trace(self._h, ptr(out, C.c_double), out.size))
        return out

    def weight_value_counts(self, values) -> np.ndarray:
        """Device census of the dense weight block: counts of each value
        (storage precision), then all other cells."""
        v = _c(values, np.float64)
        out = np.zeros(len(v) + 1, np.int64)
        check(lib.sn_weight_value_counts(self._h, ptr(v, C.c_double), len(v), ptr(out, C.c_int64)))
        return out

    def synapse_weights(self) -> np.ndarray:
        out = np.empty(self.n_synapses, np.float64)
        check(lib.sn_get_synapse_weights(self._h, ptr(out, C.c_double), self.n_synapses))
        return out

    def weight_matrix(self, n: int) -> np.ndarray:
        nl = self.stats()["n_local"]
        out = np.empty((n, nl), np.float64)
        check(lib.sn_get_weight_matrix(self._h, ptr(out, C.c_double), out.size))
        return out

    # ---- partitioned stepping ----
    def comm_init(self, uid: bytes, rank: int, world: int):
        _point_at_torch_nccl()
        buf = (C.c_uint8 * len(uid)).from_buffer_copy(uid)
        check(lib.sn_comm_init(self._h, buf, rank, world))

    def step_local(self):
        check(lib.sn_step_local(self._h))

    def spike_words(self, words: int) -> np.ndarray:
        out = np.empty(words, np.uint32)
        check(lib.sn_get_spike_words(self._h, ptr(out, C.c_uint32), words))
        return out

    def put_spike_words(self, first_word: int, words: np.ndarray):
        w = _c(words, np.uint32)
        check(lib.sn_put_spike_words(self._h, int(first_word), ptr(w, C.c_uint32), len(w)))

    def step_finish(self):
        check(lib.sn_step_finish(self._h))

    # ---- peer-to-peer exchange (fused into the neuron kernel) ----
    def p2p_handles(self) -> bytes:
        size = lib.sn_p2p_handle_size()
        buf = (C.c_uint8 * size)()
        check(lib.sn_p2p_get_handles(self._h, buf, size))
        return bytes(buf)

    def p2p_open(self, all_handles: bytes, world: int):
        buf = (C.c_uint8 * len(all_handles)).from_buffer_copy(all_handles)
        check(lib.sn_p2p_open(self._h, buf, int(world)))


def p2p_connect_local(engines) -> None:
    """Wire `engines` (ranks 0..G-1 of one process, one device) for the
    peer-to-peer exchange protocol (partition emulation)."""
    arr = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
    check(lib.sn_p2p_connect_local(arr, len(engines)))


def _point_at_torch_nccl():
    """NCCL is dlopen'ed by the engine; in a process that also imports torch
    it must be the same libnccl.so.2 torch links (the nvidia-nccl wheel), since
    the first copy loaded owns the soname.  Sets SNB_NCCL_LIB unless given."""
    if os.environ.get("SNB_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for d in (list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []):
        path = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(path):
            os.environ["SNB_NCCL_LIB"] = path
            return


def comm_unique_id() -> bytes:
    _point_at_torch_nccl()
    size = lib.sn_comm_id_size()
    buf = (C.c_uint8 * size)()
    check(lib.sn_comm_create_id(buf))
    return bytes(buf)


def partition_range(n: int, rank: int, world: int):
    f, c = C.c_int32(), C.c_int32()
    check(lib.sn_partition_range(int(n), int(rank), int(world), C.byref(f), C.byref(c)))
    return f.value, c.value


def device_count() -> int:
    return int(lib.sn_device_count())


def stdp_defaults():
    w = C.c_int32()
    check(lib.sn_stdp_defaults(C.byref(w), None, None, None, None))
    ap = np.empty(w.value, np.float64)
    am = np.empty(w.value, np.float64)
    wmin, wmax = C.c_double(), C.c_double()
    check(lib.sn_stdp_defaults(C.byref(w), ptr(ap, C.c_double), ptr(am, C.c_double),
                               C.byref(wmin), C.byref(wmax)))
    return w.value, ap, am, wmin.value, wmax.value
