"""Multi-GPU driver: one process per GPU, posts partitioned into contiguous
32-aligned ranges.  Per step the only exchange is the spike
bitmask of the step (N/8 bytes): inside the engine with NCCL
(``transport="nccl"``, one in-place ncclAllGather captured with the step), or
host-driven through ``torch.distributed`` (``transport="host"``; works with
the gloo backend, used by the CPU tests and as a fallback transport).

Rank 0 returns the merged RunResult; the raster of each rank is ascending and
the ranges are ascending, so merging is a per-step concatenation.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .engine import MatEngine, comm_unique_id, partition_range
from .model import (NetworkDef, RunResult, SimulationConfig, SpikeRaster, StimulusSchedule,
                    throw_first, validate_stimulus)


def partition_ranges(n: int, world: int) -> List[Tuple[int, int]]:
    """(first, count) per rank -- the engine's own partition (sn_partition_range)."""
    return [partition_range(n, r, world) for r in range(world)]


def words_per_rank(n: int, world: int) -> int:
    """Spike words per rank slice: rank 0's range rounded up to whole words."""
    return (max(partition_ranges(n, world)[0][1], 1) + 31) // 32


def pack_words(spikes: np.ndarray, words: int) -> np.ndarray:
    """bool spikes of a rank's posts -> its uint32 words (bit b of word w = post 32w+b)."""
    padded = np.zeros(words * 32, dtype=np.uint8)
    padded[:len(spikes)] = spikes.astype(np.uint8)
    bits = padded.reshape(words, 32)
    return (bits.astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)


def unpack_words(words: np.ndarray, n: int) -> np.ndarray:
    w = np.asarray(words, dtype=np.uint32).astype(np.uint64)
    bits = (w[:, None] >> np.arange(32, dtype=np.uint64)) & np.uint64(1)
    return bits.reshape(-1)[:n].astype(bool)


def allgather_words(local: np.ndarray, group=None) -> np.ndarray:
    """Host all-gather of every rank's spike words (equal-size slices) -> full bitmask."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.uint32).view(np.int32).copy())
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return torch.cat(out).numpy().view(np.uint32)


def broadcast_uid(uid: Optional[bytes], src: int = 0, group=None) -> bytes:
    import torch.distributed as dist
    box = [uid]
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]


def exchange_p2p_handles(mine: bytes, group=None) -> bytes:
    """All-gather every rank's 128-byte IPC handle block, rank-major, for sn_p2p_open."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    if any(len(p) != len(mine) for p in parts):
        raise RuntimeError("p2p handle blocks differ in size across ranks")
    return b"".join(parts)


def merge_rasters(parts: Sequence[Tuple[np.ndarray, np.ndarray]]) -> Tuple[np.ndarray, np.ndarray]:
    """Per-rank (steps, neurons) rasters -> one raster ascending by (step, neuron)."""
    if not parts:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    steps = np.concatenate([np.asarray(p[0], np.int32) for p in parts])
    neurons = np.concatenate([np.asarray(p[1], np.int32) for p in parts])
    order = np.lexsort((neurons, steps))
    return steps[order], neurons[order]


def gather_raster(steps: np.ndarray, neurons: np.ndarray, group=None):
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, (steps, neurons), group=group)
    return merge_rasters(parts)


def run_partitioned(net: NetworkDef, cfg: SimulationConfig, stim: Optional[StimulusSchedule] = None,
                    *, rank: int, world: int, device: int, transport: str = "nccl",
                    group=None, **engine_opts) -> Optional[RunResult]:
    """mat_run over `world` GPUs (this process = `rank`); rank 0 gets the result."""
    stim = stim or StimulusSchedule()
    if cfg.steps < 1:
        raise ValueError("mat_run: steps must be >= 1")
    a = net.to_arrays()
    n = a["threshold"].shape[0]
    throw_first("mat_run", validate_stimulus(stim, n, cfg.steps))
    eng = MatEngine(device=device, rank=rank, world=world, record_membrane=cfg.record_membrane,
                    **engine_opts)
    eng.add_neurons(a["threshold"], a["leak"], a["reset"], a["refractory"], a["axonal"])
    if a["pre"].shape[0]:
        eng.add_synapses(a["pre"], a["post"], a["weight"], a["delay"], a["stdp"])
    if cfg.stdp is not None:
        s = cfg.stdp
        eng.set_stdp(s.window, s.a_plus, s.a_minus, s.w_min, s.w_max)
    eng.setup()
    if stim.entries:
        eng.add_stimulus(*stim.to_arrays())
    if transport == "nccl":
        uid = broadcast_uid(comm_unique_id() if rank == 0 else None, group=group)
        eng.comm_init(uid, rank, world)
        eng.simulate(cfg.steps)
    elif transport == "p2p":
        eng.p2p_open(exchange_p2p_handles(eng.p2p_handles(), group), world)
        eng.simulate(cfg.steps)
    elif transport == "host":
        wpr = words_per_rank(n, world)
        for _ in range(cfg.steps):
            eng.step_local()
            mine = eng.spike_words(wpr * world)[rank * wpr:(rank + 1) * wpr]
            full = allgather_words(mine, group)
            for q in range(world):
                if q != rank:
                    eng.put_spike_words(q * wpr, full[q * wpr:(q + 1) * wpr])
            eng.step_finish()
    else:
        raise ValueError(f"unknown transport {transport!r}")
    steps, neurons = gather_raster(*eng.raster(), group=group)
    eng.close()
    if rank != 0:
        return None
    return RunResult(raster=SpikeRaster(neuron_count=n, step_count=cfg.steps,
                                        steps_array=steps, neurons_array=neurons))
