"""CPU, world_size = 2 (and 3) over gloo: the multi-rank host logic of the
N > 1 path -- post partition ranges (the engine's own sn_partition_range),
spike-word packing, the host all-gather transport and the raster merge of
paper_2305_02510_b200.distributed -- driving a numpy per-partition LIF step.
The merged raster must equal the oracle's (integer nets, delays included)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _leak(v, leak, reset):
    d = v - reset
    out = v.copy()
    pos = d > 0
    neg = d < 0
    with np.errstate(invalid="ignore"):
        out[pos] = reset[pos] + np.maximum(d[pos] - leak[pos], 0.0)
        out[neg] = reset[neg] + np.minimum(d[neg] + leak[neg], 0.0)
    return out


def _worker(rank, world, port, seeds, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch.distributed as dist
    from support import random_net, random_stim
    from paper_2305_02510_b200 import distributed as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for seed in seeds:
            net = random_net(seed, max_neurons=40, edge_prob=0.3, max_delay=4, max_axonal=1)
            a = net.to_arrays()
            n = len(a["threshold"])
            steps = 120
            stim = random_stim(seed, n, steps, 60).to_arrays()
            first, count = D.partition_ranges(n, world)[rank]
            wpr = D.words_per_rank(n, world)
            # this rank's columns of W, one matrix per effective delay
            deff = a["delay"] + a["axonal"][a["pre"]]
            dmax = int(deff.max()) if len(deff) else 1
            Wd = np.zeros((dmax + 1, n, count))
            for s in range(len(a["pre"])):
                j = a["post"][s]
                if first <= j < first + count:
                    Wd[deff[s], a["pre"][s], j - first] += a["weight"][s]
            sl = slice(first, first + count)
            v = a["reset"][sl].copy()
            cnt = np.zeros(count, np.int64)
            hist = [np.zeros(n, bool) for _ in range(dmax + 1)]   # hist[k] = s[t-1-k]
            ext_by_t = {}
            for st, nr, am in zip(*stim):
                ext_by_t.setdefault(int(st), []).append((int(nr), float(am)))
            ev_s, ev_n = [], []
            for t in range(steps):
                u = _leak(v, a["leak"][sl], a["reset"][sl])
                for d in range(1, dmax + 1):
                    u = u + hist[d - 1].astype(float) @ Wd[d]
                if t in ext_by_t:
                    ext = np.zeros(n)
                    for nr, am in ext_by_t[t]:
                        ext[nr] += am
                    u = u + ext[sl]
                s = u > a["threshold"][sl]
                refr = cnt > 0
                s[refr] = False
                cnt[refr] -= 1
                u[refr] = a["reset"][sl][refr]
                v = np.where(s, a["reset"][sl], u)
                cnt = np.where(s, a["refractory"][sl], cnt)
                full = D.unpack_words(D.allgather_words(D.pack_words(s, wpr)), world * wpr * 32)[:n]
                hist = [full] + hist[:-1]
                for j in np.nonzero(s)[0]:
                    ev_s.append(t)
                    ev_n.append(first + j)
            steps_m, neurons_m = D.gather_raster(np.array(ev_s, np.int32), np.array(ev_n, np.int32))
            results.append((seed, steps_m, neurons_m))
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_host_logic_matches_oracle(world):
    from oracle import bridge as B
    from support import random_net, random_stim
    seeds = [300, 301, 302, 7, 8]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seeds, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for seed, steps_m, neurons_m in results:
        net = random_net(seed, max_neurons=40, edge_prob=0.3, max_delay=4, max_axonal=1)
        o = B.run_oracle(net.to_arrays(), 120, random_stim(seed, net.neuron_count(), 120, 60).to_arrays())
        assert len(o["steps"]) > 0
        assert np.array_equal(steps_m, o["steps"]), seed
        assert np.array_equal(neurons_m, o["neurons"]), seed


def test_word_packing_roundtrip_and_merge():
    from paper_2305_02510_b200 import distributed as D
    rng = np.random.default_rng(0)
    for n in (1, 31, 33, 100):
        s = rng.random(n) < 0.4
        words = D.pack_words(s, (n + 31) // 32)
        assert np.array_equal(D.unpack_words(words, n), s)
    a = (np.array([0, 0, 2], np.int32), np.array([1, 5, 3], np.int32))
    b = (np.array([0, 1], np.int32), np.array([40, 33], np.int32))
    st, nr = D.merge_rasters([a, b])
    assert list(zip(st.tolist(), nr.tolist())) == [(0, 1), (0, 5), (0, 40), (1, 33), (2, 3)]


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch.distributed as dist
    from paper_2305_02510_b200 import distributed as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = D.broadcast_uid(bytes(range(128)) if rank == 0 else None)
        handles = D.exchange_p2p_handles(bytes([rank]) * 128)
        q.put((rank, uid, handles))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_communicator_id_and_p2p_handle_exchange(world):
    """bench.py's connect(): rank 0's NCCL unique id reaches every rank, and
    every rank receives all ranks' IPC handle blocks in rank order (the layout
    sn_p2p_open expects)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = b"".join(bytes([r]) * 128 for r in range(world))
    for rank, uid, handles in got:
        assert uid == bytes(range(128))
        assert handles == expect
