"""distributed.run_partitioned as real processes: two ranks over gloo (the
host transport: each step's spike words all-gathered through
torch.distributed, no kernel waits on another process, so both ranks can
share the one GPU of this box), against the reference oracle."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from paper_2305_02510_b200.model import NetworkDef, SimulationConfig, StdpConfig, StimulusSchedule
    from paper_2305_02510_b200.netgen import RandomStream, erdos_renyi_arrays, scenario_stimulus
    n, p, seed, steps = 300, 0.06, 32, 60
    pre, post = erdos_renyi_arrays(n, p, seed)
    m = len(pre)
    rs = RandomStream(seed, 9)
    k = np.arange(m, dtype=np.uint64)
    net = NetworkDef.from_arrays(np.full(n, 1.5), np.full(n, 0.3), np.zeros(n), np.ones(n, np.int32), pre, post,
                                 -0.3 + 1.2 * rs.unit_np(k), delay=(1 + rs.below_np(k + np.uint64(m), 4)),
                                 stdp=(rs.unit_np(k + np.uint64(2 * m)) < 0.7).astype(np.uint8))
    stim = scenario_stimulus(n, steps, seed, count=12, period=2, amplitude=2.5)
    return net, SimulationConfig(steps=steps, stdp=StdpConfig.defaults()), stim


def _worker(rank, world, port, storage, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_02510_b200.distributed import run_partitioned
        net, cfg, stim = _problem()
        res = run_partitioned(net, cfg, stim, rank=rank, world=world, device=0, transport="host",
                              storage=storage, precision="f64")
        if rank == 0:
            np.savez(out_path, steps=res.raster.steps_array, neurons=res.raster.neurons_array)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("storage", [1, 2])
def test_run_partitioned_two_processes_host_transport(tmp_path, storage):
    import torch.multiprocessing as mp
    from oracle import bridge as B
    out = str(tmp_path / "r0.npz")
    mp.start_processes(_worker, args=(2, _port(), storage, out), nprocs=2, start_method="spawn", join=True)
    net, cfg, stim = _problem()
    a = net.to_arrays()
    s = cfg.stdp
    o = B.run_oracle(a, cfg.steps, stim.to_arrays(), (s.window, np.array(s.a_plus), np.array(s.a_minus), s.w_min, s.w_max))
    r = np.load(out)
    assert len(o["steps"]) > 1000
    assert (o["neurons"] >= 160).sum() > 100        # rank 1 (posts 160..299) spikes too
    assert np.array_equal(r["steps"], o["steps"]) and np.array_equal(r["neurons"], o["neurons"])
