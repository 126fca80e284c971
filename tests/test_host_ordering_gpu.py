"""Host/stream ordering of the engine's synchronous uploads and reads.

The engine runs on a non-blocking stream; a pageable cudaMemcpy H2D runs on
the legacy default stream and may return before its DMA lands.  Here other
processes time-share the GPU (as pytest -n 4 did when an 8,000-case fuzz run
caught the race) and the copy engines are kept busy by large pinned H2D copies
on a side stream, while a stimulus table is uploaded right before a single
graph-captured simulate(): every run must still see the step-0 stimulus and
match the chain's known raster."""
from __future__ import annotations

import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_stimulus_upload_is_ordered_before_the_first_step():
    import torch
    from paper_2305_02510_b200.engine import MatEngine
    big = torch.empty(1 << 27, dtype=torch.uint8).pin_memory()
    dev = torch.empty(big.shape, dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    hog = ("import torch,time\n"
           "a=torch.randn(4096,4096,device='cuda'); torch.cuda.synchronize(); print('ready', flush=True)\n"
           "t=time.time()\n"
           "while time.time()-t<30: a=(a@a).clamp_(-1,1); torch.cuda.synchronize()\n")
    hogs = [subprocess.Popen([sys.executable, "-c", hog], stdout=subprocess.PIPE, text=True) for _ in range(3)]
    for h in hogs:
        h.stdout.readline()
    n, steps = 8, 30
    # chain 0 -> 1 -> ... -> 7, unit weights, threshold 0.5, no leak effect:
    # a kick of neuron 0 at step 0 fires neuron k at step k (mat_engine.cpp:168-208)
    want = [(k, k) for k in range(n)]
    try:
        _chain_trials(MatEngine, big, dev, side, n, steps, want, 96)
    finally:
        for h in hogs:
            h.kill()
            h.wait()


def _chain_trials(MatEngine, big, dev, side, n, steps, want, trials):
    import torch
    for trial in range(trials):
        eng = MatEngine(use_graphs=True, persistent=bool(trial % 2), storage=trial % 3)
        try:
            eng.add_neurons(np.full(n, 0.5), np.full(n, np.inf), np.zeros(n), np.zeros(n, np.int32))
            eng.add_synapses(np.arange(n - 1, dtype=np.int32), np.arange(1, n, dtype=np.int32), np.ones(n - 1))
            eng.setup()
            with torch.cuda.stream(side):
                for _ in range(4):
                    dev.copy_(big, non_blocking=True)
            eng.add_stimulus(np.array([0], np.int32), np.array([0], np.int32), np.array([2.0]))
            eng.simulate(steps)
            s, q = eng.raster()
        finally:
            eng.close()
        side.synchronize()
        assert list(zip(s.tolist(), q.tolist())) == want, (trial, s, q)
