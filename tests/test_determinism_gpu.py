"""Race detection without compute-sanitizer (closed on this GPU pool): each
hot kernel's case from tools/sanitize_cases.py runs several times in one
process, interleaved with other engines' work, and every repeat must be
bitwise identical -- rasters, membranes and weights -- and equal to the
oracle's raster.  The mbarrier rings (k_dense_tma), the DSMEM exchange
(k_cluster_count), the shared-memory loop (k_tiny), the 16-bit lists
(k_sparse_count16), the staged pull (k_sparse_pull) and the p2p partition
exchange are all deterministic by construction (fixed reduction orders), so
any difference is a race.  `SNB_LIB=paper_2305_02510_b200/libsnmat_checked.so`
runs the same tests on the checked build (device bounds checks, trapping
mbarrier waits; tools/build_variant.sh checked -DSNB_CHECKED)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def _run(name):
    import sanitize_cases as S
    from oracle import bridge as B
    pa, opts, want = S.CASES[name]
    arrays, stim, sd = S.problem(**pa)
    e = S.engine(arrays, sd, **opts)
    e.add_stimulus(*stim)
    e.simulate(pa["steps"])
    s, q = e.raster()
    out = (s, q, e.membrane(), e.synapse_weights(), e.stats()["sweep_kernel"])
    e.close()
    return out


@pytest.mark.parametrize("name", ["dense_tma", "dense_tma_delay", "cluster", "tiny", "count16", "sparse_pull"])
def test_repeated_runs_bitwise_identical(name):
    import sanitize_cases as S
    from oracle import bridge as B
    pa, opts, want = S.CASES[name]
    arrays, stim, sd = S.problem(**pa)
    o = B.run_oracle(arrays, pa["steps"], stim, sd)
    first = _run(name)
    assert first[4] == want
    assert np.array_equal(first[0], o["steps"]) and np.array_equal(first[1], o["neurons"])
    for rep in range(4):
        if rep % 2:   # interleave another engine's kernels between repeats
            _run("tiny")
        again = _run(name)
        for a, b in zip(first[:4], again[:4]):
            assert np.array_equal(a, b), (name, rep)


def test_p2p_partitions_repeat_identically():
    import subprocess
    outs = [subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), "p2p"],
                           capture_output=True, text=True, timeout=300) for _ in range(3)]
    for r in outs:
        assert r.returncode == 0, r.stdout + r.stderr
    assert len({r.stdout for r in outs}) == 1
