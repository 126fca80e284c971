"""The k_sparse_count8 list layout, built by the fill code itself run on the
host (tools/c16_fill_check.cu compiles csrc/k_sparse.cu's c16_fill_group for
the CPU; no GPU): every synapse of a (post, pre block) list lands exactly once
in its post's chunks of the right segment as `slot << 4 | d - 1`, the rest of
the chunks are the segment's zero slot, and the per-LDS bank assignment keeps
the shared-memory wavefronts near the matched level."""
import os
import shutil
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.skipif(shutil.which("nvcc") is None, reason="needs nvcc for the host harness")


@pytest.fixture(scope="module")
def harness():
    import c16_fill_sim as F
    tmp = tempfile.mkdtemp()
    return F, F.build_harness(tmp), tmp


@pytest.mark.parametrize("p", [0.01, 0.003, 0.05])
def test_every_synapse_placed_once_in_its_segment(harness, p):
    F, exe, tmp = harness
    groups = 24
    posts, lists, ent = F.run_fill(exe, tmp, groups, seed=int(p * 1000), p=p)
    placed = [dict() for _ in posts]          # post -> {(segment, entry): count}
    pads = 0
    for g, _, lanes in F.walk(posts, ent, groups):
        for i, _, s, row in lanes:
            for v in row.tolist():
                if v >> 4 == F.zero(s):       # the segment's zero slot: padding
                    pads += 1
                    continue
                key = (s, v)
                placed[g * F.P + i][key] = placed[g * F.P + i].get(key, 0) + 1
    for k, (pl, dm1) in enumerate(lists):
        want = {}
        for a, d in zip(pl.tolist(), dm1.tolist()):
            s = a // F.SEGP
            low = a - s * F.SEGP
            slot = low + (1 if low >= F.zero(s) else 0)
            want[(s, slot << 4 | d)] = want.get((s, slot << 4 | d), 0) + 1
        assert placed[k] == want, k
    chunks = sum(c for c, _, _ in posts)
    assert pads == 8 * chunks - sum(len(pl) for pl, _ in lists)


def test_bank_matching_keeps_wavefronts_low(harness):
    F, exe, tmp = harness
    posts, _, ent = F.run_fill(exe, tmp, 60)
    w, _ = F.wavefronts(posts, ent, 60)
    assert w < 1.6   # 1.53 with the matched fill; 1.79 with the greedy order alone
