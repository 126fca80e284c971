"""Shared-memory wavefronts per LDS of the k_sparse_count8 list layout, from
the fill code itself run on the host (tools/c16_fill_check.cu): random
cfg4-shaped lists (p = 0.01 over a 3 x 4095-pre block, delays 1..16, SUB = 4,
8 posts per warp group), the kernel's LDS order (row-major chunk stream, entry
e of every active lane's chunk per LDS), banks = 4-byte words mod 32 with
same-word broadcast.  Usage: python tools/c16_fill_sim.py [groups]"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEGP, SUB, P = 4095, 4, 8


def zero(s):
    return 4095 - 16 * s


def build_harness(tmp):
    exe = os.path.join(tmp, "c16_fill_check")
    subprocess.run(["nvcc", "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                    "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "paper_2305_02510_b200", "csrc"),
                    "-I" + os.path.join(ROOT, "include"), "-o", exe,
                    os.path.join(ROOT, "tools", "c16_fill_check.cu")], check=True, capture_output=True)
    return exe


def run_fill(exe, tmp, groups, seed=7, p=0.01):
    """Random cfg4-shaped lists of `groups` warp groups through the fill.
    Returns (posts, lists, ent): per post (C, E1, E2), its (pre_local, d-1)
    entries, and the filled 16-bit chunk stream [chunks][8]."""
    rng = np.random.default_rng(seed)
    posts, lists = [], []
    buf = [np.int32(groups).tobytes()]
    for _ in range(groups * P):
        m = rng.binomial(3 * SEGP, p)
        pl = np.sort(rng.choice(3 * SEGP, m, replace=False))
        dm1 = rng.integers(0, 16, m)
        n = np.bincount(pl // SEGP, minlength=3)
        e = np.cumsum((n + 7) // 8)
        y = int(e[0]) | int(e[1]) << 8 | int(e[2]) << 16 | int(e[2]) << 24
        posts.append((int(e[2]), int(e[0]), int(e[1])))
        lists.append((pl, dm1))
        buf += [np.array([y, m], np.uint32).tobytes(), (pl | dm1 << 16).astype(np.uint32).tobytes()]
    inp, outp = os.path.join(tmp, "in.bin"), os.path.join(tmp, "out.bin")
    with open(inp, "wb") as f:
        f.write(b"".join(buf))
    subprocess.run([exe, inp, outp], check=True)
    return posts, lists, np.fromfile(outp, np.uint16).reshape(-1, 8)


def walk(posts, ent, groups):
    """The kernel's reading order: yields (group, row, [(post i, chunk c, segment, 8 entries)])."""
    pos = 0
    for g in range(groups):
        grp = posts[g * P:(g + 1) * P]
        rows = (max(c for c, _, _ in grp) + SUB - 1) // SUB
        for r in range(rows):
            lanes = [(i, r * SUB + sl) for i in range(P) for sl in range(SUB) if r * SUB + sl < grp[i][0]]
            yield g, r, [(i, c, int(c >= grp[i][1]) + int(c >= grp[i][2]), ent[pos + q])
                         for q, (i, c) in enumerate(lanes)]
            pos += len(lanes)


def wavefronts(posts, ent, groups):
    wf, lds = 0, 0
    for _, _, lanes in walk(posts, ent, groups):
        for e in range(8):
            words = {(s << 16 | int(row[e])) >> 2 for _, _, s, row in lanes}
            wf += np.bincount([w & 31 for w in words], minlength=32).max()
            lds += 1
    return wf / lds, lds


def main(groups):
    tmp = tempfile.mkdtemp()
    exe = build_harness(tmp)
    posts, _, ent = run_fill(exe, tmp, groups)
    w, lds = wavefronts(posts, ent, groups)
    print(f"{groups} warp groups, {lds} LDS: {w:.3f} shared-memory wavefronts per LDS (ideal 1)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 200)
