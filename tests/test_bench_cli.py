"""bench.py's launcher contract on CPU: `--gpus N` outside torchrun re-execs
under torch.distributed.run only when the node has N GPUs, and a torchrun
world that disagrees with --gpus is refused (no silent single-GPU run)."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, env=env, timeout=300)


def test_gpus_n_needs_n_devices():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    r = _bench(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert "--gpus 2 needs 2 GPUs" in r.stderr


def test_world_mismatch_refused():
    r = _bench(["--gpus", "4", "--steps", "1", "--warmup", "3"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in r.stderr


def test_reference_arm_cfg1_line():
    """--impl reference on the CPU-runnable config: the reference's own loop,
    one JSON line with the contract keys and the steps actually timed."""
    import json
    from oracle import bridge as B
    if not B.ref_available():
        pytest.skip("oracle/_ref not built")
    r = _bench(["--impl", "reference", "--workload", "cfg1", "--steps", "50", "--warmup", "3"])
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["same_config"] is True and d["steps"] == 50 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["value"] == d["value"] > 0
