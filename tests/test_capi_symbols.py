"""CPU checks of the C-ABI boundary: the engine library loads without a GPU,
exports exactly what include/superneuro_mat.h declares, and fails cleanly
(status + message, no crash) when no device is present."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "superneuro_mat.h")


def header_functions():
    txt = open(HEADER).read()
    return set(re.findall(r"^SN_API\s+[\w\s\*]+?\b(sn_\w+)\s*\(", txt, flags=re.M))


def test_header_declares_the_boundary():
    fns = header_functions()
    for need in ("sn_engine_create", "sn_add_neurons", "sn_add_synapses", "sn_add_stimulus",
                 "sn_set_stdp", "sn_setup", "sn_simulate", "sn_get_raster", "sn_get_membrane",
                 "sn_get_synapse_weights", "sn_last_error", "sn_engine_destroy", "sn_comm_init"):
        assert need in fns


def test_library_exports_every_declared_symbol():
    from paper_2305_02510_b200 import _capi
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (sn_\w+)", out))
    declared = header_functions()
    assert declared <= exported, declared - exported
    assert exported <= declared, exported - declared     # nothing undocumented
    assert declared == set(_capi.SIGNATURES)             # the Python binding covers it all


def test_library_is_sm100a():
    from paper_2305_02510_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_errors_are_clean():
    import paper_2305_02510_b200 as sn
    from paper_2305_02510_b200 import _capi
    if sn.device_count() > 0:
        pytest.skip("a GPU is visible; this checks the CPU-only failure path")
    with pytest.raises((ValueError, _capi.CudaError)) as ei:
        sn.MatEngine()
    assert "device" in str(ei.value).lower() or "cuda" in str(ei.value).lower()


def test_options_and_partition_math():
    import paper_2305_02510_b200 as sn
    from paper_2305_02510_b200 import _capi
    o = _capi.Options()
    assert _capi.lib.sn_options_init(C.byref(o)) == 0
    assert o.abi_version == _capi.SN_ABI_VERSION and o.world == 1 and o.use_graphs == 1
    for n in (1, 31, 32, 100, 1000, 32000, 256000, 96000):
        for world in (1, 2, 3, 4, 8):
            parts = [sn.partition_range(n, r, world) for r in range(world)]
            firsts = [f for f, _ in parts]
            counts = [c for _, c in parts]
            assert sum(counts) == n
            for r in range(world):
                assert firsts[r] % 32 == 0 or counts[r] == 0
                if r + 1 < world and counts[r + 1]:
                    assert firsts[r] + counts[r] == firsts[r + 1]
    with pytest.raises(ValueError):
        sn.partition_range(10, 2, 2)


def test_stdp_defaults_match_reference_defaults():
    import paper_2305_02510_b200 as sn
    w, ap, am, lo, hi = sn.stdp_defaults()
    d = sn.StdpConfig.defaults()
    assert w == d.window == 20 and lo == 0.0 and hi == 1.0
    assert list(ap) == d.a_plus and list(am) == d.a_minus
    from oracle import bridge as B
    if B.ref_available():
        lib = B.ref_lib()
        rw = C.c_int32()
        rap = (C.c_double * 20)()
        ram = (C.c_double * 20)()
        rlo, rhi = C.c_double(), C.c_double()
        lib.ref_stdp_defaults(C.byref(rw), rap, ram, C.byref(rlo), C.byref(rhi))
        assert list(rap) == list(ap) and list(ram) == list(am)


def test_missing_engine_library_fails_loudly(tmp_path):
    """No CPU fallback: without libsnmat.so the package refuses to import."""
    env = dict(os.environ, SNB_LIB=str(tmp_path / "absent" / "libsnmat.so"))
    r = subprocess.run(["python", "-c", "import paper_2305_02510_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "is missing" in r.stderr and "ImportError" in r.stderr
