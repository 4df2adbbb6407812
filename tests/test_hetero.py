"""vnt::hetero — the two pieces on the training path (include/vnt/hetero.hpp):
assignment expansion into a VirtualNodeMapping (C++ suite, CPU) and the
measured B200 profile (profile_device, GPU)."""
import ctypes as C
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _host():
    import paper_2009_09523_b200 as vnt
    if not vnt.HOST_SO.exists():
        from paper_2009_09523_b200 import build as b
        b.build_host()
    vnt.load_engine()
    lib = C.CDLL(str(vnt.HOST_SO))
    lib.vnt_host_last_error.restype = C.c_char_p
    return lib


def test_cpp_hetero_suite():
    exe = ROOT / "build" / "tests" / "test_hetero"
    if not exe.exists():
        from paper_2009_09523_b200 import build as b
        b.build_host()
        b.build_cpp_tests()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_profile_device_measures_b200_steps():
    """Measured B200 curve for the cfg1 model: one point per batch size up to
    the capacity (larger sizes skipped), positive times growing with rows."""
    lib = _host()
    w = (C.c_uint64 * 3)(784, 16, 10)
    sizes = [1, 2, 4, 8, 16, 32, 64, 128]
    bs = (C.c_uint64 * len(sizes))(*sizes)
    ob, ot = (C.c_uint64 * len(sizes))(), (C.c_double * len(sizes))()
    npts, comm = C.c_uint32(), C.c_double()
    rc = lib.vnt_hetero_profile_device(w, 3, 1, 1, C.c_uint64(11), b"B200", C.c_uint64(64), bs,
                                       len(sizes), C.c_uint64(20), C.c_uint64(5), 0, 0, ob, ot,
                                       C.byref(npts), C.byref(comm))
    assert rc == 0, lib.vnt_host_last_error()
    assert npts.value == 7                         # 128 > capacity 64: skipped
    pts = [(ob[k], ot[k]) for k in range(npts.value)]
    print("B200 profile:", [(b, round(t * 1e6, 1)) for b, t in pts], "comm", comm.value)
    assert [b for b, _ in pts] == sizes[:7]
    assert all(0 < t < 0.05 for _, t in pts)
    assert comm.value >= 0
