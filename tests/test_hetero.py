"""vnt::hetero — heterogeneous planning (reference hetero.hpp / test_hetero.cpp).

CPU: the C++ suite (tests/cpp/test_hetero.cpp) and, on random instances, our
solver against the reference's own solver compiled in oracle/_ref (best
assignment, predicted time bit-for-bit, number of feasible candidates, and
the Infeasible/Config error classes).
GPU: profile_device measures real B200 step times and the solver plans from
them."""
import ctypes as C
import random
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

u64p, u32p, f64p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_double)


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


def _solve(fn, types, B, max_v=64, collect=True):
    n = len(types)
    names = (C.c_char_p * n)(*[t["name"].encode() for t in types])
    counts = (C.c_uint64 * n)(*[t["count"] for t in types])
    caps = (C.c_uint64 * n)(*[t["cap"] for t in types])
    comm = (C.c_double * n)(*[t["comm"] for t in types])
    npts = (C.c_uint32 * n)(*[len(t["points"]) for t in types])
    pb = [b for t in types for b, _ in t["points"]]
    pt = [s for t in types for _, s in t["points"]]
    pbatch = (C.c_uint64 * max(1, len(pb)))(*pb)
    ptime = (C.c_double * max(1, len(pt)))(*pt)
    ot, on, ob, ov = (C.c_uint32 * n)(), (C.c_uint64 * n)(), (C.c_uint64 * n)(), (C.c_uint64 * n)()
    nt, tm, cand = C.c_uint32(), C.c_double(), C.c_uint64()
    rc = fn(C.c_uint32(n), names, counts, caps, comm, npts, pbatch, ptime, C.c_uint64(B),
            C.c_uint64(max_v), C.c_int32(1 if collect else 0), C.byref(nt), ot, on, ob, ov,
            C.byref(tm), C.byref(cand))
    if rc:
        return rc, None
    best = [(types[ot[j]]["name"], on[j], ob[j], ov[j]) for j in range(nt.value)]
    return 0, (best, tm.value, cand.value)


def _instance(rng):
    types = []
    for name in rng.sample(["A", "B", "C", "D"], rng.randint(1, 3)):
        cap = rng.choice([2, 4, 6, 8, 12, 16, 32, 64])
        sizes = sorted(rng.sample(range(1, 65), rng.randint(1, 7)))
        fixed, per = rng.uniform(0, 0.01), rng.uniform(1e-4, 2e-3)
        # some measured-looking curves are not linear: jitter a few points
        pts = [(b, fixed + per * b * (1.0 + (rng.random() - 0.5) * 0.2 * (rng.random() < 0.5)))
               for b in sizes]
        types.append(dict(name=name, count=rng.randint(0, 4), cap=cap, comm=rng.uniform(0, 0.02),
                          points=pts))
    if all(t["count"] == 0 for t in types):
        types[0]["count"] = 1
    max_v = rng.choice([1, 2, 4, 64])
    if rng.random() < 0.25:
        return types, rng.randint(1, 96), max_v     # often infeasible
    B = 0                                           # a reachable batch
    for t in types:
        fits = [b for b, _ in t["points"] if b <= t["cap"]]
        if t["count"] and fits and rng.random() < 0.8:
            v = 2 ** rng.randint(0, min(2, max_v.bit_length() - 1))
            B += rng.randint(1, t["count"]) * rng.choice(fits) * v
    return types, max(B, 1), max_v


def test_solver_matches_reference_solver(ref):
    if ref is None:
        pytest.skip("oracle/_ref not built")
    ours = _host().vnt_hetero_solve
    theirs = ref.lib.vntref_hetero_solve
    rng = random.Random(2009)
    seen = {"ok": 0, "infeasible": 0}
    for _ in range(400):
        types, B, max_v = _instance(rng)
        a = _solve(ours, types, B, max_v)
        b = _solve(theirs, types, B, max_v)
        assert a[0] == b[0], (types, B, a, b)
        if a[0] == 0:
            assert a[1] == b[1], (types, B, a, b)   # best tuples, time (bitwise), candidate count
            seen["ok"] += 1
        else:
            assert a[0] in (2, 5)
            seen["infeasible"] += a[0] == 5
    assert seen["ok"] > 100 and seen["infeasible"] > 10


@pytest.mark.gpu
def test_profile_device_feeds_the_solver():
    """Measured B200 curve for the cfg1 model, then a plan for B=256 on 8 devices."""
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
    rc, res = _solve(lib.vnt_hetero_solve,
                     [dict(name="B200", count=8, cap=64, comm=comm.value, points=pts)], 256)
    assert rc == 0
    best, t, cand = res
    (name, n, b, v), = best
    assert name == "B200" and n * b == 256 and b % v == 0 and b // v <= 64
    times = dict(pts)
    want = times[b // v] * v + (comm.value if n >= 2 else 0.0)
    assert t == want and cand > 0
