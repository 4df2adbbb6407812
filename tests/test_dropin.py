"""The C++ drop-in `vnt::` API (include/vnt/*.hpp, libvnt.so).

CPU: C++ host tests (tests/cpp/test_host.cpp) and the host-only C-ABI
(SynthDataset, init) bit-identical to the reference oracle.
GPU: C++ drop-in tests mirroring the reference suites
(tests/cpp/test_dropin_gpu.cpp) and the drop-in Trainer, through
include/vnt_trainer.h, against the reference Trainer (oracle/_ref or port)."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
BUILD = ROOT / "build" / "tests"


def _bin(name):
    p = BUILD / name
    if not p.exists():
        from paper_2009_09523_b200 import build as b
        b.build_host()
        b.build_cpp_tests()
    return p


def _host():
    import paper_2009_09523_b200 as vnt
    if not vnt.HOST_SO.exists():
        from paper_2009_09523_b200 import build as b
        b.build_host()
    vnt.load_engine()
    lib = C.CDLL(str(vnt.HOST_SO))
    lib.vnt_host_last_error.restype = C.c_char_p
    return lib


def test_cpp_host_suite():
    r = subprocess.run([str(_bin("test_host"))], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_host_data_and_init_bit_identical_to_reference(port):
    lib = _host()
    f64p = C.POINTER(C.c_double)
    for (seed, n, i, o, start, cnt) in [(11, 64, 4, 4, 5, 20), (11, 60000, 784, 10, 59990, 16)]:
        x = np.empty((cnt, i))
        y = np.empty((cnt, o))
        assert lib.vnt_synth_batch(C.c_uint64(seed), C.c_uint64(n), C.c_uint64(i), C.c_uint64(o),
                                   C.c_uint64(start), C.c_uint64(cnt), x.ctypes.data_as(f64p),
                                   y.ctypes.data_as(f64p)) == 0
        x2, y2 = port.synth_batch(seed, n, i, o, start, cnt)
        assert np.array_equal(x, x2) and np.array_equal(y, y2)
    w = [784, 16, 10]
    wa = (C.c_uint64 * 3)(*w)
    p = np.empty(port.param_count(w))
    assert lib.vnt_init_params(wa, 3, C.c_uint64(11), p.ctypes.data_as(f64p)) == 0
    assert np.array_equal(p, port.init_params(w, 11))


@pytest.mark.gpu
def test_cpp_dropin_suite_on_gpu():
    r = subprocess.run([str(_bin("test_dropin_gpu"))], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["headline", "cfg1", "shuffled"])
def test_dropin_trainer_matches_reference_trainer(port, ref, case):
    """Trainer::step through the drop-in vs the reference's Trainer, same config,
    including a resize 8 -> 4 -> 8 (cfg5 shape) for the headline case; the
    shuffled case runs shuffled epochs (runner.cpp:47-62, rng.cpp:65-73) with
    prefetch on both sides across 7 epochs and the same resizes."""
    lib = _host()
    o = ref if ref is not None else port
    shuffle = case == "shuffled"
    if shuffle and ref is None:
        pytest.skip("shuffled epochs: the reference trainer (oracle/_ref) is the checker")
    if case in ("headline", "shuffled"):
        w, act, loss, seed, B, V, lr, ds, n, G, steps = [4, 16, 4], 1, 0, 11, 64, 8, 0.05, 11, 256, 8, 30
    else:
        w, act, loss, seed, B, V, lr, ds, n, G, steps = [784, 16, 10], 1, 1, 11, 256, 16, 0.05, 11, 60000, 1, 10
    import paper_2009_09523_b200 as vnt
    mine = vnt.Trainer(w, ["relu", "tanh", "identity"][act], ["mse", "softmax-cross-entropy"][loss], seed,
                       B, V, lr, ds, n, G, shuffle_seed=7 if shuffle else None, prefetch=shuffle)
    extra = dict(shuffle_seed=7, prefetch=True) if shuffle else {}
    t = o.trainer(w, ["relu", "tanh", "identity"][act], ["mse", "softmax-cross-entropy"][loss], seed,
                  B, V, lr, ds, n, G, **extra)
    for s in range(steps):
        if case != "cfg1" and s in (10, 20):
            k = 4 if s == 10 else 8
            mine.resize(k)
            t.resize(k)
        got = mine.step()
        want = t.step()
        assert abs(got - want) <= 2e-5 * abs(want), (s, got, want)
    assert np.abs(mine.params() - t.params()).max() <= 2e-5
    # Input statistics are fp64 in the reference's op order: bit-identical,
    # including lineages merged/seeded by the resizes (moved on the GPU).
    assert mine.local_device_count() == G
    for i in range(G):
        cnt, mean, m2 = mine.input_stats(i)
        c2, mean2, m22 = t.input_stats(i)
        assert cnt == c2 and np.array_equal(mean, mean2) and np.array_equal(m2, m22)
    mine.close()
