"""TEST INFRASTRUCTURE: ctypes access to the two CPU oracles.

* ``port`` — oracle/_build/libvntoracle.so, our plain-C restatement
  (oracle/vnt_oracle.c).  Rebuilt on demand with gcc, so it exists on the GPU box.
* ``ref``  — oracle/_ref/libvntref.so, the reference's own sources compiled in
  place (oracle/Makefile).  Built in the dev container (needs /root/reference);
  the .so travels with the snapshot.  ``None`` when absent.

Only tests/, bench.py's cpu_baseline / --impl reference legs and
__graft_entry__.smoke() may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE = ROOT / "oracle"
PORT_SO = ORACLE / "_build" / "libvntoracle.so"
REF_SO = ORACLE / "_ref" / "libvntref.so"

ACT = {"relu": 0, "tanh": 1, "identity": 2}
LOSS = {"mse": 0, "softmax-cross-entropy": 1, "ce": 1}

_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


def _widths(ws):
    arr = (C.c_uint64 * len(ws))(*ws)
    return arr, len(ws)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_f64p)


def build_port() -> Path:
    if not PORT_SO.exists() or PORT_SO.stat().st_mtime < (ORACLE / "vnt_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ORACLE), "oracle"], check=True)
    return PORT_SO


class Oracle:
    """Uniform view over either oracle library (prefix ``vo_`` or ``vntref_``)."""

    def __init__(self, kind: str):
        self.kind = kind
        if kind == "port":
            self.lib = C.CDLL(str(build_port()))
            p = "vo_"
        else:
            if not REF_SO.exists():
                raise FileNotFoundError(REF_SO)
            self.lib = C.CDLL(str(REF_SO))
            p = "vntref_"
        L = self.lib
        self._synth = getattr(L, p + "synth_batch")
        self._synth.argtypes = [C.c_uint64] * 6 + [_f64p, _f64p]
        self._init = getattr(L, p + "init_params")
        self._fb = getattr(L, p + "forward_backward")
        self._fb.argtypes = [_u64p, C.c_uint32, C.c_int, C.c_int, _f64p, _f64p, _f64p,
                             C.c_uint64, _f64p, _f64p]
        self._tc = getattr(L, p + "trainer_create")
        self._tc.restype = C.c_void_p
        self._td = getattr(L, p + "trainer_destroy")
        self._td.argtypes = [C.c_void_p]
        self._ts = getattr(L, p + "trainer_step")
        self._ts.argtypes = [C.c_void_p, _f64p]
        self._tp = getattr(L, p + "trainer_params")
        self._tp.argtypes = [C.c_void_p, _f64p, C.c_uint64]
        self._tr = getattr(L, p + "trainer_resize")
        self._tst = getattr(L, p + "trainer_input_stats")
        self._tst.argtypes = [C.c_void_p, C.c_uint32, _f64p, _f64p, _f64p, C.c_uint64]
        self.p = p

    # data.cpp:107-113
    def synth_batch(self, data_seed, dataset_size, in_w, out_w, start, count):
        x = np.empty((count, in_w), np.float64)
        y = np.empty((count, out_w), np.float64)
        rc = self._synth(data_seed, dataset_size, in_w, out_w, start, count, _ptr(x), _ptr(y))
        assert rc == 0
        return x, y

    @staticmethod
    def param_count(widths):
        return sum(widths[i] * widths[i + 1] + widths[i + 1] for i in range(len(widths) - 1))

    # model.cpp:170-183
    def init_params(self, widths, seed, act="tanh", loss="mse"):
        out = np.empty(self.param_count(widths), np.float64)
        w, n = _widths(widths)
        if self.kind == "port":
            rc = self._init(w, C.c_uint32(n), C.c_uint64(seed), _ptr(out))
        else:
            rc = self._init(w, C.c_uint32(n), C.c_int(ACT[act]), C.c_int(LOSS[loss]),
                            C.c_uint64(seed), _ptr(out))
        assert rc == 0
        return out

    # model.cpp:345-360
    def forward_backward(self, widths, act, loss, params, x, y):
        w, n = _widths(widths)
        g = np.empty(self.param_count(widths), np.float64)
        lo = C.c_double()
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        params = np.ascontiguousarray(params, np.float64)
        rc = self._fb(w, n, ACT[act], LOSS[loss], _ptr(params), _ptr(x), _ptr(y),
                      x.shape[0], _ptr(g), C.byref(lo))
        assert rc == 0
        return g, lo.value

    def forward_backward_wide(self, widths, act, loss, params, x, y, act_ext=None, tau=0.0,
                              counts=False):
        """vo_forward_backward_wide[_masked] (port only): the wide-model variant,
        examples in parallel, compensated sums (pinned to forward_backward in
        tests).  act_ext {layer: rows x width fp32 activations}: relu masks of
        near-zero pre-activations (|z| <= tau max|z|) taken from them."""
        assert self.kind == "port"
        f = self.lib.vo_forward_backward_wide_masked
        f.argtypes = self._fb.argtypes[:8] + [C.c_void_p, C.c_double, _f64p, _f64p,
                                              C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        w, n = _widths(widths)
        g = np.empty(self.param_count(widths), np.float64)
        lo = C.c_double()
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        params = np.ascontiguousarray(params, np.float64)
        keep, ptrs = [], None
        if act_ext:
            ptrs = (C.c_void_p * len(widths))()
            for l, a in act_ext.items():
                a = np.ascontiguousarray(a, np.float32)
                keep.append(a)
                ptrs[l] = a.ctypes.data
        amb, conf = C.c_uint64(), C.c_uint64()
        rc = f(w, n, ACT[act], LOSS[loss], _ptr(params), _ptr(x), _ptr(y), x.shape[0],
               C.cast(ptrs, C.c_void_p) if ptrs is not None else None, tau, _ptr(g), C.byref(lo),
               C.byref(amb), C.byref(conf))
        assert rc == 0
        if counts:
            return g, lo.value, amb.value, conf.value
        return g, lo.value

    def trainer(self, widths, act, loss, seed, global_batch, virtual_nodes, lr,
                data_seed, dataset_size, n_devices, capacity=1 << 20, parallel=False,
                shuffle_seed=None, prefetch=False):
        w, n = _widths(widths)
        if shuffle_seed is not None or prefetch:
            assert self.kind == "ref", "shuffled epochs / prefetch: reference trainer only"
            f = self.lib.vntref_trainer_create_ex
            f.restype = C.c_void_p
            h = f(w, C.c_uint32(n), C.c_int(ACT[act]), C.c_int(LOSS[loss]),
                  C.c_uint64(seed), C.c_uint64(global_batch), C.c_uint64(virtual_nodes),
                  C.c_double(lr), C.c_uint64(data_seed), C.c_uint64(dataset_size),
                  C.c_uint32(n_devices), C.c_uint64(capacity), C.c_int(1 if parallel else 0),
                  C.c_int(0 if shuffle_seed is None else 1), C.c_uint64(shuffle_seed or 0),
                  C.c_int(1 if prefetch else 0))
            assert h, "trainer_create_ex failed"
            return _Trainer(self, h, self.param_count(widths), widths[0])
        if self.kind == "port":
            h = self._tc(w, C.c_uint32(n), C.c_int(ACT[act]), C.c_int(LOSS[loss]),
                         C.c_uint64(seed), C.c_uint64(global_batch), C.c_uint64(virtual_nodes),
                         C.c_double(lr), C.c_uint64(data_seed), C.c_uint64(dataset_size),
                         C.c_uint32(n_devices))
        else:
            h = self._tc(w, C.c_uint32(n), C.c_int(ACT[act]), C.c_int(LOSS[loss]),
                         C.c_uint64(seed), C.c_uint64(global_batch), C.c_uint64(virtual_nodes),
                         C.c_double(lr), C.c_uint64(data_seed), C.c_uint64(dataset_size),
                         C.c_uint32(n_devices), C.c_uint64(capacity), C.c_int(1 if parallel else 0))
        assert h, "trainer_create failed"
        return _Trainer(self, h, self.param_count(widths), widths[0])


class _Trainer:
    def __init__(self, o: Oracle, h, P, in_w):
        self.o, self.h, self.P, self.in_w = o, h, P, in_w

    def step(self) -> float:
        lo = C.c_double()
        assert self.o._ts(self.h, C.byref(lo)) == 0
        return lo.value

    def params(self) -> np.ndarray:
        out = np.empty(self.P, np.float64)
        assert self.o._tp(self.h, _ptr(out), self.P) == 0
        return out

    def resize(self, n_devices, capacity=1 << 20):
        if self.o.kind == "port":
            rc = self.o._tr(C.c_void_p(self.h), C.c_uint32(n_devices))
        else:
            rc = self.o._tr(C.c_void_p(self.h), C.c_uint32(n_devices), C.c_uint64(capacity))
        assert rc == 0

    def input_stats(self, idx):
        cnt = C.c_double()
        mean = np.zeros(self.in_w)
        m2 = np.zeros(self.in_w)
        assert self.o._tst(self.h, idx, C.byref(cnt), _ptr(mean), _ptr(m2), self.in_w) == 0
        return cnt.value, mean, m2

    def __del__(self):
        try:
            self.o._td(self.h)
        except Exception:
            pass


def port() -> Oracle:
    return Oracle("port")


def ref():
    try:
        return Oracle("ref")
    except (FileNotFoundError, OSError):
        return None
