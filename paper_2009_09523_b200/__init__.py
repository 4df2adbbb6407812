"""B200-native virtual-node training step (VirtualFlow, arXiv 2009.09523).

Python view of the C-ABI in ``include/vnt_engine.h`` (the engine is
``libvnt_engine.so``, built in-tree by ``__graft_entry__.build()``).  This
module is host plumbing for tests and ``bench.py``; the product is the CUDA
engine plus the C++ drop-in ``vnt::`` API (``include/vnt/``, ``libvnt.so``).
There is no CPU fallback: constructing an :class:`Engine` without the built
library or without an sm_100 GPU raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
ENGINE_SO = PKG / "libvnt_engine.so"
HOST_SO = PKG / "libvnt.so"

ACTIVATIONS = {"relu": 0, "tanh": 1, "identity": 2}
LOSSES = {"mse": 0, "softmax-cross-entropy": 1}
GEMM_MODES = {"auto": 0, "ffma": 1, "tf32": 2, "3xf16": 3, "3xtf32": 3}   # 3xtf32: round-1 name

VNT_OK = 0
ERRORS = {1: "Error", 2: "ConfigError", 3: "CapacityError", 6: "ShapeError",
          7: "ConsistencyError", 8: "MigrationError", 9: "CudaError", 10: "NcclError",
          11: "NonFiniteError", 12: "RescaleRequired"}


class VntError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, 'Error')} ({code}): {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")


class _ModelDesc(C.Structure):
    _fields_ = [("layer_widths", C.POINTER(C.c_uint64)), ("num_widths", C.c_uint32),
                ("activation", C.c_int32), ("loss", C.c_int32)]


class _Options(C.Structure):
    _fields_ = [("cuda_device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("nccl_id", C.POINTER(C.c_uint8)), ("gemm_mode", C.c_int32),
                ("momentum", C.c_double), ("resident_rows", C.c_uint64),
                ("comm_ops", C.c_void_p)]


class DeviceMetrics(C.Structure):
    _fields_ = [("waves", C.c_uint64), ("examples", C.c_uint64),
                ("peak_resident", C.c_uint64), ("buffer_bytes", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class StepTimings(C.Structure):
    _fields_ = [("total_ms", C.c_float), ("forward_ms", C.c_float), ("backward_ms", C.c_float),
                ("sync_ms", C.c_float), ("update_ms", C.c_float),
                ("kernel_launches", C.c_uint32), ("rescale_retries", C.c_uint32),
                ("gemm_ms", C.c_float), ("gemm_launches", C.c_uint32), ("gemm_flops", C.c_double),
                ("passes", C.c_uint32)]

    def as_dict(self):
        return {k: (float(getattr(self, k)) if t in (C.c_float, C.c_double) else int(getattr(self, k)))
                for k, t in self._fields_}


_lib = None

_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_vp = C.c_void_p


def load_engine() -> C.CDLL:
    """Load libvnt_engine.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not ENGINE_SO.exists():
        raise ImportError(f"{ENGINE_SO} missing: run __graft_entry__.build() (no CPU fallback)")
    lib = C.CDLL(str(ENGINE_SO))
    sig = {
        "vnt_last_error": (C.c_char_p, []),
        "vnt_build_info": (C.c_char_p, []),
        "vnt_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "vnt_engine_create": (C.c_int, [C.POINTER(_ModelDesc), C.POINTER(_Options), C.POINTER(_vp)]),
        "vnt_engine_destroy": (None, [_vp]),
        "vnt_engine_param_count": (C.c_uint64, [_vp]),
        "vnt_engine_tensor_count": (C.c_uint32, [_vp]),
        "vnt_engine_scale_count": (C.c_uint32, [_vp]),
        "vnt_engine_set_params": (C.c_int, [_vp, _f64p, C.c_uint64]),
        "vnt_engine_get_params": (C.c_int, [_vp, _f64p, C.c_uint64]),
        "vnt_engine_add_device": (C.c_int, [_vp, C.c_uint64, _i32p]),
        "vnt_engine_device_count": (C.c_int, [_vp]),
        "vnt_engine_device_step": (C.c_int, [_vp, C.c_int32, _f64p, _f64p, _u64p, C.c_uint32,
                                             C.POINTER(DeviceMetrics)]),
        "vnt_engine_sync": (C.c_int, [_vp, _f64p, _f64p, _u64p]),
        "vnt_engine_sgd_apply": (C.c_int, [_vp, C.c_double]),
        "vnt_engine_take_gradient_sum": (C.c_int, [_vp, _f64p, _f64p, _u64p]),
        "vnt_engine_train_step": (C.c_int, [_vp, _f64p, _f64p, C.c_uint64, _u64p, _i32p,
                                            C.c_uint32, C.c_double, _f64p,
                                            C.POINTER(DeviceMetrics)]),
        "vnt_engine_train_step_resident": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _u64p, _i32p,
                                                     C.c_uint32, C.c_double, _f64p,
                                                     C.POINTER(DeviceMetrics)]),
        "vnt_engine_get_input_stats": (C.c_int, [_vp, C.c_int32, _f64p, _f64p, _f64p]),
        "vnt_engine_set_input_stats": (C.c_int, [_vp, C.c_int32, C.c_double, _f64p, _f64p]),
        "vnt_engine_get_scales": (C.c_int, [_vp, _i32p, C.c_uint32]),
        "vnt_engine_set_scales": (C.c_int, [_vp, _i32p, C.c_uint32]),
        "vnt_engine_last_timings": (C.c_int, [_vp, C.POINTER(StepTimings)]),
        "vnt_engine_reset_scales": (C.c_int, [_vp]),
        "vnt_engine_comm_log": (C.c_int, [_vp, _u64p, C.c_uint32, C.POINTER(C.c_uint32)]),
        "vnt_engine_regroup_ops": (C.c_int, [_vp, _vp, C.c_int32]),
        "vnt_engine_set_membership": (C.c_int, [_vp, C.c_int32, C.c_int32]),
        "vnt_engine_debug_activation": (C.c_int, [_vp, C.c_int32, C.POINTER(C.c_float), C.c_uint64]),
        "vnt_engine_prefetch": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _u64p, _i32p, C.c_uint32,
                                          C.c_int32]),
        "vnt_engine_regroup": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.c_int32]),
        "vnt_engine_stream": (_vp, [_vp]),
        "vnt_engine_device_alloc": (C.c_int, [_vp, C.c_uint64, C.POINTER(_vp)]),
        "vnt_engine_device_free": (C.c_int, [_vp, _vp]),
        "vnt_engine_memcpy_h2d": (C.c_int, [_vp, _vp, _vp, C.c_uint64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(rc: int):
    if rc != VNT_OK:
        raise VntError(rc, load_engine().vnt_last_error().decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_f64p)


def uniform_mapping(global_batch: int, total_nodes: int, n_devices: int, capacity: int = 1 << 30):
    """make_uniform_mapping (virtual_exec.cpp:71-100): node n -> device n % G."""
    if total_nodes == 0 or n_devices == 0:
        raise VntError(2, "make_uniform_mapping: need nodes and devices")
    if global_batch % total_nodes:
        raise VntError(2, "make_uniform_mapping: node count must divide batch size")
    if total_nodes < n_devices:
        raise VntError(2, "make_uniform_mapping: fewer virtual nodes than devices")
    micro = global_batch // total_nodes
    if micro > capacity:
        raise VntError(3, f"micro-batch of {micro} examples exceeds memory capacity of device gpu0")
    sizes = np.full(total_nodes, micro, np.uint64)
    dev = np.arange(total_nodes, dtype=np.int64) % n_devices
    return sizes, dev


class Engine:
    """One process's view of the virtual-node engine (one GPU)."""

    def __init__(self, widths, activation="tanh", loss="mse", cuda_device=0, rank=0,
                 world_size=1, nccl_id: bytes | None = None, gemm_mode="auto",
                 momentum=0.0, resident_rows=0, comm=None):
        """comm: a hostcomm.GlooGroup (host-callback process group, several
        processes on one GPU) instead of NCCL (rank / world_size / nccl_id)."""
        lib = load_engine()
        self.lib = lib
        self.widths = [int(w) for w in widths]
        self._w = (C.c_uint64 * len(self.widths))(*self.widths)
        desc = _ModelDesc(self._w, len(self.widths), ACTIVATIONS[activation], LOSSES[loss])
        self._nid = None
        if nccl_id is not None:
            self._nid = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._comm = comm   # keeps the callbacks alive
        opt = _Options(cuda_device, rank, world_size,
                       C.cast(self._nid, C.POINTER(C.c_uint8)) if self._nid else None,
                       GEMM_MODES[gemm_mode], momentum, resident_rows,
                       C.cast(C.pointer(comm.ops), C.c_void_p) if comm is not None else None)
        h = _vp()
        _check(lib.vnt_engine_create(C.byref(desc), C.byref(opt), C.byref(h)))
        self.h = h
        self.P = int(lib.vnt_engine_param_count(h))
        self.ntensors = int(lib.vnt_engine_tensor_count(h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.vnt_engine_destroy(self.h)
            self.h = None

    __del__ = close

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(load_engine().vnt_nccl_unique_id(buf))
        return bytes(buf)

    # ---- replica state
    def set_params(self, params):
        p = _f64(params)
        _check(self.lib.vnt_engine_set_params(self.h, _fp(p), p.size))

    def get_params(self) -> np.ndarray:
        out = np.empty(self.P, np.float64)
        _check(self.lib.vnt_engine_get_params(self.h, _fp(out), self.P))
        return out

    def add_device(self, capacity=1 << 30) -> int:
        idx = C.c_int32()
        _check(self.lib.vnt_engine_add_device(self.h, capacity, C.byref(idx)))
        return idx.value

    # ---- reference decomposition: device_step / sync_gradients / sgd_apply
    def device_step(self, device, x, y, node_sizes):
        x, y = _f64(x), _f64(y)
        ns = np.ascontiguousarray(node_sizes, np.uint64)
        m = DeviceMetrics()
        _check(self.lib.vnt_engine_device_step(self.h, device, _fp(x), _fp(y),
                                               ns.ctypes.data_as(_u64p), ns.size, C.byref(m)))
        return m.as_dict()

    def sync(self, want_grad=True):
        g = np.empty(self.P, np.float64) if want_grad else None
        ls = C.c_double()
        ex = C.c_uint64()
        _check(self.lib.vnt_engine_sync(self.h, _fp(g) if want_grad else None, C.byref(ls),
                                        C.byref(ex)))
        return g, ls.value, ex.value

    COMM_OPS = {1: "allreduce", 2: "reduce_scatter", 3: "allgather", 4: "max", 5: "count",
                6: "broadcast", 7: "send", 8: "recv"}

    def comm_log(self, cap=4096):
        """(op, offset, count) of each collective issued since the last call
        (vnt_engine_comm_log; clears the log); op named as in COMM_OPS."""
        out = np.zeros(3 * cap, np.uint64)
        n = C.c_uint32()
        _check(self.lib.vnt_engine_comm_log(self.h, out.ctypes.data_as(_u64p), cap, C.byref(n)))
        return [(self.COMM_OPS.get(int(out[3 * i]), "?"), int(out[3 * i + 1]), int(out[3 * i + 2]))
                for i in range(min(n.value, cap))]

    def take_gradient_sum(self):
        """Process-local exact gradient sum (no collective), closes the round:
        (sum[P] = double(S) * 2^-s per tensor, loss_sum, examples)."""
        g = np.empty(self.P, np.float64)
        ls = C.c_double()
        ex = C.c_uint64()
        _check(self.lib.vnt_engine_take_gradient_sum(self.h, _fp(g), C.byref(ls), C.byref(ex)))
        return g, ls.value, ex.value

    def sgd_apply(self, lr):
        _check(self.lib.vnt_engine_sgd_apply(self.h, lr))

    # ---- fused train step
    def _mapping_args(self, node_sizes, node_device):
        ns = np.ascontiguousarray(node_sizes, np.uint64)
        nd = np.ascontiguousarray(node_device, np.int32)
        assert ns.size == nd.size
        ndev = int(self.lib.vnt_engine_device_count(self.h))
        return ns, nd, (DeviceMetrics * max(ndev, 1))()

    def train_step(self, x, y, node_sizes, node_device, lr):
        x, y = _f64(x), _f64(y)
        ns, nd, pm = self._mapping_args(node_sizes, node_device)
        loss = C.c_double()
        _check(self.lib.vnt_engine_train_step(self.h, _fp(x), _fp(y), x.shape[0],
                                              ns.ctypes.data_as(_u64p), nd.ctypes.data_as(_i32p),
                                              ns.size, lr, C.byref(loss), pm))
        return loss.value, [m.as_dict() for m in pm]

    def _mapping_ptrs(self, node_sizes, node_device):
        """ctypes views of a mapping, cached for the last (node_sizes, node_device)
        objects seen (the arrays are kept alive and re-read by C every call)."""
        c = getattr(self, "_map_cache", None)
        if c is not None and c[0] is node_sizes and c[1] is node_device:
            return c[2]
        ns = np.ascontiguousarray(node_sizes, np.uint64)
        nd = np.ascontiguousarray(node_device, np.int32)
        ptrs = (ns.ctypes.data_as(_u64p), nd.ctypes.data_as(_i32p), ns.size, ns, nd)
        self._map_cache = (node_sizes, node_device, ptrs)
        return ptrs

    def train_step_ptr(self, x_ptr: int, y_ptr: int, rows: int, node_sizes, node_device, lr,
                       resident: bool):
        """x_ptr / y_ptr: fp64 host (pinned) or device pointers.  Returns the loss only
        (no per-device metrics are gathered on this hot path)."""
        nsp, ndp, n = self._mapping_ptrs(node_sizes, node_device)[:3]
        loss = C.c_double()
        if resident:
            rc = self.lib.vnt_engine_train_step_resident(self.h, _vp(x_ptr), _vp(y_ptr), rows, nsp,
                                                         ndp, n, lr, C.byref(loss), None)
        else:
            rc = self.lib.vnt_engine_train_step(self.h, C.cast(_vp(x_ptr), _f64p),
                                                C.cast(_vp(y_ptr), _f64p), rows, nsp, ndp, n, lr,
                                                C.byref(loss), None)
        _check(rc)
        return loss.value

    def prefetch_ptr(self, x_ptr: int, y_ptr: int, rows: int, node_sizes, node_device,
                     resident: bool):
        """Stage a future step's rows on the copy stream (vnt_engine_prefetch):
        call prefetch(i) once, then before each step(i) queue prefetch(i+1)."""
        nsp, ndp, n = self._mapping_ptrs(node_sizes, node_device)[:3]
        _check(self.lib.vnt_engine_prefetch(self.h, _vp(x_ptr), _vp(y_ptr), rows, nsp, ndp, n,
                                            1 if resident else 0))

    # ---- kernel state / scales / timings
    def input_stats(self, device):
        cnt = C.c_double()
        mean = np.empty(self.widths[0])
        m2 = np.empty(self.widths[0])
        _check(self.lib.vnt_engine_get_input_stats(self.h, device, C.byref(cnt), _fp(mean), _fp(m2)))
        return cnt.value, mean, m2

    def set_input_stats(self, device, count, mean, m2):
        mean, m2 = _f64(mean), _f64(m2)
        _check(self.lib.vnt_engine_set_input_stats(self.h, device, count, _fp(mean), _fp(m2)))

    def scales(self, full: bool = False) -> np.ndarray:
        """Fixed-point scale exponents per gradient tensor; full=True appends the
        split-fp16 operand exponents (vnt_engine_scale_count)."""
        n = int(self.lib.vnt_engine_scale_count(self.h)) if full else self.ntensors
        out = np.empty(n, np.int32)
        _check(self.lib.vnt_engine_get_scales(self.h, out.ctypes.data_as(_i32p), n))
        return out

    def set_scales(self, s):
        s = np.ascontiguousarray(s, np.int32)
        _check(self.lib.vnt_engine_set_scales(self.h, s.ctypes.data_as(_i32p), s.size))

    def regroup(self, rank: int, world_size: int, nccl_id: bytes | None, source_rank: int = 0):
        """Join a new process group and take the replica state from source_rank."""
        nid = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        _check(self.lib.vnt_engine_regroup(self.h, rank, world_size,
                                           C.cast(nid, C.POINTER(C.c_uint8)) if nid else None,
                                           source_rank))

    def regroup_ops(self, comm, source_rank: int = 0):
        """Join a host-callback group (hostcomm.GlooGroup) and take the replica
        state from its source_rank."""
        self._comm_new = comm
        _check(self.lib.vnt_engine_regroup_ops(self.h, C.cast(C.pointer(comm.ops), _vp),
                                               source_rank))

    def set_membership(self, member: bool, source_pool_rank: int = 0):
        """Elastic resize inside the process pool (collective over the pool)."""
        _check(self.lib.vnt_engine_set_membership(self.h, 1 if member else 0, source_pool_rank))

    def debug_activation(self, layer: int, rows: int) -> np.ndarray:
        """Hidden activations X[layer] of the last pass (diagnostics)."""
        out = np.empty((rows, self.widths[layer]), np.float32)
        _check(self.lib.vnt_engine_debug_activation(self.h, layer,
                                                    out.ctypes.data_as(C.POINTER(C.c_float)), rows))
        return out

    def timings(self) -> dict:
        t = StepTimings()
        _check(self.lib.vnt_engine_last_timings(self.h, C.byref(t)))
        return t.as_dict()

    def stream_ptr(self) -> int:
        return int(self.lib.vnt_engine_stream(self.h) or 0)


class _DevSpec(C.Structure):
    _fields_ = [("device_id", C.c_char_p), ("device_type", C.c_char_p), ("memory_capacity", C.c_uint64)]


class _RunnerCfg(C.Structure):   # vnt_runner_config (include/vnt_trainer.h)
    _fields_ = [("layer_widths", C.POINTER(C.c_uint64)), ("num_widths", C.c_uint32),
                ("activation", C.c_int32), ("loss", C.c_int32), ("seed", C.c_uint64),
                ("global_batch", C.c_uint64), ("virtual_nodes", C.c_uint64), ("lr", C.c_double),
                ("data_seed", C.c_uint64), ("dataset_size", C.c_uint64),
                ("shuffle_epochs", C.c_int32), ("shuffle_seed", C.c_uint64),
                ("devices", C.POINTER(_DevSpec)), ("num_devices", C.c_uint32),
                ("parallel_devices", C.c_int32), ("prefetch", C.c_int32), ("gemm_mode", C.c_int32),
                ("momentum", C.c_double), ("comm_ops", C.c_void_p), ("nccl_id", C.POINTER(C.c_uint8)),
                ("rank", C.c_int32), ("world_size", C.c_int32), ("cuda_device", C.c_int32),
                ("resident_rows", C.c_uint64)]


_host_lib = None


def load_host():
    """libvnt.so: the C++ drop-in vnt:: API and its C-ABI (include/vnt_trainer.h)."""
    global _host_lib
    if _host_lib is None:
        load_engine()
        if not HOST_SO.exists():
            raise ImportError(f"{HOST_SO} missing: run __graft_entry__.build()")
        _host_lib = C.CDLL(str(HOST_SO))
        _host_lib.vnt_host_last_error.restype = C.c_char_p
        _host_lib.vnt_trainer_param_count.restype = C.c_uint64
        _host_lib.vnt_trainer_device_count.restype = C.c_uint32
    return _host_lib


def _hcheck(rc: int):
    if rc != VNT_OK:
        raise VntError(rc, load_host().vnt_host_last_error().decode(errors="replace"))


class Trainer:
    """The drop-in vnt::Trainer (RunnerConfig / step / resize / params / world)
    through its C-ABI.  devices: [(device_id, memory_capacity)] or a count
    ("gpu0".. names).  comm: a hostcomm.GlooGroup for one process per rank."""

    def __init__(self, widths, activation, loss, seed, global_batch, virtual_nodes, lr, data_seed,
                 dataset_size, devices, shuffle_seed=None, prefetch=False, gemm_mode="auto",
                 momentum=0.0, comm=None, resident_rows=0, cuda_device=0):
        self.lib = load_host()
        self.widths = [int(w) for w in widths]
        self._w = (C.c_uint64 * len(self.widths))(*self.widths)
        self._devs = self._dev_array(devices)
        self._comm = comm
        cfg = _RunnerCfg(self._w, len(self.widths), ACTIVATIONS[activation], LOSSES[loss], seed,
                         global_batch, virtual_nodes, lr, data_seed, dataset_size,
                         0 if shuffle_seed is None else 1, shuffle_seed or 0, self._devs, len(self._devs),
                         0, 1 if prefetch else 0, GEMM_MODES[gemm_mode], momentum,
                         C.cast(C.pointer(comm.ops), C.c_void_p) if comm is not None else None, None,
                         comm.rank if comm is not None else 0, comm.size if comm is not None else 1,
                         cuda_device, resident_rows)
        h = C.c_void_p()
        _hcheck(self.lib.vnt_trainer_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.P = int(self.lib.vnt_trainer_param_count(h))

    @staticmethod
    def _dev_array(devices):
        if isinstance(devices, int):
            devices = [(f"gpu{i}", 1 << 20) for i in range(devices)]
        arr = (_DevSpec * len(devices))()
        for i, (name, cap) in enumerate(devices):
            arr[i] = _DevSpec(name.encode(), b"B200", cap)
        return arr

    def step(self) -> float:
        lo = C.c_double()
        _hcheck(self.lib.vnt_trainer_step(self.h, C.byref(lo), None, 0))
        return lo.value

    def resize(self, devices):
        arr = self._dev_array(devices)
        _hcheck(self.lib.vnt_trainer_resize(self.h, arr, len(arr)))

    def params(self) -> np.ndarray:
        p = np.empty(self.P)
        _hcheck(self.lib.vnt_trainer_params(self.h, p.ctypes.data_as(_f64p), self.P))
        return p

    def local_device_count(self) -> int:
        return int(self.lib.vnt_trainer_device_count(self.h))

    def input_stats(self, idx):
        cnt = C.c_double()
        mean = np.empty(self.widths[0])
        m2 = np.empty(self.widths[0])
        _hcheck(self.lib.vnt_trainer_input_stats(self.h, idx, C.byref(cnt), mean.ctypes.data_as(_f64p),
                                                 m2.ctypes.data_as(_f64p)))
        return cnt.value, mean, m2

    def close(self):
        if getattr(self, "h", None):
            self.lib.vnt_trainer_destroy(self.h)
            self.h = None

    __del__ = close


def param_count(widths) -> int:
    return sum(widths[i] * widths[i + 1] + widths[i + 1] for i in range(len(widths) - 1))


__all__ = ["Engine", "Trainer", "VntError", "uniform_mapping", "param_count", "load_engine",
           "load_host", "ENGINE_SO", "HOST_SO"]
