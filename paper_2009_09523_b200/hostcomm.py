"""Host-callback process groups for the engine (``vnt_comm_ops``, include/vnt_engine.h).

The product multi-GPU path is NCCL over NVLink (one process per GPU).  This
module backs the engine's collectives with ``torch.distributed`` on the
``gloo`` backend instead, through host buffers, so several engine processes
can share ONE GPU and still run the multi-rank code — the sharded update,
pool membership changes of an elastic resize — bit for bit as NCCL would:
every collective here is exact (int64 sums, max, byte copies).  The engine
synchronises its stream before each callback, so no kernel ever waits on
another rank's kernel.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
_RSCATTER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
_AGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
_BCAST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
_SEND = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
_RECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)


class CommOps(C.Structure):
    pass


_SPLIT = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(CommOps))
_RELEASE = C.CFUNCTYPE(None, C.c_void_p)

CommOps._fields_ = [("ctx", C.c_void_p), ("rank", C.c_int32), ("size", C.c_int32),
                    ("allreduce", _ALLREDUCE), ("reduce_scatter", _RSCATTER),
                    ("allgather", _AGATHER), ("broadcast", _BCAST), ("send", _SEND),
                    ("recv", _RECV), ("split", _SPLIT), ("release", _RELEASE)]

_groups: dict[int, "GlooGroup"] = {}   # ctx id -> live group (kept alive for the engine)


def _arr(ptr, nbytes, dtype):
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype)


def _guard(fn):
    def wrapped(*a):
        try:
            return fn(*a)
        except Exception as ex:   # a callback must not raise through C
            import traceback
            traceback.print_exc()
            print("hostcomm callback failed:", ex, flush=True)
            return 1
    return wrapped


class GlooGroup:
    """One process group: `ranks` are torch.distributed global ranks (ascending
    by group rank); None = the default (world) group."""

    _next_id = 1

    def __init__(self, group=None, ranks=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.ranks = list(range(dist.get_world_size())) if ranks is None else list(ranks)
        me = dist.get_rank()
        self.rank = self.ranks.index(me)
        self.size = len(self.ranks)
        self.id = GlooGroup._next_id
        GlooGroup._next_id += 1
        _groups[self.id] = self
        self._cbs = (_ALLREDUCE(_guard(self._allreduce)), _RSCATTER(_guard(self._reduce_scatter)),
                     _AGATHER(_guard(self._allgather)), _BCAST(_guard(self._broadcast)),
                     _SEND(_guard(self._send)), _RECV(_guard(self._recv)),
                     _SPLIT(_guard(self._split)), _RELEASE(self._release))
        self.ops = CommOps(C.c_void_p(self.id), self.rank, self.size, *self._cbs)

    # -- callbacks (host pointers into the engine's pinned staging)
    def _t(self, ptr, nbytes, dtype):
        import torch
        return torch.from_numpy(_arr(ptr, nbytes, dtype))

    def _allreduce(self, ctx, buf, count, op):
        t = self._t(buf, 8 * count, np.int64)
        # op 1 = uint64 max: the engine only max-reduces positive doubles' bit
        # patterns (< 2^63), which order the same as int64
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM if op == 0 else self.dist.ReduceOp.MAX,
                             group=self.group)
        return 0

    def _reduce_scatter(self, ctx, send, recv, count):
        t = self._t(send, 8 * count * self.size, np.int64).clone()
        self.dist.all_reduce(t, group=self.group)
        out = self._t(recv, 8 * count, np.int64)
        out.copy_(t[self.rank * count:(self.rank + 1) * count])
        return 0

    def _allgather(self, ctx, send, recv, nbytes):
        import torch
        src = self._t(send, nbytes, np.uint8)
        parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.size)]
        self.dist.all_gather(parts, src, group=self.group)
        self._t(recv, nbytes * self.size, np.uint8).copy_(torch.cat(parts))
        return 0

    def _broadcast(self, ctx, buf, nbytes, root):
        self.dist.broadcast(self._t(buf, nbytes, np.uint8), src=self.ranks[root], group=self.group)
        return 0

    def _send(self, ctx, buf, nbytes, peer):
        self.dist.send(self._t(buf, nbytes, np.uint8).clone(), dst=self.ranks[peer], group=self.group)
        return 0

    def _recv(self, ctx, buf, nbytes, peer):
        self.dist.recv(self._t(buf, nbytes, np.uint8), src=self.ranks[peer], group=self.group)
        return 0

    def _split(self, ctx, color, key, out):
        colors = [None] * self.size
        self.dist.all_gather_object(colors, (int(color), int(key), self.ranks[self.rank]),
                                    group=self.group)
        members = sorted((k, g) for c, k, g in colors if c >= 0)
        ranks = [g for _, g in members]
        # torch requires every process of the default group to create the group
        grp = self.dist.new_group(ranks=ranks, backend="gloo") if ranks else None
        if color < 0:
            out[0] = CommOps()
            return 0
        sub = GlooGroup(grp, ranks)
        out[0] = sub.ops
        return 0

    def _release(self, ctx):
        _groups.pop(int(ctx or 0), None)


def world_group() -> GlooGroup:
    """The default torch.distributed group (must be initialised, gloo)."""
    return GlooGroup()
