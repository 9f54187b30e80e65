"""Angle sharding across GPUs: one process per GPU, each owning a
contiguous block of projection angles; the volume is replicated.

* ``shard_angles`` -- the partition (ctk_shard_angles in the native library).
* ``NcclComm``     -- native NCCL communicator (libnccl.so.2 dlopen'd by libctk_b200.so);
                      the 128-byte unique id is broadcast with torch.distributed.
* ``TorchComm``    -- the same collectives as callbacks over torch.distributed (nccl or
                      gloo); scalars are all-gathered and summed in rank order.
Attach either to a Projector (``Projector.attach_comm``): A^T b partial volumes are then
sum-reduced and range-space reductions are summed over ranks inside the C++ solvers.
"""
from __future__ import annotations

import ctypes as C

from . import _lib as L
from .api import _check


def shard_angles(n_angles: int, nranks: int, rank: int):
    """Contiguous angle block [first, first + count) of `rank`."""
    lib = L.load()
    f, c = C.c_int(), C.c_int()
    _check(lib.ctk_shard_angles(n_angles, nranks, rank, C.byref(f), C.byref(c)))
    return f.value, c.value


def shard_slabs(nz: int, nranks: int, rank: int):
    """Contiguous z-slab [z0, z0 + count) of `rank` (z-slab sharding)."""
    lib = L.load()
    z, c = C.c_int(), C.c_int()
    _check(lib.ctk_shard_slabs(nz, nranks, rank, C.byref(z), C.byref(c)))
    return z.value, c.value


class NcclComm:
    def __init__(self, rank: int, nranks: int, group=None):
        import torch
        import torch.distributed as dist

        lib = L.load()
        self.lib = lib
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _check(lib.ctk_nccl_get_unique_id(C.cast(uid, C.c_void_p)))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        raw = bytes(t.cpu().tolist())
        uid = (C.c_ubyte * 128).from_buffer_copy(raw)
        h = C.c_void_p()
        _check(lib.ctk_comm_create_nccl(C.cast(uid, C.c_void_p), nranks, rank, C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.ctk_comm_destroy(h)
            self.handle = None


class TorchComm:
    """ctk_comm_callbacks over torch.distributed.  `device` is where the buffers passed to
    allreduce live ("cuda" for the product path, "cpu" for gloo tests of the host logic)."""

    def __init__(self, rank: int, nranks: int, group=None, device: str = "cuda"):
        self.rank, self.nranks, self.group, self.device = rank, nranks, group, device
        self._ar = L.ALLREDUCE(self._allreduce)
        self._ag = L.ALLGATHER(self._allgather)
        self._ex = L.EXCHANGE(self._exchange)
        self.callbacks = L.CommCallbacks(rank, nranks, self._ar, self._ag, None, self._ex)
        self._handle = None

    @property
    def handle(self):
        if self._handle is None:
            lib = L.load()
            h = C.c_void_p()
            _check(lib.ctk_comm_create(C.byref(self.callbacks), C.byref(h)))
            self._handle = h
        return self._handle

    def _wrap(self, ptr, count, dtype):
        import torch

        tdt = torch.float32 if dtype == 0 else torch.float64
        esz = 4 if dtype == 0 else 8
        if self.device == "cpu":
            import numpy as np

            arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float if dtype == 0 else C.c_double)), shape=(count,))
            return torch.from_numpy(arr)
        # wrap a raw device pointer without copying (legacy __cuda_array_interface__ route)
        class _CAI:
            __cuda_array_interface__ = {"shape": (count,), "typestr": "<f4" if dtype == 0 else "<f8",
                                        "data": (ptr, False), "version": 2}

        t = torch.as_tensor(_CAI(), device="cuda")
        assert t.element_size() == esz and t.dtype == tdt
        return t

    def _allreduce(self, ptr, count, dtype, stream, user):
        import torch.distributed as dist

        try:
            t = self._wrap(ptr, count, dtype)
            if self.device == "cpu":
                dist.all_reduce(t, group=self.group)
                return 0
            import torch

            # Run the collective on the library's stream: the kernels that produced the buffer
            # and the ones that consume the result are queued there, so the reduction is
            # ordered after the former and before the latter (NCCL enqueues on the current
            # stream).  Host-staged backends (gloo) complete synchronously on the host, so the
            # stream is drained first and the copy back is finished before returning.
            ext = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
            if dist.get_backend(self.group) == "nccl":
                with torch.cuda.stream(ext):
                    dist.all_reduce(t, group=self.group)
            else:
                ext.synchronize()
                dist.all_reduce(t, group=self.group)
                torch.cuda.synchronize()
            return 0
        except Exception:  # surfaced by the library as CTK_E_CUDA
            return 1

    def _exchange(self, ops, n_ops, dtype, stream, user):
        """Point-to-point transfers of the band-sharded range (bands.cpp): NCCL batches them
        on the library's stream; host-staged backends (gloo) copy through host memory."""
        import torch
        import torch.distributed as dist

        try:
            lst = [ops[i] for i in range(n_ops)]
            if self.device == "cpu":
                ts = [self._wrap(o.d_buf, o.count, dtype) for o in lst]
                reqs = [(dist.isend if o.is_send else dist.irecv)(t, o.peer, group=self.group) for o, t in zip(lst, ts)]
                for r in reqs:
                    r.wait()
                return 0
            ext = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
            if dist.get_backend(self.group) == "nccl":
                with torch.cuda.stream(ext):
                    p2p = [dist.P2POp(dist.isend if o.is_send else dist.irecv, self._wrap(o.d_buf, o.count, dtype),
                                      o.peer, group=self.group) for o in lst]
                    for r in dist.batch_isend_irecv(p2p):
                        r.wait()
                return 0
            ext.synchronize()
            host = [self._wrap(o.d_buf, o.count, dtype).cpu() if o.is_send else
                    torch.empty(o.count, dtype=torch.float32 if dtype == 0 else torch.float64) for o in lst]
            reqs = [(dist.isend if o.is_send else dist.irecv)(t, o.peer, group=self.group) for o, t in zip(lst, host)]
            for r in reqs:
                r.wait()
            for o, t in zip(lst, host):
                if not o.is_send:
                    self._wrap(o.d_buf, o.count, dtype).copy_(t)
            torch.cuda.synchronize()
            return 0
        except Exception:  # surfaced by the library as CTK_E_CUDA
            return 1

    def _allgather(self, value, out, user):
        import torch
        import torch.distributed as dist

        try:
            dev = "cuda" if (self.device != "cpu" and dist.get_backend(self.group) == "nccl") else "cpu"
            v = torch.tensor([value], dtype=torch.float64, device=dev)
            parts = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(self.nranks)]
            dist.all_gather(parts, v, group=self.group)
            for r in range(self.nranks):
                out[r] = float(parts[r].item())
            return 0
        except Exception:
            return 1

    def sum_scalar(self, value: float) -> float:
        """Rank-ordered sum of one scalar per rank (the library's comm_sum_scalar contract)."""
        buf = (C.c_double * self.nranks)()
        if self._allgather(value, buf, None) != 0:
            raise RuntimeError("allgather failed")
        s = 0.0
        for r in range(self.nranks):
            s += buf[r]
        return s

    def allreduce_buffer(self, ptr: int, count: int, dtype: int) -> None:
        if self._allreduce(ptr, count, dtype, None, None) != 0:
            raise RuntimeError("allreduce failed")
