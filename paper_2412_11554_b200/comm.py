"""Host-side communicators for ACCORD_COMM_HOST (include/accord.h).

The production multi-GPU path is ACCORD_COMM_NCCL (the library calls NCCL
itself). These host communicators carry the same 8-double line-search sums
and the export gather through other transports:

* TorchDistComm: torch.distributed (gloo on CPU tests, any backend);
* ThreadComm: P contexts driven by P host threads of one process (the
  one-GPU emulation of P ranks: the kernels never wait on each other, only
  the host threads meet at a barrier).

Each exposes `allreduce(user, buf, count)`, `allgatherv(user, in, in_bytes,
out, counts)` and `sendrecv(user, send, send_bytes, dst, recv, recv_bytes,
src)` (the ring of the sharded-X mode) with the C callback signatures; pass
them to AccordSolver (comm=COMM_HOST, allreduce=..., allgatherv=...,
sendrecv=...).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np


class TorchDistComm:
    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce(self, user, buf, count):
        import torch
        try:
            a = np.ctypeslib.as_array(buf, shape=(count,))
            t = torch.from_numpy(a.copy())
            self.dist.all_reduce(t, group=self.group)
            a[:] = t.numpy()
            return 0
        except Exception:
            return 1

    def allgatherv(self, user, inp, in_bytes, out, counts):
        import torch
        try:
            sizes = torch.zeros(self.world, dtype=torch.int64)
            sizes[self.rank] = int(in_bytes)
            self.dist.all_reduce(sizes, group=self.group)
            cnt = np.ctypeslib.as_array(counts, shape=(self.world,))
            cnt[:] = sizes.numpy()
            if not out:
                return 0
            mx = int(sizes.max())
            mine = torch.zeros(mx, dtype=torch.uint8)
            if in_bytes:
                mine[:in_bytes] = torch.from_numpy(
                    np.ctypeslib.as_array(C.cast(inp, C.POINTER(C.c_uint8)),
                                          shape=(in_bytes,)).copy())
            parts = [torch.zeros(mx, dtype=torch.uint8) for _ in range(self.world)]
            self.dist.all_gather(parts, mine, group=self.group)
            dst = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_uint8)),
                                        shape=(int(sizes.sum()),))
            o = 0
            for r in range(self.world):
                s = int(sizes[r])
                dst[o:o + s] = parts[r].numpy()[:s]
                o += s
            return 0
        except Exception:
            return 1


    def sendrecv(self, user, send, send_bytes, dst, recv, recv_bytes, src):
        """Ring exchange (sharded-X mode) over torch.distributed point-to-point."""
        import torch
        try:
            out = torch.from_numpy(np.ctypeslib.as_array(
                C.cast(send, C.POINTER(C.c_uint8)), shape=(send_bytes,)).copy()) \
                if send_bytes else torch.zeros(0, dtype=torch.uint8)
            inb = torch.zeros(recv_bytes, dtype=torch.uint8)
            ops = [self.dist.P2POp(self.dist.isend, out, dst, group=self.group),
                   self.dist.P2POp(self.dist.irecv, inb, src, group=self.group)]
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
            if recv_bytes:
                dstv = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                             shape=(recv_bytes,))
                dstv[:] = inb.numpy()
            return 0
        except Exception:
            return 1


class ThreadComm:
    """P ranks = P host threads of one process (one context each)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.tls = threading.local()

    def bind(self, rank):
        """Call from the thread that drives rank `rank` before using it."""
        self.tls.rank = rank

    def _exchange(self, value):
        r = self.tls.rank
        self.slots[r] = value
        self.barrier.wait()
        vals = list(self.slots)
        self.barrier.wait()
        return vals

    def allreduce(self, user, buf, count):
        try:
            a = np.ctypeslib.as_array(buf, shape=(count,))
            vals = self._exchange(a.copy())
            tot = np.zeros(count)
            for v in vals:          # fixed rank order: identical sums on every rank
                tot += v
            a[:] = tot
            return 0
        except Exception:
            return 1

    def allgatherv(self, user, inp, in_bytes, out, counts):
        try:
            mine = bytes(np.ctypeslib.as_array(C.cast(inp, C.POINTER(C.c_uint8)),
                                               shape=(in_bytes,))) if in_bytes else b""
            vals = self._exchange(mine)
            cnt = np.ctypeslib.as_array(counts, shape=(self.world,))
            cnt[:] = [len(v) for v in vals]
            if out:
                blob = b"".join(vals)
                dst = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_uint8)),
                                            shape=(len(blob),))
                dst[:] = np.frombuffer(blob, dtype=np.uint8)
            return 0
        except Exception:
            return 1

    def sendrecv(self, user, send, send_bytes, dst, recv, recv_bytes, src):
        """Ring exchange of the sharded-X mode: every rank deposits its block
        for `dst` and takes the one `src` deposited for it."""
        try:
            mine = bytes(np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)),
                                               shape=(send_bytes,))) if send_bytes else b""
            vals = self._exchange((dst, mine))
            to, blob = vals[src]
            if to != self.tls.rank or len(blob) != recv_bytes:
                return 1
            if recv_bytes:
                dstv = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                             shape=(recv_bytes,))
                dstv[:] = np.frombuffer(blob, dtype=np.uint8)
            return 0
        except Exception:
            return 1
