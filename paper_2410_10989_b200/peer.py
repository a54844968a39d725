"""Symmetric peer-memory buffers and the token-sharded grad_w all-reduce over them.

One `PeerBuffer` per rank: a device allocation (control page + data) made by the library
(`lk_peer_alloc`), whose CUDA IPC handle every rank exchanges once through the process group
(`all_gather_object`: torch.distributed is the plumbing) and maps (`lk_peer_open`).  After
that, `all_reduce_(t, lo, hi)` sums elements [lo, hi) of a view `t` of the data across ranks
with one kernel (`lk_peer_allreduce`, csrc/peer.cu) that reads and writes the peers' buffers
directly over NVLink -- the replacement for the NCCL all-reduce of the token-sharded dW
(SURVEY §8(e), §2.1).  The sum is in fp32 in rank order, rounded once: bit-identical on every
rank and every run.

Rules the kernel's flags rely on (include/liger_b200.h, lk_peer_allreduce): every rank makes
the same calls in the same order on one stream per buffer, so epochs agree.  A timed-out call
poisons the buffer: `check()` raises and the buffer must be re-created.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import torch
import torch.distributed as dist

from . import errors
from ._utils import check, dtype_code, lib

CTL_BYTES = 4096  # LK_PEER_CTL_BYTES
HANDLE_BYTES = 64  # LK_PEER_HANDLE_BYTES
MAX_PEERS = 16  # LK_PEER_MAX


class PeerTimeout(errors.CudaError):
    """A peer all-reduce waited longer than its timeout for another rank (a rank died or made
    a different sequence of calls)."""


class _CudaArray:
    """__cuda_array_interface__ over the buffer's data region; keeps the PeerBuffer alive for
    as long as a tensor view exists."""

    def __init__(self, owner: "PeerBuffer", nbytes: int):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (owner.base + CTL_BYTES, False), "version": 2}


class PeerBuffer:
    """A symmetric buffer of `nbytes` data bytes on `device`, mapped by every rank of `group`."""

    def __init__(self, nbytes: int, group=None, device: Optional[torch.device] = None,
                 timeout_s: float = 120.0):
        self.device = torch.device(device if device is not None else torch.cuda.current_device())
        if self.device.type != "cuda":
            raise errors.ExtensionMissing("PeerBuffer needs a CUDA device; there is no CPU fallback")
        self.dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > MAX_PEERS:
            raise errors.UnsupportedOption(f"world size {self.world} > LK_PEER_MAX {MAX_PEERS}")
        self.nbytes = int(nbytes)
        self.timeout_ns = int(timeout_s * 1e9)
        self.epoch = 0
        self.poisoned = False
        L = lib()
        base = C.c_void_p()
        handle = (C.c_ubyte * HANDLE_BYTES)()
        check(L.lk_peer_alloc(self.dev_index, self.nbytes, C.byref(base), handle))
        self.base = int(base.value)
        handles: list = [None] * self.world
        with torch.cuda.device(self.dev_index):  # NCCL's object gather stages on the current device
            dist.all_gather_object(handles, bytes(handle), group=group)
        self._opened = []
        ptrs = []
        try:
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self.base)
                    continue
                p = C.c_void_p()
                check(L.lk_peer_open(self.dev_index, (C.c_ubyte * HANDLE_BYTES).from_buffer_copy(h), C.byref(p)))
                self._opened.append(int(p.value))
                ptrs.append(int(p.value))
        except Exception:
            self.close()
            raise
        self._bases = (C.c_void_p * self.world)(*ptrs)
        self._data = torch.as_tensor(_CudaArray(self, self.nbytes), device=self.device)

    def tensor(self, shape, dtype: torch.dtype) -> torch.Tensor:
        """A contiguous view of the data region (this rank's copy) as `shape` / `dtype`."""
        n = 1
        for d in shape:
            n *= int(d)
        esize = torch.empty((), dtype=dtype).element_size()
        if n * esize > self.nbytes:
            raise errors.SizeMismatch(f"{tuple(shape)} {dtype} needs {n * esize} bytes > buffer {self.nbytes}")
        return self._data[: n * esize].view(dtype).view(*shape)

    def all_reduce_(self, t: torch.Tensor, lo: int = 0, hi: Optional[int] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Sum flattened elements [lo, hi) of `t` (a view from `tensor()`) over the ranks, in
        place, on `stream` (default: the current stream).  Enqueues one kernel; no host sync."""
        if self.poisoned:
            raise PeerTimeout("a previous peer all-reduce on this buffer timed out; re-create it")
        if not t.is_contiguous():
            raise errors.NonContiguousInput("peer all-reduce needs a contiguous view")
        off = t.data_ptr() - self.base
        n_all = t.numel()
        hi = n_all if hi is None else int(hi)
        lo = int(lo)
        if not (0 <= lo <= hi <= n_all) or off < CTL_BYTES or off + n_all * t.element_size() > CTL_BYTES + self.nbytes:
            raise errors.SizeMismatch("peer all-reduce range outside the buffer")
        if self.world == 1 or hi == lo:
            return t
        self.epoch += 1
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().lk_peer_allreduce(self._bases, self.world, self.rank, off + lo * t.element_size(), hi - lo,
                                      dtype_code(t), self.epoch, self.timeout_ns, st))
        return t

    def check(self) -> None:
        """Host-synchronous: raise PeerTimeout if a call on this buffer timed out."""
        torch.cuda.synchronize(self.device)  # the calls run on side streams
        err = C.c_int(0)
        check(lib().lk_peer_status(self.dev_index, C.c_void_p(self.base), 0, C.byref(err)))
        if err.value:
            self.poisoned = True
            raise PeerTimeout(f"peer all-reduce timed out on rank {self.rank} (epoch <= {self.epoch})")

    def close(self) -> None:
        L = lib()
        for p in getattr(self, "_opened", []):
            L.lk_peer_close(self.dev_index, C.c_void_p(p))
        self._opened = []
        if getattr(self, "base", 0):
            torch.cuda.synchronize(self.device)
            L.lk_peer_free(self.dev_index, C.c_void_p(self.base))
            self.base = 0


_BUFFERS: dict = {}


def buffer_for(nbytes: int, device: torch.device, group=None, tag: str = "") -> PeerBuffer:
    """The cached symmetric buffer of `nbytes` for (`tag`, group, device), created collectively on
    first use: every rank must reach the first call with the same arguments."""
    key = (tag, id(group), torch.device(device).index, int(nbytes))
    buf = _BUFFERS.get(key)
    if buf is None or buf.poisoned:
        buf = PeerBuffer(nbytes, group=group, device=device)
        _BUFFERS[key] = buf
    return buf


def grad_w_buffer(weight: torch.Tensor, group=None) -> PeerBuffer:
    """The cached symmetric buffer that holds grad_w for `weight`'s shape (token-sharded mode)."""
    return buffer_for(weight.numel() * weight.element_size(), weight.device, group, "grad_w")


__all__ = ["PeerBuffer", "PeerTimeout", "buffer_for", "grad_w_buffer", "CTL_BYTES", "MAX_PEERS"]
