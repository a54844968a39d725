"""Torch plumbing around the C ABI: device checks, dtype codes, streams, workspaces.

PyTorch only provides device memory (caching allocator) and the current stream;
all arithmetic on the path happens in the sm_100a library.
"""

from __future__ import annotations

import torch

from . import _capi, errors

_DTYPE_CODE = {torch.float32: _capi.LK_F32, torch.bfloat16: _capi.LK_BF16, torch.float16: _capi.LK_F16}

# Read the device-side out-of-range target count after CE/FLCE and raise
# TargetOutOfRange like the reference (rowfuse/ops.py:496-498).  Costs one 16-byte
# device->host read per call (Liger syncs on .item() as well).
CHECK_TARGETS = True


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPE_CODE[t.dtype]
    except KeyError:
        raise errors.ShapeMismatch(f"unsupported dtype {t.dtype}; expected float32, bfloat16 or float16") from None


def require_cuda(*tensors: torch.Tensor | None) -> None:
    """Every operand on CUDA and on the same device (the kernels launch on one device and read
    their operands through plain device pointers)."""
    dev = None
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise errors.ExtensionMissing(
                "paper_2410_10989_b200 runs only on CUDA (sm_100a); got a tensor on "
                f"{t.device}. There is no CPU fallback."
            )
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise errors.ShapeMismatch(f"operands on different devices: {dev} and {t.device}")


def require_contiguous(name: str, t: torch.Tensor) -> None:
    if not t.is_contiguous():
        raise errors.NonContiguousInput(f"{name} must be contiguous (rowfuse/core.py:210-215)")


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_of(t: torch.Tensor) -> int:
    # raw cudaStream_t of the tensor's device's current stream (the C call behind
    # torch.cuda.current_stream(dev).cuda_stream, without building a Stream object)
    if _raw_stream is not None:
        return _raw_stream(t.get_device())
    return torch.cuda.current_stream(t.device).cuda_stream


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def lib():
    return _capi.load()


def device_guard(fn):
    """Run `fn` with the current CUDA device set to that of its first CUDA tensor argument: the
    library launches on the current device (as torch ops do under their device guard)."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        for a in args if not kwargs else list(args) + list(kwargs.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                dev = a.get_device()
                if dev == torch.cuda.current_device():  # common case: no device switch
                    return fn(*args, **kwargs)
                with torch.cuda.device(dev):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)

    return wrapped


def check(rc: int) -> None:
    _capi.check(rc)


def as_targets(target: torch.Tensor) -> torch.Tensor:
    if target.dtype not in (torch.int64, torch.int32, torch.int16, torch.uint8, torch.int8):
        raise errors.ShapeMismatch(f"targets must be integer class ids, got {target.dtype}")
    t = target.reshape(-1)
    if t.dtype != torch.int64:
        t = t.to(torch.int64)
    return t.contiguous()


def stage_target_stats(stats: torch.Tensor):
    """Copy the device (n_valid, n_out_of_range) counts to pinned host memory right after the
    kernel that produced them, and record an event.  The range check at the end of the call
    (`raise_if_staged_out_of_range`) then waits for that small kernel only, not for the whole op
    behind it, so the host goes on to launch the next op while the GEMMs run.  None when the
    check is off or under graph capture."""
    if not CHECK_TARGETS or not stats.is_cuda or torch.cuda.is_current_stream_capturing():
        return None
    host = torch.empty(2, dtype=torch.int64, pin_memory=True)  # torch's caching host allocator
    host.copy_(stats[:2], non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(stats.device))
    return host, ev


def count_and_stage_targets(t: torch.Tensor, vocab: int, ignore_index: int):
    """lk_count_targets into a fresh device pair, staged for the host check (see above)."""
    if not CHECK_TARGETS or t.numel() == 0 or torch.cuda.is_current_stream_capturing():
        return None
    counts = torch.empty(2, dtype=torch.int64, device=t.device)
    check(lib().lk_count_targets(t.data_ptr(), t.numel(), vocab, ignore_index, counts.data_ptr(), stream_of(t)))
    return stage_target_stats(counts)


def raise_if_staged_out_of_range(staged, vocab: int) -> None:
    if staged is None:
        return
    host, ev = staged
    ev.synchronize()
    n = int(host[1])
    if n > 0:
        raise errors.TargetOutOfRange(f"{n} target(s) outside [0, {vocab}) that are not ignore_index")
