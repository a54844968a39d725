"""Token-sharded and vocab-parallel FLCE on the CUDA kernels, world_size 2 on one GPU (GPU).

Both ranks share cuda:0 and talk over gloo (which all-reduces CUDA tensors), so the
sharded paths -- count / loss / dW all-reduce (token-sharded) and row-statistics / dX
all-reduce with tcgen05 local GEMMs (vocab-parallel) -- run their real kernels and are
compared with the float64 oracle on the full problem.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(bt=384, h=256, v=3000, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (v, h)) / math.sqrt(h) * 3
    t = rng.integers(0, v, bt)
    t[rng.random(bt) < 0.1] = -100
    return x, w, t


def _worker(rank, port, mode, kw, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2410_10989_b200  # noqa: F401
        from oracle import liger_ref
        from paper_2410_10989_b200.distributed import shard_rows, token_sharded_flce, vocab_parallel_flce, vocab_shard
        from tests.conftest import rel_close

        dev = torch.device("cuda:0")
        kw = dict(kw)
        x, w, t = _problem()
        if kw.pop("_ignore_first_half", False):
            t[: len(t) // 2] = -100  # rank 0's whole token shard is ignore_index
        dtype = kw.pop("_dtype", torch.bfloat16)
        zero_rows = kw.pop("_rank0_no_rows", False)
        if "_min_skipped" in kw:  # exercise the kept-row path at test sizes
            import paper_2410_10989_b200.fused_linear_cross_entropy as flce_mod

            flce_mod.COMPACT_MIN_SKIPPED = kw.pop("_min_skipped")
        tol = 1e-4 if dtype == torch.float32 else 2e-2
        xb = torch.tensor(x, dtype=dtype, device=dev)
        wb = torch.tensor(w, dtype=dtype, device=dev)
        tb = torch.tensor(t, device=dev)
        ref_kw = {k: v for k, v in kw.items() if k not in ("dw_slices", "dx_reduce_dtype", "comm")}
        if "ce_weight" in kw:  # numpy class weights: the oracle's `weight`, the library's ce_weight tensor
            ref_kw["weight"] = ref_kw.pop("ce_weight")
            kw["ce_weight"] = torch.tensor(kw["ce_weight"], dtype=torch.float32, device=dev)
        ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(xb.double().cpu().numpy(), wb.double().cpu().numpy(), t, **ref_kw)
        if mode == "token":
            lo, hi = shard_rows(len(t), rank, WORLD)
            if zero_rows:  # rank 0 holds no tokens at all (library BT == 0 path)
                lo, hi = (0, 0) if rank == 0 else (0, len(t))
            loss, gx, gw = token_sharded_flce(xb[lo:hi].contiguous(), wb, tb[lo:hi], chunk_rows=128, **kw)
            gx_ref, gw_ref = rgx[lo:hi], rgw
        else:
            sh = vocab_shard(w.shape[0], rank, WORLD)
            loss, gx, gw = vocab_parallel_flce(xb, wb[sh.offset:sh.offset + sh.size].contiguous(), tb, sh,
                                               chunk_rows=160, **kw)
            gx_ref, gw_ref = rgx, rgw[sh.offset:sh.offset + sh.size]
        torch.cuda.synchronize()
        if kw.get("reduction") == "none":  # per-row losses of this rank's own tokens
            ref_loss = liger_ref.flce(xb.double().cpu().numpy()[lo:hi], wb.double().cpu().numpy(), t[lo:hi],
                                      **ref_kw)[1]
            lv = loss.float().cpu().numpy()
        else:
            lv = float(loss.float().item())
        checks = [("loss", lv, ref_loss), ("gx", gx.float().cpu().numpy(), gx_ref),
                  ("gw", gw.float().cpu().numpy(), gw_ref)]
        bad = [(n, rel_close(a, b, tol)[1]) for n, a, b in checks if not rel_close(a, b, tol)[0]]
        ign = (tb == -100).nonzero().flatten()
        if mode == "vocab" and not torch.all(gx[ign] == 0):
            bad.append(("ignored rows of dX not zero", 0))
        out[rank] = "ok" if not bad else repr(bad)
    except Exception as e:  # pragma: no cover - reported to the parent
        out[rank] = repr(e)
    finally:
        dist.destroy_process_group()


def _run(mode, kw):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_port(), mode, kw, out), nprocs=WORLD, join=True)
    assert dict(out) == {0: "ok", 1: "ok"}, dict(out)


_CW = np.random.default_rng(5).random(3000) + 0.2


@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1, softcap=30.0), dict(ce_weight=_CW),
                                dict(ce_weight=_CW, label_smoothing=0.1), dict(_ignore_first_half=True),
                                # slice events on the SIMT (fp32) path, on a rank with no
                                # rows (BT == 0 early return) and beyond the slice limit
                                dict(_dtype=torch.float32), dict(_rank0_no_rows=True),
                                dict(_rank0_no_rows=True, _dtype=torch.float32), dict(dw_slices=40),
                                dict(reduction="none"), dict(reduction="sum", dw_slices=7),
                                # grad_w summed by the peer-memory kernel (csrc/peer.cu) instead of
                                # the collective: sliced, unsliced, fp32, a rank with no rows
                                dict(comm="peer"), dict(comm="peer", dw_slices=1),
                                dict(comm="peer", dw_slices=7, label_smoothing=0.1),
                                dict(comm="peer", _dtype=torch.float32), dict(comm="peer", _rank0_no_rows=True),
                                # each rank's ignore_index rows skipped (kept-row path)
                                dict(_min_skipped=1), dict(_min_skipped=1, comm="peer"),
                                dict(_min_skipped=1, reduction="none"), dict(_min_skipped=1, _ignore_first_half=True)])
def test_token_sharded_cuda_world2(kw):
    _run("token", kw)


@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1, softcap=30.0), dict(lse_square_scale=1e-4),
                                dict(_ignore_first_half=True), dict(dx_reduce_dtype=torch.float32),
                                dict(_dtype=torch.float32), dict(_min_skipped=1),
                                dict(_min_skipped=1, _ignore_first_half=True, label_smoothing=0.1),
                                # dX partials summed by the peer-memory kernel (csrc/peer.cu)
                                dict(comm="peer"), dict(comm="peer", _min_skipped=1),
                                dict(comm="peer", dx_reduce_dtype=torch.float32)])
def test_vocab_parallel_cuda_world2(kw):
    _run("vocab", kw)


def _sync_free_worker(rank, port, mode, out, skip=False):
    """One-rank NCCL group: the sharded call must enqueue every kernel and collective without a
    device->host sync (the dW all-reduce overlap was defeated by an .item())."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        from paper_2410_10989_b200.distributed import token_sharded_flce, vocab_parallel_flce, vocab_shard

        x, w, t = _problem(bt=1024, h=512, v=4096)
        xb = torch.tensor(x, dtype=torch.bfloat16, device=dev)
        wb = torch.tensor(w, dtype=torch.bfloat16, device=dev)
        tb = torch.tensor(t, device=dev)
        sh = vocab_shard(wb.shape[0], 0, 1)

        def call():
            if mode == "token":
                # skip=True: the kept-row path with the count on the device (the default mode)
                return token_sharded_flce(xb, wb, tb, chunk_rows=256, check_targets=False, skip_ignored_rows=skip)
            return vocab_parallel_flce(xb, wb, tb, sh, chunk_rows=256, check_targets=False, skip_ignored_rows=False)

        ref = call()  # warm (workspace allocation, tensor-map encode, NCCL communicator)
        torch.cuda.synchronize()
        torch.cuda.set_sync_debug_mode("error")
        try:
            got = call()
        finally:
            torch.cuda.set_sync_debug_mode(0)
        torch.cuda.synchronize()
        same = all(torch.equal(a, b) for a, b in zip(ref, got))
        out[0] = "ok" if same else "second call differs"
    except Exception as e:  # pragma: no cover
        out[0] = repr(e)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,skip", [("token", False), ("vocab", False), ("token", True)])
def test_sharded_calls_have_no_host_sync(mode, skip):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.spawn(_sync_free_worker, args=(_port(), mode, out, skip), nprocs=1, join=True)
    assert dict(out) == {0: "ok"}, dict(out)
