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
        xb = torch.tensor(x, dtype=torch.bfloat16, device=dev)
        wb = torch.tensor(w, dtype=torch.bfloat16, device=dev)
        tb = torch.tensor(t, device=dev)
        ref_kw = dict(kw)
        if "ce_weight" in kw:  # numpy class weights: the oracle's `weight`, the library's ce_weight tensor
            ref_kw["weight"] = ref_kw.pop("ce_weight")
            kw["ce_weight"] = torch.tensor(kw["ce_weight"], dtype=torch.float32, device=dev)
        ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(xb.double().cpu().numpy(), wb.double().cpu().numpy(), t, **ref_kw)
        if mode == "token":
            lo, hi = shard_rows(len(t), rank, WORLD)
            loss, gx, gw = token_sharded_flce(xb[lo:hi].contiguous(), wb, tb[lo:hi], chunk_rows=128, **kw)
            gx_ref, gw_ref = rgx[lo:hi], rgw
        else:
            sh = vocab_shard(w.shape[0], rank, WORLD)
            loss, gx, gw = vocab_parallel_flce(xb, wb[sh.offset:sh.offset + sh.size].contiguous(), tb, sh,
                                               chunk_rows=160, **kw)
            gx_ref, gw_ref = rgx, rgw[sh.offset:sh.offset + sh.size]
        torch.cuda.synchronize()
        checks = [("loss", float(loss.float().item()), ref_loss), ("gx", gx.float().cpu().numpy(), gx_ref),
                  ("gw", gw.float().cpu().numpy(), gw_ref)]
        bad = [(n, rel_close(a, b, 2e-2)[1]) for n, a, b in checks if not rel_close(a, b, 2e-2)[0]]
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
                                dict(ce_weight=_CW, label_smoothing=0.1), dict(_ignore_first_half=True)])
def test_token_sharded_cuda_world2(kw):
    _run("token", kw)


@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1, softcap=30.0), dict(lse_square_scale=1e-4),
                                dict(_ignore_first_half=True)])
def test_vocab_parallel_cuda_world2(kw):
    _run("vocab", kw)
