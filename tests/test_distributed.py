"""Token-sharded and vocab-parallel FLCE host logic, world_size 2 over gloo on CPU.

The collective choreography in paper_2410_10989_b200.distributed (count all-reduce,
loss / dW all-reduce; per-row statistics all-reduce, dX all-reduce) is exercised with
the float64 oracle standing in for the CUDA stages, and the result is compared with
the single-process oracle on the same global inputs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import liger_ref
from paper_2410_10989_b200.distributed import (
    VocabShard,
    shard_rows,
    token_sharded_flce,
    vocab_parallel_flce,
    vocab_shard,
)

WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem(bt=24, h=6, v=11, seed=0, ignore_first_half=False):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (v, h)) * 1.5
    t = rng.integers(0, v, bt)
    t[rng.random(bt) < 0.25] = -100
    if ignore_first_half:
        t[: bt // 2] = -100  # at world 2, rank 0's whole token shard is ignore_index
    return x, w, t


# ---------------------------------------------------------- oracle stages
def oracle_count(t, vocab=None, ignore_index=-100):
    return torch.tensor([int((t != ignore_index).sum()), 0], dtype=torch.int64)


def oracle_local_flce(x, w, t, counts, ignore_index=-100, reduction="mean", **kw):
    n = int(counts[0])
    loss, rows, _, g = liger_ref.ce(x.numpy() @ w.numpy().T, t.numpy(), ignore_index=ignore_index,
                                    reduction="sum", **kw)
    scale = 1.0 / max(n, 1) if reduction == "mean" else 1.0
    g = g * scale
    lv = torch.tensor(rows) if reduction == "none" else torch.tensor(loss * scale, dtype=torch.float64)
    return lv, torch.tensor(g @ w.numpy()), torch.tensor(g.T @ x.numpy())


class OracleVocabOps:
    def count(self, t, vocab, ignore_index):
        return oracle_count(t, vocab, ignore_index)

    def logits_stats(self, x, w_shard, t, shard, softcap, ignore_index):
        z = x.numpy() @ w_shard.numpy().T
        if softcap:
            z = softcap * np.tanh(z / softcap)
        m = z.max(axis=1)
        s = np.exp(z - m[:, None]).sum(axis=1)
        sz = z.sum(axis=1)
        tl = t.numpy() - shard.offset
        inr = (tl >= 0) & (tl < shard.size)
        zt = np.where(inr, z[np.arange(len(tl)), np.clip(tl, 0, shard.size - 1)], 0.0)
        return torch.tensor(np.stack([m, s, sz, zt], axis=1)), torch.tensor(z)

    def combine_stats(self, gathered):
        g = gathered.numpy()
        m = g[:, :, 0].max(axis=0)
        s = (g[:, :, 1] * np.exp(g[:, :, 0] - m[None, :])).sum(axis=0)
        return torch.tensor(np.stack([m, s, g[:, :, 2].sum(axis=0), g[:, :, 3].sum(axis=0)], axis=1))

    def backward(self, x, w_shard, t, shard, stats_g, buf, n_valid, gw_acc, accumulate, *, ignore_index,
                 label_smoothing, lse_square_scale, softcap, reduction, gx_out=None):
        z = buf.numpy()
        st = stats_g.numpy()
        m, s, sz, zt = st[:, 0], st[:, 1], st[:, 2], st[:, 3]
        lse = m + np.log(s)
        tn = t.numpy()
        valid = tn != ignore_index
        eps = label_smoothing / shard.total
        scale = 1.0 / max(int(n_valid[0]), 1) if reduction == "mean" else 1.0
        loss = lse - zt
        if label_smoothing > 0:
            loss = loss * (1 - label_smoothing) + label_smoothing * lse - eps * sz
        loss = (loss + lse_square_scale * lse * lse) * scale
        loss = np.where(valid, loss, 0.0)
        g = np.exp(z - m[:, None]) / s[:, None] * (1 + 2 * lse_square_scale * lse[:, None]) - eps
        tl = tn - shard.offset
        hit = valid & (tl >= 0) & (tl < shard.size)
        g[np.nonzero(hit)[0], tl[hit]] -= 1 - label_smoothing
        g *= scale
        if softcap:
            g *= 1 - (z / softcap) ** 2
        g[~valid] = 0
        gw = torch.tensor(g.T @ x.numpy())
        if accumulate:
            gw_acc += gw
        else:
            gw_acc.copy_(gw)
        return torch.tensor(loss), torch.tensor(g @ w_shard.numpy())


# ------------------------------------------------------------------ workers
def _worker(rank, port, mode, kw, out, world=WORLD, prob=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, t = problem(**(prob or {}))
        ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t, **kw)
        if mode == "token":
            lo, hi = shard_rows(len(t), rank, world)
            loss, gx, gw = token_sharded_flce(torch.tensor(x[lo:hi]), torch.tensor(w), torch.tensor(t[lo:hi]),
                                              count_fn=oracle_count, local_fn=oracle_local_flce, **kw)
            if kw.get("reduction") == "none":  # this rank's own per-row losses, never summed across ranks
                ref_rows = liger_ref.flce(x[lo:hi], w, t[lo:hi], **kw)[1]
                assert loss.shape == (hi - lo,)
                np.testing.assert_allclose(loss.numpy(), ref_rows, rtol=1e-12, atol=1e-14)
            else:
                np.testing.assert_allclose(loss.item(), ref_loss, rtol=1e-12)
            np.testing.assert_allclose(gx.numpy(), rgx[lo:hi], rtol=1e-10, atol=1e-14)
            np.testing.assert_allclose(gw.numpy(), rgw, rtol=1e-10, atol=1e-14)
        else:
            sh = vocab_shard(w.shape[0], rank, world)
            loss, gx, gw = vocab_parallel_flce(torch.tensor(x), torch.tensor(w[sh.offset:sh.offset + sh.size]),
                                               torch.tensor(t), sh, chunk_rows=7, ops=OracleVocabOps(), **kw)
            np.testing.assert_allclose(loss.item(), ref_loss, rtol=1e-6)  # per-row losses are kept in fp32
            np.testing.assert_allclose(gx.numpy(), rgx, rtol=1e-10, atol=1e-14)
            np.testing.assert_allclose(gw.numpy(), rgw[sh.offset:sh.offset + sh.size], rtol=1e-10, atol=1e-14)
        out[rank] = "ok"
    except Exception as e:  # pragma: no cover - reported to the parent
        out[rank] = repr(e)
    finally:
        dist.destroy_process_group()


def run_world(mode, kw, world=WORLD, prob=None):
    port = free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(port, mode, kw, out, world, prob), nprocs=world, join=True)
    assert dict(out) == {r: "ok" for r in range(world)}, dict(out)


def test_shard_rows_cover_exactly():
    for n in (1, 7, 24, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert vocab_shard(128256, 7, 8) == VocabShard(112224, 16032, 128256)


@pytest.mark.parametrize("kw", [dict(), dict(reduction="sum"), dict(label_smoothing=0.1)])
def test_token_sharded_world2_matches_single_process(kw):
    run_world("token", kw)


@pytest.mark.parametrize("kw", [dict(), dict(softcap=3.0, label_smoothing=0.1), dict(lse_square_scale=1e-3)])
def test_vocab_parallel_world2_matches_single_process(kw):
    run_world("vocab", kw)


def test_token_sharded_reduction_none_ragged_world3():
    """reduction='none' returns each rank's own per-row losses (ragged 9/8/8 shards): the
    per-row vectors are not all-reduced element-wise across ranks."""
    run_world("token", dict(reduction="none"), world=3, prob=dict(bt=25))


@pytest.mark.parametrize("mode", ["token", "vocab"])
def test_world3_ragged_shards(mode):
    """Uneven splits on both axes: 25 tokens -> 9/8/8 rows, 11 classes -> 4/4/3 vocab columns."""
    run_world(mode, dict(label_smoothing=0.05), world=3, prob=dict(bt=25))


@pytest.mark.parametrize("mode", ["token", "vocab"])
def test_world2_rank_with_only_ignored_tokens(mode):
    """A rank whose token shard is all ignore_index contributes zero loss/dX but still joins
    every collective; the mean denominator is the global valid count."""
    run_world(mode, dict(), prob=dict(ignore_first_half=True))


@pytest.mark.parametrize("mode", ["token", "vocab"])
def test_world4_matches_single_process(mode):
    """Four ranks (the 8xB200 box's scaling points are 1/2/4/8): ragged token and vocab shards,
    smoothing + softcap on the vocab path, against the single-process oracle."""
    kw = dict(label_smoothing=0.1) if mode == "token" else dict(softcap=3.0, label_smoothing=0.1)
    run_world(mode, kw, world=4, prob=dict(bt=30))
