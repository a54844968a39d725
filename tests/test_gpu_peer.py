"""Peer-memory all-reduce (csrc/peer.cu, peer.py) with 2 and 3 ranks sharing cuda:0 (GPU).

The ranks are separate processes, so their buffers are distinct allocations mapped into each
other through CUDA IPC exactly as on an NVLink node; only the wires differ (same-device
memory instead of NVLink).  gloo carries the handle exchange.  Checked: the sum is the fp32
rank-order sum rounded once, bit for bit, on every rank; ragged lengths, 16-byte-unaligned
ranges (scalar path), repeated calls (epochs), every dtype; and a missing peer ends in
PeerTimeout instead of a hung GPU.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(rank, trial, n, dtype):
    g = torch.Generator().manual_seed(1000 * trial + rank)
    return (torch.randn(n, generator=g) * (1 + rank)).to(dtype)


def _expected(world, trial, n, dtype):
    acc = torch.zeros(n, dtype=torch.float32)
    for r in range(world):
        acc = acc + _inputs(r, trial, n, dtype).float()  # rank order, fp32
    return acc.to(dtype)


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_10989_b200.peer import PeerBuffer, PeerTimeout

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        bad = []
        if case == "timeout":
            buf = PeerBuffer(1 << 16, device=dev, timeout_s=0.5)
            t = buf.tensor((1000,), torch.bfloat16)
            if rank == 0:  # the other ranks never call: rank 0's kernel must give up, not hang
                buf.all_reduce_(t)
                try:
                    buf.check()
                    bad.append("no PeerTimeout")
                except PeerTimeout:
                    pass
                try:
                    buf.all_reduce_(t)
                    bad.append("poisoned buffer accepted a call")
                except PeerTimeout:
                    pass
            dist.barrier()
        else:
            buf = PeerBuffer(4 << 20, device=dev)
            side = torch.cuda.Stream(device=dev)
            trial = 0
            for dtype in (torch.bfloat16, torch.float32, torch.float16):
                for n, cuts in ((100_003, (0, 100_003)), (262_144, (0, 65_536, 131_072, 262_144)),
                                (50_001, (0, 7, 20_001, 50_001)), (5, (0, 5)), (1, (0, 1))):
                    trial += 1
                    t = buf.tensor((n,), dtype)
                    t.copy_(_inputs(rank, trial, n, dtype).to(dev))
                    torch.cuda.synchronize()
                    for lo, hi in zip(cuts[:-1], cuts[1:]):  # slices, like the per-slice dW calls
                        buf.all_reduce_(t, lo, hi, stream=side)
                    torch.cuda.synchronize()
                    got = t.cpu()
                    if not torch.equal(got.view(torch.int16 if dtype != torch.float32 else torch.int32),
                                       _expected(world, trial, n, dtype).view(
                                           torch.int16 if dtype != torch.float32 else torch.int32)):
                        bad.append((str(dtype), n, cuts))
            buf.check()
        out[rank] = "ok" if not bad else repr(bad)
    except Exception as e:  # pragma: no cover - reported to the parent
        out[rank] = repr(e)
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.spawn(_worker, args=(world, _port(), case, out), nprocs=world, join=True)
    assert dict(out) == {r: "ok" for r in range(world)}, dict(out)


@pytest.mark.parametrize("world", [2, 3])
def test_peer_allreduce_bitwise(world):
    _run(world, "sum")


def test_peer_allreduce_missing_peer_times_out():
    _run(2, "timeout")
