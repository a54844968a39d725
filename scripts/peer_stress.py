"""Stress of the peer-memory all-reduce flag protocol: W processes on cuda:0 (IPC mappings),
N back-to-back calls of varying sizes and offsets on one side stream, each checked bit for bit
against the fp32 rank-order sum at the end of every 50 calls.

    python scripts/peer_stress.py [world] [calls]"""

import os
import socket
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, calls, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_10989_b200.peer import PeerBuffer

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    buf = PeerBuffer(8 << 20, device=dev, timeout_s=60)
    side = torch.cuda.Stream()
    bad = 0
    t0 = time.time()
    for c in range(calls):
        n = 1000 + (c * 7919) % 200000
        g = torch.Generator().manual_seed(c * 97 + rank)
        t = buf.tensor((n,), torch.bfloat16)
        t.copy_((torch.randn(n, generator=g) * (rank + 1)).to(torch.bfloat16).to(dev))
        torch.cuda.synchronize()
        lo = (c * 13) % 64
        buf.all_reduce_(t, lo, n, stream=side)
        if c % 50 == 49 or c == calls - 1:
            torch.cuda.synchronize()
            want = torch.zeros(n - lo)
            for r in range(world):
                gr = torch.Generator().manual_seed(c * 97 + r)
                want = want + (torch.randn(n, generator=gr) * (r + 1)).to(torch.bfloat16).float()[lo:]
            bad += int(not torch.equal(t[lo:].cpu().view(torch.int16), want.to(torch.bfloat16).view(torch.int16)))
        else:
            torch.cuda.synchronize()
    buf.check()
    out[rank] = f"calls {calls}, bad {bad}, {time.time() - t0:.1f} s, epoch {buf.epoch}"
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(worker, args=(world, port, calls, out), nprocs=world, join=True)
    print(dict(out))
