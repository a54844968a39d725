#!/usr/bin/env python
"""FLCE fwd+bwd benchmark at the Llama-3-8B lm_head shape (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one fused-linear-cross-entropy forward+backward over one synthetic batch
(BT=8192 tokens, H=4096, V=128256, bf16, 10% ignore_index targets): loss, grad_x and
grad_w, i.e. 6*BT*H*V = 2.58e13 FLOP.  Under torchrun (N>1) every rank runs the
token-sharded mode on its own 8192 tokens (weak scaling) with the NCCL dW all-reduce.

Keys beyond the base contract:
  roofline      dominant kernel = the tcgen05 GEMM (logits + backward launches); achieved =
                algorithmic FLOP / summed CUDA-event durations of those launches in the timed
                region; peak from MEASURED_PEAKS.json (sustained: launched inside a long step).
  cpu_baseline  the oracle port of rowfuse.flce_forward_backward (numpy f32, all host threads)
                on a bounded 256-token sample (one reference-plan chunk) of the same shape, rank 0 at N=1 only.
  e2e           the public module LigerFusedLinearCrossEntropyLoss + autograd backward with
                X/targets copied from pinned host memory every step (on a side stream, one
                step ahead, double-buffered) and the loss read back with .item() every step.
  --impl reference  times the reference's CPU algorithm (oracle port, f32) on the box's host
                cores; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BT, H, V = 8192, 4096, 128256
IGNORE_FRAC = 0.1
METRIC = "FLCE fwd+bwd tokens/s & peak mem @Llama-3-8B head; % tensor/HBM roofline"
WORKLOAD = "cfg2: Llama-3-8B lm_head FLCE fwd+bwd, BT=8192 tokens, H=4096, V=128256, bf16, 10% ignore_index"
# --config cfg4 (BASELINE.json configs[3]; not the headline line): Gemma-2-9B head
CFG4 = dict(hidden=3584, vocab=256000, softcap=30.0, label_smoothing=0.1,
            workload="cfg4: Gemma-2-9B lm_head FLCE fwd+bwd, BT=8192 tokens, H=3584, V=256000, softcap 30, "
                     "label_smoothing 0.1, bf16, 10% ignore_index")


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [s.strip() for s in line.split(",")]))

    def mark(self, which):
        setattr(self, which, time.monotonic())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        rows = [r for ts, r in self.rows if t0 is None or (t0 - 0.1 <= ts <= t1 + 0.25)]
        if not rows and self.rows:  # region shorter than the sampling period: nearest sample
            rows = [min(self.rows, key=lambda tr: abs(tr[0] - (t0 or 0)))[1]]
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 7:
                for n, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU baseline
def cpu_flce_sample(rows: int, reps: int = 2):
    """Oracle port of rowfuse.flce_forward_backward at f32 on `rows` tokens of the cfg2 shape."""
    import numpy as np

    from oracle import rowfuse_port as rp  # CPU baseline leg only

    rng = np.random.default_rng(0)
    x = (rng.random((rows, H), dtype=np.float32) * 2 - 1)
    w_hv = (rng.random((H, V), dtype=np.float32) * 2 - 1) / np.float32(64.0)
    t = rng.integers(0, V, rows)
    plan = rp.plan_chunk_rows(BT, V, H)  # the reference's chunk at the full batch (256 rows)
    rp.flce_forward_backward(x[:8], w_hv, t[:8], chunk_rows=plan)  # warm
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=plan)
        times.append(time.perf_counter() - t0)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return statistics.median(times), cores


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import numpy as np

    from oracle import rowfuse_port as rp  # --impl reference: the reference's CPU algorithm

    rows = args.ref_rows
    rng = np.random.default_rng(0)
    x = rng.random((rows, H), dtype=np.float32) * 2 - 1
    w_hv = (rng.random((H, V), dtype=np.float32) * 2 - 1) / np.float32(64.0)
    t = rng.integers(0, V, rows)
    plan = rp.plan_chunk_rows(BT, V, H)  # the chunk the reference uses at BT=8192 (256 rows)
    for _ in range(args.warmup):
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=plan)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=plan)
    el = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    value = rows * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "bt_per_step": rows, "hidden": H, "vocab": V,
                   "sample": f"{rows} tokens of the cfg2 shape per step = one reference-plan chunk "
                             f"(plan_chunks(8192, 128256, 4096) = 256 rows)",
                   "parallelism": "host threads (numpy/OpenBLAS)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"{rows} tokens/step, rowfuse.flce_forward_backward restated in numpy f32 "
                                   f"(oracle/rowfuse_port.py), chunk = plan_chunks at BT=8192"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2410_10989_b200 as lk
    from paper_2410_10989_b200 import _capi, _utils
    from paper_2410_10989_b200.distributed import token_sharded_flce, vocab_parallel_flce, vocab_shard
    from paper_2410_10989_b200.fused_linear_cross_entropy import (
        flce_plan,
        flce_workspace_bytes,
        fused_linear_cross_entropy_forward,
    )

    rank, world, local = env_rank()
    vocab_mode = args.mode == "vocab"
    # Test hook for the multi-rank code path on a 1-GPU box: LK_BENCH_SHARE_GPU=1 puts every
    # rank on cuda:0 over gloo (NCCL refuses two ranks per device).  Numbers from it are not
    # bench values.
    share = os.environ.get("LK_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1 or vocab_mode:
        torch.cuda.set_device(local)
        if world == 1:  # vocab-parallel at N=1: a one-rank group so the same code path runs
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        elif share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    L = _capi.load()
    bt, h, v = args.bt, args.hidden, args.vocab
    opts = dict(softcap=args.softcap, label_smoothing=args.label_smoothing)
    workload = CFG4["workload"] if args.config == "cfg4" else WORKLOAD

    # token mode: every rank its own BT tokens (weak scaling); vocab mode: one global problem,
    # W rows sharded over ranks (strong scaling of the GEMM work)
    g = torch.Generator(device=dev).manual_seed(1000 + (0 if vocab_mode else rank))
    x = (torch.rand(bt, h, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, h, device=dev, generator=g) * 2 - 1) / 64.0).to(torch.bfloat16)
    t = torch.randint(0, v, (bt,), device=dev, generator=g)
    t[torch.rand(bt, device=dev, generator=g) < IGNORE_FRAC] = -100
    chunk = args.chunk_rows or flce_plan(bt, h, v)[0]
    if vocab_mode:
        shard = vocab_shard(v, rank, world)
        w = w[shard.offset:shard.offset + shard.size].contiguous()

    def step():
        if vocab_mode:
            return vocab_parallel_flce(x, w, t, shard, chunk_rows=chunk, **opts)
        if world > 1:
            return token_sharded_flce(x, w, t, chunk_rows=chunk, **opts)
        return fused_linear_cross_entropy_forward(x, w, t, chunk_rows=chunk, compute_grad_input=True, **opts,
                                                  compute_grad_weight=True)

    def barrier():
        if world > 1:
            dist.barrier()

    clk = ClockSampler(local).__enter__()  # started early: nvidia-smi needs ~0.5 s to emit samples
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # peak memory of one step (untimed): SURVEY §8(d) definition
    torch.cuda.reset_peak_memory_stats(dev)
    base = torch.cuda.memory_allocated(dev)
    out = step()
    torch.cuda.synchronize()
    peak_extra = torch.cuda.max_memory_allocated(dev) - base
    del out
    out_bytes = bt * h * 2 + w.shape[0] * h * 2
    ws_bytes = flce_workspace_bytes(bt, h, v, torch.bfloat16, chunk, True)
    logits_chunk_bytes = chunk * (-(-v // 64) * 64) * 2

    # ---- timed region (device-resident inputs) ----
    L.lk_profile_enable(1)
    L.lk_profile_collect(None, None)
    n0 = L.lk_launch_count()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark("t0")
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    clk.mark("t1")
    clk.__exit__()
    barrier()
    launches = (L.lk_launch_count() - n0) / args.steps
    L.lk_profile_enable(0)
    import ctypes as C

    ms4 = (C.c_double * 4)()
    cnt4 = (C.c_int64 * 4)()
    L.lk_profile_collect(ms4, cnt4)
    ms = ev0.elapsed_time(ev1)
    tmax = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    tokens_per_step = bt if vocab_mode else world * bt
    value = tokens_per_step * args.steps / (ms / 1e3)
    flop_step = 6.0 * bt * h * v / (world if vocab_mode else 1)  # per rank

    # ---- e2e through the public module, host buffers, H2D/D2H inside the timed region ----
    xh = x.cpu().pin_memory()
    th = t.cpu().pin_memory()
    wp = torch.nn.Parameter(w.clone())
    loss_fn = lk.LigerFusedLinearCrossEntropyLoss(chunk_rows=chunk, **opts)

    # Inputs of step i+1 are copied host->device on a side stream while step i computes
    # (double-buffered), as a training input pipeline does; every step still moves its own
    # X and targets from pinned host memory and reads its loss back.
    copy_stream = torch.cuda.Stream(device=dev)
    bufs = [(torch.empty_like(x), torch.empty_like(t)) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    state = {"i": 0}

    def stage_copy(i):
        xb, tb = bufs[i % 2]
        with torch.cuda.stream(copy_stream):
            xb.copy_(xh, non_blocking=True)
            tb.copy_(th, non_blocking=True)
            ready[i % 2].record(copy_stream)

    def e2e_step():
        i = state["i"]
        if i == 0:
            stage_copy(0)
        stage_copy(i + 1)  # next step's inputs in flight during this step
        cur = torch.cuda.current_stream(dev)
        cur.wait_event(ready[i % 2])
        xd, td = bufs[i % 2]
        xd.record_stream(cur)
        xd = xd.detach().requires_grad_(True)
        state["i"] = i + 1
        if vocab_mode:
            loss, gx, gw = vocab_parallel_flce(xd.detach(), wp.detach(), td, shard, chunk_rows=chunk, **opts)
            val = loss.item()
        elif world > 1:
            loss, gx, gw = token_sharded_flce(xd, wp, td, chunk_rows=chunk, **opts)
            val = loss.item()
        else:
            loss = loss_fn(wp, xd, td)
            loss.backward()
            val = loss.item()
        wp.grad = None
        return val

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    ems = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
    e2e_value = tokens_per_step * args.steps / (float(ems.item()) / 1e3)

    peaks, peak_src = measured_peaks()
    gemm_ms = (ms4[0] + ms4[2]) / args.steps
    achieved = flop_step / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    peak_sus = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    # DRAM bytes of the GEMM launches from the committed ncu --set full capture of one step
    # (scripts/profile_json.py): per launch on average, like `achieved`
    traffic, traffic_step = None, None
    prof = ROOT / "profiles" / "r01_flce_step.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic, traffic_step = pj.get("gemm_dram_bytes_per_launch"), pj.get("dram_bytes_per_step")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, cores = cpu_flce_sample(args.cpu_rows)
        cpu = {"value": args.cpu_rows / sec, "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": f"{args.cpu_rows} tokens of the cfg2 shape (H=4096, V=128256) = one reference-plan "
                         f"chunk, oracle port of rowfuse.flce_forward_backward in numpy f32, median of 2"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if vocab_mode else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform X, W, 10% ignore_index targets)",
            "config": {
                "workload": workload, "bt_per_gpu": bt, "hidden": h, "vocab": v, "chunk_rows": chunk,
                "softcap": args.softcap, "label_smoothing": args.label_smoothing,
                "num_chunks": -(-bt // chunk), "global_tokens": tokens_per_step,
                "parallelism": (f"vocab-parallel vp{world}" if vocab_mode else
                                (f"token-sharded dp{world}" if world > 1 else "single GPU")),
                "l2": "inputs larger than L2 (W = 1.05 GB bf16 re-streamed every chunk)",
            },
            "roofline": {
                "bound": "tensor", "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s",
                "frac": (achieved / peak_sus) if achieved else None, "traffic": traffic,
                "kernel": "tc2::gemm2_kernel<bf16> (CTA-pair tcgen05; logits + backward launches)",
                "traffic_unit": "DRAM bytes per GEMM launch (avg over one step's launches, ncu)",
                "traffic_per_step": traffic_step,
                "algorithmic_flop_per_step": flop_step,
                "peak_source": f"{peak_src} bf16_tflops_sustained", "peak_burst": float(peaks["bf16_tflops"]),
                "frac_of_burst": (achieved / float(peaks["bf16_tflops"])) if achieved else None,
                "step_tflops": flop_step / (ms / args.steps / 1e3) / 1e12,
                "stage_ms_per_step": {"logits_gemm": ms4[0] / args.steps, "finalize": ms4[1] / args.steps,
                                      "backward_gemm": ms4[2] / args.steps, "other": ms4[3] / args.steps},
            },
            "peak_mem": {"peak_extra_bytes": peak_extra, "outputs_bytes": out_bytes,
                         "peak_extra_minus_outputs": peak_extra - out_bytes, "workspace_bytes": ws_bytes,
                         "logits_chunk_bytes": logits_chunk_bytes, "dw_fp32_accumulator_bytes": v * h * 4,
                         "full_logits_bytes_avoided": bt * v * 2},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": bt * h * 2 + bt * 8,
                    "d2h_bytes_per_step": 4,
                    "api": ("distributed.vocab_parallel_flce" if vocab_mode else
                            "distributed.token_sharded_flce" if world > 1 else
                            "LigerFusedLinearCrossEntropyLoss + backward()"),
                    "h2d_pipeline": "each step's X/targets copied from pinned host memory on a side stream, "
                                    "double-buffered one step ahead; loss read back with .item() every step"},
            "gpu_launches": launches * args.steps,
            "gpu_launches_per_step": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1 or vocab_mode:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--bt", type=int, default=BT)
    ap.add_argument("--hidden", type=int, default=H)
    ap.add_argument("--vocab", type=int, default=V)
    ap.add_argument("--chunk-rows", type=int, default=0)
    ap.add_argument("--config", choices=["cfg2", "cfg4"], default="cfg2",
                    help="cfg2 = Llama-3-8B head (headline); cfg4 = Gemma-2-9B head with softcap 30 + smoothing 0.1")
    ap.add_argument("--softcap", type=float, default=None)
    ap.add_argument("--label-smoothing", type=float, default=0.0)
    ap.add_argument("--mode", choices=["token", "vocab"], default="token",
                    help="multi-GPU shard mode: token-sharded (default, weak scaling) or vocab-parallel (strong)")
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--ref-rows", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.config == "cfg4":
        args.hidden, args.vocab = CFG4["hidden"], CFG4["vocab"]
        args.softcap, args.label_smoothing = CFG4["softcap"], CFG4["label_smoothing"]
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
