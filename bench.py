#!/usr/bin/env python
"""FLCE fwd+bwd benchmark at the Llama-3-8B lm_head shape (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg4|cfg5] [--mode token|vocab]

One step = one fused-linear-cross-entropy forward+backward over one synthetic batch
(BT=8192 tokens, H=4096, V=128256, bf16, 10% ignore_index targets): loss, grad_x and
grad_w, i.e. 6*BT*H*V = 2.58e13 FLOP.

Multi-GPU (one process per GPU over NCCL).  `--gpus N` without a torchrun environment
re-launches itself under `torch.distributed.run` with N ranks on 127.0.0.1; under torchrun
the env (RANK/WORLD_SIZE/LOCAL_RANK) is used as is.  The batch is ONE seed-0 global batch
generated identically on every rank and split by rows with distributed.shard_rows:
  cfg2 (default)  token-sharded weak scaling: N x 8192 global tokens, 8192 per rank, full W
                  replica per rank, NCCL all-reduce of dW overlapped with the last chunk.
  cfg5            token-sharded strong scaling: 65536 global tokens (BASELINE configs[4]),
                  65536/N per rank.
  --mode vocab    vocab-parallel strong scaling of one 8192-token batch (W rows sharded).

The device-resident loop passes check_targets=False (the out-of-range target count is still
computed on the device every step; its host read would stall the next step's launch) and
makes one checked, untimed call afterwards on the same batch.

Keys beyond the base contract:
  roofline      dominant kernel = the tcgen05 GEMM (logits + backward launches); achieved =
                executed FLOP (6 * kept rows * H * V: the ignore_index rows are skipped, see
                variants.all_rows) / summed CUDA-event durations of those launches in the timed
                region; peak from MEASURED_PEAKS.json (sustained: launched inside a long step);
                traffic = ncu DRAM bytes per GEMM launch for THIS config (profiles/r02_traffic.json,
                scripts/traffic_capture.py), null when no capture exists for the config.
  cpu_baseline  the oracle port of rowfuse.flce_forward_backward (numpy f32, all host threads)
                on a bounded 256-token sample of the same shape, rowfuse's protocol (3 warm-ups,
                10 repeats, median and q20/q80; rowfuse/bench.py:46-48, 315-324); plus `cfg1`:
                BASELINE configs[0] on all cores and at OPENBLAS_NUM_THREADS=1, beside the
                GPU's fp32 FLCE on the same cfg1 inputs.  Rank 0 at N=1 only.
  e2e           the public module LigerFusedLinearCrossEntropyLoss + autograd backward with
                X/targets copied from pinned host memory every step (on a side stream, one
                step ahead, double-buffered) and every step's loss copied back to pinned host
                memory inside the timed region, read on the host one step later.
  variants      accum_dtype=torch.float32 (fp32 dW accumulator) tokens/s and peak memory;
                all_rows: skip_ignored_rows=False (every row through the GEMMs).
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
# --config cfg5 (BASELINE.json configs[4]): one 65536-token global batch split across the ranks
CFG5_BT = 65536
CFG5_WORKLOAD = ("cfg5: token-sharded FLCE fwd+bwd, BT=65536 global tokens split across ranks, H=4096, "
                 "V=128256, bf16, 10% ignore_index, NCCL dW all-reduce")


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
REF_WARMUP, REF_REPEATS = 3, 10  # rowfuse/bench.py:46-48


def quantiles(times):
    """median and [0.2, 0.8] quantiles (rowfuse/bench.py:315-324)."""
    import numpy as np

    a = np.asarray(times, dtype=np.float64)
    return float(np.median(a)), float(np.quantile(a, 0.2)), float(np.quantile(a, 0.8))


def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cfg2_sample_inputs(rows, hidden=H, vocab=V):
    import numpy as np

    rng = np.random.default_rng(0)
    x = (rng.random((rows, hidden), dtype=np.float32) * 2 - 1)
    w_hv = (rng.random((hidden, vocab), dtype=np.float32) * 2 - 1) / np.float32(64.0)
    t = rng.integers(0, vocab, rows)
    return x, w_hv, t


def cfg1_inputs_np():
    """BASELINE configs[0] / SURVEY §8(d) cfg1: BT=1024, H=512, V=4096, fp32, seed 0, W_hv ~ U(-1,1)/sqrt(H)."""
    import numpy as np

    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (1024, 512)).astype(np.float32)
    w_hv = (rng.uniform(-1, 1, (512, 4096)) / math.sqrt(512)).astype(np.float32)
    t = rng.integers(0, 4096, 1024)
    return x, w_hv, t


def time_port(x, w_hv, t, chunk, warmup=REF_WARMUP, repeats=REF_REPEATS):
    from oracle import rowfuse_port as rp  # CPU baseline leg only

    for _ in range(warmup):
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=chunk)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=chunk)
        times.append(time.perf_counter() - t0)
    return quantiles(times)


def cpu_cfg1_worker():
    """Child process: cfg1 on the port with the thread count fixed by its environment."""
    x, w_hv, t = cfg1_inputs_np()
    med, q20, q80 = time_port(x, w_hv, t, None)
    print(json.dumps({"median_ms": 1e3 * med, "q20_ms": 1e3 * q20, "q80_ms": 1e3 * q80,
                      "tokens_per_s": 1024 / med, "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                      "cores": host_cores()}))


def cpu_cfg1(one_thread: bool):
    env = dict(os.environ)
    if one_thread:
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            env[k] = "1"
    else:
        env.pop("OPENBLAS_NUM_THREADS", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cpu-cfg1-worker"], capture_output=True,
                         text=True, env=env, timeout=600, cwd=ROOT)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode != 0 or not lines:
        return {"error": out.stderr[-300:]}
    d = json.loads(lines[-1])
    d["threads"] = 1 if one_thread else d["cores"]
    return d


def cpu_baseline_line(rows):
    """cfg2-shape bounded sample (same workload as the GPU line) + cfg1 on all cores / 1 thread."""
    from oracle import rowfuse_port as rp  # CPU baseline leg only

    x, w_hv, t = cfg2_sample_inputs(rows)
    plan = rp.plan_chunk_rows(BT, V, H)  # the reference's chunk at the full batch (256 rows)
    med, q20, q80 = time_port(x, w_hv, t, plan)
    return {"value": rows / med, "unit": "tokens/s", "cores": host_cores(), "kind": "port",
            "sample": f"{rows} tokens of the cfg2 shape (H=4096, V=128256; f32, no ignored targets: rowfuse has "
                      f"no ignore_index) per call = one reference-plan chunk; oracle port of "
                      f"rowfuse.flce_forward_backward in numpy f32 on all host threads; rowfuse protocol "
                      f"{REF_WARMUP} warm-ups + {REF_REPEATS} repeats, median",
            "median_ms": 1e3 * med, "q20_ms": 1e3 * q20, "q80_ms": 1e3 * q80,
            "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
            "cfg1": {"workload": "BASELINE configs[0]: BT=1024, H=512, V=4096, fp32, seed 0, default plan "
                                 "(128-row chunks), no ignored targets",
                     "all_cores": cpu_cfg1(False), "one_thread": cpu_cfg1(True)}}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import rowfuse_port as rp  # --impl reference: the reference's CPU algorithm

    rows = args.ref_rows
    hidden, vocab = args.hidden, args.vocab
    x, w_hv, t = cfg2_sample_inputs(rows, hidden, vocab)
    plan = rp.plan_chunk_rows(BT, vocab, hidden)  # the chunk the reference uses at BT=8192
    for _ in range(args.warmup):
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=plan)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rp.flce_forward_backward(x, w_hv, t, chunk_rows=plan)
        times.append(time.perf_counter() - t0)
    el = sum(times)
    med, q20, q80 = quantiles(times)
    cores = host_cores()
    value = rows * args.steps / el
    cfg = "cfg4" if args.config == "cfg4" else "cfg2"
    workload = (f"{cfg}-shape FLCE fwd+bwd sample on the host CPU: {rows} tokens per step, H={hidden}, V={vocab}, "
                f"f32, mean reduction, no ignored targets / softcap / smoothing (rowfuse implements none of them)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform X, W; uniform targets)",
        "config": {"workload": workload, "bt_per_step": rows, "hidden": hidden, "vocab": vocab, "chunk_rows": plan,
                   "sample": f"{rows} tokens of the {cfg} shape per step = one reference-plan chunk "
                             f"(plan_chunks({BT}, {vocab}, {hidden}) = {plan} rows); the full 8192-token step "
                             f"would take ~{8192 / max(value, 1e-9):.0f} s",
                   "parallelism": f"host threads (numpy/OpenBLAS, {cores} cores)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"{rows} tokens/step, rowfuse.flce_forward_backward restated in numpy f32 "
                                   f"(oracle/rowfuse_port.py; the Python reference cannot travel to the GPU box), "
                                   f"chunk = plan_chunks at BT=8192",
                         "median_ms": 1e3 * med, "q20_ms": 1e3 * q20, "q80_ms": 1e3 * q80},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def traffic_for(bt, h, v, softcap, skipped=False):
    """ncu DRAM bytes per GEMM launch for this rank's local FLCE shape (and row schedule: the
    kept-row path or all rows), captured by scripts/traffic_capture.py into
    profiles/r02_traffic.json; None when not captured."""
    prof = ROOT / "profiles" / "r02_traffic.json"
    if not prof.exists():
        return None, None, None
    try:
        d = json.loads(prof.read_text()).get(f"bt{bt}_h{h}_v{v}_cap{float(softcap or 0.0):g}"
                                             + ("_kept" if skipped else ""))
    except Exception:
        return None, None, None
    if not d or "error" in d:
        return None, None, None
    return d.get("gemm_dram_bytes_per_launch"), d.get("gemm_dram_bytes_per_step"), d.get("source")


def gpu_cfg1_fp32(dev):
    """The library's fp32 FLCE on the cfg1 inputs, rowfuse's protocol (CUDA events)."""
    import torch

    from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward

    x, w_hv, t = cfg1_inputs_np()
    xd = torch.tensor(x, device=dev)
    wd = torch.tensor(w_hv.T.copy(), device=dev)
    td = torch.tensor(t, device=dev)

    def call():
        return fused_linear_cross_entropy_forward(xd, wd, td, compute_grad_input=True, compute_grad_weight=True)

    for _ in range(REF_WARMUP):
        call()
    torch.cuda.synchronize()
    times = []
    for _ in range(REF_REPEATS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    med, q20, q80 = quantiles(times)
    return {"median_ms": 1e3 * med, "q20_ms": 1e3 * q20, "q80_ms": 1e3 * q80, "tokens_per_s": 1024 / med,
            "tflops": 6.0 * 1024 * 512 * 4096 / med / 1e12,
            "path": "fp32 FLCE through fused_linear_cross_entropy_forward (includes the host-side range check): "
                    "bf16 tensor cores on 3-piece split operands, segmented fp32 accumulation of dX"}


def gpu_cfg2_fp32(dev, steps=3):
    """fp32 FLCE at the cfg2 shape (X, W, grads in fp32): the split-operand tensor-core path."""
    import torch

    from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward

    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.rand(BT, H, device=dev, generator=g) * 2 - 1
    w = (torch.rand(V, H, device=dev, generator=g) * 2 - 1) / 64.0
    t = torch.randint(0, V, (BT,), device=dev, generator=g)
    t[torch.rand(BT, device=dev, generator=g) < IGNORE_FRAC] = -100

    def call():
        return fused_linear_cross_entropy_forward(x, w, t, compute_grad_input=True, compute_grad_weight=True)

    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    flop = 6.0 * BT * H * V
    return {"value": BT / (ms / 1e3), "unit": "tokens/s", "steps": steps, "ms_per_step": ms,
            "algorithmic_tflops": flop / (ms / 1e3) / 1e12,
            "note": "fp32 inputs/outputs at the cfg2 shape; GEMMs on the bf16 tensor cores over 3-piece split "
                    "operands (6 piece products per product, K' = 6K), dX accumulated in 32-k-block segments "
                    "summed in fp32; algorithmic_tflops counts 6*BT*H*V"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2410_10989_b200 as lk
    from paper_2410_10989_b200 import _capi
    from paper_2410_10989_b200.distributed import shard_rows, token_sharded_flce, vocab_parallel_flce, vocab_shard
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
    h, v = args.hidden, args.vocab
    opts = dict(softcap=args.softcap, label_smoothing=args.label_smoothing)
    strong = args.config == "cfg5"
    # ONE seed-0 global batch, generated identically on every rank, split by rows
    if vocab_mode:
        global_bt = args.bt
    elif strong:
        global_bt = CFG5_BT
    else:
        global_bt = args.bt * world
    lo, hi = (0, global_bt) if vocab_mode else shard_rows(global_bt, rank, world)
    bt = hi - lo
    g = torch.Generator(device=dev).manual_seed(0)
    xg = (torch.rand(global_bt, h, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, h, device=dev, generator=g) * 2 - 1) / 64.0).to(torch.bfloat16)
    tg = torch.randint(0, v, (global_bt,), device=dev, generator=g)
    tg[torch.rand(global_bt, device=dev, generator=g) < args.ignore_frac] = -100
    x, t = xg[lo:hi].contiguous(), tg[lo:hi].contiguous()
    del xg, tg
    chunk = args.chunk_rows or flce_plan(bt, h, v)[0]
    # one GPU: the library plans its own chunks (on the kept rows when ignored rows are skipped)
    call_chunk = args.chunk_rows or None
    if vocab_mode:
        shard = vocab_shard(v, rank, world)
        w = w[shard.offset:shard.offset + shard.size].contiguous()
    workload = {"cfg4": CFG4["workload"], "cfg5": CFG5_WORKLOAD}.get(args.config, WORKLOAD)

    prep_stream = torch.cuda.Stream(device=dev)

    def step(accum_dtype=None, check=False, skip=None):
        # device-resident loop: the out-of-range target count is computed on the device every
        # step; its host read (a sync that would leave the GPU idle while the next step is
        # launched) is done once, untimed, by the checked call after the loop
        if vocab_mode:
            out = vocab_parallel_flce(x, w, t, shard, chunk_rows=chunk, accum_dtype=accum_dtype,
                                      check_targets=check, skip_ignored_rows=skip, comm=args.comm, **opts)
        elif world > 1:
            out = token_sharded_flce(x, w, t, chunk_rows=call_chunk, accum_dtype=accum_dtype,
                                     check_targets=check, comm=args.comm, skip_ignored_rows=skip, **opts)
        else:
            out = fused_linear_cross_entropy_forward(x, w, t, chunk_rows=call_chunk, compute_grad_input=True, **opts,
                                                     compute_grad_weight=True, accum_dtype=accum_dtype,
                                                     check_targets=check, skip_ignored_rows=skip)
        # the next step's batch (the same resident targets) gets its kept-row compaction on a
        # side stream, as an input pipeline would prepare it: the next call reads its count
        # without waiting for this step's GEMMs (lk.prepare_kept_rows)
        if skip is not False:
            lk.prepare_kept_rows(t, stream=prep_stream)
        return out

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(ms):
        tm = torch.tensor([ms], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        return float(tm.item())

    clk = ClockSampler(local).__enter__()  # started early: nvidia-smi needs ~0.5 s to emit samples
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def peak_of(accum_dtype=None):
        """peak memory of one step beyond its inputs (untimed): SURVEY §8(d) definition"""
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        out = step(accum_dtype)
        torch.cuda.synchronize()
        pk = torch.cuda.max_memory_allocated(dev) - base
        del out
        return pk

    peak_extra = peak_of()
    out_bytes = bt * h * 2 + w.shape[0] * h * 2
    ws_bytes = flce_workspace_bytes(bt, h, v, torch.bfloat16, chunk, True)
    logits_chunk_bytes = chunk * (-(-v // 64) * 64) * 2

    def timed(n, accum_dtype=None, skip=None):
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(n):
            step(accum_dtype, skip=skip)
        ev1.record()
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1))

    # ---- timed region (device-resident inputs) ----
    L.lk_profile_enable(1)
    L.lk_profile_collect(None, None)
    n0 = L.lk_launch_count()
    clk.mark("t0")
    ms = timed(args.steps)
    clk.mark("t1")
    clk.__exit__()
    launches = (L.lk_launch_count() - n0) / args.steps
    L.lk_profile_enable(0)
    step(check=True)  # the host-side target range check of the timed steps' (identical) batch
    import ctypes as C

    ms4 = (C.c_double * 4)()
    cnt4 = (C.c_int64 * 4)()
    L.lk_profile_collect(ms4, cnt4)
    tokens_per_step = bt if vocab_mode else global_bt
    value = tokens_per_step * args.steps / (ms / 1e3)
    flop_step = 6.0 * bt * h * v / (world if vocab_mode else 1)  # per rank
    # ignored-row skipping (single-GPU path, fused_linear_cross_entropy._forward_kept_rows):
    # the GEMMs run on the kept rows only, so the roofline counts the FLOPs actually executed
    n_ignored = int((t == -100).sum().item())
    from paper_2410_10989_b200 import fused_linear_cross_entropy as flce_mod

    skipping = (flce_mod.SKIP_IGNORED_ROWS and n_ignored > 0
                and n_ignored >= max(flce_mod.COMPACT_MIN_SKIPPED, bt // 64))
    flop_exec = 6.0 * (bt - n_ignored) * h * v / (world if vocab_mode else 1) if skipping else flop_step
    # the rows the kept-row call plans its chunks for: all row slots with the device count (the
    # default), the kept rows with the host count
    plan_rows = bt - n_ignored if (skipping and not flce_mod.KEPT_ROWS_DEVICE_COUNT) else bt
    if skipping and not args.chunk_rows and not vocab_mode:
        chunk = flce_plan(plan_rows, h, v)[0]
    if skipping:
        ws_bytes = flce_workspace_bytes(plan_rows, h, v, torch.bfloat16, chunk, True)
        logits_chunk_bytes = chunk * (-(-v // 64) * 64) * 2
    n_chunks = -(-plan_rows // chunk)

    # ---- variant: fp32 dW accumulator (accum_dtype=torch.float32), untimed peak + timed steps ----
    variants = None
    if not args.no_variants:
        pk32 = peak_of(torch.float32)
        vsteps = max(3, args.steps // 4)
        ms32 = timed(vsteps, torch.float32)
        variants = {"accum_fp32": {"value": tokens_per_step * vsteps / (ms32 / 1e3), "unit": "tokens/s",
                                   "steps": vsteps, "ms_per_step": ms32 / vsteps,
                                   "peak_extra_minus_outputs": pk32 - out_bytes,
                                   "note": "accum_dtype=torch.float32: grad_w accumulated across chunks in an "
                                           "fp32 workspace (V*H*4 bytes), one final rounding"}}
        if skipping:
            ms_full = timed(vsteps, skip=False)
            variants["all_rows"] = {"value": tokens_per_step * vsteps / (ms_full / 1e3), "unit": "tokens/s",
                                    "steps": vsteps, "ms_per_step": ms_full / vsteps,
                                    "note": "skip_ignored_rows=False: the GEMMs also run on the ignore_index rows "
                                            "(the upstream Liger / reference schedule)"}
        if world == 1 and args.config == "cfg2" and not vocab_mode and args.bt == BT:
            variants["fp32_cfg2"] = gpu_cfg2_fp32(dev)

    # ---- e2e through the public module, host buffers, H2D/D2H inside the timed region ----
    xh = x.cpu().pin_memory()
    th = t.cpu().pin_memory()
    wp = torch.nn.Parameter(w.clone())
    loss_fn = lk.LigerFusedLinearCrossEntropyLoss(chunk_rows=call_chunk, **opts)

    # Inputs of step i+1 are copied host->device on a side stream while step i computes
    # (double-buffered), as a training input pipeline does; every step still moves its own
    # X and targets from pinned host memory and reads its loss back.
    copy_stream = torch.cuda.Stream(device=dev)
    bufs = [(torch.empty_like(x), torch.empty_like(t)) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    state = {"i": 0, "pending": None}
    # each step's loss goes device->host into pinned memory on the compute stream (inside the
    # timed region) and is read on the host one step later, as a training loop logs its loss,
    # so the read does not stall the launch of the next step
    loss_host = [torch.empty((), dtype=torch.float32).pin_memory() for _ in range(2)]
    loss_ready = [torch.cuda.Event() for _ in range(2)]
    e2e_losses = []

    def read_pending():
        j = state["pending"]
        if j is not None:
            loss_ready[j % 2].synchronize()
            e2e_losses.append(float(loss_host[j % 2]))
            state["pending"] = None

    def stage_copy(i):
        xb, tb = bufs[i % 2]
        with torch.cuda.stream(copy_stream):
            xb.copy_(xh, non_blocking=True)
            tb.copy_(th, non_blocking=True)
            # the input pipeline also enqueues the kept-row compaction of the targets it just
            # landed (lk.prepare_kept_rows), so the step's FLCE call does not wait on the GPU
            lk.prepare_kept_rows(tb, stream=copy_stream)
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
            loss, gx, gw = vocab_parallel_flce(xd.detach(), wp.detach(), td, shard, chunk_rows=chunk, comm=args.comm,
                                               **opts)
        elif world > 1:
            loss, gx, gw = token_sharded_flce(xd, wp, td, chunk_rows=call_chunk, comm=args.comm, **opts)
        else:
            loss = loss_fn(wp, xd, td)
            loss.backward()
        loss_host[i % 2].copy_(loss.detach().float(), non_blocking=True)
        loss_ready[i % 2].record(cur)
        read_pending()  # the previous step's loss (its copy finished long ago)
        state["pending"] = i
        wp.grad = None

    for _ in range(max(1, args.warmup)):
        e2e_step()
    read_pending()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    read_pending()
    assert all(math.isfinite(v) for v in e2e_losses), "non-finite loss in the e2e loop"
    e2e_value = tokens_per_step * args.steps / (max_over_ranks(e0.elapsed_time(e1)) / 1e3)

    peaks, peak_src = measured_peaks()
    gemm_ms = (ms4[0] + ms4[2]) / args.steps
    achieved = flop_exec / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    peak_sus = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    traffic, traffic_step, traffic_src = (None, None, None) if vocab_mode else traffic_for(bt, h, v, args.softcap, skipping)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args.cpu_rows)
        cpu["cfg1"]["gpu_fp32"] = gpu_cfg1_fp32(dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (vocab_mode or strong) else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform X, W, 10% ignore_index targets; "
                                                          "one seed-0 global batch split by rows across ranks)",
            "config": {
                "workload": workload, "ignore_frac": args.ignore_frac, "bt_per_gpu": bt, "hidden": h, "vocab": v, "chunk_rows": chunk,
                "softcap": args.softcap, "label_smoothing": args.label_smoothing,
                "num_chunks": n_chunks, "global_tokens": tokens_per_step,
                "parallelism": (f"vocab-parallel vp{world}" if vocab_mode else
                                (f"token-sharded dp{world}" if world > 1 else "single GPU")),
                "collectives": (None if world == 1 else
                                "per chunk: all_gather of row statistics + async dX all-reduce (bf16)" if vocab_mode
                                else "count all-reduce; dW all-reduce (bf16) overlapped with the last chunk's "
                                     "dW GEMM slices; loss all-reduce"),
                "grad_w_comm": None if world == 1 else
                (("NCCL" if args.comm == "nccl" else "peer-memory kernel (csrc/peer.cu: fp32 rank-order sum over "
                  "IPC-mapped buffers)") + (" per chunk, dX partials" if vocab_mode else " per dW slice")),
                "l2": "inputs larger than L2 (W = 1.05 GB bf16 re-streamed every chunk)",
                "ignore_index_rows": ("skipped: the chunk loop runs on the kept rows (outputs of ignored rows "
                                      "written as the full call leaves them); each step's kept-row compaction "
                                      "is enqueued on a side stream during the previous step "
                                      "(lk.prepare_kept_rows), inside the timed region" if skipping else "computed"),
            },
            "roofline": {
                "bound": "tensor", "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s",
                "frac": (achieved / peak_sus) if achieved else None, "traffic": traffic,
                "kernel": "tc2::gemm2_kernel<bf16> (CTA-pair tcgen05; logits + backward launches)",
                "traffic_unit": "DRAM bytes per GEMM launch (avg over one step's launches, ncu, this config)",
                "traffic_per_step": traffic_step, "traffic_source": traffic_src,
                "algorithmic_flop_per_step": flop_step, "executed_flop_per_step": flop_exec,
                "ignored_rows": n_ignored, "ignored_rows_skipped": skipping,
                "peak_source": f"{peak_src} bf16_tflops_sustained", "peak_burst": float(peaks["bf16_tflops"]),
                "frac_of_burst": (achieved / float(peaks["bf16_tflops"])) if achieved else None,
                "step_tflops": flop_exec / (ms / args.steps / 1e3) / 1e12,
                "stage_ms_per_step": {"logits_gemm": ms4[0] / args.steps, "finalize": ms4[1] / args.steps,
                                      "backward_gemm": ms4[2] / args.steps, "other": ms4[3] / args.steps},
            },
            "peak_mem": {"peak_extra_bytes": peak_extra, "outputs_bytes": out_bytes,
                         "peak_extra_minus_outputs": peak_extra - out_bytes, "workspace_bytes": ws_bytes,
                         "logits_chunk_bytes": logits_chunk_bytes, "dw_fp32_accumulator_bytes": v * h * 4,
                         "full_logits_bytes_avoided": bt * v * 2},
            "variants": variants,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": bt * h * 2 + bt * 8,
                    "d2h_bytes_per_step": 4,
                    "api": ("distributed.vocab_parallel_flce" if vocab_mode else
                            "distributed.token_sharded_flce" if world > 1 else
                            "LigerFusedLinearCrossEntropyLoss + backward()"),
                    "h2d_pipeline": "each step's X/targets copied from pinned host memory on a side stream, "
                                    "double-buffered one step ahead; every step's loss copied device->host "
                                    "(pinned, on the compute stream, inside the timed region) and read on the "
                                    "host one step later; the side stream also enqueues the targets' kept-row "
                                    "compaction (lk.prepare_kept_rows) after their copy; the forward's "
                                    "target-range check reads a count "
                                    "staged to pinned memory before the GEMMs every step, so the host waits "
                                    "for the count kernel only (Liger's n_non_ignore .item() waits for it too)"},
            "gpu_launches": launches * args.steps,
            "gpu_launches_per_step": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1 or vocab_mode:
        dist.destroy_process_group()


def free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv):
    """`--gpus N` outside torchrun: re-run this script under torch.distributed.run with N ranks."""
    share = os.environ.get("LK_BENCH_SHARE_GPU") == "1"
    if not share:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(ROOT / "bench.py"), *argv]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--bt", type=int, default=BT, help="tokens per GPU (cfg2/cfg4) or of the vocab-mode batch")
    ap.add_argument("--hidden", type=int, default=H)
    ap.add_argument("--vocab", type=int, default=V)
    ap.add_argument("--chunk-rows", type=int, default=0)
    ap.add_argument("--config", choices=["cfg2", "cfg4", "cfg5"], default="cfg2",
                    help="cfg2 = Llama-3-8B head, 8192 tokens/GPU (headline, weak scaling); cfg4 = Gemma-2-9B "
                         "head with softcap 30 + smoothing 0.1; cfg5 = 65536 global tokens (strong scaling)")
    ap.add_argument("--softcap", type=float, default=None)
    ap.add_argument("--label-smoothing", type=float, default=0.0)
    ap.add_argument("--ignore-frac", type=float, default=IGNORE_FRAC,
                    help="fraction of targets set to ignore_index (the headline config uses 0.1)")
    ap.add_argument("--mode", choices=["token", "vocab"], default="token",
                    help="multi-GPU shard mode: token-sharded (default) or vocab-parallel (strong)")
    ap.add_argument("--comm", choices=["nccl", "peer"], default="nccl",
                    help="N>1: the dW (token mode) or dX (vocab mode) all-reduce by NCCL or by the peer-memory "
                         "kernel (csrc/peer.cu)")
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--ref-rows", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--cpu-cfg1-worker", action="store_true", help=argparse.SUPPRESS)
    argv = sys.argv[1:]
    args = ap.parse_args(argv)
    if args.cpu_cfg1_worker:
        cpu_cfg1_worker()
        return 0
    if args.config == "cfg4":
        args.hidden, args.vocab = CFG4["hidden"], CFG4["vocab"]
        args.softcap, args.label_smoothing = CFG4["softcap"], CFG4["label_smoothing"]
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args, argv)
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
