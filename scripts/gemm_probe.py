"""Diagnose the tcgen05 GEMM on one tile: prints how the result relates to the expected
product (exact, transposed operand, row/column permutation, zero) for each layout.
Usage (GPU box): python scripts/gemm_probe.py"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_10989_b200 import _capi  # noqa: E402


def run(a, b, m, n, k, layout, tc=True):
    d = torch.full((m, n), float("nan"), device="cuda")
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    rc = _capi.load().lk_gemm_test(a.data_ptr(), b.data_ptr(), d.data_ptr(), m, n, k, layout, 1, int(tc),
                                   ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    if rc:
        print("rc", rc, _capi.load().lk_last_error())
    return d


def main():
    torch.manual_seed(0)
    for (m, n, k) in [(128, 256, 64), (128, 256, 16), (128, 256, 128), (256, 512, 256)]:
        A = torch.randint(-2, 3, (m, k), device="cuda").to(torch.bfloat16)
        B = torch.randint(-2, 3, (k, n), device="cuda").to(torch.bfloat16)
        ref = A.float() @ B.float()
        for layout, cg in [(l, c) for c in (1, 2) for l in (0, 1, 2)]:
            if layout == 0:
                a, b = A.contiguous(), B.t().contiguous()
            elif layout == 1:
                a, b = A.contiguous(), B.contiguous()
            else:
                a, b = A.t().contiguous(), B.contiguous()
            d = run(a, b, m, n, k, layout, tc=cg)
            eq = (d == ref)
            info = f"m{m} n{n} k{k} layout{layout} cg{cg}: exact={bool(eq.all())} frac={eq.float().mean().item():.4f}"
            if not eq.all():
                nan = torch.isnan(d).float().mean().item()
                zero = (d == 0).float().mean().item()
                rows_ok = eq.all(dim=1).float().mean().item()
                cols_ok = eq.all(dim=0).float().mean().item()
                info += f" nan={nan:.3f} zero={zero:.3f} rows_ok={rows_ok:.3f} cols_ok={cols_ok:.3f}"
                bad = torch.nonzero(~eq)[:3].tolist()
                info += f" first_bad={bad}"
                for (r, c) in bad[:2]:
                    info += f" d[{r},{c}]={d[r, c].item()} ref={ref[r, c].item()}"
                # does each output row appear somewhere in ref (row permutation)?
                if m <= 256:
                    match_rows = 0
                    for r in range(min(m, 64)):
                        match_rows += int(((ref == d[r]).all(dim=1)).any().item())
                    info += f" rows_found_in_ref={match_rows}/64"
            print(info, flush=True)
        simt = run(A.contiguous(), B.t().contiguous(), m, n, k, 0, tc=False)
        print(f"  simt exact={bool((simt == ref).all())}", flush=True)


if __name__ == "__main__":
    main()
