"""Chunk planning for the FLCE row loop.

`ChunkPlan` / `plan_chunks` restate the reference rule (rowfuse/flce.py:31-78,
PAPER.md:272): chunk_rows = 2^ceil(log2(ceil(BT / ceil(V / H)))), validated the
same way (power of two, <= next_pow2(BT), consistent chunk count).  The B200
library uses a larger default (`b200_plan`) because
every chunk is one more pass of the dW GEMM over all of grad_w; any plan can be passed
explicitly, which is the reference's sanctioned override (ChunkPlan.with_chunk_rows,
rowfuse/flce.py:58-66; "plan_chunks is advisory").
"""

from __future__ import annotations

from dataclasses import dataclass


def next_pow2(n: int) -> int:
    return 1 if n <= 1 else 1 << (n - 1).bit_length()


@dataclass(frozen=True)
class ChunkPlan:
    chunk_rows: int
    num_chunks: int
    total_rows: int
    scale_ratio: float

    def __post_init__(self) -> None:
        if self.total_rows < 1:
            raise ValueError(f"total_rows must be >= 1, got {self.total_rows}")
        c = self.chunk_rows
        if c < 1 or (c & (c - 1)) != 0:
            raise ValueError(f"chunk_rows must be a power of two >= 1, got {c}")
        if c > next_pow2(self.total_rows):
            raise ValueError(f"chunk_rows {c} exceeds next power of two above {self.total_rows} rows")
        want = -(-self.total_rows // c)
        if self.num_chunks != want:
            raise ValueError(f"num_chunks {self.num_chunks} inconsistent, expected {want}")

    @classmethod
    def with_chunk_rows(cls, total_rows: int, chunk_rows: int) -> "ChunkPlan":
        return cls(chunk_rows=chunk_rows, num_chunks=-(-total_rows // chunk_rows), total_rows=total_rows,
                   scale_ratio=chunk_rows / total_rows)


def plan_chunks(total_rows: int, vocab_size: int, hidden_size: int) -> ChunkPlan:
    """The reference/Liger chunk rule (LK/ops/fused_linear_cross_entropy.py:52-58 is identical)."""
    if total_rows < 1 or vocab_size < 1 or hidden_size < 1:
        raise ValueError(
            f"dimensions must be >= 1, got rows={total_rows}, vocab={vocab_size}, hidden={hidden_size}")
    vocab_per_hidden = -(-vocab_size // hidden_size)
    raw = -(-total_rows // vocab_per_hidden)
    return ChunkPlan.with_chunk_rows(total_rows, next_pow2(raw))


@dataclass(frozen=True)
class B200Plan:
    """The library's chunk plan: chunk_rows need not be a power of two (whole 256-row tiles,
    or the whole batch), num_chunks = ceil(total_rows / chunk_rows)."""

    chunk_rows: int
    num_chunks: int
    total_rows: int

    def __post_init__(self) -> None:
        if self.total_rows < 1 or self.chunk_rows < 1 or self.chunk_rows > self.total_rows:
            raise ValueError(f"bad plan: {self.chunk_rows} rows per chunk for {self.total_rows} rows")
        if self.num_chunks != -(-self.total_rows // self.chunk_rows):
            raise ValueError(f"num_chunks {self.num_chunks} inconsistent with {self.chunk_rows} / {self.total_rows}")


def b200_plan(total_rows: int, vocab_size: int, hidden_size: int, elem_bytes: int = 2) -> B200Plan:
    """Host restatement of the library's default (flce.cu b200_chunk_rows): the fewest chunks
    of at most 3072 rows (4096 when BT > 16384) and a 1.5 GiB logits buffer (1 GiB for fp32),
    split evenly in 256-row tiles; never below the reference's rule (capped by the buffer)."""
    ref = plan_chunks(total_rows, vocab_size, hidden_size).chunk_rows
    ldz = -(-vocab_size // 64) * 64
    cap_bytes = (1 << 30) if elem_bytes == 4 else (3 << 29)  # 1.5 GiB (1 GiB for fp32 logits)
    cap_rows = max(256, cap_bytes // (ldz * elem_bytes) // 256 * 256)
    c_max = min(4096 if total_rows > 2048 * 8 else 3072, cap_rows)
    if total_rows <= c_max:
        c = total_rows
    else:
        nch = -(-total_rows // c_max)
        tiles = -(-total_rows // 256)
        c = -(-tiles // nch) * 256
    c = max(c, min(ref, cap_rows))
    c = max(1, min(c, max(total_rows, 1)))
    return B200Plan(chunk_rows=c, num_chunks=-(-total_rows // c), total_rows=total_rows)
