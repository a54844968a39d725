"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/liger_b200.h declares, validates arguments into the reference's error
taxonomy, and the Python surface matches liger_kernel's signatures."""

import ctypes as C
import inspect
import re
from pathlib import Path

import pytest
import torch

import paper_2410_10989_b200 as lk
from paper_2410_10989_b200.chunking import b200_plan
from paper_2410_10989_b200 import _capi, errors

HEADER = Path(__file__).resolve().parents[1] / "include" / "liger_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.SIGNATURES), "ctypes binding out of sync with the header"
    assert lib.lk_has_tcgen05() == 1
    assert b"sm_100a" in lib.lk_version()


def test_flce_args_struct_matches_header_field_order():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    body = re.search(r"typedef struct \{(.*?)\} lk_flce_args;", text, flags=re.S).group(1)
    names = []
    for stmt in body.split(";"):
        stmt = stmt.strip()
        if stmt:
            names += re.findall(r"(\w+)\s*(?:,|$)", stmt)
    assert names == [f[0] for f in _capi.FlceArgs._fields_]


def test_plan_and_workspace_queries():
    lib = _capi.load()
    c, n = C.c_int64(), C.c_int64()
    assert lib.lk_flce_plan(8192, 4096, 128256, 1, C.byref(c), C.byref(n)) == 0
    assert (c.value, n.value) == (2816, 3)
    assert lib.lk_flce_plan(1024, 512, 4096, 0, C.byref(c), C.byref(n)) == 0
    assert (c.value, n.value) == (1024, 1)
    assert lib.lk_flce_plan(0, 4096, 128256, 1, C.byref(c), C.byref(n)) == 3  # SIZE_MISMATCH
    chunk = 2816 * 128256 * 2
    dw_acc = 128256 * 4096 * 4
    # default (LK_ACCUM_AUTO, 3 chunks): grad_w accumulates in bf16 -> workspace ~ one logits chunk
    ws = lib.lk_flce_workspace_bytes(8192, 4096, 128256, 1, 0, 1)
    assert chunk < ws < chunk + 64 * 2**20
    assert lib.lk_flce_workspace_bytes_ex(8192, 4096, 128256, 1, 0, 1, _capi.LK_ACCUM_AUTO) == ws
    assert lib.lk_flce_workspace_bytes_ex(8192, 4096, 128256, 1, 0, 1, _capi.LK_ACCUM_WEIGHT_DTYPE) == ws
    ws32 = lib.lk_flce_workspace_bytes_ex(8192, 4096, 128256, 1, 0, 1, _capi.LK_ACCUM_FP32)
    assert chunk + dw_acc < ws32 < chunk + dw_acc + 64 * 2**20
    # more than 8 chunks: auto falls back to the fp32 accumulator
    assert lib.lk_flce_workspace_bytes(8192, 4096, 128256, 1, 512, 1) > dw_acc
    assert lk.flce_plan(8192, 4096, 128256) == (2816, 3)
    # the legacy size queries cover the exact-call query for the default options, fp32 included
    # (fp32 runs on split operands with 3 pieces by default: 6 terms along K)
    for dt, (bt, h, v) in ((0, (1024, 512, 4096)), (0, (300, 264, 5003)), (1, (8192, 4096, 128256))):
        a = _capi.FlceArgs(bt=bt, hidden=h, vocab=v, dtype=dt, grad_x=1, grad_w=1)
        exact = lib.lk_flce_workspace_bytes_for(C.byref(a))
        assert lib.lk_flce_workspace_bytes(bt, h, v, dt, 0, 1) >= exact
        assert lib.lk_flce_workspace_bytes_ex(bt, h, v, dt, 0, 1, _capi.LK_ACCUM_AUTO) >= exact
    for bt in (1, 3000, 7373, 8192, 16384, 65536, 32768 + 5):  # the host restatement agrees with the library
        for h, v in ((4096, 128256), (3584, 256000), (512, 4096)):
            p = b200_plan(bt, v, h)
            assert lk.flce_plan(bt, h, v) == (p.chunk_rows, p.num_chunks), (bt, h, v)


def test_status_codes_map_to_reference_exceptions():
    lib = _capi.load()
    rc = lib.lk_rope(None, None, None, None, 1, 4, 2, 2, 7, 1, 1, 1, 0, None)
    assert rc == 4
    with pytest.raises(errors.OddHeadDim):
        _capi.check(rc)
    assert "even" in lib.lk_last_error().decode()
    rc = lib.lk_rope(None, None, None, None, 2, 4, 2, 2, 8, 3, 1, 1, 0, None)
    with pytest.raises(errors.ShapeMismatch):
        _capi.check(rc)
    rc = lib.lk_cross_entropy_fwd(None, 2, None, 4, 8, 1, -100, 0.0, 0.0, 0.0, 1, 1, None, None, None, None,
                                  None, 0, None)
    with pytest.raises(errors.NonContiguousInput):
        _capi.check(rc)
    rc = lib.lk_swiglu_fwd(None, None, None, -1, 1, None)
    with pytest.raises(errors.SizeMismatch):
        _capi.check(rc)
    assert issubclass(errors.TargetOutOfRange, IndexError)
    assert issubclass(errors.ShapeMismatch, ValueError)


def test_no_cpu_fallback():
    x = torch.randn(4, 8)
    t = torch.zeros(4, dtype=torch.long)
    with pytest.raises(errors.ExtensionMissing):
        lk.LigerCrossEntropyLoss()(x, t)
    with pytest.raises(errors.ExtensionMissing):
        lk.LigerFusedLinearCrossEntropyLoss()(torch.randn(16, 8), x, t)
    with pytest.raises(errors.ExtensionMissing):
        lk.LigerRMSNorm(8)(x)
    with pytest.raises(errors.ExtensionMissing):
        lk.liger_swiglu(x, x)
    with pytest.raises(errors.ExtensionMissing):
        lk.LigerLayerNorm(8)(x)


def _params(obj):
    sig = inspect.signature(obj)
    return [(p.name, p.default) for p in sig.parameters.values() if p.name not in ("self", "ctx")]


@pytest.mark.parametrize(
    "ours,theirs",
    [
        ("LigerCrossEntropyLoss.__init__", "liger_kernel.transformers.cross_entropy.LigerCrossEntropyLoss.__init__"),
        ("LigerCrossEntropyLoss.forward", "liger_kernel.transformers.cross_entropy.LigerCrossEntropyLoss.forward"),
        ("LigerFusedLinearCrossEntropyLoss.forward",
         "liger_kernel.transformers.fused_linear_cross_entropy.LigerFusedLinearCrossEntropyLoss.forward"),
        ("LigerRMSNorm.__init__", "liger_kernel.transformers.rms_norm.LigerRMSNorm.__init__"),
        ("LigerRMSNorm.forward", "liger_kernel.transformers.rms_norm.LigerRMSNorm.forward"),
        ("liger_rotary_pos_emb", "liger_kernel.transformers.rope.liger_rotary_pos_emb"),
        ("LigerSwiGLUMLP.__init__", "liger_kernel.transformers.swiglu.LigerSwiGLUMLP.__init__"),
        ("LigerGEGLUMLP.__init__", "liger_kernel.transformers.geglu.LigerGEGLUMLP.__init__"),
        ("LigerCrossEntropyFunction.forward", "liger_kernel.ops.cross_entropy.LigerCrossEntropyFunction.forward"),
        ("LigerLayerNorm.__init__", "liger_kernel.transformers.layer_norm.LigerLayerNorm.__init__"),
        ("LigerLayerNorm.forward", "liger_kernel.transformers.layer_norm.LigerLayerNorm.forward"),
        ("LigerLayerNormFunction.forward", "liger_kernel.ops.layer_norm.LigerLayerNormFunction.forward"),
        ("liger_layer_norm", "liger_kernel.transformers.functional.liger_layer_norm"),
    ],
)
def test_signatures_match_liger(ours, theirs):
    lk_mod = pytest.importorskip("liger_kernel.transformers")  # noqa: F841  (third-party, signature source only)
    import importlib

    def resolve(path, root=None):
        parts = path.split(".")
        if root is None:
            for i in range(len(parts), 0, -1):
                try:
                    obj = importlib.import_module(".".join(parts[:i]))
                    break
                except Exception:
                    continue
            rest = parts[i:]
        else:
            obj, rest = root, parts
        for p in rest:
            obj = getattr(obj, p)
        return obj

    a = _params(resolve(ours, lk))
    b = _params(resolve(theirs))
    assert a == b


def test_flce_module_signature_is_liger_plus_chunk_override():
    pytest.importorskip("liger_kernel.transformers")
    from liger_kernel.transformers.fused_linear_cross_entropy import LigerFusedLinearCrossEntropyLoss as Ref

    ours = _params(lk.LigerFusedLinearCrossEntropyLoss.__init__)
    assert ours[:-1] == _params(Ref.__init__)
    assert ours[-1] == ("chunk_rows", None)


def test_benchrecord_schema_round_trip(tmp_path):
    """GPU bench results use rowfuse's BenchRecord CSV schema (rowfuse/bench.py:84-159), so
    `rowfuse report` can merge them with CPU runs."""
    from paper_2410_10989_b200 import benchrecord as br

    assert br.FIELDS == ("op", "variant", "rows", "cols", "hidden", "dtype", "repeats", "workers", "median_s",
                         "q20_s", "q80_s", "peak_bytes")
    recs = [br.BenchRecord("linear_ce", "fused", 128, 40960, 256, "bf16", 10, 0, 1.25e-4, 1.2e-4, 1.3e-4, 12345)]
    p = tmp_path / "r.csv"
    br.write_records(p, recs)
    assert br.read_records(p) == recs
    assert p.read_text().splitlines()[0] == ",".join(br.FIELDS)
    bad = tmp_path / "bad.csv"
    bad.write_text("op,variant\nx,y\n")
    with pytest.raises(br.SchemaMismatch):
        br.read_records(bad)
    assert br.default_shapes("rmsnorm")[0] == (256, 4096, 0)
    assert br.default_shapes("linear_ce")[-1] == (128, 163840, 256)


def test_benchrecord_csv_reads_with_the_reference_reader(tmp_path):
    """Where the reference tree exists (the build container), its own reader accepts our CSV."""
    import os
    import sys

    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference tree not present (GPU box)")
    from paper_2410_10989_b200 import benchrecord as br

    p = tmp_path / "r.csv"
    br.write_records(p, [br.BenchRecord("rmsnorm", "fused", 256, 4096, 0, "bf16", 10, 0, 2e-5, 1.9e-5, 2.2e-5, 4096)])
    sys.path.insert(0, src)
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.dont_write_bytecode = True
    try:
        from rowfuse.bench import read_records, summarize
    finally:
        sys.path.remove(src)
    recs = read_records(p)
    assert recs[0].op == "rmsnorm" and recs[0].median_s == 2e-5
    assert summarize(recs)[0]["fused_median_s"] == 2e-5


def test_peer_allreduce_validates_before_touching_the_device():
    """lk_peer_allreduce rejects bad arguments with LK_INVALID_ARGUMENT before any CUDA call
    (so this runs without a GPU), and the constants agree with the Python mirror."""
    from paper_2410_10989_b200 import peer

    text = HEADER.read_text()
    for name, val in (("LK_PEER_MAX", peer.MAX_PEERS), ("LK_PEER_CTL_BYTES", peer.CTL_BYTES),
                      ("LK_PEER_HANDLE_BYTES", peer.HANDLE_BYTES)):
        assert re.search(rf"#define {name} {val}\b", text), name
    lib = _capi.load()
    bases = (C.c_void_p * 2)(4096 * 16, 4096 * 32)
    ok = dict(bases=bases, world=2, rank=0, offset=4096, n=100, dtype=_capi.LK_BF16, epoch=1, timeout=0)

    def call(**over):
        a = dict(ok, **over)
        return lib.lk_peer_allreduce(a["bases"], a["world"], a["rank"], a["offset"], a["n"], a["dtype"], a["epoch"],
                                     a["timeout"], None)

    for bad in (dict(world=0), dict(world=peer.MAX_PEERS + 1), dict(rank=2), dict(rank=-1), dict(dtype=7),
                dict(n=-1), dict(epoch=0), dict(offset=100), dict(offset=4097),
                dict(bases=(C.c_void_p * 2)(4096, None))):
        assert call(**bad) == 8, bad  # LK_INVALID_ARGUMENT
    assert lib.lk_peer_alloc(0, 16, None, None) == 8
    assert lib.lk_peer_status(0, None, 0, None) == 8


def test_token_sharded_rejects_unknown_comm():
    from paper_2410_10989_b200.distributed import token_sharded_flce

    with pytest.raises(ValueError, match="comm must be"):
        token_sharded_flce(torch.zeros(2, 8), torch.zeros(4, 8), torch.zeros(2, dtype=torch.int64), comm="mpi")


def test_compaction_entry_points_validate_arguments():
    lib = _capi.load()
    assert lib.lk_compact_rows(None, -1, -100, None, None, None, None) == 8
    assert lib.lk_compact_rows(None, 10, -100, None, None, None, None) == 8
    assert lib.lk_gather_rows(None, 4, 3, None, 4, None, 0, None) == 8  # element width 3
    assert lib.lk_gather_rows(None, -1, 2, None, 4, None, 0, None) == 8
    assert lib.lk_gather_rows(None, 0, 2, None, 4, None, 0, None) == 0  # nothing to copy
    assert lib.lk_gather_rows(None, 4, 2, None, 4, None, 0, None) == 8
