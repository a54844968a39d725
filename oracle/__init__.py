"""CPU oracle for the Liger hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package, and only as the checker or the timed CPU baseline.
The product path (paper_2410_10989_b200) never imports it and has no CPU fallback.

Modules
  rowfuse_port : numpy restatement of the reference package `rowfuse` 0.1.0
                 (/root/reference/pkg/src/rowfuse): chunked FLCE, in-place streaming
                 cross entropy, RMSNorm, RoPE, SwiGLU/GeGLU, chunk planning.  Each
                 function cites the reference file:line it follows.  Pinned against
                 golden vectors produced by the reference itself
                 (tests/golden/make_golden.py -> tests/golden/rowfuse_golden.npz).
  liger_ref    : float64 restatement of the semantics the reference does not have
                 (ignore_index, label_smoothing, softcap, z-loss, reduction='none',
                 the Liger (V, H) weight layout, cos/sin RoPE tables, RMSNorm casting
                 modes).  Parity for these is pinned against torch-CPU float64
                 F.cross_entropy in tests/test_oracle.py — the reference has no
                 code for them (SURVEY §8(c) "parity unpinned" rows).
"""
