"""Paper-shaped synthetic workloads: C2 (547 kernels / 18,217
instances / 6 apps), C3 (TVM-style GEMM/conv, 1M), C4 (cuDNN-like, 16+ pointer
args) and the replication used for C5 and the bench.

Inputs only: kernel summaries are built from templates of common GPU kernels
(what the paper's analyzer would emit for them), launch records from per-app
"programs" that reuse buffers the way applications do.  Nothing here computes a
range, an overlap or a verdict.  Per-app kernel counts, kernel-level classes and
NI reasons are the paper's (Table 3 l.1235-1277, Table 4 l.1304-1318);
the instance counts per app are Table 3's; everything else (templates, sizes,
aliasing rates) is this generator's choice, stated in DESIGN.md §8.
"""
from __future__ import annotations

import numpy as np

from .golden import bx, desc, kernel, term
from .records import REC_DTYPE, RecordBuilder

PTR_HI = (1 << 56) - 1
I32_HI = (1 << 31) - 1

# (name, kernels, instances, (IDEM, NONIDEM, COND), NONIDEM reasons (IF, PE, NA, SO))
APPS = [
    ("Rodinia", 40, 4527, (4, 23, 13), (7, 2, 3, 11)),
    ("Parboil", 25, 1033, (1, 15, 9), (1, 1, 3, 10)),
    ("TVM", 308, 609, (0, 0, 308), (0, 0, 0, 0)),
    ("PyTorch", 66, 1570, (3, 22, 41), (0, 16, 5, 1)),
    ("TensorRT", 58, 478, (0, 17, 41), (0, 12, 4, 1)),
    ("FT", 50, 10000, (8, 19, 23), (0, 12, 4, 3)),
]

# Generator knobs per app: probability that a COND instance runs in place (a
# write pointer equal to a read pointer), share of launches
# that go to NONIDEM kernels, and probability that a guarded non-parameter
# (opaque) access is switched on.  Calibrated with scripts/c2_mix.py
# (oracle only) so that the instance-level I/NI mix lands near Table 3.
KNOBS = {
    "Rodinia": dict(p_alias=0.02, ni_share=0.05, p_opaque_on=0.1),
    "Parboil": dict(p_alias=0.7, ni_share=0.35, p_opaque_on=0.6),
    "TVM": dict(p_alias=0.0, ni_share=0.0, p_opaque_on=0.0),
    "PyTorch": dict(p_alias=0.25, ni_share=0.35, p_opaque_on=0.5),
    "TensorRT": dict(p_alias=0.05, ni_share=0.45, p_opaque_on=0.3),
    "FT": dict(p_alias=0.06, ni_share=0.22, p_opaque_on=0.15),
}


def ptr_pre(names):
    return [{"op": n, "lo": 0, "hi": PTR_HI} for n in names]


def rng_pick(rng, xs):
    return xs[int(rng.integers(0, len(xs)))]


class Alloc:
    """Bump allocator of 256-byte aligned device VAs in [2^32, 2^44)."""

    def __init__(self, rng):
        self.rng = rng
        self.next = (1 << 32) + int(rng.integers(0, 1 << 20)) * 256

    def buf(self, nbytes):
        p = self.next
        self.next += ((int(nbytes) + 255) // 256) * 256 + 256 * int(self.rng.integers(1, 64))
        assert self.next < (1 << 44)
        return p


# ---------------------------------------------------------------------------
# Kernel templates.  Each returns (summary-without-id, sampler); the sampler
# draws one launch (args, grid, block) given the program state.
# ---------------------------------------------------------------------------

def t_elementwise(rng, *, nin=None, width=None, grid_stride=None):
    nin = nin or int(rng.integers(1, 4))
    w = width or rng_pick(rng, [2, 4, 4, 4, 8])
    gs = grid_stride if grid_stride is not None else rng.random() < 0.3
    params = [("out", "ptr")] + [(f"in{i}", "ptr") for i in range(nin)] + [("N", "i32")]
    if gs:  # for (i = gidx; i < N; i += gdim*bdim): i in [0, N-1] (induction)
        v = {"ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["N"]))]}}
        t = [term(w, (), "ind0")]
    else:   # if (gidx < N): gidx in [0, min(N-1, gdim*bdim-1)] (tightening, l.1023-1026)
        v = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
        t = [term(w, (), "gidx.x")]
    ds = [desc("W", w, "out", t, v)] + [desc("R", w, f"in{i}", t, v) for i in range(nin)]
    pre = ptr_pre([p for p, k in params if k == "ptr"]) + [{"op": "N", "lo": 0, "hi": I32_HI}]
    bdim = rng_pick(rng, [128, 256, 512, 1024])

    def sample(rng, st):
        N = st.size(rng)
        g = min(max(1, (N + bdim - 1) // bdim), 65535 * 4) if not gs else rng_pick(rng, [148, 296, 592, 1184])
        ptrs = st.bufs(["out"] + [f"in{i}" for i in range(nin)], N * w)
        if nin and st.alias(rng):
            ptrs[0] = ptrs[1 + int(rng.integers(0, nin))]
        return ptrs + [N], (g, 1, 1), (bdim, 1, 1)

    return ("elementwise", params, ds, pre, []), sample


def t_bias_act(rng):
    w = 4
    params = [("out", "ptr"), ("in", "ptr"), ("bias", "ptr"), ("N", "i32"), ("C", "i32")]
    v = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
    vb = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]},
          "fr0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["C"]))]}}  # gidx % C -> fresh in [0, C-1]
    ds = [desc("W", w, "out", [term(w, (), "gidx.x")], v),
          desc("R", w, "in", [term(w, (), "gidx.x")], v),
          desc("R", w, "bias", [term(w, (), "fr0")], vb)]
    pre = ptr_pre(["out", "in", "bias"]) + [{"op": "N", "lo": 0, "hi": I32_HI},
                                            {"op": "C", "lo": 1, "hi": 1 << 20}]
    bdim = rng_pick(rng, [256, 512, 1024])

    def sample(rng, st):
        C = st.hidden
        N = C * st.rows(rng)
        ptrs = st.bufs(["out", "in", "bias"], N * w, small={"bias": C * w})
        if st.alias(rng):
            ptrs[0] = ptrs[1]
        return ptrs + [N, C], ((N + bdim - 1) // bdim, 1, 1), (bdim, 1, 1)

    return ("add_bias_act", params, ds, pre, []), sample


def t_rowop(rng, *, kind=None):
    """softmax / layernorm / row reduction: one block per row of M columns."""
    kind = kind or rng_pick(rng, ["softmax", "layernorm", "reduce"])
    w = rng_pick(rng, [2, 4])
    params = [("out", "ptr"), ("in", "ptr")]
    if kind == "layernorm":
        params += [("gamma", "ptr"), ("beta", "ptr")]
    params += [("M", "i32")]
    v = {"bid.x": {"lo": [], "hi": []}, "ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["M"]))]}}
    row = [term(w, ("M",), "bid.x"), term(w, (), "ind0")]
    ds = [desc("R", w, "in", row, v)]
    if kind == "reduce":
        ds.append(desc("W", w, "out", [term(w, (), "bid.x")], {"bid.x": {"lo": [], "hi": []}}))
    else:
        ds.append(desc("W", w, "out", row, v))
    if kind == "layernorm":
        vi = {"ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["M"]))]}}
        ds += [desc("R", w, "gamma", [term(w, (), "ind0")], vi),
               desc("R", w, "beta", [term(w, (), "ind0")], vi)]
    pre = ptr_pre([p for p, k in params if k == "ptr"]) + [{"op": "M", "lo": 1, "hi": 1 << 16}]
    bdim = rng_pick(rng, [128, 256, 1024])
    # each thread keeps its M / bdim columns in registers: the loop is unrolled
    # at most 32 times, so the summary holds only while M <= 32 bdim (the
    # global condition of an unbounded loop)
    glob = [{"op": "M", "lo": 1, "hi": 32 * bdim}]

    def sample(rng, st):
        M = st.hidden
        R = st.rows(rng)
        names = [p for p, k in params if k == "ptr"]
        ptrs = st.bufs(names, R * M * w, small={"gamma": M * w, "beta": M * w, "out": R * M * w})
        if st.alias(rng) and kind != "reduce":
            ptrs[0] = ptrs[1]  # in-place normalisation
        return ptrs + [M], (R, 1, 1), (bdim, 1, 1)

    return (kind, params, ds, pre, glob), sample


def t_stencil2d(rng):
    w = 4
    r = int(rng.integers(1, 3))
    params = [("out", "ptr"), ("in", "ptr"), ("W", "i32"), ("H", "i32")]
    v2 = {"bid.x": {"lo": [], "hi": []}, "bid.y": {"lo": [], "hi": []},
          "tid.x": {"lo": [], "hi": []}, "tid.y": {"lo": [], "hi": []}}
    vr = dict(v2)
    vr["ind0"] = {"lo": [bx(-r)], "hi": [bx(r)]}
    vr["ind1"] = {"lo": [bx(-r)], "hi": [bx(r)]}
    cell = [term(16 * w, ("W",), "bid.y"), term(w, ("W",), "tid.y"), term(16 * w, (), "bid.x"),
            term(w, (), "tid.x")]
    ds = [desc("R", w, "in", cell + [term(w, ("W",), "ind0"), term(w, (), "ind1")], vr),
          desc("W", w, "out", cell, v2)]
    pre = ptr_pre(["out", "in"]) + [{"op": "W", "lo": 1, "hi": 1 << 15}, {"op": "H", "lo": 1, "hi": 1 << 15},
                                    {"op": "gdim.x", "lo": 1, "hi": 1 << 12}, {"op": "gdim.y", "lo": 1, "hi": 1 << 12}]

    def sample(rng, st):
        Wd = rng_pick(rng, [256, 512, 1024, 2048])
        Hd = rng_pick(rng, [256, 512, 1024, 2048])
        pad = (r * Wd + r) * w
        ptrs = st.bufs(["out", "in"], Wd * Hd * w + 2 * pad, offset={"in": pad})
        if st.alias(rng):
            ptrs[0] = ptrs[1]
        return ptrs + [Wd, Hd], ((Wd + 15) // 16, (Hd + 15) // 16, 1), (16, 16, 1)

    return ("stencil2d", params, ds, pre, []), sample


def t_interleave(rng):
    """Red-black / even-odd update (PAPER l.1174-1177 pattern): reads odd, writes even."""
    w = rng_pick(rng, [4, 8])
    params = [("A", "ptr"), ("N", "i32")]
    v = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
    ds = [desc("R", w, "A", [term(2 * w, (), "gidx.x"), term(w)], v),
          desc("W", w, "A", [term(2 * w, (), "gidx.x")], v)]
    pre = ptr_pre(["A"]) + [{"op": "N", "lo": 0, "hi": 1 << 28}]

    def sample(rng, st):
        N = st.size(rng) // 2 + 1
        return st.bufs(["A"], 2 * N * w) + [N], ((N + 255) // 256, 1, 1), (256, 1, 1)

    return ("redblack", params, ds, pre, []), sample


def t_gather(rng):
    """Embedding lookup / indirect gather: the table address depends on memory
    contents (non-parameter address), guarded by a flag."""
    w = 4
    params = [("out", "ptr"), ("table", "ptr"), ("ids", "ptr"), ("N", "i32"), ("H", "i32"),
              ("use_table", "i32")]
    v = {"bid.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}, "ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["H"]))]}}
    ds = [desc("R", 4, "ids", [term(4, (), "bid.x")], {"bid.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}),
          desc("R", w, "table", [], v, guard=[{"a": "use_table", "cmp": "!=", "b": 0}], opaque=True),
          desc("W", w, "out", [term(w, ("H",), "bid.x"), term(w, (), "ind0")], v)]
    pre = ptr_pre(["out", "table", "ids"]) + [{"op": "N", "lo": 0, "hi": I32_HI},
                                              {"op": "H", "lo": 1, "hi": 1 << 16},
                                              {"op": "use_table", "lo": -I32_HI - 1, "hi": I32_HI}]

    def sample(rng, st):
        H = st.hidden
        N = st.rows(rng)
        ptrs = st.bufs(["out", "table", "ids"], N * H * w, small={"ids": N * 4})
        on = 1 if rng.random() < st.knobs["p_opaque_on"] else 0
        return ptrs + [N, H, on], (N, 1, 1), (rng_pick(rng, [128, 256]), 1, 1)

    return ("gather", params, ds, pre, []), sample


def t_transpose(rng):
    w = rng_pick(rng, [2, 4])
    params = [("out", "ptr"), ("in", "ptr"), ("W", "i32"), ("H", "i32")]
    v2 = {"bid.x": {"lo": [], "hi": []}, "bid.y": {"lo": [], "hi": []},
          "tid.x": {"lo": [], "hi": []}, "tid.y": {"lo": [], "hi": []}}
    ds = [desc("R", w, "in", [term(32 * w, ("W",), "bid.y"), term(w, ("W",), "tid.y"),
                              term(32 * w, (), "bid.x"), term(w, (), "tid.x")], v2),
          desc("W", w, "out", [term(32 * w, ("H",), "bid.x"), term(w, ("H",), "tid.x"),
                               term(32 * w, (), "bid.y"), term(w, (), "tid.y")], v2)]
    pre = ptr_pre(["out", "in"]) + [{"op": "W", "lo": 1, "hi": 1 << 16}, {"op": "H", "lo": 1, "hi": 1 << 16},
                                    {"op": "gdim.x", "lo": 1, "hi": 1 << 11}, {"op": "gdim.y", "lo": 1, "hi": 1 << 11}]

    def sample(rng, st):
        Wd = rng_pick(rng, [64, 128, 256, 512, 768, 1024])
        Hd = rng_pick(rng, [64, 128, 256, 512, 1024])
        ptrs = st.bufs(["out", "in"], Wd * Hd * w)
        return ptrs + [Wd, Hd], ((Wd + 31) // 32, (Hd + 31) // 32, 1), (32, 32, 1)

    return ("transpose", params, ds, pre, []), sample


def t_attention(rng):
    """Decoder self-attention over a KV cache: reads steps [0, step-1] (or
    [0, step]), appends at `step` (FT masked multi-head attention)."""
    w = 2
    incl = rng.random() < 0.5
    params = [("out", "ptr"), ("q", "ptr"), ("kc", "ptr"), ("vc", "ptr"), ("step", "i32"),
              ("maxlen", "i32"), ("D", "i32")]
    hi_s = bx(0, (1, ["step"])) if incl else bx(-1, (1, ["step"]))
    v = {"bid.x": {"lo": [], "hi": []}, "tid.x": {"lo": [], "hi": []}, "ind0": {"lo": [bx(0)], "hi": [hi_s]}}
    vt = {"bid.x": {"lo": [], "hi": []}, "tid.x": {"lo": [], "hi": []}}
    cache = [term(w, ("maxlen", "D"), "bid.x"), term(w, ("D",), "ind0"), term(w, (), "tid.x")]
    app = [term(w, ("maxlen", "D"), "bid.x"), term(w, ("D", "step")), term(w, (), "tid.x")]
    vec = [term(w, ("D",), "bid.x"), term(w, (), "tid.x")]
    ds = [desc("R", w, "q", vec, vt), desc("R", w, "kc", cache, v), desc("R", w, "vc", cache, v),
          desc("W", w, "kc", app, vt), desc("W", w, "vc", app, vt), desc("W", w, "out", vec, vt)]
    pre = ptr_pre(["out", "q", "kc", "vc"]) + [{"op": "step", "lo": 0, "hi": 1 << 16},
                                               {"op": "maxlen", "lo": 1, "hi": 1 << 16},
                                               {"op": "D", "lo": 1, "hi": 1024}]
    glob = [{"op": "step", "lo": 0, "hi": 4095}]

    def sample(rng, st):
        D = 64
        heads = st.hidden // D
        maxlen = 1024
        step = int(st.step)
        ptrs = st.bufs(["out", "q", "kc", "vc"], heads * D * w,
                       small={"kc": heads * maxlen * D * w, "vc": heads * maxlen * D * w})
        return ptrs + [step, maxlen, D], (heads, 1, 1), (D, 1, 1)

    return ("masked_mha", params, ds, pre, glob), sample


def t_scan(rng):
    w = 4
    params = [("out", "ptr"), ("in", "ptr"), ("sums", "ptr"), ("N", "i32")]
    v = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
    ds = [desc("R", w, "in", [term(w, (), "gidx.x")], v),
          desc("W", w, "out", [term(w, (), "gidx.x")], v),
          desc("W", w, "sums", [term(w, (), "bid.x")], {"bid.x": {"lo": [], "hi": []}},
               guard=[{"a": "gdim.x", "cmp": ">", "b": 1}])]
    pre = ptr_pre(["out", "in", "sums"]) + [{"op": "N", "lo": 0, "hi": I32_HI}]

    def sample(rng, st):
        N = st.size(rng)
        g = (N + 1023) // 1024
        ptrs = st.bufs(["out", "in", "sums"], N * w, small={"sums": g * w})
        if st.alias(rng):
            ptrs[0] = ptrs[1]
        return ptrs + [N], (g, 1, 1), (1024, 1, 1)

    return ("scan", params, ds, pre, []), sample


def t_gemm_tvm(rng, *, concat=False, small=False):
    """TVM-generated tiled GEMM / implicit-GEMM conv: constant shapes, only
    pointer arguments, fixed launch (TVM kernels are
    induction-variable loops over loop-invariant expressions).  ``small``: shapes
    the exact (enumerating) verifier finishes on (row f2's Base)."""
    es = rng_pick(rng, [2, 4])
    if small:
        M = int(rng_pick(rng, [16, 32, 49, 64]))
        N = int(rng_pick(rng, [16, 32, 64]))
        K = int(rng_pick(rng, [16, 32, 64]))
    else:
        M = int(rng_pick(rng, [64, 128, 256, 512, 1024, 3136, 784, 196, 49]))
        N = int(rng_pick(rng, [64, 128, 256, 512, 1024, 2048]))
        K = int(rng_pick(rng, [64, 128, 256, 576, 1152, 2304]))
    TM, TN = rng_pick(rng, [(32, 32), (64, 64), (16, 64), (64, 16), (8, 8)])
    M = ((M + TM - 1) // TM) * TM
    N = ((N + TN - 1) // TN) * TN
    TY, TX = (min(8, TM), min(8, TN))
    RM, RN = TM // TY, TN // TX
    bias = rng.random() < 0.5
    params = [("A", "ptr"), ("B", "ptr"), ("C", "ptr")] + ([("bias", "ptr")] if bias else [])
    vA = {"bid.y": {"lo": [], "hi": []}, "tid.y": {"lo": [], "hi": []},
          "ind1": {"lo": [bx(0)], "hi": [bx(RM - 1)]}, "ind0": {"lo": [bx(0)], "hi": [bx(K - 1)]}}
    vB = {"bid.x": {"lo": [], "hi": []}, "tid.x": {"lo": [], "hi": []},
          "ind2": {"lo": [bx(0)], "hi": [bx(RN - 1)]}, "ind0": {"lo": [bx(0)], "hi": [bx(K - 1)]}}
    vC = {"bid.x": {"lo": [], "hi": []}, "tid.x": {"lo": [], "hi": []}, "bid.y": {"lo": [], "hi": []},
          "tid.y": {"lo": [], "hi": []}, "ind1": {"lo": [bx(0)], "hi": [bx(RM - 1)]},
          "ind2": {"lo": [bx(0)], "hi": [bx(RN - 1)]}}
    ldc = 2 * N if concat else N  # write into one half of a concatenated buffer
    rowsC = [term(es * ldc * TM, (), "bid.y"), term(es * ldc * RM, (), "tid.y"), term(es * ldc, (), "ind1")]
    colsC = [term(es * TN, (), "bid.x"), term(es * RN, (), "tid.x"), term(es, (), "ind2")]
    ds = [desc("R", es, "A", [term(es * K * TM, (), "bid.y"), term(es * K * RM, (), "tid.y"),
                              term(es * K, (), "ind1"), term(es, (), "ind0")], vA),
          desc("R", es, "B", [term(es * N, (), "ind0"), term(es * TN, (), "bid.x"),
                              term(es * RN, (), "tid.x"), term(es, (), "ind2")], vB),
          desc("W", es, "C", rowsC + colsC + ([term(es * N)] if concat else []), vC)]
    if bias:
        ds.append(desc("R", es, "bias", colsC, {k: vC[k] for k in ("bid.x", "tid.x", "ind2")}))
    if concat:  # also reads the other half (e.g. a residual slice of the same buffer)
        ds.append(desc("R", es, "C", rowsC + colsC, vC))
    pre = ptr_pre([p for p, _ in params]) + [
        {"op": "gdim.x", "lo": N // TN, "hi": N // TN}, {"op": "gdim.y", "lo": M // TM, "hi": M // TM},
        {"op": "bdim.x", "lo": TX, "hi": TX}, {"op": "bdim.y", "lo": TY, "hi": TY}]
    name = "tvm_concat_dense" if concat else "tvm_dense"

    def sample(rng, st):
        ptrs = st.bufs(["A", "B", "C", "bias"][:len(params)], 0,
                       small={"A": M * K * es, "B": K * N * es, "C": M * ldc * es, "bias": N * es})
        return ptrs, (N // TN, M // TM, 1), (TX, TY, 1)

    return (name, params, ds, pre, []), sample


def t_tvm_fused_ew(rng, small=False):
    """TVM fused elementwise/pooling with constant sizes (no scalar arguments)."""
    w = rng_pick(rng, [2, 4])
    nin = int(rng.integers(1, 4))
    n = int(rng_pick(rng, [1024, 2048, 4096] if small else [50176, 100352, 200704, 401408, 802816]))
    bd = rng_pick(rng, [256, 512, 1024])
    g = (n + bd - 1) // bd
    params = [("out", "ptr")] + [(f"in{i}", "ptr") for i in range(nin)]
    v = {"gidx.x": {"lo": [], "hi": [bx(n - 1)]}}
    ds = [desc("W", w, "out", [term(w, (), "gidx.x")], v)] + \
         [desc("R", w, f"in{i}", [term(w, (), "gidx.x")], v) for i in range(nin)]
    pre = ptr_pre([p for p, _ in params]) + [{"op": "gdim.x", "lo": g, "hi": g},
                                             {"op": "bdim.x", "lo": bd, "hi": bd}]

    def sample(rng, st):
        return st.bufs([p for p, _ in params], n * w), (g, 1, 1), (bd, 1, 1)

    return ("tvm_fused_ew", params, ds, pre, []), sample


def t_cudnn_like(rng, *, nptr=None):
    """Library kernel with many pointer arguments (C4): per-tensor read sites,
    output/workspace writes, scalar strides."""
    nptr = nptr or int(rng.integers(16, 49))
    nw = max(4, nptr // 4)
    nr = nptr - nw
    nsc = int(rng.integers(2, 5))
    params = [(f"p{i}", "ptr") for i in range(nptr)] + [(f"s{i}", "i32") for i in range(nsc)]
    descs = []
    for i in range(nptr):
        kind = "W" if i >= nr else "R"
        w = rng_pick(rng, [2, 4, 8, 16])
        s = f"s{int(rng.integers(0, nsc))}"
        v = {"bid.x": {"lo": [], "hi": []}, "tid.x": {"lo": [], "hi": []},
             "ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, [s]))]}}
        descs.append(desc(kind, w, f"p{i}", [term(w, ("bdim.x", s), "bid.x"), term(w, (s,), "tid.x"),
                                            term(w, (), "ind0")], v))
    pre = ptr_pre([f"p{i}" for i in range(nptr)]) + [{"op": f"s{i}", "lo": 1, "hi": 1 << 12} for i in range(nsc)] \
        + [{"op": "gdim.x", "lo": 1, "hi": 1 << 16}]

    def sample(rng, st):
        sc = [int(rng_pick(rng, [8, 16, 32, 64])) for _ in range(nsc)]
        g, b = int(rng_pick(rng, [64, 128, 256, 512])), int(rng_pick(rng, [128, 256]))
        size = g * b * 64 * 16
        ptrs = st.bufs([f"p{i}" for i in range(nptr)], size)
        if st.alias(rng):
            ptrs[nr + int(rng.integers(0, nw))] = ptrs[int(rng.integers(0, nr))]
        return ptrs + sc, (g, 1, 1), (b, 1, 1)

    return ("cudnn_like", params, descs, pre, []), sample


def t_multi_tensor(rng, *, kind=None, ntensor=None):
    """Multi-tensor-apply kernels (fused optimizers, foreach ops, multi-tensor
    norms): one launch touches T tensors of a parameter list, each through its
    own pointer argument (sizes shared by groups of 4 tensors), so the summary
    has 150-300 symbolic addresses and |R| x |W| > 4096 -- the wide (K2) path
    of SURVEY §8 row a8.  (<= 192 parameters per kernel, the loader's limit.)
      foreach_binary: o_i = a_i op b_i        (R a_i, R b_i, W o_i; T 48-56)
      adam_fused:     p, m, v updated in place (R p g m v, W p m v; T 24-44)
      l2norm:         ws[i] = |x_i|            (R x_i, W ws + 8 i; T 80-150)"""
    kind = kind or rng_pick(rng, ["foreach_binary"] * 6 + ["l2norm"] * 3 + ["adam_fused"] * 1)
    T = ntensor or int({"foreach_binary": rng.integers(48, 57), "adam_fused": rng.integers(24, 45),
                        "l2norm": rng.integers(80, 151)}[kind])
    ins, outs = {"foreach_binary": (["a", "b"], ["o"]), "adam_fused": (["p", "g", "m", "v"], ["p", "m", "v"]),
                 "l2norm": (["x"], [])}[kind]
    names = sorted(set(ins + outs), key=(ins + outs).index)
    ns = (T + 3) // 4
    params = [(f"{l}{i}", "ptr") for l in names for i in range(T)] + [(f"n{j}", "i64") for j in range(ns)]
    if kind == "l2norm":
        params.append(("ws", "ptr"))
    descs = []
    for i in range(T):
        v = {"ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, [f"n{i // 4}"]))]}}
        for l in ins:
            descs.append(desc("R", 4, f"{l}{i}", [term(4, (), "ind0")], v))
        for l in outs:
            descs.append(desc("W", 4, f"{l}{i}", [term(4, (), "ind0")], v))
        if kind == "l2norm":
            descs.append(desc("W", 8, "ws", [term(8 * i)], {}))
    ptrs = [p for p, k in params if k == "ptr"]
    pre = ptr_pre(ptrs) + [{"op": f"n{j}", "lo": 0, "hi": 1 << 28} for j in range(ns)]
    groups = []  # parameter groups the kernel is launched on (a training loop repeats them)

    def sample(rng, st):
        if len(groups) < 3 and (not groups or rng.random() < 0.3):
            n = [int(2 ** rng.uniform(8, 20)) for _ in range(ns)]
            bufs = {p: st.alloc.buf(8 * T if p == "ws" else 4 * n[int(p[1:]) // 4]) for p in ptrs}
            groups.append((n, bufs))
        n, bufs = groups[int(rng.integers(0, len(groups)))]
        pv = dict(bufs)
        if outs and st.alias(rng):
            # an output tensor aliases an input tensor of the list (in-place use)
            pv[f"{outs[0]}{int(rng.integers(0, T))}"] = pv[f"{ins[-1]}{int(rng.integers(0, T))}"]
        if kind == "l2norm" and st.alias(rng):
            pv["ws"] = pv[f"x{int(rng.integers(0, T))}"]  # workspace inside a read tensor
        args = [pv[p] for p in ptrs if p != "ws"] + n + ([pv["ws"]] if kind == "l2norm" else [])
        return args, (int(rng_pick(rng, [64, 148, 296, 592])), 1, 1), (512, 1, 1)

    return (f"mt_{kind}", params, descs, pre, []), sample


def t_fused_heavy(rng):
    """Heavily fused kernel of a DL framework (C2-heavy, SURVEY §8F "2-40
    descriptors per COND kernel, R x W of 4-100"): residual + bias + norm +
    activation + dropout-style fusions reading 6-30 tensors of an [R, H] layout
    (full tensors at row bid, per-column vectors), writing 2-4 outputs (full
    tensors and per-row statistics)."""
    w = rng_pick(rng, [2, 4])
    nfull = int(rng.integers(3, 16))
    nvec = int(rng.integers(3, 15))
    nout = int(rng.integers(2, 5))
    ins = [f"x{i}" for i in range(nfull)] + [f"v{i}" for i in range(nvec)]
    outs = [f"y{i}" for i in range(nout)]
    params = [(p, "ptr") for p in outs + ins] + [("H", "i32")]
    v = {"bid.x": {"lo": [], "hi": []}, "ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["H"]))]}}
    vv = {"ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["H"]))]}}
    row = [term(w, ("H",), "bid.x"), term(w, (), "ind0")]
    ds = [desc("R", w, f"x{i}", row, v) for i in range(nfull)]
    ds += [desc("R", w, f"v{i}", [term(w, (), "ind0")], vv) for i in range(nvec)]
    for j in range(nout):
        if j == nout - 1 and nout > 2:  # per-row statistic (mean / rstd)
            ds.append(desc("W", 4, f"y{j}", [term(4, (), "bid.x")], {"bid.x": {"lo": [], "hi": []}}))
        else:
            ds.append(desc("W", w, f"y{j}", row, v))
    pre = ptr_pre(outs + ins) + [{"op": "H", "lo": 1, "hi": 1 << 16}]
    bdim = rng_pick(rng, [128, 256, 512])

    def sample(rng, st):
        H = st.hidden
        R = st.rows(rng)
        ptrs = st.bufs(outs + ins, R * H * w, small={**{f"v{i}": H * w for i in range(nvec)}, outs[-1]: R * 4})
        if st.alias(rng):  # in-place residual update
            ptrs[0] = ptrs[nout + int(rng.integers(0, nfull))]
        return ptrs + [H], (R, 1, 1), (bdim, 1, 1)

    return ("fused_heavy", params, ds, pre, []), sample


def _violate(prng, k, args, p_pre, p_glob):
    """~0.5 % of the launches break a precondition (PAPER.md
    l.976-979: a value outside the range the analyzer assumed) and loop kernels
    sometimes run past their global condition (l.743-752): an argument set just
    past the bound of one check, kept inside every other check on it.  Inputs
    only: the code these launches get is the oracle's business."""
    names = [p["name"] for p in k["params"]]
    kinds = {p["name"]: p["kind"] for p in k["params"]}

    def typemax(nm):
        return I32_HI if kinds[nm] == "i32" else (1 << 63) - 1

    if k["glob"] and prng.random() < p_glob:
        c = k["glob"][int(prng.integers(0, len(k["glob"])))]
        if c["op"] in kinds:
            v = c["hi"] + 1
            if v <= typemax(c["op"]) and all(pc["lo"] <= v <= pc["hi"] for pc in k["pre"] if pc["op"] == c["op"]):
                args = list(args)
                args[names.index(c["op"])] = v
                return args
    if prng.random() < p_pre:
        cs = [c for c in k["pre"] if c["op"] in kinds and c["hi"] + 1 <= typemax(c["op"])]
        if cs:
            c = cs[int(prng.integers(0, len(cs)))]
            args = list(args)
            args[names.index(c["op"])] = c["hi"] + 1
    return args


def t_shortcut(rng, cls, reason=None):
    """Kernel-level I / NI kernels: memset-like writes; the
    validator returns their class without computing."""
    w = 4
    if cls == "IDEM":
        params = [("out", "ptr"), ("N", "i32")]
        v = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
        ds = [desc("W", w, "out", [term(w, (), "gidx.x")], v)]
    else:
        params = [("A", "ptr"), ("B", "ptr"), ("N", "i32")]
        v = {"gidx.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
        ds = [desc("R", w, "A", [term(w, (), "gidx.x")], v), desc("W", w, "A", [term(w, (), "gidx.x")], v)]
    pre = ptr_pre([p for p, k in params if k == "ptr"]) + [{"op": "N", "lo": 0, "hi": I32_HI}]

    def sample(rng, st):
        N = st.size(rng)
        names = [p for p, k in params if k == "ptr"]
        return st.bufs(names, N * w) + [N], ((N + 255) // 256, 1, 1), (256, 1, 1)

    name = "fill" if cls == "IDEM" else {"IF": "indirect_call", "PE": "lib_gemm", "NA": "ptr_chase",
                                         "SO": "inplace_update", "ATOMIC": "atomic_hist"}[reason]
    return (name, params, ds, pre, []), sample


MENUS = {
    "Rodinia": [t_elementwise, t_stencil2d, t_interleave, t_gather, t_scan, t_transpose, t_rowop, t_bias_act],
    "Parboil": [t_stencil2d, t_elementwise, t_gather, t_rowop, t_interleave],
    "TVM": [t_gemm_tvm, t_gemm_tvm, t_tvm_fused_ew],
    "PyTorch": [t_elementwise, t_bias_act, t_rowop, t_transpose, t_gather, t_scan],
    "TensorRT": [t_elementwise, t_bias_act, t_rowop, t_gemm_tvm, t_transpose],
    "FT": [t_bias_act, t_rowop, t_attention, t_transpose, t_gather, t_elementwise],
}


class ProgState:
    """Buffers and sizes of one running program (an app phase)."""

    def __init__(self, rng, alloc, knobs, hidden):
        self.alloc = alloc
        self.knobs = knobs
        self.hidden = hidden
        self.step = 0
        self._bufs = {}
        self.sizes = [int(x) for x in rng.choice([1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 3 << 18],
                                                 size=4)]

    def size(self, rng):
        return self.sizes[int(rng.integers(0, len(self.sizes)))]

    def rows(self, rng):
        return int(rng_pick(rng, [1, 8, 32, 128, 512]))

    def alias(self, rng):
        return rng.random() < self.knobs["p_alias"]

    def bufs(self, names, nbytes, small=None, offset=None):
        out = []
        for nm in names:
            want = (small or {}).get(nm, nbytes)
            key = (nm, want)
            if key not in self._bufs:
                self._bufs[key] = self.alloc.buf(max(want, 256) * 2)
            out.append(self._bufs[key] + (offset or {}).get(nm, 0))
        return out


# Launch-share multipliers: templates that are always (or mostly) range-
# overestimated are rarer in real traces (PAPER Table 5: RO is 310 of 18,217).
TEMPLATE_WEIGHT = {"redblack": 0.08, "masked_mha": 0.35, "tvm_concat_dense": 1.0}


def _weights(rng, samplers, knobs):
    """Zipf-like launch weights; NONIDEM/IDEM kernels get `ni_share` in total."""
    w = 1.0 / np.arange(1, len(samplers) + 1) ** 1.1
    rng.shuffle(w)
    w = w * np.array([s[4] for s in samplers])
    is_short = np.array([s[2] for s in samplers])
    w_cond, w_short = w * ~is_short, w * is_short
    wt = w_cond / max(w_cond.sum(), 1e-12) * (1 - knobs["ni_share"])
    if w_short.sum() > 0:
        wt = wt + w_short / w_short.sum() * knobs["ni_share"]
    return wt / wt.sum()


def _finish(kid, name, params, ds, pre, glob, cls="COND", reason=None):
    return kernel(kid, name, params, ds, pre=pre, glob=glob, cls=cls, reason=reason)


# launch shares of the SURVEY §8F boundary cases (separate generator stream,
# so the rest of the trace is the same with or without them)
P_PRE_VIOLATION = 0.005
P_GLOB_VIOLATION = 0.05


def make_c2(seed=23661, violations=True, heavy=False):
    """C2: returns (summary, rec, args, meta) with meta['app'][i] the app index
    of record i and meta['ptr_mask'] marking pointer argument slots.
    ``violations``: plant ~0.5 % precondition violations and global-condition
    violations on loop kernels (False gives round 1's mix).
    ``heavy``: C2-heavy, a third of the PyTorch / TensorRT / FT COND kernels
    are heavily fused (6-30 reads, 2-4 writes: up to 34 descriptors)."""
    rng = np.random.default_rng(seed)
    prng = np.random.default_rng(seed + 1000)  # boundary cases (violations / heavy choice)
    alloc = Alloc(rng)
    kernels, rows_app, launches = [], [], []
    kid = 0
    for ai, (app, nk, ninst, (n_i, n_ni, n_c), (r_if, r_pe, r_na, r_so)) in enumerate(APPS):
        knobs = KNOBS[app]
        samplers = []  # (kernel id, sampler, is_shortcut)
        ni_reasons = ["IF"] * r_if + ["PE"] * r_pe + ["NA"] * r_na + ["SO"] * r_so
        for j in range(nk):
            if j < n_i:
                (nm, p, d, pre, gl), smp = t_shortcut(rng, "IDEM")
                k = _finish(kid, f"{app}.{nm}{j}", p, d, pre, gl, cls="IDEM")
                short = True
            elif j < n_i + n_ni:
                reason = ni_reasons[j - n_i]
                (nm, p, d, pre, gl), smp = t_shortcut(rng, "NONIDEM", reason)
                k = _finish(kid, f"{app}.{nm}{j}", p, d, pre, gl, cls="NONIDEM", reason=reason)
                short = True
            else:
                menu = MENUS[app]
                if heavy and app in ("PyTorch", "TensorRT", "FT") and prng.random() < 1 / 3:
                    (nm, p, d, pre, gl), smp = t_fused_heavy(prng)
                elif app == "TVM" and rng.random() < 0.015:
                    (nm, p, d, pre, gl), smp = t_gemm_tvm(rng, concat=True)
                else:
                    (nm, p, d, pre, gl), smp = menu[int(rng.integers(0, len(menu)))](rng)
                k = _finish(kid, f"{app}.{nm}{j}", p, d, pre, gl)
                short = False
            kernels.append(k)
            samplers.append((kid, smp, short, k, TEMPLATE_WEIGHT.get(nm, 1.0)))
            kid += 1
        launches.append((ai, app, knobs, samplers, ninst))
    # Launch sequences: programs of 2-6 kernels iterated, concatenated per app.
    b = RecordBuilder()
    ptr_mask = []
    for ai, app, knobs, samplers, ninst in launches:
        hidden = int(rng_pick(rng, [256, 512, 768, 1024]))
        st = ProgState(rng, alloc, knobs, hidden)
        wt = _weights(rng, samplers, knobs)
        if app == "FT":
            # GPT-2 decode: a fixed launch sequence replayed (50 kernels,
            # 10,000 instances): every kernel once plus weighted draws, 100 per replay
            seq = list(range(len(samplers))) + [int(x) for x in rng.choice(len(samplers), size=50, p=wt)]
            rng.shuffle(seq)
            order = (seq * (ninst // len(seq) + 1))[:ninst]
        elif app == "TVM":
            order = list(range(len(samplers))) * 2
            order = order[:ninst] + [int(x) for x in rng.integers(0, len(samplers), size=max(0, ninst - len(order)))]
        else:
            # every kernel launched at least once; the rest by Zipf-like weights
            extra = rng.choice(len(samplers), size=ninst - len(samplers), p=wt)
            order = list(range(len(samplers))) + [int(x) for x in extra]
            # group into programs: sort by a random program key so launches of one
            # program are adjacent, as in an application's phases
            prog_of = rng.integers(0, max(1, len(samplers) // 3), size=len(samplers))
            order.sort(key=lambda j: (prog_of[j], rng.random()))
        for step, j in enumerate(order):
            st.step = step % 1024
            k_id, smp, short, k, _ = samplers[j]
            args, grid, block = smp(rng, st)
            if violations and not short:
                args = _violate(prng, k, args, P_PRE_VIOLATION, P_GLOB_VIOLATION)
            b.add(k_id, args, grid=grid, block=block)
            rows_app.append(ai)
            ptr_mask.extend(p["kind"] == "ptr" for p in k["params"])
    rec, args = b.build()
    summary = {"version": 1, "kernels": kernels}
    meta = {"app": np.array(rows_app, np.int8), "ptr_mask": np.array(ptr_mask, bool),
            "apps": [a[0] for a in APPS]}
    return summary, rec, args, meta


def make_c4(seed=23663, n=1 << 12, n_kernels=32):
    """C4: cuDNN-like kernels with 16-48 pointer args (~1% aliased writes)."""
    rng = np.random.default_rng(seed)
    alloc = Alloc(rng)
    ks, smps = [], []
    for kid in range(n_kernels):
        (nm, p, d, pre, gl), smp = t_cudnn_like(rng)
        ks.append(_finish(kid, f"{nm}{kid}", p, d, pre, gl))
        smps.append(smp)
    st = ProgState(rng, alloc, dict(p_alias=0.01, ni_share=0, p_opaque_on=0), 512)
    b = RecordBuilder()
    ptr_mask = []
    for i in range(n):
        j = int(rng.integers(0, n_kernels))
        args, grid, block = smps[j](rng, st)
        b.add(j, args, grid=grid, block=block)
        ptr_mask.extend(p["kind"] == "ptr" for p in ks[j]["params"])
    rec, args = b.build()
    return {"version": 1, "kernels": ks}, rec, args, {"ptr_mask": np.array(ptr_mask, bool)}


def make_wide(seed=23665, n=1 << 12, n_kernels=16):
    """Wide family ("instances with many pointer arguments"):
    multi-tensor-apply kernels with 80-400 symbolic addresses, all beyond 4096
    read x write pairs (auto-routed to the K2 sort + sweep path); ~5 % of the
    launches alias an output (or the workspace) to an input tensor."""
    rng = np.random.default_rng(seed)
    alloc = Alloc(rng)
    ks, smps = [], []
    for kid in range(n_kernels):
        (nm, p, d, pre, gl), smp = t_multi_tensor(rng)
        ks.append(_finish(kid, f"{nm}{kid}", p, d, pre, gl))
        smps.append(smp)
    st = ProgState(rng, alloc, dict(p_alias=0.05, ni_share=0, p_opaque_on=0), 512)
    b = RecordBuilder()
    ptr_mask = []
    for i in range(n):
        j = int(rng.integers(0, n_kernels))
        args, grid, block = smps[j](rng, st)
        b.add(j, args, grid=grid, block=block)
        ptr_mask.extend(p["kind"] == "ptr" for p in ks[j]["params"])
    rec, args = b.build()
    return {"version": 1, "kernels": ks}, rec, args, {"ptr_mask": np.array(ptr_mask, bool)}


def make_c3(seed=23662, n=1 << 14, n_kernels=64, small=False):
    """C3 base: TVM-style tiled GEMM/conv and fused elementwise kernels with
    affine strided ranges, some RO-prone (concatenated outputs).  ``small``:
    the small-grid subset the exact verifier enumerates (rows a10, f2)."""
    rng = np.random.default_rng(seed)
    alloc = Alloc(rng)
    ks, smps = [], []
    for kid in range(n_kernels):
        r = rng.random()
        if r < 0.1:
            (nm, p, d, pre, gl), smp = t_gemm_tvm(rng, concat=True, small=small)
        elif r < 0.75:
            (nm, p, d, pre, gl), smp = t_gemm_tvm(rng, small=small)
        else:
            (nm, p, d, pre, gl), smp = t_tvm_fused_ew(rng, small=small)
        ks.append(_finish(kid, f"{nm}{kid}", p, d, pre, gl))
        smps.append(smp)
    st = ProgState(rng, alloc, dict(p_alias=0.0, ni_share=0, p_opaque_on=0), 512)
    b = RecordBuilder()
    ptr_mask = []
    order = np.repeat(np.arange(n_kernels), (n + n_kernels - 1) // n_kernels)[:n]
    for j in order:
        args, grid, block = smps[j](rng, st)
        b.add(int(j), args, grid=grid, block=block)
        ptr_mask.extend(p["kind"] == "ptr" for p in ks[j]["params"])
    rec, args = b.build()
    return {"version": 1, "kernels": ks}, rec, args, {"ptr_mask": np.array(ptr_mask, bool)}


def replicate(rec, args, ptr_mask, copies, delta=1 << 37):
    """Tile a base trace `copies` times; replica r moves every pointer argument
    by r * delta (keeps the preconditions; verdicts are translation invariant,
    SURVEY §8E G9).  Returns packed (rec, args)."""
    n, a = len(rec), len(args)
    R = np.empty(n * copies, dtype=REC_DTYPE)
    A = np.empty(a * copies, dtype=np.int64)
    for r in range(copies):
        blk = R[r * n:(r + 1) * n]
        blk[:] = rec
        blk["arg_off"] += r * a
        A[r * a:(r + 1) * a] = args + ptr_mask.astype(np.int64) * (r * delta)
    return R, A
