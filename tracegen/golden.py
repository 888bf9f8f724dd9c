"""Hand-written access summaries for the paper's worked examples.

Each summary is the canonical JSON IR that the paper's offline
analyzer would have produced.  These are *inputs*: no expected verdicts live
here (the pinned expectations are in tests/golden/*.json with citations).

Kernels (ids are fixed so golden record files can refer to them):
  0 vectorAdd  PAPER.md l.296-301, l.592-596 (Fig. 1): A written, B and C read
  1 vectorSet  PAPER.md l.324-327: write-only -> kernel-level idempotent
  2 vectorInc  PAPER.md l.328-330: reads and writes A[idx] -> NONIDEM (SO)
  3 relu       PAPER.md l.776-791, 943-947, 1059-1069 (Fig. 4): per-thread loop of
               N elements, global condition N<=32, compacted to 2 descriptors
  4 stride_ro  PAPER.md l.1174-1177: reads {1,3,5}, writes {0,2,4}
  5 tighten    PAPER.md l.1012-1014, 1023-1026: path condition tid<N
  6 modfresh   PAPER.md l.990-992: A+tid%10 -> A+v, v in [0,9]
  7 opaque_na  PAPER.md l.755-765, 1149-1159: an address read from memory
  8 atomic     PAPER.md l.771-773: contains an atomic -> NONIDEM (ATOMIC)
  9 opaque_io  PAPER.md l.755-765, 1486-1491: opaque reads AND writes (an offset
               from __constant__ memory, the NA type (3)), each under its own
               runtime-checkable guard, next to plain reads and writes
"""
from __future__ import annotations

PTR_PRE_HI = (1 << 56) - 1  # "A < 2^56"


def bx(k0=0, *prods):
    """bexpr k0 + sum(k * prod(f)); prods are (k, [operands])."""
    return {"k0": int(k0), "p": [{"k": int(k), "f": list(f)} for k, f in prods]}


def term(k, f=(), var=None, div=1):
    return {"k": int(k), "f": list(f), "var": var, "div": int(div)}


def desc(kind, width, base, terms, vars=None, guard=None, opaque=False):
    return {
        "kind": kind,
        "width": width,
        "opaque": opaque,
        "base": base,
        "guard": guard or [],
        "vars": vars or {},
        "terms": terms,
    }


def ptr_pre(*names):
    return [{"op": n, "lo": 0, "hi": PTR_PRE_HI} for n in names]


def kernel(kid, name, params, desc_list, pre=(), glob=(), cls="COND", reason=None):
    return {
        "id": kid,
        "name": name,
        "params": [{"name": n, "kind": k} for n, k in params],
        "class": cls,
        "reason": reason,
        "pre": list(pre),
        "glob": list(glob),
        "desc": desc_list,
    }


GIDX = {"gidx.x": {"lo": [], "hi": []}}


def vector_add(kid=0):
    # A[idx] = B[idx] + C[idx], idx = bid*bdim + tid (Fig. 1)
    t = [term(4, (), "gidx.x")]
    return kernel(
        kid, "vectorAdd", [("A", "ptr"), ("B", "ptr"), ("C", "ptr")],
        [desc("W", 4, "A", t, GIDX), desc("R", 4, "B", t, GIDX), desc("R", 4, "C", t, GIDX)],
        pre=ptr_pre("A", "B", "C"),
    )


def vector_set(kid=1):
    t = [term(4, (), "gidx.x")]
    return kernel(kid, "vectorSet", [("A", "ptr")], [desc("W", 4, "A", t, GIDX)],
                  pre=ptr_pre("A"), cls="IDEM")


def vector_inc(kid=2):
    t = [term(4, (), "gidx.x")]
    return kernel(kid, "vectorInc", [("A", "ptr")],
                  [desc("R", 4, "A", t, GIDX), desc("W", 4, "A", t, GIDX)],
                  pre=ptr_pre("A"), cls="NONIDEM", reason="SO")


def relu(kid=3):
    # A[(bid*bdim+tid)*N + i], i in [0, N-1]
    v = {"bid.x": {"lo": [], "hi": []}, "tid.x": {"lo": [], "hi": []},
         "ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["N"]))]}}
    t = [term(4, ("bdim.x", "N"), "bid.x"), term(4, ("N",), "tid.x"), term(4, (), "ind0")]
    return kernel(
        kid, "relu", [("A", "ptr"), ("B", "ptr"), ("N", "i32")],
        [desc("R", 4, "A", t, v), desc("W", 4, "B", t, v)],
        pre=ptr_pre("A", "B") + [{"op": "N", "lo": 0, "hi": (1 << 10) - 1}],
        glob=[{"op": "N", "lo": -(1 << 63), "hi": 32}],  # "N<=32"
    )


def stride_ro(kid=4):
    # read A[2*tid+1], write A[2*tid] (bytes)
    v = {"tid.x": {"lo": [], "hi": []}}
    return kernel(
        kid, "stride_ro", [("A", "ptr")],
        [desc("R", 1, "A", [term(2, (), "tid.x"), term(1)], v),
         desc("W", 1, "A", [term(2, (), "tid.x")], v)],
        pre=ptr_pre("A"),
    )


def tighten(kid=5):
    # if (tid < N) B[tid] = A[tid]; tid in [0, min(N-1, bdim-1)]
    v = {"tid.x": {"lo": [], "hi": [bx(-1, (1, ["N"]))]}}
    t = [term(4, (), "tid.x")]
    return kernel(
        kid, "tighten", [("A", "ptr"), ("B", "ptr"), ("N", "i64")],
        [desc("R", 4, "A", t, v), desc("W", 4, "B", t, v)],
        pre=ptr_pre("A", "B") + [{"op": "N", "lo": 0, "hi": 1 << 31}],
    )


def modfresh(kid=6):
    # B[tid] = A[tid % 10]: A + 4*v, v = tid%10 in [0, 9]
    v = {"tid.x": {"lo": [], "hi": []},
         "fr0": {"lo": [bx(0)], "hi": [bx(9)], "def": {"src": "tid.x", "mod": 10}}}
    return kernel(
        kid, "modfresh", [("A", "ptr"), ("B", "ptr")],
        [desc("R", 4, "A", [term(4, (), "fr0")], v),
         desc("W", 4, "B", [term(4, (), "tid.x")], {"tid.x": {"lo": [], "hi": []}})],
        pre=ptr_pre("A", "B"),
    )


def opaque_na(kid=7):
    # out[tid] = *pp (address read from memory) when flag != 0
    return kernel(
        kid, "opaque_na", [("pp", "ptr"), ("out", "ptr"), ("flag", "i32")],
        [desc("R", 8, "pp", [], {}),
         desc("R", 4, None, [], {"tid.x": {"lo": [], "hi": []}}, opaque=True,
              guard=[{"a": "flag", "cmp": "!=", "b": 0}]),
         desc("W", 4, "out", [term(4, (), "tid.x")], {"tid.x": {"lo": [], "hi": []}})],
        pre=ptr_pre("pp", "out") + [{"op": "flag", "lo": -(1 << 31), "hi": (1 << 31) - 1}],
    )


def opaque_io(kid=9):
    # __constant__ int c_off;   (a non-parameter variable, PAPER.md l.1489-1491 type (3))
    # k(int* out, const int* src, int rflag, int wflag) {
    #   int v = 0;
    #   if (rflag == 1) v = src[tid];            // R src + 4*tid
    #   if (rflag == 2) v = src[c_off + tid];    // R opaque
    #   if (wflag == 1) out[c_off + tid] = v;    // W opaque
    #   if (wflag == 2) out[tid] = v;            // W out + 4*tid
    # }
    t = {"tid.x": {"lo": [], "hi": []}}
    i32 = {"lo": -(1 << 31), "hi": (1 << 31) - 1}
    return kernel(
        kid, "opaque_io", [("out", "ptr"), ("src", "ptr"), ("rflag", "i32"), ("wflag", "i32")],
        [desc("R", 4, "src", [term(4, (), "tid.x")], t, guard=[{"a": "rflag", "cmp": "==", "b": 1}]),
         desc("R", 4, None, [], t, opaque=True, guard=[{"a": "rflag", "cmp": "==", "b": 2}]),
         desc("W", 4, None, [], t, opaque=True, guard=[{"a": "wflag", "cmp": "==", "b": 1}]),
         desc("W", 4, "out", [term(4, (), "tid.x")], t, guard=[{"a": "wflag", "cmp": "==", "b": 2}])],
        pre=ptr_pre("out", "src") + [dict(op="rflag", **i32), dict(op="wflag", **i32)],
    )


def atomic_k(kid=8):
    return kernel(kid, "atomicHist", [("H", "ptr")],
                  [desc("W", 4, "H", [term(4, (), "gidx.x")], GIDX)],
                  pre=ptr_pre("H"), cls="NONIDEM", reason="ATOMIC")


def golden_summary():
    return {
        "version": 1,
        "kernels": [vector_add(), vector_set(), vector_inc(), relu(), stride_ro(),
                    tighten(), modfresh(), opaque_na(), atomic_k(), opaque_io()],
    }


# C1: vectorAdd, gdim=4, bdim=128, 8 records.
C1_ARGS = [
    (0x1000, 0x2000, 0x3000),  # r0 distinct
    (0x1000, 0x2000, 0x1000),  # r1 C aliases A
    (0x1000, 0x1000, 0x3000),  # r2 B aliases A
    (0x1000, 0x2000, 0x2000),  # r3 B = C (read/read alias)
    (0x1800, 0x1000, 0x3000),  # r4 touching extents
    (0x17FC, 0x1000, 0x3000),  # r5 4-byte overlap
    (0x1000, 0x2000, 0x802),   # r6 overlap only through the access width
    (1 << 56, 0x2000, 0x3000),  # r7 violates A < 2^56
]


def c1_records():
    from .records import RecordBuilder

    b = RecordBuilder()
    for a in C1_ARGS:
        b.add(0, a, grid=(4,), block=(128,))
    return b.build()
