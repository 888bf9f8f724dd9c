"""Plain CPU oracle for Picker's runtime validation (arXiv 2410.23661).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_2410_23661_b200/) never imports it, and this module imports nothing from
the product path: the two share no code.

It is deliberately slow and obvious: exact Python integers (no wrap-around), the
plain definitions written out, in the order of the paper's Fig. 3 pseudocode as
the prose describes it: global condition first, then the
concrete addresses of every symbolic address, then the read/write overlap.

Two functions:

* ``oracle_interval(kernel, rec)`` -- the optimized validator's result: one range
  [LB, UB] per symbolic address (descriptor), ``LB = min over the variable box of
  Addr`` (the definition of LB(args)), byte extent
  [LB, UB + width - 1] (byte granularity, l.140-141 "for every byte"), then the
  R/W overlap rule (l.658-666).  The min/max is taken by brute force over the
  box when the box is small, otherwise per variable (the address is a sum of
  one-variable terms, so the box minimum is the sum of per-variable minima); a
  per-variable range that is too large to enumerate is evaluated at its two
  endpoints, which is exact because every such variable's terms are checked here
  to be monotone in the same direction (the monotonicity the
  analyzer proves offline); a non-monotone large variable raises.
* ``oracle_exact(kernel, rec, cap)`` -- the strawman (Fig. 3 / l.717-730): enumerate
  every point of every descriptor's variable box, build the set of read bytes
  and the set of written bytes, intersect the sets.

Readings of points the paper leaves open are DESIGN.md §4 (Q1-Q21); each is
cited at the line that implements it.
"""
from __future__ import annotations

import itertools

# ---- verdict codes (identical on the GPU) --------------------
IDEM_CHECKED = 0
IDEM_KERNEL = 1
NI_KERNEL = {"SO": 2, "ATOMIC": 3, "IF": 4, "PE": 5, "NA": 6}
NI_PRECOND = 7
NI_GLOBAL = 8
NI_OPAQUE = 9
NI_OVERLAP = 10
EXACT_SKIPPED = 11
ERR_ARITY = 0xFE
ERR_KERNEL = 0xFF

IDEMPOTENT_CODES = (IDEM_CHECKED, IDEM_KERNEL)

DIMS = ("gdim.x", "gdim.y", "gdim.z", "bdim.x", "bdim.y", "bdim.z")
# CUDA launch limits (reading Q21): a record outside them is conservatively NI (code 7).
DIM_MAX = {"gdim.x": 2**31 - 1, "gdim.y": 65535, "gdim.z": 65535,
           "bdim.x": 1024, "bdim.y": 1024, "bdim.z": 64}
BLOCK_MAX_THREADS = 1024

# whole-box enumeration of at most 2^20 points, else per-variable
# enumeration of ranges of at most 2^20 values, else the endpoints.  2^12 here
# (the oracle's first value; 2^20 costs minutes per C2 trace in pure Python);
# tests/test_oracle_pins.py::test_box_vs_per_variable pins that the three
# methods give the same extents on every random summary.
BRUTE_BOX_POINTS = 1 << 12   # whole-box enumeration up to this many points
BRUTE_VAR_POINTS = 1 << 12   # per-variable enumeration up to this range size


class OracleUnsupported(Exception):
    """The summary falls outside what the oracle can decide exactly."""


# ---- summary access ---------------------------------------------------------

def index_summary(summary):
    """Map kernel id -> kernel dict (the JSON IR)."""
    return {int(k["id"]): k for k in summary["kernels"]}


def decode_record(rec_row, args):
    """Decode one numpy record row + the args pool into plain Python values."""
    return {
        "kernel_id": int(rec_row["kernel_id"]),
        "nargs": int(rec_row["nargs"]),
        "grid": (int(rec_row["grid_x"]), int(rec_row["grid_y"]), int(rec_row["grid_z"])),
        "block": (int(rec_row["block_x"]), int(rec_row["block_y"]), int(rec_row["block_z"])),
        "arg_off": int(rec_row["arg_off"]),
        "args_pool": args,
    }


def _values(kernel, rec):
    """Concrete values of every operand: launch arguments and dimensions.

    i32 parameters take the low 32 bits of their slot, sign-extended (SURVEY §8A.1:
    "i32 values are sign-extended into the 64-bit arg slot"); ptr and i64 slots
    are read as signed 64-bit integers.
    """
    vals = {}
    pool = rec["args_pool"]
    for i, p in enumerate(kernel["params"]):
        v = int(pool[rec["arg_off"] + i])
        if p["kind"] == "i32":
            v &= 0xFFFFFFFF
            if v >= 1 << 31:
                v -= 1 << 32
        vals[p["name"]] = v
    for name, v in zip(DIMS, rec["grid"] + rec["block"]):
        vals[name] = v
    return vals


def _operand(vals, x):
    return x if isinstance(x, int) else vals[x]


def _prod(vals, factors):
    r = 1
    for f in factors:
        r *= _operand(vals, f)
    return r


def _bexpr(vals, e):
    """bexpr = k0 + sum_j k_j * prod(f_j)."""
    return e["k0"] + sum(p["k"] * _prod(vals, p["f"]) for p in e["p"])


def _cmp(a, op, b):
    return {"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b,
            "==": a == b, "!=": a != b}[op]


# ---- variable boxes -----------------------------------------------------------

def _structural(var, vals):
    """Implicit thread-space bounds (min/max over bid, tid)."""
    kind, _, axis = var.partition(".")
    if kind == "tid":
        return 0, vals["bdim." + axis] - 1
    if kind == "bid":
        return 0, vals["gdim." + axis] - 1
    if kind == "gidx":
        return 0, vals["gdim." + axis] * vals["bdim." + axis] - 1
    return None  # induction / fresh variables declare their own bounds


def var_box(d, vals):
    """[lo, hi] of every variable of descriptor d for this instance.

    lo = max(structural lo, declared lo bexprs), hi = min(structural hi, declared
    hi bexprs): the path-condition tightening of PAPER.md l.1023-1026
    ("[0, min(N-1, bdim-1)]"), induction ranges l.1063/1066-1067 ("from 0 to N-1"),
    fresh ranges l.990-992 ("[0, 9]").
    """
    box = {}
    for var, spec in d["vars"].items():
        los = [_bexpr(vals, e) for e in spec.get("lo", [])]
        his = [_bexpr(vals, e) for e in spec.get("hi", [])]
        s = _structural(var, vals)
        if s is not None:
            los.append(s[0])
            his.append(s[1])
        if not los or not his:
            raise OracleUnsupported(f"variable {var} has no lower or upper bound")
        box[var] = (max(los), min(his))
    return box


def _phi(x, div):
    return x // div  # floor division by a positive constant (monotone), SURVEY §8A.1


def _addr(d, vals, point):
    """Concrete address of descriptor d at one point of its variable box."""
    a = vals[d["base"]] if d["base"] is not None else 0
    for t in d["terms"]:
        c = t["k"] * _prod(vals, t["f"])
        if t["var"] is None:
            a += c
        else:
            a += c * _phi(point[t["var"]], t.get("div", 1))
    return a


def _box_points(box):
    n = 1
    for lo, hi in box.values():
        n *= hi - lo + 1
    return n


def interval_extent(d, vals, box):
    """Byte extent [LB, UB + width - 1] of an active, non-opaque descriptor.

    LB(args) = min over the box of Addr; UB the max.
    """
    if _box_points(box) <= BRUTE_BOX_POINTS:
        names = list(box)
        addrs = [
            _addr(d, vals, dict(zip(names, pt)))
            for pt in itertools.product(*(range(lo, hi + 1) for lo, hi in box.values()))
        ]
        lb, ub = min(addrs), max(addrs)
    else:
        # Addr = base + const terms + sum_v g_v(x_v): the minimum over a box of a sum
        # of functions of distinct variables is the sum of their minima.
        zero = {v: 0 for v in box}
        base = _addr({"base": d["base"], "terms": [t for t in d["terms"] if t["var"] is None]},
                     vals, zero)
        lb = ub = base
        for v, (lo, hi) in box.items():
            ts = [t for t in d["terms"] if t["var"] == v]
            if not ts:
                continue
            coefs = [t["k"] * _prod(vals, t["f"]) for t in ts]

            def g(x, ts=ts, coefs=coefs):
                return sum(c * _phi(x, t.get("div", 1)) for c, t in zip(coefs, ts))

            if hi - lo + 1 <= BRUTE_VAR_POINTS:
                gs = [g(x) for x in range(lo, hi + 1)]
                lb += min(gs)
                ub += max(gs)
            else:
                if all(c >= 0 for c in coefs) or all(c <= 0 for c in coefs):
                    ends = (g(lo), g(hi))  # monotone in x: extremes at the endpoints
                    lb += min(ends)
                    ub += max(ends)
                else:
                    raise OracleUnsupported(f"non-monotone large variable {v}")
    return lb, ub + d["width"] - 1


# ---- the shared prefix of both validators -------------------------------------

def _prefix(kernels, rec, through_idem=False):
    """Steps common to oracle_interval and oracle_exact.

    Returns (code, None) when the verdict is decided before any address is
    computed, else (None, (kernel, vals, active)) where active is a list of
    (descriptor, box) for descriptors whose guard holds and whose box is nonempty.
    ``through_idem``: evaluate a kernel-level idempotent kernel like a COND one
    (its writes matter to a multi-kernel window, reading Q23).
    """
    k = kernels.get(rec["kernel_id"])
    if k is None:
        return ERR_KERNEL, None
    if rec["nargs"] != len(k["params"]) or rec["arg_off"] + rec["nargs"] > len(rec["args_pool"]):
        return ERR_ARITY, None
    # Kernel-level shortcuts: "The validator directly returns kernel-level
    # idempotency without performing the validation".
    if k["class"] == "IDEM" and not through_idem:
        return IDEM_KERNEL, None
    if k["class"] == "NONIDEM":
        return NI_KERNEL[k["reason"]], None
    vals = _values(k, rec)
    # Preconditions: "If an instance violates these constraints, Picker would
    # conservatively treat it as non-idempotent".  The CUDA
    # launch limits on the dimensions are implicit preconditions (reading Q21).
    for name in DIMS:
        if not 1 <= vals[name] <= DIM_MAX[name]:
            return NI_PRECOND, None
    if vals["bdim.x"] * vals["bdim.y"] * vals["bdim.z"] > BLOCK_MAX_THREADS:
        return NI_PRECOND, None
    for c in k["pre"]:
        if not c["lo"] <= vals[c["op"]] <= c["hi"]:
            return NI_PRECOND, None
    # Global condition (Fig. 3 lines 1-2; unbounded loops l.743-752).
    for c in k["glob"]:
        if not c["lo"] <= vals[c["op"]] <= c["hi"]:
            return NI_GLOBAL, None
    active = []
    for d in k["desc"]:
        # Path conditions over launch arguments only (Fig. 3 lines 6-7).
        if not all(_cmp(_operand(vals, g["a"]), g["cmp"], _operand(vals, g["b"])) for g in d["guard"]):
            continue
        box = var_box(d, vals)
        if any(lo > hi for lo, hi in box.values()):
            continue  # empty thread/loop range: the site never executes (reading Q5)
        active.append((d, box))
    return None, (k, vals, active)


def _opaque_rule(active):
    """Non-parameter addresses "could be any concrete value" and overlap any other
    address; an opaque read needs some active write and an
    opaque write some active read (reading Q8)."""
    kinds = {(d["kind"], d["opaque"]) for d, _ in active}
    has_r = any(k == "R" for k, _ in kinds)
    has_w = any(k == "W" for k, _ in kinds)
    return (("R", True) in kinds and has_w) or (("W", True) in kinds and has_r)


def congruence(d, vals, box):
    """Stride-aware range (reading Q24): every address of an
    active descriptor is congruent to r modulo g.

    The terms on one variable with one divisor form a group C * phi(x), C the sum
    of their coefficients.  g = gcd of |C| over the groups whose phi takes more
    than one value on the box; the other groups are constants.  g = 0: the
    descriptor is a single address r.  Otherwise 0 <= r < g.  This is the
    congruence class the paper's RO example needs (reads
    {1,3,5} and writes {0,2,4} are both stride 2, residues 1 and 0).
    """
    const = vals[d["base"]] if d["base"] is not None else 0
    groups = {}
    for t in d["terms"]:
        c = t["k"] * _prod(vals, t["f"])
        if t["var"] is None:
            const += c
        else:
            key = (t["var"], t.get("div", 1))
            groups[key] = groups.get(key, 0) + c
    g = 0
    for (v, div), c in groups.items():
        lo, hi = box[v]
        if _phi(lo, div) == _phi(hi, div):
            const += c * _phi(lo, div)
        else:
            g = _gcd(g, abs(c))
    return g, (const % g if g else const)


def _gcd(a, b):
    while b:
        a, b = b, a % b
    return a


def may_collide(r_cong, r_width, w_cong, w_width):
    """Can an address a = r (mod gR) touching [a, a + wR - 1] share a byte with
    an address b = r' (mod gW) touching [b, b + wW - 1]?  b - a ranges over
    (r' - r) + gcd(gR, gW) * Z; a shared byte needs -(wW - 1) <= b - a <= wR - 1."""
    (gr, rr), (gw, rw) = r_cong, w_cong
    G = _gcd(gr, gw)
    lo, hi = -(w_width - 1), r_width - 1
    if G == 0:
        return lo <= rw - rr <= hi
    return (rw - rr - lo) % G <= hi - lo


def oracle_interval(kernels, rec, stride=False):
    """Verdict code of the range-based validator for one instance.

    ``stride``: the stride-aware variant (row f4): a read/write pair whose byte
    intervals intersect is an overlap only if their congruence classes can also
    share a byte (``may_collide``)."""
    code, st = _prefix(kernels, rec)
    if code is not None:
        return code
    _, vals, active = st
    if _opaque_rule(active):
        return NI_OPAQUE
    reads, writes = [], []
    for d, box in active:
        e = interval_extent(d, vals, box)
        cg = congruence(d, vals, box) if stride else None
        (reads if d["kind"] == "R" else writes).append((e, cg, d["width"]))
    # "an instance is considered non-idempotent if there exists any overlap in the
    # read and write addresses ... regardless of the access order";
    # closed byte intervals, touching is not overlapping (reading Q4).
    for r, rc, rw in reads:
        for w, wc, ww in writes:
            if r[0] <= w[1] and w[0] <= r[1]:
                if not stride or may_collide(rc, rw, wc, ww):
                    return NI_OVERLAP
    return IDEM_CHECKED


def extents(kernels, rec):
    """Active (kind, lb, ub) extents of one instance (for tests and diagnostics)."""
    code, st = _prefix(kernels, rec)
    if code is not None:
        return code, []
    _, vals, active = st
    out = []
    for d, box in active:
        if d["opaque"]:
            out.append((d["kind"], None, None))
        else:
            lb, ub = interval_extent(d, vals, box)
            out.append((d["kind"], lb, ub))
    return None, out


def _points(d, box):
    """Every point of the descriptor's box; fresh variables with a definition take
    their defining value ("A+tid%10" -> "A+var")."""
    free = [v for v in box if "def" not in d["vars"][v]]
    derived = [v for v in box if "def" in d["vars"][v]]
    for pt in itertools.product(*(range(box[v][0], box[v][1] + 1) for v in free)):
        p = dict(zip(free, pt))
        for v in derived:
            df = d["vars"][v]["def"]
            s = p[df["src"]]
            p[v] = s % df["mod"] if "mod" in df else s & df["and"]
        yield p


def exact_points(kernels, rec):
    """Total number of enumerated points of the active non-opaque descriptors."""
    code, st = _prefix(kernels, rec)
    if code is not None:
        return 0
    _, _, active = st
    total = 0
    for d, box in active:
        if not d["opaque"]:
            free = {v: b for v, b in box.items() if "def" not in d["vars"][v]}
            total += _box_points(free)
    return total


def oracle_exact(kernels, rec, cap=1 << 20):
    """Strawman verdict: per-thread address enumeration and set intersection
    (Fig. 3).  Code 11 when the active non-opaque symbolic
    addresses have more than ``cap`` points in total ("the point
    count exceeds the cap"; reading Q22)."""
    code, st = _prefix(kernels, rec)
    if code is not None:
        return code
    _, vals, active = st
    if _opaque_rule(active):
        return NI_OPAQUE
    if exact_points(kernels, rec) > cap:
        return EXACT_SKIPPED
    rbytes, wbytes = set(), set()
    for d, box in active:
        target = rbytes if d["kind"] == "R" else wbytes
        for p in _points(d, box):
            a = _addr(d, vals, p)
            target.update(range(a, a + d["width"]))
    return NI_OVERLAP if rbytes & wbytes else IDEM_CHECKED


def oracle_batch(summary, rec_array, args, fn=oracle_interval, **kw):
    """Apply fn to every record of a packed batch; returns a list of codes."""
    kernels = index_summary(summary)
    return [fn(kernels, decode_record(r, args), **kw) for r in rec_array]


def _mp_chunk(job):
    summary, rec, args, fn_name, kw = job
    return oracle_batch(summary, rec, args, globals()[fn_name], **kw)


def oracle_batch_mp(summary, rec_array, args, fn=oracle_interval, processes=None, **kw):
    """oracle_batch over a multiprocessing pool (same results, more cores)."""
    import multiprocessing as mp
    import warnings
    import os

    processes = processes or os.cpu_count() or 1
    n = len(rec_array)
    if processes <= 1 or n < 256:
        return oracle_batch(summary, rec_array, args, fn, **kw)
    step = (n + processes * 4 - 1) // (processes * 4)
    jobs = [(summary, rec_array[i:i + step], args, fn.__name__, kw) for i in range(0, n, step)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", DeprecationWarning)
        pool = mp.get_context("fork").Pool(processes)
    with pool:
        parts = pool.map(_mp_chunk, jobs)
    return [c for p in parts for c in p]


# ---- multi-kernel idempotency (reading Q23) ----------------

SEQ_SEQUENTIAL, SEQ_CONCURRENT = 0, 1


def oracle_sequence(kernels, recs, mode=SEQ_SEQUENTIAL):
    """Idempotency of a list of launches as one unit.

    "First, Picker predicts the read and write addresses of each GPU kernel
    instance.  Second, [it] sorts the instances by their launch order, and then
    checks the clobber anti-dependency across the instances" (sequential list);
    for "concurrently executed GPU kernel instances, [it checks] the overlap of
    read and write addresses among all concurrent instances".

    Reading Q23: the first instance (launch order) whose single-instance check is
    decided before any address (unknown kernel, arity, kernel-level NI class,
    precondition, global condition) decides the list; kernel-level idempotent
    instances take part with their writes.  Otherwise, with instances i (reads)
    and j (writes): sequential requires i <= j (a write can clobber a byte read
    by the same or an earlier instance; an earlier write cannot be trusted to
    cover the byte, the extents over-approximate), concurrent takes every pair.
    Opaque rule first (9), then overlap (10), else 0.
    """
    inst = []
    for rec in recs:
        code, st = _prefix(kernels, rec, through_idem=True)
        if code is not None:
            return code
        _, vals, active = st
        inst.append([(d["kind"], d["opaque"], None if d["opaque"] else interval_extent(d, vals, box))
                     for d, box in active])

    def ordered(i, j):
        return mode == SEQ_CONCURRENT or i <= j

    for i, a in enumerate(inst):  # reads of i
        for j, b in enumerate(inst):  # writes of j
            if not ordered(i, j):
                continue
            if any(k == "R" and o for k, o, _ in a) and any(k == "W" for k, _, _ in b):
                return NI_OPAQUE
            if any(k == "R" for k, _, _ in a) and any(k == "W" and o for k, o, _ in b):
                return NI_OPAQUE
    for i, a in enumerate(inst):
        for j, b in enumerate(inst):
            if not ordered(i, j):
                continue
            for kr, orr, r in a:
                if kr != "R" or orr:
                    continue
                for kw, ow, w in b:
                    if kw == "W" and not ow and r[0] <= w[1] and w[0] <= r[1]:
                        return NI_OVERLAP
    return IDEM_CHECKED


def oracle_windows(summary, rec_array, args, window, mode=SEQ_SEQUENTIAL):
    """oracle_sequence over consecutive windows of ``window`` records."""
    kernels = index_summary(summary)
    recs = [decode_record(r, args) for r in rec_array]
    return [oracle_sequence(kernels, recs[w:w + window], mode) for w in range(0, len(recs), window)]


# ---- row f3: consumer models on the verdicts (§7.5 l.1612-1690) ------

MODEL_MAX_READS = 128  # reading Q25: more active read extents -> input size unknown
MODEL_HIST_BUCKETS = 129  # preemption-latency histogram: 1 us buckets, last = >= 128 us


def oracle_input_bytes(kernels, rec):
    """Bytes an Asymmetric-Resilience checkpoint copies for one instance: "AR
    checkpoints the input buffer of every GPU kernel instance" (PAPER.md
    l.1620-1622), read as the length of the union of the instance's active,
    non-opaque read extents (reading Q25).  Returns None (unknown) when the
    extents are not computable: unknown kernel, arity, a kernel-level NONIDEM
    class (no verified summary), a failing launch limit / precondition / global
    condition, an opaque read, or more than MODEL_MAX_READS read extents."""
    code, st = _prefix(kernels, rec, through_idem=True)
    if code is not None:
        return None
    _, vals, active = st
    ext = []
    for d, box in active:
        if d["kind"] != "R":
            continue
        if d["opaque"]:
            return None
        ext.append(interval_extent(d, vals, box))
    if len(ext) > MODEL_MAX_READS:
        return None
    merged = []  # union of closed intervals: merge in lb order
    for lb, ub in sorted(ext):
        if merged and lb <= merged[-1][1] + 1:
            merged[-1][1] = max(merged[-1][1], ub)
        else:
            merged.append([lb, ub])
    return sum(ub - lb + 1 for lb, ub in merged)


def oracle_models(summary, rec_array, args, codes, ctx_bytes, kill_ns=1000, save_bytes_per_us=1000):
    """AR checkpoint bytes and Chimera preemption latency.

    AR: without idempotency every instance's input is checkpointed; with it only
    the non-idempotent ones (codes other than 0 and 1).  Instances whose input
    size is unknown count 0 bytes and are counted in ``unknown_input``.
    Chimera: preempting an idempotent instance kills it (``kill_ns``, "less than
    1 microsecond", l.1677-1679); a non-idempotent one saves its context,
    ``ctx_bytes * 1000 // save_bytes_per_us`` ns.  Integer nanoseconds; the
    histogram has 1 us buckets (bucket 128 = 128 us and above)."""
    K = index_summary(summary)
    out = {"n": len(rec_array), "n_idem": 0, "ckpt_bytes_all": 0, "ckpt_bytes_ni": 0, "unknown_input": 0,
           "preempt_ns_without": 0, "preempt_ns_with": 0,
           "hist_without": [0] * MODEL_HIST_BUCKETS, "hist_with": [0] * MODEL_HIST_BUCKETS}
    for row, code, cb in zip(rec_array, codes, ctx_bytes):
        r = decode_record(row, args)
        idem = int(code) in IDEMPOTENT_CODES
        b = oracle_input_bytes(K, r)
        if b is None:
            out["unknown_input"] += 1
            b = 0
        out["ckpt_bytes_all"] += b
        if not idem:
            out["ckpt_bytes_ni"] += b
        out["n_idem"] += idem
        save = int(cb) * 1000 // save_bytes_per_us
        lat = kill_ns if idem else save
        out["preempt_ns_without"] += save
        out["preempt_ns_with"] += lat
        out["hist_without"][min(save // 1000, MODEL_HIST_BUCKETS - 1)] += 1
        out["hist_with"][min(lat // 1000, MODEL_HIST_BUCKETS - 1)] += 1
    return out
