"""Host-side checks of the specialised-module generator (jit.cpp) that need no
GPU: NVRTC compiles for sm_100a here.  Correctness of the generated code is
pinned on the GPU (tests/test_gpu_codegen.py); these check which code the
generator emits from the loader's proofs and the summary's paths."""
import re

import pytest

from tracegen import golden, workloads
from tracegen.edges import edge_summary


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


def _shape_bodies(src):
    return dict(re.findall(r"uint8_t (ks\d+)\((.*?)\n}\n", src, re.S))


def test_narrow_multiplies_only_where_proved(pk):
    """A coefficient of 2^31 - 1 or -2^31 on bid.x (< 2^31 - 1) is int32 on both
    factors: one 32x32->64 multiply (mulw); 2^31, -2^31 - 1 and gidx.x
    (up to 2^41) keep the 64-bit multiply."""
    s = edge_summary()
    r, msg, src = pk.compile_summaries(s, want_source=True)
    assert r > 0, msg
    assert "mulw(" in src and "mul64(" in src
    for k in s["kernels"]:
        sub = {"version": 1, "kernels": [k]}
        r, msg, src = pk.compile_summaries(sub, want_source=True)
        assert r == 1, msg
        body = next(iter(_shape_bodies(src).values()))
        # the write site (1 x tid.x) is int32 everywhere; the read site decides
        coef = k["desc"][0]["terms"][0]["k"] if k["name"].startswith("edge") else None
        if coef in ((1 << 31) - 1, -(1 << 31)):
            assert "mul64(" not in body, (k["name"], body)
        elif coef is not None:
            assert "mul64(" in body, (k["name"], body)
        if k["name"] == "gidx":
            assert "mul64(" in body and "mulw(" not in body
        if k["name"] == "argcoef1":  # s0 (int32) x tid.x
            assert "mul64(" not in body
        if k["name"] == "argcoef2":  # 2 * s0 may reach 2^32
            assert "mul64(" in body


def test_unused_paths_left_out(pk):
    """Without wide kernels the module is built without the K2 path; with one,
    the path is there."""
    s = golden.golden_summary()
    _, _, src = pk.compile_summaries(s, want_source=True)
    assert "#define PICKER_NO_WIDE 1" in src
    assert "eval_generic(" not in src.split("struct JitDispatch")[1]


def test_launch_limits_once_and_packed_constants(pk):
    """The CUDA launch limits are checked in the dispatch, not in each shape;
    per-kernel constants are read as int32 words with 128-bit loads."""
    s = workloads.make_c3()[0]  # 64 kernels in 14 shapes: constants vary within a shape
    r, msg, src = pk.compile_summaries(s, want_source=True)
    assert r > 0, msg
    bodies = _shape_bodies(src)
    assert bodies and all("launch_limits_rec" not in b for b in bodies.values())
    assert src.count("launch_limits_rec(r)") >= 1
    assert "__ldg(K +" not in src  # no scalar 64-bit constant loads left
    varying = [b for b in bodies.values() if "kv[" in b]
    assert varying and all("reinterpret_cast<const int4*>(K)" in b for b in varying)


def test_contradictory_preconditions_compile(pk):
    """a kernel whose pre/glob box is empty (N in [5, 3])
    verifies (every record fails a check -> code 7/8 before any address); the
    generator must route it to the table path instead of emitting specialised
    code from variable signs it never computed."""
    k = golden.relu(0)
    k["pre"] = [p for p in k["pre"] if p["op"] != "N"] + [{"op": "N", "lo": 5, "hi": 3}]
    s = {"version": 1, "kernels": [k, golden.vector_add(1)]}
    assert pk.verify_summaries(s)[0] == 2
    r, msg, src = pk.compile_summaries(s, want_source=True)
    assert r == 1, msg  # one specialised shape (vectorAdd); relu takes the table path
    # the same kernel alone (no specialised kernel in the module at all)
    r, msg, _ = pk.compile_summaries({"version": 1, "kernels": [k]}, want_source=True)
    assert r == 0, msg
