"""C-ABI library: loads, exports every declared symbol, and the loader's
verification accepts/rejects summaries as specified.  CPU only
(no compute calls)."""
import copy
import json
import os
import re

import pytest

from tracegen import golden
from tracegen.synth import random_summary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


def test_exports_every_declared_symbol(pk):
    from paper_2410_23661_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "picker.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(picker_\w+)\(", hdr, re.M))
    assert {"picker_create", "picker_load_summaries", "picker_validate_batch",
            "picker_exact_check", "picker_destroy", "picker_last_error"} <= declared
    for name in declared:
        assert hasattr(_lib.lib, name), name
        assert name in _lib.SIGNATURES, name


def test_golden_verifies(pk):
    n, msg = pk.verify_summaries(golden.golden_summary())
    assert n == 10, msg


@pytest.mark.parametrize("seed", range(6))
def test_random_summaries_verify(pk, seed):
    s = random_summary(seed, n_kernels=24)
    n, msg = pk.verify_summaries(s)
    assert n == 24, msg


def _relu():
    return {"version": 1, "kernels": [golden.relu(0)]}


def _mut(f):
    s = _relu()
    f(s["kernels"][0])
    return s


EUNSAFE, EFORMAT = -3, -2


@pytest.mark.parametrize("name,mut,status", [
    ("no pointer precondition", lambda k: k.update(pre=[p for p in k["pre"] if p["op"] != "A"]), EUNSAFE),
    ("unbounded i64 factor", lambda k: (k["params"].append({"name": "M", "kind": "i64"}),
                                        k["desc"][0]["terms"].append({"k": 1, "f": ["M"], "var": "tid.x"})), EUNSAFE),
    ("possible overflow", lambda k: k["desc"][0]["terms"].append(
        {"k": 1 << 40, "f": ["N", "bdim.x"], "var": "bid.x"}), EUNSAFE),
    ("mixed signs on one variable", lambda k: k["desc"][0]["terms"].append(
        {"k": -1, "f": [], "var": "tid.x"}), EUNSAFE),
    ("IDEM kernel that reads", lambda k: k.update({"class": "IDEM"}), EUNSAFE),
    ("fresh range misses its definition", lambda k: k["desc"][0]["vars"].update(
        {"fr0": {"lo": [{"k0": 0, "p": []}], "hi": [{"k0": 3, "p": []}], "def": {"src": "tid.x", "mod": 10}}}),
     EUNSAFE),
    ("unknown operand", lambda k: k["desc"][0]["terms"].append({"k": 1, "f": ["Q"], "var": None}), EFORMAT),
    ("gidx and tid on one axis", lambda k: k["desc"][0]["vars"].update({"gidx.x": {"lo": [], "hi": []}}), EFORMAT),
    ("undeclared term variable", lambda k: k["desc"][0]["terms"].append({"k": 1, "f": [], "var": "ind3"}), EFORMAT),
    ("induction without bounds", lambda k: k["desc"][0]["vars"].update({"ind1": {"lo": [], "hi": []}}), EFORMAT),
    ("bad width", lambda k: k["desc"][0].update(width=0), EFORMAT),
    ("bad kind", lambda k: k["desc"][0].update(kind="X"), EFORMAT),
    ("unknown reason", lambda k: k.update({"class": "NONIDEM", "reason": "ZZ"}), EFORMAT),
    ("literal outside int64", lambda k: k["pre"].append({"op": "N", "lo": 0, "hi": 1 << 64}), EFORMAT),
])
def test_loader_rejects(pk, name, mut, status):
    s = _mut(mut)
    r, msg = pk.verify_summaries(s)
    assert r == status, (name, r, msg)
    assert msg


def test_loader_accepts_single_term_of_unknown_sign(pk):
    """One term of either sign on a variable is still exact at the endpoints."""
    s = _mut(lambda k: (k["pre"].append({"op": "N", "lo": -4, "hi": 20}),
                        k["desc"][0]["terms"].__setitem__(0, {"k": 4, "f": ["bdim.x", "N"], "var": "bid.x"})))
    k = s["kernels"][0]
    k["pre"] = [p for p in k["pre"] if not (p["op"] == "N" and p["lo"] == 0)]
    r, msg = pk.verify_summaries(s)
    # bid.x carries one N-scaled term (sign unknown) -> accepted; tid.x carries
    # 4*N as well, alone -> accepted.
    assert r == 1, msg


def test_bad_json(pk):
    for t in [b"", b"{", b'{"kernels": [1.5]}', b'{"kernels": [}', b"[]", b'{"version": 2, "kernels": []}']:
        r, msg = pk.verify_summaries(t)
        assert r == EFORMAT, (t, r, msg)


def test_duplicate_kernel_id(pk):
    s = {"version": 1, "kernels": [golden.relu(3), golden.vector_add(3)]}
    assert pk.verify_summaries(s)[0] == EFORMAT


def test_empty_summary(pk):
    assert pk.verify_summaries({"version": 1, "kernels": []})[0] == 0
