"""The reference's own kernel corpus through the generic IR backend (femgpu_ir_*).

Fixtures: tests/golden/corpus/<name>_<raw|opt>.{json,npz}, made by
oracle/make_corpus.py from the reference itself -- every kernel of
corpus::all_json() (/root/reference/proj/tests/kernels.hpp:321-342: poisson,
fig2, mass, helmholtz, elastic, interp*, padded*, linear, divsigma, callsigma,
noreduction, twostmt, imperfect, ...) and plan_kernel_json(0..19) (:348-363),
raw and femopt-optimized with the reference's default options, with the
outputs of femopt's emitted C (``emitc_*``) and of its interpreter on the raw
kernel (``interp_*``).

The bar is the reference's own (test_backend.cpp:167-182, comparator :22-35,
max |a-b| / max(|a|, |b|, 1)): raw emission within 1e-12 of the interpreter,
optimized emission within 1e-10 -- and, stronger, the GPU output bit-identical
to femopt's emitted C of the same IR (same printed arithmetic, no contraction).
"""
import glob
import json
import os

import numpy as np
import pytest

from paper_1604_05872_b200 import emit_cuda

GOLD = os.path.join(os.path.dirname(__file__), "golden", "corpus")
CASES = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLD, "*.json")))
REF_NAMES = ("poisson", "poisson_small", "fig2", "mass", "mass_big", "helmholtz", "elastic",
             "interp6", "interp2", "interp2mix", "padded", "padded_e", "linear", "divsigma",
             "callsigma", "noreduction", "twostmt", "imperfect")


def load(case):
    with open(os.path.join(GOLD, case + ".json")) as f:
        js = f.read()
    return js, json.loads(js), np.load(os.path.join(GOLD, case + ".npz"))


def worst_error(a, b):
    """test_backend.cpp:22-35."""
    a, b = np.asarray(a).reshape(-1), np.asarray(b).reshape(-1)
    assert a.shape == b.shape
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))


def test_corpus_complete():
    names = {c.rsplit("_", 1)[0] for c in CASES}
    assert set(REF_NAMES) <= names
    assert {f"plan{v}" for v in range(20)} <= names
    assert all(f"{n}_raw" in CASES and f"{n}_opt" in CASES for n in names)


@pytest.mark.parametrize("case", CASES)
def test_corpus_generates_and_compiles(case):
    """femgpu_ir_create parses, generates and NVRTC-compiles every corpus kernel
    (no GPU needed); the argument lists are emit_c's (emit_c.cpp:137-140)."""
    js, d, _ = load(case)
    K = emit_cuda.IRKernel(js)
    tabs = d["tables"]
    assert K.outputs == sorted(d["outputs"])
    assert K.inputs == sorted(n for n, t in tabs.items()
                              if t.get("provenance", "input") != "preevaluated")
    assert K.constants == sorted((d.get("constants") or {}).keys())
    assert "fma(" not in K.source


def _strategies(case):
    js, _, _ = load(case)
    out = ["thread"]
    try:
        emit_cuda.IRKernel(js, strategy="warp")
        out.append("warp")
    except emit_cuda.IRError:
        pass
    return out


STRATS = [(c, s) for c in CASES for s in _strategies(c)]


@pytest.mark.gpu
@pytest.mark.parametrize("case,strategy", STRATS)
def test_corpus_on_gpu(case, strategy):
    pytest.importorskip("torch")
    js, d, z = load(case)
    K = emit_cuda.IRKernel(js, strategy=strategy)
    got = K.run_ir_tables(d)
    tol = 1e-12 if case.endswith("_raw") else 1e-10
    for o in d["outputs"]:
        g = got[o].reshape(-1)
        assert np.array_equal(g, z[f"emitc_{o}"].reshape(-1)), \
            f"{case}/{o} ({strategy}): not bit-identical to femopt's emitted C"
        assert worst_error(g, z[f"interp_{o}"]) < tol
