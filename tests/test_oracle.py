"""Pin the oracle: the C restatement (oracle/femoracle.c) vs the reference.

The golden fixtures were produced by the reference itself (femopt built from
/root/reference in oracle/_ref/): its optimized emitted C (``A``, and
``A_tensor``/``A_unbounded`` for other femopt plans) and its interpreter on the
raw IR (``A_interp``; proj/src/interp.cpp:125-154).  The port must agree with
all of them; CPU only.
"""
import json
import os

import numpy as np
import pytest

import port
from paper_1604_05872_b200 import fe, ir

CONFIGS = ["c1", "c2", "c3", "c4", "c5"]


def frob_rel(A, R):
    A = np.asarray(A).reshape(len(A), -1)
    R = np.asarray(R).reshape(len(R), -1)
    return float(np.max(np.linalg.norm(A - R, axis=1) / np.linalg.norm(R, axis=1)))


def load(golden_dir, name):
    z = np.load(os.path.join(golden_dir, f"{name}.npz"))
    tabs = fe.Tables(X=z["X"], W=z["W"], B=z["B"], D=z["D"], P=z["P"])
    with open(os.path.join(golden_dir, f"{name}.json")) as f:
        meta = json.load(f)
    return z, tabs, meta


@pytest.mark.parametrize("name", CONFIGS)
def test_port_matches_reference_golden(name, golden_dir):
    z, tabs, meta = load(golden_dir, name)
    cfg = fe.CONFIGS[name]
    A = port.assemble(cfg, tabs, z["coords"], z["coeffs"])
    assert frob_rel(A, z["A"]) < 1e-13
    assert frob_rel(A[: len(z["A_interp"])], z["A_interp"]) < 1e-13
    # the reference's own emitted-vs-interpreter agreement recorded at generation
    assert meta["emitted_vs_interp_frob_rel"] < 1e-13


@pytest.mark.parametrize("name", CONFIGS)
def test_golden_inputs_are_the_configs(name, golden_dir):
    """Fixture inputs equal the front end's seeded inputs (same generator)."""
    z, tabs, _ = load(golden_dir, name)
    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg, ncells=z["coords"].shape[0])
    assert np.array_equal(coords, z["coords"])
    assert np.array_equal(coeffs, z["coeffs"])
    t = fe.tables(cfg)
    for k in ("W", "B", "D", "P"):
        assert np.allclose(getattr(t, k), z[k], rtol=0, atol=1e-14)


def test_flop_counts_recorded(golden_dir):
    """femopt's flop counts (F_alg ingredients) for the fixture kernels."""
    for name in CONFIGS:
        _, _, meta = load(golden_dir, name)
        for plan, p in meta["plans"].items():
            assert 0 < p["flops_per_cell"] <= p["flops_raw_per_cell"]


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(port.HERE), "oracle", "_ref",
                                                    "libfemopt_ref.so")),
                    reason="reference oracle not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_port_vs_live_reference_interpreter(name):
    import refbridge as rb

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=2, shard=3)
    blocks = {o: rb.interpret(ir.dumps(k), o) for o, k in ir.build(cfg, coords, coeffs, tabs)}
    R = ir.assemble_blocks(cfg, blocks, 2)
    assert frob_rel(port.assemble(cfg, tabs, coords, coeffs), R) < 1e-13


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(port.HERE), "oracle", "_ref",
                                                    "libfemopt_ref.so")),
                    reason="reference oracle not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c5"])
def test_vector_port_vs_live_reference_interpreter(name):
    # the element-vector oracle (port.assemble_vector) against the reference's own
    # interpreter (interp.cpp:125-154) on the arity-1 IR of the same form
    import refbridge as rb

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=3, shard=5)
    oname, k = ir.build_vector(cfg, coords, coeffs, tabs)
    R = np.asarray(rb.interpret(ir.dumps(k), oname)).reshape(3, -1)
    V = port.assemble_vector(cfg, tabs, coords, coeffs)
    assert V.shape == R.shape
    assert frob_rel(V, R) < 1e-13


def test_reference_acceptance_suite():
    """The reference's own acceptance binary (proj/tests/acceptance.cpp) passes."""
    import subprocess

    exe = os.path.join(os.path.dirname(port.HERE), "oracle", "_ref", "acceptance")
    if not os.path.exists(exe):
        pytest.skip("reference acceptance binary not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0
    assert out.stdout.count("PASS") == 10
