"""The generic femopt-IR -> CUDA backend (paper_1604_05872_b200/emit_cuda.py).

Parity reference: tests/golden/ir/<case>.{json,npz} -- the kernel IR (raw, or
femopt-optimized) and femopt's own outputs on it: its emitted C compiled with
-ffp-contract=off (``emitc_*``) and its interpreter (``interp_*``), made by
oracle/make_ir_golden.py.  The generated kernels follow emit_c's statement and
operand order and are compiled without FMA contraction, so they must agree
with femopt's emitted C bit for bit.
"""
import glob
import json
import os

import numpy as np
import pytest

from paper_1604_05872_b200 import emit_cuda, fe, ir

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ir")
CASES = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLD, "*.json")))


def load(case):
    with open(os.path.join(GOLD, case + ".json")) as f:
        js = f.read()
    return js, json.loads(js), np.load(os.path.join(GOLD, case + ".npz"))


def test_fixtures_present():
    assert len(CASES) >= 10
    for kind in ("matrix", "load", "residual", "block"):
        assert any(f"_{kind}" in c for c in CASES), kind


@pytest.mark.parametrize("case", CASES)
def test_generate_and_nvrtc_compile(case):
    # femgpu_ir_create parses, generates and NVRTC-compiles for sm_100a: no GPU needed
    js, d, _ = load(case)
    K = emit_cuda.IRKernel(js)
    tabs = d["tables"]
    assert K.outputs == sorted(d["outputs"])
    assert K.inputs == sorted(n for n, t in tabs.items()
                              if t.get("provenance", "input") != "preevaluated")
    assert K.constants == sorted((d.get("constants") or {}).keys())
    assert K.per_cell
    src = K.source
    for n in tabs:
        if tabs[n].get("provenance") == "preevaluated":
            assert f"__device__ const double t_{n}[" in src
    assert "fma(" not in src  # the emitted arithmetic only


def test_bad_ir_is_rejected():
    cfg = fe.CONFIGS["c1"]
    coords, coeffs = fe.cell_inputs(cfg, ncells=2)
    k = ir.build(cfg, coords, coeffs)[0][1]
    bad = json.loads(ir.dumps(k))
    bad["statements"][-1]["rhs"] = ["*", "nosuchscalar", 1.0]
    with pytest.raises(emit_cuda.IRError):
        emit_cuda.IRKernel(bad)
    bad = json.loads(ir.dumps(k))
    bad["statements"][-1]["rhs"] = ["call", "system", 1.0]
    with pytest.raises(emit_cuda.IRError):
        emit_cuda.IRKernel(bad)
    with pytest.raises(emit_cuda.IRError):
        emit_cuda.IRKernel('{"indices": {"e": 2}, "loops": [')


# ----------------------------------------------------------------------------
# on the GPU
# ----------------------------------------------------------------------------
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


def test_warp_mapping_applies_to_the_larger_nests():
    assert sum(s == "warp" for _, s in STRATS) >= 8


@pytest.mark.gpu
@pytest.mark.parametrize("case,strategy", STRATS)
def test_matches_femopt_emitted_c(case, strategy):
    pytest.importorskip("torch")
    js, d, z = load(case)
    K = emit_cuda.IRKernel(js, strategy=strategy)
    got = K.run_ir_tables(d)
    for o in d["outputs"]:
        ref_c = z[f"emitc_{o}"].reshape(-1)
        ref_i = z[f"interp_{o}"].reshape(-1)
        g = got[o].reshape(-1)
        scale = np.abs(ref_i).max()
        assert np.abs(g - ref_i).max() <= 1e-13 * scale
        assert np.array_equal(g, ref_c), \
            f"{case}/{o} ({strategy}): not bit-identical to femopt's emitted C"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
def test_generic_backend_matches_fast_path(name):
    # the raw femopt IR of a BASELINE form, compiled by emit_cuda, against the
    # hand-written kernel on the same cells
    torch = pytest.importorskip("torch")
    from paper_1604_05872_b200 import femgpu

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    E = 777
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    k = ir.build(cfg, coords, coeffs, tabs=tabs)[0][1]
    got = emit_cuda.IRKernel(k).run_ir_tables(k)["A"].reshape(E, cfg.n, cfg.n)
    dev = torch.device("cuda:0")
    out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    femgpu.Form.from_config(cfg, tabs).assemble(torch.from_numpy(coords).to(dev),
                                                torch.from_numpy(coeffs).to(dev), out)
    torch.cuda.synchronize()
    A = out.cpu().numpy()
    rel = np.linalg.norm((got - A).reshape(E, -1), axis=1) / np.linalg.norm(A.reshape(E, -1), axis=1)
    assert rel.max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c4", "c5"])
def test_residual_derivative_is_the_jacobian(name):
    # d r / d u (central differences of the arity-1 residual kernel, generic
    # backend) against the arity-2 Jacobian of the fast path
    torch = pytest.importorskip("torch")
    from paper_1604_05872_b200 import femgpu

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    E = 6
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    nd = 3 * cfg.ns  # unknown dofs: w (c4) or u (c5), component-blocked
    rng = np.random.default_rng(3)
    delta = rng.uniform(-1, 1, size=(E, nd))
    eps = 1e-6 if name == "c4" else 1e-5

    def residual(cf):
        oname, k = ir.build_vector(cfg, coords, cf, tabs)
        return emit_cuda.IRKernel(k).run_ir_tables(k)[oname].reshape(E, nd)

    cp, cm = coeffs.copy(), coeffs.copy()
    cp[:, :nd] += eps * delta
    cm[:, :nd] -= eps * delta
    fd = (residual(cp) - residual(cm)) / (2 * eps)
    dev = torch.device("cuda:0")
    out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    femgpu.Form.from_config(cfg, tabs).assemble(torch.from_numpy(coords).to(dev),
                                                torch.from_numpy(coeffs).to(dev), out)
    torch.cuda.synchronize()
    Jd = np.einsum("ejk,ek->ej", out.cpu().numpy(), delta)
    rel = np.linalg.norm(fd - Jd, axis=1) / np.linalg.norm(Jd, axis=1)
    assert rel.max() < 1e-7, rel


# ----------------------------------------------------------------------------
# femopt's own optimized kernels of the BASELINE configs (oracle/make_ir_full.py)
IR_FULL = os.path.join(os.path.dirname(__file__), "golden", "ir_full")
FULL_CASES = sorted(f[:-len(".json.gz")] for f in os.listdir(IR_FULL)) if os.path.isdir(IR_FULL) else []


def _load_full(case):
    import gzip

    with gzip.open(os.path.join(IR_FULL, case + ".json.gz"), "rt") as f:
        return json.load(f)


def test_full_config_ir_fixtures():
    # every config has femopt's optimized kernels for each reference-arm plan
    assert {c.split("_")[0] for c in FULL_CASES} >= {"c1", "c2", "c3", "c4", "c5"}
    for case in FULL_CASES:
        d = _load_full(case)
        cfg = fe.CONFIGS[d["config"]]
        outs = [k["output"] for k in d["kernels"]]
        assert outs == (["A"] if cfg.kind != fe.BURGERS else
                        [f"A{c}{e}" for c in range(3) for e in range(3)])
        for k in d["kernels"]:
            assert k["flops_per_cell"] <= k["flops_raw_per_cell"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", FULL_CASES)
def test_femopt_optimized_kernel_on_gpu_matches_fast_path(case):
    # femopt's optimized kernel of a BASELINE config, run by the generic backend
    # on fresh cells (e-tables at run time), against the hand-written kernel
    torch = pytest.importorskip("torch")
    from paper_1604_05872_b200 import femgpu

    d = _load_full(case)
    cfg = fe.CONFIGS[d["config"]]
    E = 333
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    dev = torch.device("cuda:0")
    et = {k: torch.from_numpy(v).to(dev) for k, v in ir.e_tables(cfg, coords, coeffs).items()}
    got = np.zeros((E, cfg.n, cfg.n))
    for kk in d["kernels"]:
        k = kk["ir"]
        K = emit_cuda.IRKernel(k)
        inputs = {n: et[n] if n in et else torch.tensor(np.asarray(k["tables"][n]["values"]),
                                                        device=dev) for n in K.inputs}
        (o,) = K.outputs
        out = torch.zeros(K.size(0, o, E), dtype=torch.float64, device=dev)
        K.run({o: out}, inputs, k.get("constants", {}), E)
        blk = out.cpu().numpy()
        if o == "A":
            got[:] = blk.reshape(E, cfg.n, cfg.n)
        else:
            c, e, ns = int(o[1]), int(o[2]), cfg.ns
            got[:, c * ns:(c + 1) * ns, e * ns:(e + 1) * ns] = blk.reshape(E, ns, ns)
    ref = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    femgpu.Form.from_config(cfg).assemble(torch.from_numpy(coords).to(dev),
                                          torch.from_numpy(coeffs).to(dev), ref)
    A = ref.cpu().numpy()
    rel = np.linalg.norm((got - A).reshape(E, -1), axis=1) / np.linalg.norm(A.reshape(E, -1), axis=1)
    assert rel.max() < 1e-12


# ----------------------------------------------------------------------------
# GEMM mapping of femopt's pre-evaluated (tensor) nests
# ----------------------------------------------------------------------------
def _gemm_ok(js):
    try:
        emit_cuda.IRKernel(js, strategy="gemm")
        return True
    except emit_cuda.IRError:
        return False


GEMM_CASES = [c for c in CASES if _gemm_ok(load(c)[0])]


def test_gemm_mapping_applies_to_tensor_plans():
    # femopt's G-factored (fully pre-evaluated) plans are GEMM-shaped; raw nests are not
    assert any("gfac_opt" in c for c in GEMM_CASES)
    assert not any(c.endswith("_raw") for c in GEMM_CASES)
    for case in FULL_CASES:
        d = _load_full(case)
        strat = [emit_cuda.IRKernel(k["ir"]).strategy for k in d["kernels"]]
        if case in ("c2_tensor",):
            assert strat == ["gemm"]
        if case == "c5_unbounded":
            assert "gemm" in strat


@pytest.mark.gpu
@pytest.mark.parametrize("case", GEMM_CASES)
def test_gemm_mapping_matches_emitted_c(case):
    pytest.importorskip("torch")
    js, d, z = load(case)
    got = emit_cuda.IRKernel(js, strategy="gemm").run_ir_tables(d)
    for o in d["outputs"]:
        ref = z[f"emitc_{o}"]
        g = got[o].reshape(ref.shape)
        E = int(d["indices"]["e"])
        G, R = g.reshape(E, -1), ref.reshape(E, -1)
        rel = np.linalg.norm(G - R, axis=1) / np.linalg.norm(R, axis=1)
        assert rel.max() < 1e-12, rel.max()


@pytest.mark.gpu
def test_gemm_mapping_chunks_on_the_full_tensor_plan():
    # femopt's P3 Helmholtz tensor plan (200 pre-evaluated tables of 20x20) through the
    # GEMM mapping on more cells than one chunk (2^17), against the hand-written kernel
    torch = pytest.importorskip("torch")
    from paper_1604_05872_b200 import femgpu

    d = _load_full("c2_tensor")
    cfg = fe.CONFIGS["c2"]
    E = (1 << 17) + 77
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    dev = torch.device("cuda:0")
    et = {k: torch.from_numpy(v).to(dev) for k, v in ir.e_tables(cfg, coords, coeffs).items()}
    k = d["kernels"][0]["ir"]
    K = emit_cuda.IRKernel(k)
    assert K.strategy == "gemm"
    inputs = {n: et[n] if n in et else torch.tensor(np.asarray(k["tables"][n]["values"]),
                                                    device=dev) for n in K.inputs}
    out = torch.full((E, cfg.n, cfg.n), 0.25, dtype=torch.float64, device=dev)  # += contract
    K.run({"A": out}, inputs, k.get("constants", {}), E)
    ref = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    femgpu.Form.from_config(cfg).assemble(torch.from_numpy(coords).to(dev),
                                          torch.from_numpy(coeffs).to(dev), ref)
    torch.cuda.synchronize()
    G = (out - 0.25).reshape(E, -1)
    R = ref.reshape(E, -1)
    rel = ((G - R).norm(dim=1) / R.norm(dim=1)).max().item()
    assert rel < 1e-12, rel


def _synthetic_tensor_ir(E=37, nj=6, nk=5, nt=40, seed=3):
    """A femopt-shaped pre-evaluated nest: preheader scalars, then
    OUT[e][j][k] += sum_t T_t * p_t with tables stored [j][k] or [k][j] and products
    of temporaries, constants and numbers."""
    rng = np.random.default_rng(seed)
    tables = {"x0": {"dims": ["e"], "values": list(rng.uniform(0.5, 1.5, E))},
              "x1": {"dims": ["e"], "values": list(rng.uniform(0.5, 1.5, E))}}
    stmts = [{"lhs": ["a"], "op": "=", "rhs": ["*", ["sym", "x0", "e"], ["sym", "x1", "e"]]},
             {"lhs": ["b"], "op": "=", "rhs": ["+", ["sym", "x0", "e"], -0.25]}]
    terms = []
    for t in range(nt):
        name = f"T{t}"
        if t % 3 == 0:  # stored transposed
            tables[name] = {"dims": ["k", "j"], "provenance": "preevaluated",
                            "values": list(rng.uniform(-1, 1, nk * nj))}
            sym = ["sym", name, "k", "j"]
        else:
            tables[name] = {"dims": ["j", "k"], "provenance": "preevaluated",
                            "values": list(rng.uniform(-1, 1, nj * nk))}
            sym = ["sym", name, "j", "k"]
        factors = [sym, "a"] if t % 2 else ["b", sym, "c0", 0.5]
        terms.append(["*", *factors])
    nest = {"loop": {"index": "j", "begin": 0, "end": nj, "body": [
        {"loop": {"index": "k", "begin": 0, "end": nk, "body": [
            {"lhs": ["A", "e", "j", "k"], "op": "+=", "rhs": ["+", *terms]}]}}]}}
    return {"indices": {"e": E, "j": nj, "k": nk}, "tables": tables,
            "constants": {"c0": 1.75}, "outputs": ["A"],
            "body": [{"loop": {"index": "e", "class": "orderfree", "begin": 0, "end": E,
                               "body": stmts + [nest]}}]}


def test_gemm_mapping_detects_transposed_tables():
    d = _synthetic_tensor_ir()
    assert emit_cuda.IRKernel(d, strategy="gemm").strategy == "gemm"
    assert emit_cuda.IRKernel(d).strategy != "gemm"  # 40 x 30 < 2048 multiply-adds: AUTO keeps thread/warp
    bad = json.loads(json.dumps(d))
    bad["body"][0]["loop"]["body"][-1]["loop"]["body"][0]["loop"]["body"][0]["rhs"][1].append(
        ["sym", "x0", "e"])  # an e-table inside the nest: not a pure tensor contraction
    with pytest.raises(emit_cuda.IRError):
        emit_cuda.IRKernel(bad, strategy="gemm")


@pytest.mark.gpu
def test_gemm_mapping_matches_thread_mapping_on_synthetic_plan():
    pytest.importorskip("torch")
    d = _synthetic_tensor_ir(E=301)
    ref = emit_cuda.IRKernel(d, strategy="thread").run_ir_tables(d)["A"].reshape(301, -1)
    got = emit_cuda.IRKernel(d, strategy="gemm").run_ir_tables(d)["A"].reshape(301, -1)
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-13
