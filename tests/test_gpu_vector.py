"""Element vectors (femgpu_assemble_vector, csrc/vector.cu) against the numpy oracle
port.assemble_vector, which tests/test_oracle.py pins to the reference's own
interpreter (interp.cpp:125-154) on the arity-1 IR of each form."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1604_05872_b200 import fe, femgpu, ir  # noqa: E402

TOL = 1e-12  # Frobenius-relative per element vector (FP64, summation order differs)
VECTOR_CONFIGS = ["c1", "c2", "c4", "c5"]


def frob_rel(A, R):
    A = np.asarray(A).reshape(len(A), -1)
    R = np.asarray(R).reshape(len(R), -1)
    return float(np.max(np.linalg.norm(A - R, axis=1) / np.linalg.norm(R, axis=1)))


def _run(form, cfg, coords, coeffs, out=None, accumulate=False):
    dev = torch.device("cuda:0")
    E = coords.shape[0]
    if out is None:
        out = torch.empty((E, cfg.n), dtype=torch.float64, device=dev)
    form.assemble_vector(torch.from_numpy(coords).to(dev), torch.from_numpy(coeffs).to(dev), out,
                         accumulate=accumulate)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("name", VECTOR_CONFIGS)
@pytest.mark.parametrize("ncells", [1, 31, 301])
def test_vector_parity(name, ncells):
    import port

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=ncells, shard=2)
    form = femgpu.Form.from_config(cfg, tabs)
    out = _run(form, cfg, coords, coeffs)
    assert frob_rel(out.cpu().numpy(), port.assemble_vector(cfg, tabs, coords, coeffs)) < TOL


@pytest.mark.parametrize("name", VECTOR_CONFIGS)
def test_vector_accumulate(name):
    import port

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=133)
    form = femgpu.Form.from_config(cfg, tabs)
    R = port.assemble_vector(cfg, tabs, coords, coeffs)
    # prior contents of the size of the result (the += contract of emit_c.cpp:129)
    base = np.random.default_rng(3).uniform(-1, 1, R.shape) * np.abs(R).max(axis=1, keepdims=True)
    out = torch.from_numpy(base.copy()).to("cuda:0")
    out = _run(form, cfg, coords, coeffs, out=out, accumulate=True)
    assert frob_rel(out.cpu().numpy(), base + R) < TOL


@pytest.mark.parametrize("name", VECTOR_CONFIGS)
def test_vector_matches_generic_ir_backend(name):
    # the same arity-1 form through the generic backend (bit-identical to femopt's
    # emitted C on the golden IRs)
    from paper_1604_05872_b200 import emit_cuda

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=77, shard=1)
    oname, k = ir.build_vector(cfg, coords, coeffs, tabs)
    G = emit_cuda.IRKernel(k).run_ir_tables(k)[oname].reshape(77, -1)
    form = femgpu.Form.from_config(cfg, tabs)
    out = _run(form, cfg, coords, coeffs)
    assert frob_rel(out.cpu().numpy(), G) < TOL


@pytest.mark.parametrize("name", VECTOR_CONFIGS)
def test_vector_full_mesh_sampled(name):
    # BASELINE mesh size: sampled cells against the oracle; Helmholtz: linear in f
    import port

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg)
    E = coords.shape[0]
    form = femgpu.Form.from_config(cfg, tabs)
    out = _run(form, cfg, coords, coeffs).cpu().numpy()
    idx = np.r_[0:5, E // 3, E // 2, E - 131:E]
    assert frob_rel(out[idx], port.assemble_vector(cfg, tabs, coords[idx], coeffs[idx])) < TOL
    if cfg.kind == fe.HELMHOLTZ:
        out2 = _run(form, cfg, coords, 2.0 * coeffs + 1.0).cpu().numpy()
        ones = _run(form, cfg, coords, np.ones_like(coeffs)).cpu().numpy()
        assert frob_rel(out2, 2.0 * out + ones) < TOL


def test_vector_zero_states():
    # w = 0: F = I, E = 0, S = 0 -> r = 0; u = 0 -> Burgers r = 0 (exactly)
    for name, zero in (("c4", slice(0, 30)), ("c5", slice(0, 60))):
        cfg = fe.CONFIGS[name]
        coords, coeffs = fe.cell_inputs(cfg, ncells=40)
        coeffs = coeffs.copy()
        coeffs[:, zero] = 0.0
        form = femgpu.Form.from_config(cfg)
        out = _run(form, cfg, coords, coeffs).cpu().numpy()
        assert np.all(out == 0.0), name


def test_vector_unsupported_and_empty():
    cfg = fe.CONFIGS["c3"]
    form = femgpu.Form.from_config(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=4)
    with pytest.raises(femgpu.FemgpuError):
        _run(form, cfg, coords, coeffs)
    cfg = fe.CONFIGS["c4"]
    form = femgpu.Form.from_config(cfg)
    dev = torch.device("cuda:0")
    out = torch.full((4, cfg.n), 7.0, dtype=torch.float64, device=dev)
    x = torch.zeros((4, 12), dtype=torch.float64, device=dev)
    c = torch.zeros((4, cfg.ncoef), dtype=torch.float64, device=dev)
    form.assemble_vector(x, c, out, ncells=0)
    torch.cuda.synchronize()
    assert bool((out == 7.0).all())
