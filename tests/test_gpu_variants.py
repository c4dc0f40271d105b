"""GPU parity beyond the five BASELINE configs: the other element/quadrature
shapes the kernels are instantiated for, and the schedule-selection contract.
All through the C ABI, checked against the C oracle (tests/test_oracle.py pins
the oracle to the reference)."""
from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

TOL = 1e-12


def frob_rel(A, R):
    A = np.asarray(A).reshape(len(A), -1)
    R = np.asarray(R).reshape(len(R), -1)
    return float(np.max(np.linalg.norm(A - R, axis=1) / np.linalg.norm(R, axis=1)))


def run(cfg, E=257, schedule=femgpu.SCHED_AUTO):
    import port

    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    form = femgpu.Form.from_config(cfg, tabs, schedule=schedule)
    dev = torch.device("cuda:0")
    out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    form.assemble(torch.from_numpy(coords).to(dev), torch.from_numpy(coeffs).to(dev), out)
    torch.cuda.synchronize()
    return form, out.cpu().numpy(), port.assemble(cfg, tabs, coords, coeffs)


VARIANTS = {
    # Helmholtz P2 with a P2 coefficient (tensor kernel <10,10>), exact degree 6
    "helm_p2_p2": replace(fe.CONFIGS["c2"], name="helm_p2_p2", degree=2, quad_degree=6, N=4,
                          coef_degree=2, coef_ranges=(("f", 10, 1, 0.5, 1.5, 11),)),
    # Helmholtz P2 with a P1 coefficient (tensor kernel <10,4>)
    "helm_p2_p1": replace(fe.CONFIGS["c2"], name="helm_p2_p1", degree=2, quad_degree=5, N=4,
                          coef_degree=1, coef_ranges=(("f", 4, 1, 0.5, 1.5, 11),)),
    # elasticity with the degree-5 rule (pair kernel, Q = 27)
    "elas_q27": replace(fe.CONFIGS["c3"], name="elas_q27", quad_degree=5, N=4),
    # St Venant-Kirchhoff with the degree-3 rule (pair kernel, Q = 8)
    "svk_q8": replace(fe.CONFIGS["c4"], name="svk_q8", quad_degree=3, N=4),
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_parity(name):
    cfg = VARIANTS[name]
    form, A, R = run(cfg)
    assert frob_rel(A, R) < TOL
    assert np.abs(A - A.transpose(0, 2, 1)).max() <= 1e-13 * np.abs(A).max()


def test_elasticity_tensor_accumulate_and_ragged():
    import port

    cfg = fe.CONFIGS["c3"]
    tabs = fe.tables(cfg)
    form = femgpu.Form.from_config(cfg, tabs, schedule=femgpu.SCHED_TENSOR)
    dev = torch.device("cuda:0")
    for E in (1, 4, 6, 11, 37):
        coords, coeffs = fe.cell_inputs(cfg, ncells=E)
        R = port.assemble(cfg, tabs, coords, coeffs)
        x = torch.from_numpy(coords).to(dev)
        c = torch.from_numpy(coeffs).to(dev)
        out = torch.full((E, cfg.n, cfg.n), 1.5, dtype=torch.float64, device=dev)
        form.assemble(x, c, out, accumulate=True)
        torch.cuda.synchronize()
        assert frob_rel(out.cpu().numpy() - 1.5, R) < 1e-11


@pytest.mark.parametrize("name", ["c4", "svk_q8"])
def test_svk_tensor_core_quadrature(name):
    # St Venant-Kirchhoff with the sum over points on the DMMA pipe (svk_mma.cu), on
    # request: several 8-cell tiles per CTA (E > 148 x 8) with a ragged last tile,
    # the accumulate contract and ragged small meshes
    import port

    cfg = fe.CONFIGS["c4"] if name == "c4" else VARIANTS[name]
    tabs = fe.tables(cfg)
    form = femgpu.Form.from_config(cfg, tabs, schedule=femgpu.SCHED_QUADRATURE_MMA)
    assert form.info["kernel_name"] == "svk_mma_kernel"
    assert form.info["schedule"] == "quadrature_mma"
    dev = torch.device("cuda:0")
    for E in ((1, 7, 9, 3 * 148 * 8 + 5) if name == "c4" else (1, 13, 383)):
        coords, coeffs = fe.cell_inputs(cfg, ncells=E)
        R = port.assemble(cfg, tabs, coords, coeffs)
        x = torch.from_numpy(coords).to(dev)
        c = torch.from_numpy(coeffs).to(dev)
        out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
        form.assemble(x, c, out)
        torch.cuda.synchronize()
        A = out.cpu().numpy()
        assert frob_rel(A, R) < TOL, E
        assert np.array_equal(A, A.transpose(0, 2, 1))
        out.fill_(1.5)
        form.assemble(x, c, out, accumulate=True)
        torch.cuda.synchronize()
        assert frob_rel(out.cpu().numpy() - 1.5, R) < 1e-11, E


def test_burgers_quadrature_schedule():
    # the Burgers Jacobian in the quadrature schedule (burgers_quad.cu), on request:
    # several passes of the persistent grid (E > 148 x 12), ragged sizes, accumulate
    import port

    cfg = fe.CONFIGS["c5"]
    tabs = fe.tables(cfg)
    form = femgpu.Form.from_config(cfg, tabs, schedule=femgpu.SCHED_QUADRATURE)
    assert form.info["kernel_name"] == "burgers_quad_kernel"
    dev = torch.device("cuda:0")
    for E in (1, 13, 2 * 148 * 12 + 7):
        coords, coeffs = fe.cell_inputs(cfg, ncells=E)
        R = port.assemble(cfg, tabs, coords, coeffs)
        x = torch.from_numpy(coords).to(dev)
        c = torch.from_numpy(coeffs).to(dev)
        out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
        form.assemble(x, c, out)
        torch.cuda.synchronize()
        assert frob_rel(out.cpu().numpy(), R) < TOL, E
        out.fill_(1.5)
        form.assemble(x, c, out, accumulate=True)
        torch.cuda.synchronize()
        assert frob_rel(out.cpu().numpy() - 1.5, R) < 1e-11, E


def test_schedule_contract():
    # Helmholtz and elasticity have both schedules (AUTO: tensor resp. quadrature,
    # the faster ones, tests/test_schedule.py); St Venant-Kirchhoff only quadrature
    f = femgpu.Form.from_config(fe.CONFIGS["c2"], schedule=femgpu.SCHED_QUADRATURE)
    assert f.info["schedule"] == "quadrature" and f.info["kernel_name"] == "helm_quad_kernel"
    assert femgpu.Form.from_config(fe.CONFIGS["c2"]).info["kernel_name"] == "helm_tensor_kernel"
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.Form.from_config(fe.CONFIGS["c4"], schedule=femgpu.SCHED_TENSOR)
    assert e.value.code == 14
    f = femgpu.Form.from_config(fe.CONFIGS["c2"], schedule=femgpu.SCHED_TENSOR)
    assert f.info["schedule"] == "tensor"
    f = femgpu.Form.from_config(fe.CONFIGS["c4"], schedule=femgpu.SCHED_QUADRATURE)
    assert f.info["schedule"] == "quadrature" and f.info["kernel_name"] == "pair_svk_ws_kernel"
    f = femgpu.Form.from_config(fe.CONFIGS["c4"], schedule=femgpu.SCHED_QUADRATURE_MMA)
    assert f.info["schedule"] == "quadrature_mma" and f.info["kernel_name"] == "svk_mma_kernel"
    with pytest.raises(femgpu.FemgpuError):
        femgpu.Form.from_config(fe.CONFIGS["c2"], schedule=femgpu.SCHED_QUADRATURE_MMA)
    f = femgpu.Form.from_config(fe.CONFIGS["c3"])
    assert f.info["schedule"] == "quadrature"
    f = femgpu.Form.from_config(fe.CONFIGS["c3"], schedule=femgpu.SCHED_TENSOR)
    assert f.info["schedule"] == "tensor" and f.info["kernel_name"] == "elas_tensor_kernel"


@pytest.mark.parametrize("name", ["c3", "elas_q27"])
def test_elasticity_tensor_schedule(name):
    # the DMMA pre-evaluated kernel (elasticity.cu), on request
    cfg = fe.CONFIGS["c3"] if name == "c3" else VARIANTS[name]
    cfg = replace(cfg, N=4)
    form, A, R = run(cfg, schedule=femgpu.SCHED_TENSOR)
    assert form.info["kernel_name"] == "elas_tensor_kernel"
    assert frob_rel(A, R) < TOL
    assert np.abs(A - A.transpose(0, 2, 1)).max() <= 1e-13 * np.abs(A).max()


def test_unsupported_shapes_fail_loudly():
    # P3 Helmholtz with a P2 coefficient has no tensor-kernel instantiation: TENSOR
    # fails loudly, AUTO takes the quadrature kernel (any coefficient degree)
    cfg = replace(fe.CONFIGS["c2"], N=3, coef_degree=2, coef_ranges=(("f", 10, 1, 0.5, 1.5, 11),))
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.Form.from_config(cfg, schedule=femgpu.SCHED_TENSOR)
    assert e.value.code == 14
    form, A, R = run(cfg, E=97)
    assert form.info["kernel_name"] == "helm_quad_kernel"
    assert frob_rel(A, R) < TOL
    # no vector-form kernel for P1 vector elements (ns = 4)
    cfg = replace(fe.CONFIGS["c3"], degree=1)
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.Form.from_config(cfg)
    assert e.value.code == 14
    # inconsistent table shapes: elasticity needs P1 mu/lambda (nc == 4)
    t = fe.tables(fe.CONFIGS["c3"])
    bad = fe.Tables(X=t.X, W=t.W, B=t.B, D=t.D, P=t.B)
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.Form(fe.ELASTICITY, bad)
    assert e.value.code == 8
    # Burgers needs dt != 0
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.Form(fe.BURGERS, fe.tables(fe.CONFIGS["c5"]), consts=(0.01, 0.0))
    assert e.value.code == 9


def test_misaligned_device_pointer_rejected():
    cfg = fe.CONFIGS["c1"]
    form = femgpu.Form.from_config(cfg)
    dev = torch.device("cuda:0")
    buf = torch.zeros(4096, dtype=torch.float64, device=dev)
    with pytest.raises(femgpu.FemgpuError) as e:
        form.assemble(buf.data_ptr() + 8, buf.data_ptr(), buf.data_ptr(), ncells=4)
    assert e.value.code == 9
