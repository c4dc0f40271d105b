"""Schedule choice per form: the library's cost model and the
kernels it chooses between.

femopt picks, per monomial, pre-evaluation (tensor) or sharing elimination
(quadrature) by its own flop counts (theta_pre vs theta_se,
/root/reference/proj/src/cost.cpp:61-116; plan search driver.cpp:47-106).
femgpu ranks every kernel it has for a form by predicted time -- roofline time
of the kernel's flops and bytes on the device divided by the kernel's measured
efficiency -- and AUTO takes the fastest (femgpu_form_schedules).  These tests
check the ranking on CPU and, on the GPU, that the quadrature alternative of
the Helmholtz form (helm_quad_kernel) meets the parity bar and that the AUTO
choice is the faster kernel measured on the BASELINE meshes.
"""
import numpy as np
import pytest

from paper_1604_05872_b200 import fe, femgpu

TOL = 1e-12
EXPECT = {"c1": "helm_p1_kernel", "c2": "helm_tensor_kernel", "c3": "pair_ws_kernel",
          "c4": "pair_svk_ws_kernel", "c5": "burgers_kernel"}


@pytest.mark.parametrize("name", sorted(EXPECT))
def test_auto_ranking(name):
    r = femgpu.schedules(fe.CONFIGS[name])
    assert r and sum(x["chosen"] for x in r) == 1
    assert r[0]["chosen"] and r[0]["kernel"] == EXPECT[name]
    t = [x["predicted_ns_per_cell"] for x in r]
    assert t == sorted(t)
    for x in r:
        roof = max(x["flops_per_cell"] / x["peak_flops"], x["bytes_per_cell"] / x["peak_bytes"])
        assert x["predicted_ns_per_cell"] == pytest.approx(roof / x["efficiency"] * 1e9)
        assert 0 < x["efficiency"] <= 1


def test_explicit_schedules():
    c2 = fe.CONFIGS["c2"]
    q = femgpu.schedules(c2, schedule=femgpu.SCHED_QUADRATURE)
    assert [x["kernel"] for x in q if x["chosen"]] == ["helm_quad_kernel"]
    t = femgpu.schedules(c2, schedule=femgpu.SCHED_TENSOR)
    assert [x["kernel"] for x in t if x["chosen"]] == ["helm_tensor_kernel"]
    c3 = fe.CONFIGS["c3"]
    t = femgpu.schedules(c3, schedule=femgpu.SCHED_TENSOR)
    assert [x["kernel"] for x in t if x["chosen"]] == ["elas_tensor_kernel"]
    # no tensor schedule exists for the nonlinear St Venant--Kirchhoff tangent
    s = femgpu.schedules(fe.CONFIGS["c4"], schedule=femgpu.SCHED_TENSOR)
    assert not any(x["chosen"] for x in s)
    # the flop-minimal plan is the tensor one for P3 Helmholtz (femopt: 160 k vs 408 k)
    a = femgpu.schedules(c2)
    assert a[0]["flops_per_cell"] < a[1]["flops_per_cell"] / 3


# ----------------------------------------------------------------------------
# GPU
# ----------------------------------------------------------------------------
def _run(form, cfg, coords, coeffs, accumulate_into=None):
    import torch

    dev = torch.device("cuda:0")
    x = torch.from_numpy(np.ascontiguousarray(coords)).to(dev)
    c = torch.from_numpy(np.ascontiguousarray(coeffs)).to(dev)
    if accumulate_into is None:
        out = torch.full((coords.shape[0], cfg.n, cfg.n), float("nan"), dtype=torch.float64,
                         device=dev)
        form.assemble(x, c, out)
    else:
        out = torch.from_numpy(np.ascontiguousarray(accumulate_into)).to(dev)
        form.assemble(x, c, out, accumulate=True)
    torch.cuda.synchronize()
    return out


def _frob(A, R):
    A = np.asarray(A).reshape(len(A), -1)
    R = np.asarray(R).reshape(len(R), -1)
    return float(np.max(np.linalg.norm(A - R, axis=1) / np.linalg.norm(R, axis=1)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_quadrature_kernel_vs_reference(name, golden_dir):
    """helm_quad_kernel against femopt's emitted C: the golden fixture, a
    multi-tile window and (c2) every cell of the BASELINE mesh."""
    import parity

    cfg = fe.CONFIGS[name]
    z = np.load(f"{golden_dir}/{name}.npz")
    tabs = fe.Tables(X=z["X"], W=z["W"], B=z["B"], D=z["D"], P=z["P"])
    form = femgpu.Form.from_config(cfg, tabs, schedule=femgpu.SCHED_QUADRATURE)
    assert form.info["kernel_name"] == "helm_quad_kernel"
    A = _run(form, cfg, z["coords"], z["coeffs"]).cpu().numpy()
    assert _frob(A, z["A"]) < TOL
    form = femgpu.Form.from_config(cfg, schedule=femgpu.SCHED_QUADRATURE)
    coords, coeffs = fe.cell_inputs(cfg)
    if name == "c1":
        coords, coeffs = coords[:3 * 148 * 32 + 19], coeffs[:3 * 148 * 32 + 19]
    out = _run(form, cfg, coords, coeffs)
    r = parity.check(cfg, coords, coeffs, lambda a, b: out[a:b].cpu().numpy())
    assert r["cells_checked"] == coords.shape[0] and r["max_frob_rel"] < TOL, r


@pytest.mark.gpu
def test_quadrature_kernel_ragged_and_accumulate():
    import port

    cfg = fe.CONFIGS["c2"]
    form = femgpu.Form.from_config(cfg, schedule=femgpu.SCHED_QUADRATURE)
    for E in (1, 31, 33, 97):
        coords, coeffs = fe.cell_inputs(cfg, ncells=E)
        A = _run(form, cfg, coords, coeffs).cpu().numpy()
        assert _frob(A, port.assemble(cfg, fe.tables(cfg), coords, coeffs)) < TOL
    coords, coeffs = fe.cell_inputs(cfg, ncells=70)
    A1 = _run(form, cfg, coords, coeffs).cpu().numpy()
    base = np.random.default_rng(5).uniform(-1, 1, size=A1.shape)
    A2 = _run(form, cfg, coords, coeffs, accumulate_into=base).cpu().numpy()
    assert np.allclose(A2, base + A1, rtol=1e-15, atol=1e-15 * np.abs(A1).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_auto_choice_is_the_faster_measured(name):
    """On the BASELINE mesh, the kernel AUTO picks runs faster than the other
    schedule's kernel (timed with CUDA events over a CUDA-graph replay)."""
    import torch

    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg)
    dev = torch.device("cuda:0")
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    out = torch.empty((coords.shape[0], cfg.n, cfg.n), dtype=torch.float64, device=dev)
    times = {}
    scheds = ((femgpu.SCHED_QUADRATURE, femgpu.SCHED_QUADRATURE_MMA) if name == "c4"
              else (femgpu.SCHED_TENSOR, femgpu.SCHED_QUADRATURE))
    for sched in scheds:
        form = femgpu.Form.from_config(cfg, schedule=sched)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            for _ in range(3):
                form.assemble(x, c, out, stream=s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(5):
                    form.assemble(x, c, out, stream=s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize(dev)
        times[form.info["kernel_name"]] = e0.elapsed_time(e1) / 5
    auto = femgpu.Form.from_config(cfg).info["kernel_name"]
    assert auto == min(times, key=times.get), times
