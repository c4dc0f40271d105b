"""Run-to-run bit identity of the warp-specialised kernels on their full BASELINE
meshes.  Their producer/consumer rings, staging handoffs and TMA stores are
synchronised by mbarriers and named barriers; a missing wait would show up as an
element matrix that differs between launches (compute-sanitizer's race checks
are not available on the GPU pool).  Each kernel runs 12 times back to back on
one stream, the last mesh cell trimmed so the final tile is ragged."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

CASES = [("c1", femgpu.SCHED_AUTO), ("c2", femgpu.SCHED_AUTO), ("c3", femgpu.SCHED_AUTO),
         ("c4", femgpu.SCHED_AUTO), ("c4", femgpu.SCHED_QUADRATURE_MMA), ("c5", femgpu.SCHED_AUTO)]


@pytest.mark.parametrize("name,sched", CASES)
def test_repeat_launches_bit_identical(name, sched):
    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg)
    E = coords.shape[0] - 7
    form = femgpu.Form.from_config(cfg, schedule=sched)
    dev = torch.device("cuda:0")
    x = torch.from_numpy(coords[:E]).to(dev)
    c = torch.from_numpy(coeffs[:E]).to(dev)
    ref = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    out = torch.empty_like(ref)
    form.assemble(x, c, ref)
    for i in range(12):
        out.fill_(float("nan"))
        form.assemble(x, c, out)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), (name, form.info["kernel_name"], i)
