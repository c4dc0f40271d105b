"""GPU robustness beyond the BASELINE meshes: inverted cells, element-matrix
index ranges past 2^31 doubles, and launches on several streams at once.
Checked against the C oracle (pinned to the reference by tests/test_oracle.py)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

TOL = 1e-12
CONFIGS = ["c1", "c2", "c3", "c4", "c5"]


def frob_rel(A, R):
    A = np.asarray(A).reshape(len(A), -1)
    R = np.asarray(R).reshape(len(R), -1)
    return float(np.max(np.linalg.norm(A - R, axis=1) / np.linalg.norm(R, axis=1)))


@pytest.mark.parametrize("name", CONFIGS)
def test_inverted_cells(name):
    # negative Jacobian determinant on every other cell (vertices 1 and 2
    # swapped): the forms integrate with |det J|, like the reference IR
    import port

    cfg = fe.CONFIGS[name]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=67)
    x = coords.reshape(-1, 4, 3).copy()
    x[::2, [1, 2]] = x[::2, [2, 1]]
    coords = x.reshape(-1, 12)
    form = femgpu.Form.from_config(cfg, tabs)
    dev = torch.device("cuda:0")
    out = torch.empty((coords.shape[0], cfg.n, cfg.n), dtype=torch.float64, device=dev)
    form.assemble(torch.from_numpy(coords).to(dev), torch.from_numpy(coeffs).to(dev), out)
    torch.cuda.synchronize()
    assert frob_rel(out.cpu().numpy(), port.assemble(cfg, tabs, coords, coeffs)) < TOL


def _device_inputs(cfg, E, dev, seed=7):
    """E jittered unit-scale tetrahedra and coefficient dofs, generated on the device."""
    g = torch.Generator(device=dev).manual_seed(seed)
    ref = torch.tensor([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], dtype=torch.float64, device=dev)
    coords = ref + 0.1 * (torch.rand((E, 12), generator=g, dtype=torch.float64, device=dev) - 0.5)
    coeffs = 0.5 + torch.rand((E, cfg.ncoef), generator=g, dtype=torch.float64, device=dev)
    if cfg.kind == fe.HYPERELASTICITY:  # small displacement dofs
        coeffs[:, : 3 * cfg.ns] = 0.1 * (coeffs[:, : 3 * cfg.ns] - 1.0)
    return coords, coeffs


@pytest.mark.parametrize("name", ["c1", "c5"])
def test_element_matrix_index_past_2_31(name):
    # E * n * n > 2^31 doubles: 64-bit offsets in every kernel's output path
    import port

    cfg = fe.CONFIGS[name]
    E = (1 << 31) // (cfg.n * cfg.n) + 4099
    dev = torch.device("cuda:0")
    free, _ = torch.cuda.mem_get_info()
    need = E * (cfg.n * cfg.n + 12 + cfg.ncoef) * 8
    if need > 0.8 * free:
        pytest.skip("not enough device memory")
    coords, coeffs = _device_inputs(cfg, E, dev)
    out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    out[-300:] = float("nan")
    tabs = fe.tables(cfg)
    form = femgpu.Form.from_config(cfg, tabs)
    form.assemble(coords, coeffs, out)
    torch.cuda.synchronize()
    idx = np.r_[0:3, E // 2, E - 300:E]
    R = port.assemble(cfg, tabs, coords[idx].cpu().numpy(), coeffs[idx].cpu().numpy())
    assert frob_rel(out[idx].cpu().numpy(), R) < TOL


def test_concurrent_streams_and_threads():
    # one form per thread, each on its own stream; the form handle's device
    # tables are shared read-only state
    import port

    results = {}
    dev = torch.device("cuda:0")

    def run(name):
        cfg = fe.CONFIGS[name]
        tabs = fe.tables(cfg)
        coords, coeffs = fe.cell_inputs(cfg, ncells=301)
        form = femgpu.Form.from_config(cfg, tabs)
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            x = torch.from_numpy(coords).to(dev, non_blocking=False)
            c = torch.from_numpy(coeffs).to(dev, non_blocking=False)
            out = torch.empty((coords.shape[0], cfg.n, cfg.n), dtype=torch.float64, device=dev)
            for _ in range(3):
                form.assemble(x, c, out, stream=s.cuda_stream)
        s.synchronize()
        results[name] = frob_rel(out.cpu().numpy(), port.assemble(cfg, tabs, coords, coeffs))

    threads = [threading.Thread(target=run, args=(n,)) for n in CONFIGS]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert set(results) == set(CONFIGS)
    assert max(results.values()) < TOL, results


_FIRST_LAUNCH_RACE = r"""
import sys, threading
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1604_05872_b200 import fe, femgpu
dev = torch.device("cuda:0")
torch.cuda.init()
jobs = []
for name in ("c1", "c2", "c3", "c4", "c5"):
    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg, ncells=97)
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    for _ in range(4):  # four threads per kernel race its first launch
        form = femgpu.Form.from_config(cfg)
        out = torch.empty((97, cfg.n, cfg.n), dtype=torch.float64, device=dev)
        jobs.append((name, form, x, c, out))
torch.cuda.synchronize()
gate = threading.Barrier(len(jobs))
errors = []
def run(job):
    name, form, x, c, out = job
    s = torch.cuda.Stream(device=dev)
    gate.wait()
    try:
        form.assemble(x, c, out, stream=s.cuda_stream)
        s.synchronize()
    except Exception as e:  # noqa: BLE001
        errors.append(f"{name}: {e}")
threads = [threading.Thread(target=run, args=(j,)) for j in jobs]
for t in threads: t.start()
for t in threads: t.join()
assert not errors, errors
for name in ("c1", "c2", "c3", "c4", "c5"):
    outs = [j[4].cpu().numpy() for j in jobs if j[0] == name]
    assert all(np.array_equal(outs[0], o) for o in outs[1:]), name
print("ok")
"""


def test_first_launch_race_fresh_process():
    # the per-(kernel, device) setup (dynamic shared memory attribute, __constant__
    # tables) must be complete before any thread's first launch: a fresh process,
    # 20 threads released together into their first assemble call
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FIRST_LAUNCH_RACE, root], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_kernel_argv_rejects_foreign_reference_tables():
    """femgpu_kernel_argv: reference tables that differ from the form's would give
    results the emitted C would not compute -> INCONSISTENT_LAYOUT (code 8)."""
    from paper_1604_05872_b200 import ir

    for name in ("c1", "c4", "c5"):
        cfg = fe.CONFIGS[name]
        tabs = fe.tables(cfg)
        form = femgpu.Form.from_config(cfg, tabs)
        coords, coeffs = fe.cell_inputs(cfg, ncells=5)
        kernels = ir.build(cfg, coords, coeffs, tabs)
        tables = {}
        for _, k in kernels:
            for tname, t in k["tables"].items():
                tables[tname] = np.array(t["values"])
        consts = kernels[0][1].get("constants", {})
        onames, tnames, cnames = form.argnames()
        per = form.n * form.n // len(onames)
        outs = [np.zeros(5 * per) for _ in onames]
        args = [tables[t] for t in tnames]
        form.kernel_argv(5, outs, args, [consts[c] for c in cnames])  # the form's own: OK
        for victim in [t for t in tnames if t[0] in "WBDP"][:3]:
            bad = [a.copy() for a in args]
            bad[tnames.index(victim)][0] += 1e-9
            with pytest.raises(femgpu.FemgpuError) as e:
                form.kernel_argv(5, outs, bad, [consts[c] for c in cnames])
            assert e.value.code == 8 and victim in e.value.message


def test_python_mirror_validates_buffers():
    """Wrong dtype / shape / layout / device / argument counts raise
    FemgpuError(9) before any pointer reaches native code."""
    cfg = fe.CONFIGS["c2"]
    form = femgpu.Form.from_config(cfg)
    dev = torch.device("cuda:0")
    E = 40
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    good = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    form.assemble(x, c, good)
    bad_outs = [torch.empty((E, cfg.n, cfg.n), dtype=torch.float32, device=dev),
                torch.empty((E - 1, cfg.n, cfg.n), dtype=torch.float64, device=dev),
                torch.empty((E, cfg.n, cfg.n + 1), dtype=torch.float64, device=dev),
                torch.empty((cfg.n, E, cfg.n), dtype=torch.float64, device=dev).transpose(0, 1),
                torch.empty((E, cfg.n, cfg.n), dtype=torch.float64)]
    for o in bad_outs:
        with pytest.raises(femgpu.FemgpuError) as e:
            form.assemble(x, c, o)
        assert e.value.code == 9
    with pytest.raises(femgpu.FemgpuError) as e:
        form.assemble(x, c[:, :5].contiguous(), good)
    assert e.value.code == 9
    with pytest.raises(femgpu.FemgpuError) as e:
        form.assemble_host(coords, coeffs, np.zeros((E, cfg.n, cfg.n), dtype=np.float32))
    assert e.value.code == 9
    onames, tnames, cnames = form.argnames()
    with pytest.raises(femgpu.FemgpuError) as e:
        form.kernel_argv(E, [np.zeros(E * cfg.n * cfg.n)], [np.zeros(E)] * (len(tnames) - 1))
    assert e.value.code == 9
    with pytest.raises(femgpu.FemgpuError) as e:
        form.kernel_argv(E, [np.zeros(E * cfg.n * cfg.n, dtype=np.float32)],
                         [np.zeros(E)] * len(tnames))
    assert e.value.code == 9


def test_assemble_csr_one_form_many_streams():
    """femgpu_assemble_csr from several threads on distinct streams with ONE form
    (its element-matrix scratch is shared): every call's CSR values equal the
    single-stream result up to atomic reordering."""
    from paper_1604_05872_b200 import mesh

    cfg = fe.CONFIGS["c2"]
    ga = mesh.GlobalAssembler(cfg, N=6)
    coef = torch.from_numpy(ga.mesh.global_coeffs()).to(ga.dev)
    ga.gather(coef)
    torch.cuda.synchronize()
    ref = torch.zeros_like(ga.vals)
    ga.form.assemble_csr(ga.coords, ga.coeffs, ga.pos, ref)
    torch.cuda.synchronize()
    results, errors = {}, []

    def run(i):
        try:
            s = torch.cuda.Stream(device=ga.dev)
            with torch.cuda.stream(s):
                v = torch.zeros_like(ga.vals)
                for _ in range(4):
                    v.zero_()
                    ga.form.assemble_csr(ga.coords, ga.coeffs, ga.pos, v, stream=s)
            s.synchronize()
            results[i] = v
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=run, args=(i,)) for i in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    scale = float(ref.abs().max())
    for v in results.values():
        assert float((v - ref).abs().max()) <= 1e-13 * scale
