"""Either side of the path: global node numbering,
gather of per-cell inputs from global vectors, CSR pattern, symbolic (positions)
and numeric (scatter-add) assembly.  Host reference: numpy gather and a scipy
COO -> CSR sum of the same element matrices."""
import numpy as np
import pytest

from paper_1604_05872_b200 import fe, mesh

CONFIGS = ["c1", "c2", "c3", "c4", "c5"]


def node_positions(g, p):
    """Unjittered physical position of every (cell, local node) of degree p."""
    N = g.N
    vid = g.cells
    lat = np.stack([vid % (N + 1), (vid // (N + 1)) % (N + 1), vid // (N + 1) ** 2], -1) / N
    nodes = np.asarray(fe.lagrange_nodes(p), dtype=np.float64)
    w = np.stack([p - nodes.sum(1), nodes[:, 0], nodes[:, 1], nodes[:, 2]], 1) / p
    return np.einsum("nv,evx->enx", w, lat)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_node_numbering_is_conforming(p):
    g = mesh.GlobalMesh(fe.CONFIGS["c1"], N=3)
    M, nn = g.node_map(p)
    X = node_positions(g, p).reshape(-1, 3)
    ids = M.reshape(-1)
    assert nn == (p * 3 + 1) ** 3
    # one position per global node, every node used
    first = np.full((nn, 3), np.nan)
    first[ids] = X
    assert np.abs(first[ids] - X).max() < 1e-14
    assert np.unique(ids).size == nn
    # no cell lists a node twice
    assert all(np.unique(r).size == r.size for r in M)


def test_topology_matches_cube_mesh():
    g = mesh.GlobalMesh(fe.CONFIGS["c2"], N=4)
    assert np.array_equal(g.V[g.cells], fe.cube_mesh(4))


@pytest.mark.parametrize("name", CONFIGS)
def test_csr_pattern_covers_element_matrices(name):
    cfg = fe.CONFIGS[name]
    g = mesh.GlobalMesh(cfg, N=2)
    row_ptr, col_idx, nd = g.csr_pattern()
    dof, nd2 = g.dof_map()
    assert nd == nd2 and row_ptr[-1] == col_idx.size
    for r in range(0, nd, max(1, nd // 97)):
        c = col_idx[row_ptr[r]:row_ptr[r + 1]]
        assert np.all(np.diff(c) > 0)
    A = np.random.default_rng(0).uniform(size=(g.E, cfg.n, cfg.n))
    v = g.assemble_csr_host(A, row_ptr, col_idx)  # asserts every entry is in the pattern
    assert np.isclose(v.sum(), A.sum())


# ----------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", CONFIGS)
def test_gather_assemble_scatter(name):
    torch = pytest.importorskip("torch")
    cfg = fe.CONFIGS[name]
    ga = mesh.GlobalAssembler(cfg, N=3)
    g = ga.mesh
    coef_np = g.global_coeffs()
    coef = torch.from_numpy(coef_np).to(ga.dev)
    vals = ga.assemble(coef, fused=False).clone()
    fused = ga.assemble(coef, fused=True).clone()
    torch.cuda.synchronize()
    # gather: exact copies
    _, cidx, _ = g.coef_layout()
    assert np.array_equal(ga.coords.cpu().numpy().reshape(-1, 4, 3), g.V[g.cells])
    assert np.array_equal(ga.coeffs.cpu().numpy()[:, :cidx.shape[1]], coef_np[cidx])
    # scatter-add: the host sum of the same element matrices (atomics reorder
    # the additions: equal up to rounding)
    row_ptr, col_idx, _ = g.csr_pattern()
    ref = g.assemble_csr_host(ga.A.cpu().numpy(), row_ptr, col_idx)
    got = vals.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    # femgpu_assemble_csr (fused epilogue for Helmholtz, kernel + scatter otherwise)
    assert np.abs(fused.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()
    # the element matrices are the path's own (pinned by the parity suite)
    if cfg.kind != fe.BURGERS:
        M = ga.form.assemble_host(ga.coords.cpu().numpy(), ga.coeffs.cpu().numpy())
        assert np.array_equal(M, ga.A.cpu().numpy())


@pytest.mark.gpu
def test_positions_reject_entries_outside_the_pattern():
    torch = pytest.importorskip("torch")
    from paper_1604_05872_b200 import femgpu

    cfg = fe.CONFIGS["c1"]
    g = mesh.GlobalMesh(cfg, N=2)
    row_ptr, col_idx, _ = g.csr_pattern()
    dof, _ = g.dof_map()
    dev = torch.device("cuda:0")
    col_bad = col_idx.copy()
    col_bad[row_ptr[1]:row_ptr[2]] += 1000  # row 1 no longer holds its columns
    pos = torch.empty((g.E, cfg.n, cfg.n), dtype=torch.int64, device=dev)
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.csr_positions(torch.from_numpy(dof.astype(np.int32)).to(dev),
                             torch.from_numpy(row_ptr).to(dev),
                             torch.from_numpy(col_bad).to(dev), pos)
    assert e.value.code == 8
