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


def row_gather_host(g, A, row_ptr, col_idx):
    """The row-gather assembly's arithmetic on the host (test infrastructure):
    for every row, zero, then add its incident element rows in inc order -- the
    order femgpu_csr_gather_rows uses, so the sums are bit-identical."""
    inc_ptr, inc, maxlen = g.row_incidence()
    dof, nd = g.dof_map()
    E, n = dof.shape
    Ar = A.reshape(E * n, n)
    # column -> offset inside the row (the symbolic step femgpu_csr_row_offsets does)
    rows = dof.reshape(-1)
    loc = np.empty((E * n, n), dtype=np.int64)
    for t0 in range(0, E * n, 4096):
        t = np.arange(t0, min(E * n, t0 + 4096))
        cols = dof[t // n]                                     # [T][n] column dofs
        for i, tt in enumerate(t):
            b, e_ = row_ptr[rows[tt]], row_ptr[rows[tt] + 1]
            loc[tt] = np.searchsorted(col_idx[b:e_], cols[i])
    vals = np.zeros(col_idx.size)
    cnt = np.diff(inc_ptr)
    for s_ in range(int(cnt.max())):
        r = np.nonzero(cnt > s_)[0]
        t = inc[inc_ptr[r] + s_]
        idx = row_ptr[r][:, None] + loc[t]
        vals[idx] = vals[idx] + Ar[t]
    return vals, maxlen


@pytest.mark.parametrize("name", CONFIGS)
def test_row_incidence_plan(name):
    cfg = fe.CONFIGS[name]
    g = mesh.GlobalMesh(cfg, N=2)
    inc_ptr, inc, maxlen = g.row_incidence()
    dof, nd = g.dof_map()
    row_ptr, col_idx, _ = g.csr_pattern()
    assert inc_ptr.size == nd + 1 and inc_ptr[-1] == dof.size
    assert np.array_equal(np.sort(inc), np.arange(dof.size))        # every element row once
    flat = dof.reshape(-1)
    seg = np.repeat(np.arange(nd), np.diff(inc_ptr))
    assert np.array_equal(flat[inc], seg)                            # row r's element rows
    assert np.all(np.diff(inc)[np.diff(seg) == 0] > 0)               # ascending inside a row
    assert maxlen == np.diff(row_ptr).max() <= 65536
    # the row-gather arithmetic equals the scipy COO -> CSR sum
    A = np.random.default_rng(1).uniform(-1, 1, size=(g.E, cfg.n, cfg.n))
    got, _ = row_gather_host(g, A, row_ptr, col_idx)
    ref = g.assemble_csr_host(A, row_ptr, col_idx)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


# ----------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", CONFIGS)
def test_row_gather_assembly(name):
    # atomic-free assembly: bit-identical to the host sum in the plan's order,
    # reproducible run to run, and += honoured
    torch = pytest.importorskip("torch")
    cfg = fe.CONFIGS[name]
    ga = mesh.GlobalAssembler(cfg, N=3)
    g = ga.mesh
    coef = torch.from_numpy(g.global_coeffs()).to(ga.dev)
    rows = ga.assemble(coef, mode="rows").clone()
    again = ga.assemble(coef, mode="rows").clone()
    torch.cuda.synchronize()
    row_ptr, col_idx, _ = g.csr_pattern()
    ref, _ = row_gather_host(g, ga.A.cpu().numpy(), row_ptr, col_idx)
    assert np.array_equal(rows.cpu().numpy(), ref)
    assert np.array_equal(again.cpu().numpy(), ref)
    atomics = ga.assemble(coef, mode="scatter").clone()
    torch.cuda.synchronize()
    assert np.abs(atomics.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()
    from paper_1604_05872_b200 import femgpu

    inc_ptr, inc, loc, maxlen = ga.row_plan()
    acc = rows.clone()
    femgpu.csr_gather_rows(ga.row_ptr, inc_ptr, inc, loc, maxlen, ga.A, acc, accumulate=True)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), ref + ref)


@pytest.mark.gpu
def test_row_offsets_reject_entries_outside_their_row():
    torch = pytest.importorskip("torch")
    from paper_1604_05872_b200 import femgpu

    cfg = fe.CONFIGS["c3"]
    ga = mesh.GlobalAssembler(cfg, N=2)
    pos = ga.pos.clone()
    pos[0, 0, 0] = ga.row_ptr[-1].item() + 5   # outside row dof[0][0]
    loc = torch.empty(pos.shape, dtype=torch.uint16, device=ga.dev)
    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.csr_row_offsets(ga.dof, ga.row_ptr, pos, loc)
    assert e.value.code == 8


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
