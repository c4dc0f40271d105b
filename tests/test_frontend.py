"""Front-end self-checks (SURVEY.md §7 "Hard parts": nothing in the reference
pins basis tabulation, quadrature or meshes, so they are checked here)."""
from math import factorial

import numpy as np
import pytest

from paper_1604_05872_b200 import fe, ir


@pytest.mark.parametrize("m", [2, 3, 5])
def test_quadrature_exact_to_degree(m):
    X, W = fe.tet_quadrature(m)
    assert W.shape == (m ** 3,)
    assert abs(W.sum() - 1 / 6) < 1e-15
    for a in range(2 * m):
        for b in range(2 * m - a):
            for c in range(2 * m - a - b):
                exact = factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 3)
                got = (W * X[:, 0] ** a * X[:, 1] ** b * X[:, 2] ** c).sum()
                assert abs(got - exact) < 1e-15


def test_points_per_degree():
    assert [fe.points_for_degree(d) for d in (3, 5, 8, 9)] == [2, 3, 5, 5]
    assert [fe.CONFIGS[c].nq for c in ("c1", "c2", "c3", "c4", "c5")] == [8, 125, 8, 27, 125]


@pytest.mark.parametrize("k", [1, 2, 3])
def test_lagrange_basis(k):
    nodes = np.array(fe.lagrange_nodes(k), dtype=float) / k
    n = (k + 1) * (k + 2) * (k + 3) // 6
    assert nodes.shape == (n, 3)
    B, D = fe.lagrange_tabulate(k, nodes)
    assert np.abs(B - np.eye(n)).max() < 1e-14          # Kronecker property
    X, _ = fe.tet_quadrature(3)
    B, D = fe.lagrange_tabulate(k, X)
    assert np.abs(B.sum(1) - 1).max() < 1e-13           # partition of unity
    assert np.abs(D.sum(2)).max() < 1e-12               # gradients sum to zero
    # derivative check by central differences
    h = 1e-6
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        Bp, _ = fe.lagrange_tabulate(k, X + e)
        Bm, _ = fe.lagrange_tabulate(k, X - e)
        assert np.abs((Bp - Bm) / (2 * h) - D[a]).max() < 1e-6


def test_p1_vertex_order_matches_geometry():
    B, D = fe.lagrange_tabulate(1, np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]))
    assert np.array_equal(B, np.eye(4))
    assert np.array_equal(D[:, 0, :], np.array([[-1, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 0, 1.0]]))


@pytest.mark.parametrize("N", [1, 3, 8])
def test_cube_mesh(N):
    x = fe.cube_mesh(N)
    assert x.shape == (6 * N ** 3, 4, 3)
    J = np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]], axis=-1)
    vol = np.abs(np.linalg.det(J)) / 6
    assert abs(vol.sum() - 1.0) < 1e-12
    assert vol.min() > 0.2 / (6 * N ** 3)  # jitter keeps every tet well shaped
    assert x.min() == 0.0 and x.max() == 1.0
    # jitter bounded by 0.1 h
    grid = np.round(x * N)
    assert np.abs(x * N - grid).max() <= 0.1 + 1e-12


def test_mesh_and_dofs_deterministic():
    a = fe.cell_inputs(fe.CONFIGS["c4"], ncells=100)
    b = fe.cell_inputs(fe.CONFIGS["c4"], ncells=100)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    full = fe.cell_inputs(fe.CONFIGS["c4"].with_N(4))
    pre = fe.cell_inputs(fe.CONFIGS["c4"].with_N(4), ncells=50)
    assert np.array_equal(full[0][:50], pre[0]) and np.array_equal(full[1][:50], pre[1])
    other = fe.cell_inputs(fe.CONFIGS["c4"].with_N(4), shard=1)
    assert not np.array_equal(full[0], other[0])


def test_config_arithmetic():
    c = fe.CONFIGS
    assert [c[k].ncells for k in c] == [1572864, 663552, 663552, 196608, 196608]
    assert [c[k].n for k in c] == [4, 20, 30, 30, 60]
    assert [c[k].bytes_per_cell() for k in c] == [256, 3456, 7360, 7600, 29376]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_ir_is_valid_json_schema(name):
    cfg = fe.CONFIGS[name]
    coords, coeffs = fe.cell_inputs(cfg, ncells=2)
    for out, k in ir.build(cfg, coords, coeffs):
        assert set(k) <= {"indices", "loops", "tables", "constants", "statements", "outputs"}
        assert k["outputs"] == [out]
        for t in k["tables"].values():
            size = int(np.prod([k["indices"][d] for d in t["dims"]]))
            assert len(t["values"]) == size
        o, tabs, cons = ir.argument_order(k)
        assert tabs == sorted(tabs)
