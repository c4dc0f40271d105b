"""Finite-element front end: quadrature, Lagrange tabulation, meshes, inputs.

The reference (femopt) has no finite-element front end -- its input is "a
kernel IR file, not a variational form" whose
tables arrive pre-tabulated (proj/README.md:68-100, ``tables``).  Everything
the BASELINE configs need therefore lives here, written once and shared by
the IR generator (``ir.py``), the C-ABI host mirror (``femgpu.py``), the
tests and ``bench.py``:

* collapsed Gauss--Jacobi quadrature on the reference tetrahedron
  (m = ceil((d+1)/2) points per direction, Q = m^3);
* equispaced Lagrange P1/P2/P3 basis values and reference gradients, with the
  Vandermonde inverse computed in exact rational arithmetic so the tables are
  the correctly rounded values of the exact basis on every host;
* the jittered unit-cube mesh, N^3 hexes x 6 Kuhn tets, cell-major FP64
  coordinates ``[E][4][3]``;
* seeded per-cell coefficient dofs, cell-major ``[E][ndof]``.

All arrays are float64 and C-contiguous.  Randomness uses numpy's PCG64 with
fixed seeds, so the host, the GPU and the CPU baseline see identical bytes.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache

import numpy as np

# ----------------------------------------------------------------------------
# Quadrature
# ----------------------------------------------------------------------------


def gauss_jacobi_01(m: int, a: int) -> tuple[np.ndarray, np.ndarray]:
    """m-point Gauss rule on [0,1] for the weight (1-t)^a (exact to 2m-1)."""
    from scipy.special import roots_jacobi

    x, w = roots_jacobi(m, float(a), 0.0)  # weight (1-x)^a on [-1,1]
    t = (x + 1.0) / 2.0
    return np.ascontiguousarray(t), np.ascontiguousarray(w / 2.0 ** (a + 1))


@lru_cache(maxsize=None)
def tet_quadrature(m: int) -> tuple[np.ndarray, np.ndarray]:
    """Collapsed (Duffy) Gauss--Jacobi rule on the reference tet.

    Reference tet: (0,0,0),(1,0,0),(0,1,0),(0,0,1).  Map (u,v,w) in [0,1]^3 to
    x = u(1-v)(1-w), y = v(1-w), z = w with Jacobian (1-v)(1-w)^2; the (1-v)
    and (1-w)^2 factors are absorbed into Jacobi weights.  A polynomial of
    total degree d is exact when 2m-1 >= d.  Returns X [Q,3], W [Q] with
    sum(W) = 1/6; point order is u slowest, w fastest.
    """
    tu, wu = gauss_jacobi_01(m, 0)
    tv, wv = gauss_jacobi_01(m, 1)
    tw, ww = gauss_jacobi_01(m, 2)
    pts, wts = [], []
    for iu in range(m):
        for iv in range(m):
            for iw in range(m):
                u, v, w = tu[iu], tv[iv], tw[iw]
                pts.append((u * (1.0 - v) * (1.0 - w), v * (1.0 - w), w))
                wts.append(wu[iu] * wv[iv] * ww[iw])
    X = np.array(pts, dtype=np.float64)
    W = np.array(wts, dtype=np.float64)
    X.setflags(write=False)
    W.setflags(write=False)
    return X, W


def points_for_degree(d: int) -> int:
    """Points per collapsed direction for exactness at total degree d."""
    return (d + 2) // 2  # ceil((d+1)/2)


# ----------------------------------------------------------------------------
# Lagrange basis on the reference tetrahedron
# ----------------------------------------------------------------------------


@lru_cache(maxsize=None)
def lagrange_nodes(k: int) -> tuple[tuple[int, int, int], ...]:
    """Equispaced lattice nodes (integer coords / k), vertices first.

    Vertex order matches the cell vertex order v0..v3 of the geometry map, so
    P1 dof a lives at vertex a.  The remaining nodes follow in lexicographic
    order of their lattice coordinates.
    """
    lat = [(a, b, c) for c in range(k + 1) for b in range(k + 1) for a in range(k + 1)
           if a + b + c <= k]
    verts = [(0, 0, 0), (k, 0, 0), (0, k, 0), (0, 0, k)]
    rest = sorted(p for p in lat if p not in verts)
    return tuple(verts + rest)


def _monomials(k: int) -> list[tuple[int, int, int]]:
    return [(a, b, c) for t in range(k + 1) for c in range(t + 1) for b in range(t + 1 - c)
            for a in [t - b - c]]


@lru_cache(maxsize=None)
def lagrange_coefficients(k: int) -> tuple[tuple[tuple[int, int, int], ...], np.ndarray]:
    """Monomial coefficients C[m, n] of basis function n (exact, then rounded)."""
    nodes = lagrange_nodes(k)
    mons = _monomials(k)
    n = len(nodes)
    # Vandermonde V[i, m] = x_i^a y_i^b z_i^c, exact rationals.
    V = [[Fraction(1) for _ in range(n)] for _ in range(n)]
    for i, (p, q, r) in enumerate(nodes):
        x, y, z = Fraction(p, k), Fraction(q, k), Fraction(r, k)
        for m, (a, b, c) in enumerate(mons):
            V[i][m] = x ** a * y ** b * z ** c
    # Gauss-Jordan inverse over Q.
    M = [row[:] + [Fraction(int(i == j)) for j in range(n)] for i, row in enumerate(V)]
    for col in range(n):
        piv = next(r for r in range(col, n) if M[r][col] != 0)
        M[col], M[piv] = M[piv], M[col]
        inv = 1 / M[col][col]
        M[col] = [v * inv for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                f = M[r][col]
                M[r] = [vr - f * vc for vr, vc in zip(M[r], M[col])]
    # phi_n(x) = sum_m C[m, n] mon_m(x), with C = V^{-1}.
    C = np.array([[float(M[m][n + j]) for j in range(n)] for m in range(n)], dtype=np.float64)
    return tuple(mons), C


def lagrange_tabulate(k: int, X: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Basis values B[Q,n] and reference gradients D[3,Q,n] at points X[Q,3]."""
    mons, C = lagrange_coefficients(k)
    X = np.asarray(X, dtype=np.float64)
    Q = X.shape[0]
    n = C.shape[1]

    def powv(v, e):
        return np.ones(Q) if e == 0 else v ** e

    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    Mv = np.zeros((Q, len(mons)))
    Md = np.zeros((3, Q, len(mons)))
    for m, (a, b, c) in enumerate(mons):
        Mv[:, m] = powv(x, a) * powv(y, b) * powv(z, c)
        if a:
            Md[0, :, m] = a * powv(x, a - 1) * powv(y, b) * powv(z, c)
        if b:
            Md[1, :, m] = b * powv(x, a) * powv(y, b - 1) * powv(z, c)
        if c:
            Md[2, :, m] = c * powv(x, a) * powv(y, b) * powv(z, c - 1)
    B = np.ascontiguousarray(Mv @ C)
    D = np.ascontiguousarray(np.stack([Md[d] @ C for d in range(3)]))
    # Constant-gradient cases (P1) come out exact; tiny round-off in higher
    # degrees is fine: every consumer reads these same tables.
    assert B.shape == (Q, n)
    return B, D


# ----------------------------------------------------------------------------
# Mesh and per-cell inputs
# ----------------------------------------------------------------------------

_KUHN = list(itertools.permutations(range(3)))  # 6 tets per hex


def cube_mesh(N: int, seed: int = 1604, jitter: float = 0.1) -> np.ndarray:
    """Jittered unit cube, N^3 hexes x 6 Kuhn tets -> coords [E][4][3].

    Interior vertices move by U[-jitter*h, +jitter*h] per coordinate (h=1/N),
    drawn from PCG64(seed) in vertex order; boundary vertices stay put.  Cells
    are ordered hex-major (x fastest), the 6 tets of a hex consecutive.
    """
    V, cells = cube_topology(N, seed, jitter)
    return np.ascontiguousarray(V[cells])


def cube_topology(N: int, seed: int = 1604, jitter: float = 0.1):
    """The mesh of ``cube_mesh`` as vertices V [nv][3] and cells [E][4] (vertex ids,
    id = (k (N+1) + j)(N+1) + i for lattice point (i, j, k))."""
    h = 1.0 / N
    g = np.arange(N + 1, dtype=np.float64) * h
    zz, yy, xx = np.meshgrid(g, g, g, indexing="ij")
    V = np.stack([xx, yy, zz], axis=-1).reshape(-1, 3)  # vertex id = (k*(N+1)+j)*(N+1)+i
    rng = np.random.Generator(np.random.PCG64(seed))
    jit = rng.uniform(-jitter * h, jitter * h, size=V.shape)
    ii = np.arange(N + 1)
    interior_1d = (ii > 0) & (ii < N)
    interior = (interior_1d[:, None, None] & interior_1d[None, :, None]
                & interior_1d[None, None, :]).reshape(-1)
    V = V + jit * interior[:, None]

    def vid(i, j, k):
        return (k * (N + 1) + j) * (N + 1) + i

    hi, hj, hk = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    hi, hj, hk = hk.reshape(-1), hj.reshape(-1), hi.reshape(-1)  # x fastest
    cells = np.empty((N ** 3, 6, 4), dtype=np.int64)
    for t, perm in enumerate(_KUHN):
        off = np.zeros(3, dtype=np.int64)
        cells[:, t, 0] = vid(hi, hj, hk)
        for s in range(3):
            off[perm[s]] += 1
            cells[:, t, s + 1] = vid(hi + off[0], hj + off[1], hk + off[2])
    cells = cells.reshape(-1, 4)
    return V, cells


def draw_dofs(E: int, ndof: int, lo: float, hi: float, seed: int) -> np.ndarray:
    """Seeded per-cell dofs U[lo,hi], cell-major [E][ndof]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.ascontiguousarray(rng.uniform(lo, hi, size=(E, ndof)))


# ----------------------------------------------------------------------------
# The five BASELINE configs
# ----------------------------------------------------------------------------

HELMHOLTZ, ELASTICITY, HYPERELASTICITY, BURGERS = 1, 2, 3, 4
KIND_NAMES = {HELMHOLTZ: "helmholtz", ELASTICITY: "elasticity",
              HYPERELASTICITY: "hyperelasticity", BURGERS: "burgers"}


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config: form, element, quadrature and mesh."""

    name: str
    kind: int
    degree: int          # Lagrange degree of test/trial space (scalar or vector)
    vector: bool
    quad_degree: int     # total integrand degree the rule must integrate exactly
    N: int               # cube resolution -> 6 N^3 cells
    coef_degree: int     # degree of the pre-multiplying coefficients (0: none)
    consts: tuple = ()   # (nu, dt) for Burgers
    description: str = ""
    coef_ranges: tuple = field(default_factory=tuple)  # ((name, ndof_per_comp, ncomp, lo, hi, seed), ...)

    @property
    def m(self) -> int:
        return points_for_degree(self.quad_degree)

    @property
    def nq(self) -> int:
        return self.m ** 3

    @property
    def ns(self) -> int:
        """Scalar dofs per component."""
        k = self.degree
        return (k + 1) * (k + 2) * (k + 3) // 6

    @property
    def n(self) -> int:
        """Element-matrix dimension."""
        return self.ns * (3 if self.vector else 1)

    @property
    def ncells(self) -> int:
        return 6 * self.N ** 3

    @property
    def ncoef(self) -> int:
        return sum(nd * nc for (_, nd, nc, _, _, _) in self.coef_ranges)

    def with_N(self, N: int) -> "Config":
        from dataclasses import replace
        return replace(self, N=N)

    def bytes_per_cell(self) -> int:
        """Compulsory HBM bytes: coords + coefficient dofs + element matrix."""
        return 8 * (12 + self.ncoef + self.n * self.n)


def _p(k):
    return (k + 1) * (k + 2) * (k + 3) // 6


CONFIGS: dict[str, Config] = {
    "c1": Config("c1", HELMHOLTZ, 1, False, 3, 64, 1,
                 description="Helmholtz P1, P1 f, 64^3x6",
                 coef_ranges=(("f", _p(1), 1, 0.5, 1.5, 11),)),
    "c2": Config("c2", HELMHOLTZ, 3, False, 9, 48, 3,
                 description="Helmholtz P3, P3 f, 48^3x6",
                 coef_ranges=(("f", _p(3), 1, 0.5, 1.5, 11),)),
    "c3": Config("c3", ELASTICITY, 2, True, 3, 48, 1,
                 description="linear elasticity vec-P2, P1 mu/lambda, 48^3x6",
                 coef_ranges=(("mu", 4, 1, 0.5, 2.0, 21), ("lam", 4, 1, 0.5, 2.0, 22))),
    "c4": Config("c4", HYPERELASTICITY, 2, True, 5, 32, 1,
                 description="St Venant-Kirchhoff Jacobian vec-P2, w vec-P2, P1 mu/lambda, 32^3x6",
                 coef_ranges=(("w", _p(2), 3, -0.05, 0.05, 31), ("mu", 4, 1, 0.5, 2.0, 32),
                              ("lam", 4, 1, 0.5, 2.0, 33))),
    "c5": Config("c5", BURGERS, 3, True, 8, 32, 0, consts=(0.01, 0.1),
                 description="Burgers Jacobian vec-P3, u vec-P3, nu=0.01, dt=0.1, 32^3x6",
                 coef_ranges=(("u", _p(3), 3, -1.0, 1.0, 41),)),
}


@dataclass
class Tables:
    """Reference tables of one config (the IR's input tables)."""

    X: np.ndarray   # [Q,3] quadrature points
    W: np.ndarray   # [Q]
    B: np.ndarray   # [Q,ns] test/trial scalar basis values
    D: np.ndarray   # [3,Q,ns] reference gradients
    P: np.ndarray   # [Q,nc] coefficient basis (P1 for mu/lambda; = B otherwise)


def tables(cfg: Config) -> Tables:
    X, W = tet_quadrature(cfg.m)
    B, D = lagrange_tabulate(cfg.degree, X)
    if cfg.kind in (ELASTICITY, HYPERELASTICITY):
        P, _ = lagrange_tabulate(1, X)
    elif cfg.kind == HELMHOLTZ:
        P, _ = lagrange_tabulate(cfg.coef_degree, X)
    else:
        P = B
    return Tables(X=np.asarray(X), W=np.asarray(W), B=B, D=D, P=np.ascontiguousarray(P))


def cell_inputs(cfg: Config, ncells: int | None = None, shard: int = 0):
    """Seeded cell-major inputs (coords [E][4][3], coeffs [E][ncoef]).

    The mesh is the config's jittered cube (shard s uses jitter seed
    1604+s and coefficient seeds offset by 1000*s, so weak-scaling shards are
    distinct meshes of identical shape).  ``ncells`` truncates to the first
    cells (parity tests); the full mesh is 6 N^3 cells.
    """
    coords = cube_mesh(cfg.N, seed=1604 + shard)
    E = coords.shape[0] if ncells is None else min(ncells, coords.shape[0])
    coords = np.ascontiguousarray(coords[:E])
    parts = []
    for (_, nd, nc, lo, hi, seed) in cfg.coef_ranges:
        # PCG64 fills row-major, so a prefix of cells gets the same dofs as
        # the full mesh would.
        parts.append(draw_dofs(E, nd * nc, lo, hi, seed + 1000 * shard))
    coeffs = np.ascontiguousarray(np.concatenate(parts, axis=1)) if parts else np.zeros((E, 0))
    return coords, coeffs
