"""Global mesh data either side of the path.

The reference's element kernels read pre-gathered per-cell tables
(/root/reference/proj/tests/kernels.hpp:186-188) and stop at the element
matrix; a FEM code around them gathers geometry and coefficient
dofs from global vectors before the path and scatter-adds A_e into a global
sparse matrix after it.  This module is the host-side setup for those two
steps on the BASELINE meshes (the kernels are femgpu_gather /
femgpu_csr_positions / femgpu_scatter_add in csrc/global.cu):

  * global Lagrange node numbering of degree p on the Kuhn cube mesh, by the
    integer lattice the P_p nodes of the unjittered mesh sit on (lattice step
    h/p): node (a,b,c)/p of a cell lies at sum_v (p lambda_v) x_v with
    p lambda = (p-a-b-c, a, b, c) -- so neighbours agree on shared nodes by
    construction, whatever their local vertex order;
  * vector fields are component-blocked: dof (c, node) = c * nnodes + node,
    matching the element matrix's row (c, j) = c * ns + j;
  * the CSR pattern of the global matrix (rows sorted, columns sorted).
"""
from __future__ import annotations

import numpy as np

from . import fe

DEG_OF_NDOF = {4: 1, 10: 2, 20: 3}


class GlobalMesh:
    def __init__(self, cfg: fe.Config, N: int | None = None, shard: int = 0):
        self.cfg = cfg
        self.N = cfg.N if N is None else int(N)
        self.V, self.cells = fe.cube_topology(self.N, seed=1604 + shard)
        self.E = self.cells.shape[0]
        self._nodes: dict[int, tuple[np.ndarray, int]] = {}

    # -- numbering ------------------------------------------------------------
    def node_map(self, p: int) -> tuple[np.ndarray, int]:
        """(map [E][ns(p)] int64 global node ids, number of nodes) for degree p."""
        if p not in self._nodes:
            N = self.N
            vid = self.cells                                   # [E][4]
            lat = np.stack([vid % (N + 1), (vid // (N + 1)) % (N + 1),
                            vid // (N + 1) ** 2], axis=-1)     # [E][4][3]
            nodes = np.asarray(fe.lagrange_nodes(p), dtype=np.int64)  # [ns][3] (a,b,c)
            w = np.stack([p - nodes.sum(1), nodes[:, 0], nodes[:, 1], nodes[:, 2]], axis=1)
            L = np.einsum("nv,evx->enx", w, lat)               # lattice coords, step h/p
            M = p * N + 1
            key = (L[..., 2] * M + L[..., 1]) * M + L[..., 0]
            uniq, inv = np.unique(key.reshape(-1), return_inverse=True)
            self._nodes[p] = (inv.reshape(self.E, -1).astype(np.int64), int(uniq.size))
        return self._nodes[p]

    def dof_map(self) -> tuple[np.ndarray, int]:
        """The form's dof map [E][n] (component-blocked for vector forms), ndofs."""
        cfg = self.cfg
        M, nn = self.node_map(cfg.degree)
        if not cfg.vector:
            return M, nn
        return np.concatenate([M + c * nn for c in range(3)], axis=1), 3 * nn

    def coef_layout(self):
        """Global coefficient vector layout: per field (name, degree, ncomp, offset,
        size) and the per-cell index map [E][ncoef] into the concatenated vector."""
        fields, idx, off = [], [], 0
        for (name, nd, nc, lo, hi, seed) in self.cfg.coef_ranges:
            p = DEG_OF_NDOF[nd]
            M, nn = self.node_map(p)
            fields.append((name, p, nc, off, nn * nc, lo, hi, seed))
            for c in range(nc):
                idx.append(M + off + c * nn)
            off += nn * nc
        cidx = np.concatenate(idx, axis=1) if idx else np.zeros((self.E, 0), dtype=np.int64)
        return fields, cidx, off

    def global_coeffs(self, shard: int = 0) -> np.ndarray:
        """Seeded global coefficient vector (per field and component, U[lo, hi])."""
        fields, _, size = self.coef_layout()
        g = np.empty(size)
        for (name, p, nc, off, n, lo, hi, seed) in fields:
            rng = np.random.Generator(np.random.PCG64(seed + 7919 + 1000 * shard))
            g[off:off + n] = rng.uniform(lo, hi, size=n)
        return g

    # -- sparsity ---------------------------------------------------------------
    def csr_pattern(self) -> tuple[np.ndarray, np.ndarray, int]:
        """(row_ptr int64 [ndofs+1], col_idx int32 [nnz], ndofs) of the global matrix."""
        cfg = self.cfg
        M, nn = self.node_map(cfg.degree)
        ns = M.shape[1]
        r = np.repeat(M, ns, axis=1).reshape(-1)
        c = np.tile(M, (1, ns)).reshape(-1)
        key = np.unique(r * nn + c)
        rows, cols = key // nn, key % nn
        counts = np.bincount(rows, minlength=nn)
        if not cfg.vector:
            row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            return row_ptr, cols.astype(np.int32), nn
        # vector: row (a, r) holds columns (b, c) for b = 0..2 -- 3x the scalar row
        sptr = np.concatenate([[0], np.cumsum(counts)])
        row_len = 3 * counts
        row_ptr = np.concatenate([[0], np.cumsum(np.tile(row_len, 3))]).astype(np.int64)
        cols3 = np.empty(3 * 3 * cols.size, dtype=np.int64)
        # per scalar row: [cols, cols + nn, cols + 2nn], then the same for each a
        seg = np.repeat(np.arange(nn), counts)
        pos_in_row = np.arange(cols.size) - sptr[seg]
        for a in range(3):
            base = row_ptr[a * nn + seg]
            for b in range(3):
                cols3[base + b * counts[seg] + pos_in_row] = cols + b * nn
        return row_ptr, cols3.astype(np.int32), 3 * nn

    def row_incidence(self) -> tuple[np.ndarray, np.ndarray, int]:
        """For the atomic-free assembly (femgpu_csr_gather_rows): inc_ptr int64
        [ndofs+1] and inc int32 [E*n], the element-row ids e*n + j with dof_map[e][j]
        == r for each global row r, in ascending id order; and the longest CSR row."""
        dof, nd = self.dof_map()
        flat = dof.reshape(-1)
        inc = np.argsort(flat, kind="stable").astype(np.int32)
        inc_ptr = np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=nd))]).astype(np.int64)
        row_ptr, _, _ = self.csr_pattern()
        return inc_ptr, inc, int(np.diff(row_ptr).max())

    # -- host reference (test infrastructure for the scatter) -------------------
    def assemble_csr_host(self, A: np.ndarray, row_ptr: np.ndarray, col_idx: np.ndarray):
        """Sum of the element matrices into the CSR pattern, on the host (scipy)."""
        import scipy.sparse as sp

        dof, nd = self.dof_map()
        E, n = dof.shape
        rows = np.repeat(dof, n, axis=1).reshape(-1)
        cols = np.tile(dof, (1, n)).reshape(-1)
        S = sp.coo_matrix((A.reshape(-1), (rows, cols)), shape=(nd, nd)).tocsr()
        S.sum_duplicates()
        S = S.tocoo()
        pattern_rows = np.repeat(np.arange(nd, dtype=np.int64), np.diff(row_ptr))
        pkey = pattern_rows * nd + col_idx.astype(np.int64)       # sorted
        skey = S.row.astype(np.int64) * nd + S.col.astype(np.int64)
        at = np.searchsorted(pkey, skey)
        assert np.all(at < pkey.size) and np.array_equal(pkey[np.minimum(at, pkey.size - 1)], skey), \
            "element matrix entries outside the pattern"
        vals = np.zeros(col_idx.size)
        vals[at] = S.data
        return vals


class GlobalAssembler:
    """gather -> femgpu_assemble -> scatter-add on the device, for one config
    mesh: the device-side setup (index maps, CSR pattern, positions) is built
    once; ``assemble(coef)`` then runs the three kernels for a global coefficient
    vector and returns the CSR values (a torch tensor)."""

    def __init__(self, cfg: fe.Config, N: int | None = None, device="cuda:0", form=None):
        import torch

        from . import femgpu

        self.cfg, self.mesh = cfg, GlobalMesh(cfg, N)
        dev = self.dev = torch.device(device)
        g = self.mesh
        dof, self.ndofs = g.dof_map()
        self.fields, cidx, self.ncoef_global = g.coef_layout()
        row_ptr, col_idx, _ = g.csr_pattern()
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
        self.V = t(g.V, np.float64)
        self.cells = t(g.cells, np.int32)
        self.coef_idx = t(cidx, np.int32)
        self.dof = t(dof, np.int32)
        self.row_ptr = t(row_ptr, np.int64)
        self.col_idx = t(col_idx, np.int32)
        E, n = g.E, dof.shape[1]
        self.coords = torch.empty((E, 12), dtype=torch.float64, device=dev)
        self.coeffs = torch.empty((E, max(1, cidx.shape[1])), dtype=torch.float64, device=dev)
        self.A = torch.empty((E, n, n), dtype=torch.float64, device=dev)
        self.pos = torch.empty((E, n, n), dtype=torch.int64, device=dev)
        femgpu.csr_positions(self.dof, self.row_ptr, self.col_idx, self.pos)
        self.vals = torch.zeros(col_idx.size, dtype=torch.float64, device=dev)
        self.form = form if form is not None else femgpu.Form.from_config(cfg)
        self._rows = None

    def row_plan(self):
        """(inc_ptr, inc, loc, max_row_len) of the atomic-free row assembly, built once."""
        if self._rows is None:
            import torch

            from . import femgpu

            inc_ptr, inc, maxlen = self.mesh.row_incidence()
            loc = torch.empty(self.pos.shape, dtype=torch.uint16, device=self.dev)
            femgpu.csr_row_offsets(self.dof, self.row_ptr, self.pos, loc)
            self._rows = (torch.from_numpy(inc_ptr).to(self.dev), torch.from_numpy(inc).to(self.dev),
                          loc, maxlen)
        return self._rows

    def gather(self, coef, stream=None):
        from . import femgpu

        femgpu.gather(self.V, self.cells, coef, self.coef_idx, self.coords, self.coeffs, stream)

    def assemble(self, coef, stream=None, fused: bool = True, mode: str | None = None):
        """CSR values of the global matrix for global coefficient vector ``coef``.
        ``mode`` (default from ``fused``): "fused" -- element kernel and scatter in one
        call (femgpu_assemble_csr); "scatter" -- A_e materialised in ``self.A``, then
        FP64-atomic scatter-add; "rows" -- A_e materialised, then the atomic-free
        row-gather assembly (femgpu_csr_gather_rows; bit-reproducible)."""
        from . import femgpu

        import contextlib

        import torch

        mode = mode or ("fused" if fused else "scatter")
        # every step runs on `stream`, the zeroing of the CSR values included
        # (on torch's current stream it could overlap the atomics)
        ctx = torch.cuda.stream(stream) if isinstance(stream, torch.cuda.Stream) else \
            contextlib.nullcontext()
        if stream is not None and not isinstance(stream, torch.cuda.Stream):
            raise TypeError("stream must be a torch.cuda.Stream or None")
        self.gather(coef, stream)
        if mode == "fused":
            with ctx:
                self.vals.zero_()
            self.form.assemble_csr(self.coords, self.coeffs, self.pos, self.vals, stream=stream)
        elif mode == "scatter":
            with ctx:
                self.vals.zero_()
            self.form.assemble(self.coords, self.coeffs, self.A, stream=stream)
            femgpu.scatter_add(self.A, self.pos, self.vals, stream)
        elif mode == "rows":
            inc_ptr, inc, loc, maxlen = self.row_plan()
            self.form.assemble(self.coords, self.coeffs, self.A, stream=stream)
            femgpu.csr_gather_rows(self.row_ptr, inc_ptr, inc, loc, maxlen, self.A, self.vals,
                                   stream=stream)
        else:
            raise ValueError(f"unknown assembly mode {mode!r}")
        return self.vals
