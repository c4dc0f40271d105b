"""Host mirror of the femgpu C ABI (include/femgpu.h) -- ctypes, no torch types.

This is the Python face of the drop-in boundary.  It mirrors the reference's
two interfaces for the element-kernel path:

* libfemopt's library conventions (/root/reference/proj/include/femopt.h):
  int return codes 0..11 with femopt's meanings, a thread-local last-error
  message, handle objects that own native state -> ``FemgpuError`` carrying
  ``.code`` and the native message, ``Form`` owning a ``femgpu_form*``;
* the emitted element kernel `void kernel(double* outputs..., const double*
  tables..., double constants...)` called through the harness's uniform
  `kernel_argv(o, t, c)` (proj/tests/test_backend.cpp:62-98) ->
  ``Form.kernel_argv`` with the same argument order (emit_c.cpp:137-140) and
  the same `+=` semantics.

The CUDA path is the only path: if ``libfemgpu.so`` is missing this module
raises at load time; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import fe

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfemgpu.so")

SCHED_AUTO, SCHED_TENSOR, SCHED_QUADRATURE, SCHED_QUADRATURE_MMA = 0, 1, 2, 3
SCHEDULE_NAMES = {SCHED_AUTO: "auto", SCHED_TENSOR: "tensor", SCHED_QUADRATURE: "quadrature",
                  SCHED_QUADRATURE_MMA: "quadrature_mma"}

ERROR_NAMES = {
    0: "OK", 1: "PARSE", 2: "UNKNOWN_LOOP", 3: "NOT_FEM_NEST", 4: "NON_DISTRIBUTABLE",
    5: "NON_SEPARABLE", 6: "NOT_NORMAL_FORM", 7: "TOO_MANY_MONOMIALS", 8: "INCONSISTENT_LAYOUT",
    9: "INVALID_ARG", 10: "IO", 11: "INTERNAL", 12: "CUDA", 13: "NO_DEVICE", 14: "UNSUPPORTED",
}

# Every symbol include/femgpu.h declares (checked by tests/test_abi.py).
EXPORTS = ("femgpu_form_create", "femgpu_form_free", "femgpu_form_get_info",
           "femgpu_form_schedules", "femgpu_assemble",
           "femgpu_assemble_vector",
           "femgpu_assemble_host", "femgpu_kernel_argv", "femgpu_kernel_argc",
           "femgpu_kernel_argname", "femgpu_gather", "femgpu_csr_positions",
           "femgpu_scatter_add", "femgpu_csr_row_offsets", "femgpu_csr_gather_rows", "femgpu_assemble_csr", "femgpu_ir_create", "femgpu_ir_free", "femgpu_ir_get_info",
           "femgpu_ir_argname", "femgpu_ir_arg_size", "femgpu_ir_source", "femgpu_ir_launch",
           "femgpu_ir_argv", "femgpu_last_error", "femgpu_version")


class FemgpuError(RuntimeError):
    """A non-zero femgpu return code (femopt.h:20-33 meanings for 1..11)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"femgpu error {code} ({ERROR_NAMES.get(code, '?')}): {message}")
        self.code = code
        self.message = message


class FormDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("nq", C.c_int), ("ns", C.c_int), ("nc", C.c_int),
                ("W", C.POINTER(C.c_double)), ("B", C.POINTER(C.c_double)),
                ("D", C.POINTER(C.c_double)), ("P", C.POINTER(C.c_double)),
                ("consts", C.c_double * 4), ("schedule", C.c_int)]


class ScheduleInfo(C.Structure):
    _fields_ = [("kernel_name", C.c_char * 64), ("schedule", C.c_int), ("pipe", C.c_int),
                ("flops_per_cell", C.c_double), ("bytes_per_cell", C.c_double),
                ("peak_flops", C.c_double), ("peak_bytes", C.c_double),
                ("efficiency", C.c_double), ("predicted_ns_per_cell", C.c_double),
                ("chosen", C.c_int)]


class FormInfo(C.Structure):
    _fields_ = [("n", C.c_int), ("ncoef", C.c_int), ("schedule", C.c_int),
                ("flops_per_cell", C.c_double), ("bytes_per_cell", C.c_double),
                ("kernels_per_launch", C.c_int), ("kernel_name", C.c_char * 64)]


_lib = None


def lib():
    """Load libfemgpu.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ "
                                    "as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, dp = C.c_void_p, C.POINTER(C.c_double)
        L.femgpu_form_create.argtypes = [C.POINTER(FormDesc), C.POINTER(vp)]
        L.femgpu_form_free.argtypes = [vp]
        L.femgpu_form_free.restype = None
        L.femgpu_form_get_info.argtypes = [vp, C.POINTER(FormInfo)]
        L.femgpu_form_schedules.argtypes = [C.POINTER(FormDesc), C.POINTER(ScheduleInfo), C.c_int,
                                            C.POINTER(C.c_int)]
        L.femgpu_assemble.argtypes = [vp, C.c_long, vp, vp, vp, C.c_int, vp]
        L.femgpu_assemble_vector.argtypes = [vp, C.c_long, vp, vp, vp, C.c_int, vp]
        L.femgpu_assemble_host.argtypes = [vp, C.c_long, dp, dp, dp, C.c_int]
        L.femgpu_kernel_argv.argtypes = [vp, C.c_long, C.POINTER(dp), C.POINTER(dp), dp]
        L.femgpu_kernel_argc.argtypes = [vp, C.c_int, C.POINTER(C.c_int)]
        L.femgpu_kernel_argname.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.femgpu_last_error.restype = C.c_char_p
        L.femgpu_version.restype = C.c_char_p
        L.femgpu_gather.argtypes = [C.c_long, C.c_int, vp, vp, vp, vp, vp, vp, vp]
        L.femgpu_csr_positions.argtypes = [C.c_long, C.c_int, vp, vp, vp, vp, vp]
        L.femgpu_scatter_add.argtypes = [C.c_long, vp, vp, vp, vp]
        L.femgpu_csr_row_offsets.argtypes = [C.c_long, C.c_int, vp, vp, vp, vp, vp]
        L.femgpu_csr_gather_rows.argtypes = [C.c_long, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp,
                                             C.c_int, vp]
        L.femgpu_assemble_csr.argtypes = [vp, C.c_long, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise FemgpuError(rc, lib().femgpu_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _devptr(x):
    """Device pointer of a torch CUDA tensor (or an int)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _invalid(msg: str):
    raise FemgpuError(9, msg)


def _check_dev(t, name: str, rows: int, per_row: int, dtype: str = "float64"):
    """Validate a device tensor before its pointer reaches native code: CUDA,
    ``dtype``, C-contiguous, >= ``rows`` rows of ``per_row`` elements.  Raw
    integer pointers pass through unchecked (the caller vouches for them)."""
    if t is None or isinstance(t, int):
        return
    import torch

    if not isinstance(t, torch.Tensor):
        _invalid(f"{name}: expected a torch CUDA tensor or a raw device pointer")
    if not t.is_cuda:
        _invalid(f"{name}: tensor is not on a CUDA device")
    if t.dtype != getattr(torch, dtype):
        _invalid(f"{name}: dtype {t.dtype}, expected torch.{dtype}")
    if not t.is_contiguous():
        _invalid(f"{name}: tensor must be C-contiguous")
    if rows > 0 and (t.dim() == 0 or t.shape[0] < rows or t.numel() < rows * per_row):
        _invalid(f"{name}: shape {tuple(t.shape)} holds fewer than {rows} x {per_row} elements")
    if rows > 0 and t.numel() != t.shape[0] * per_row:
        _invalid(f"{name}: {tuple(t.shape)[1:]} per row, expected {per_row} elements")


def _check_host(a, name: str, rows: int, per_row: int):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        _invalid(f"{name}: expected a C-contiguous float64 numpy array")
    if a.size < rows * per_row or (rows > 0 and a.size != a.shape[0] * per_row):
        _invalid(f"{name}: shape {a.shape}, expected [{rows}] x {per_row} elements")


def _desc(kind: int, tables: "fe.Tables", consts=(), schedule: int = SCHED_AUTO):
    """A femgpu_form_desc over (kept-alive) contiguous copies of the tables."""
    keep = [np.ascontiguousarray(tables.W, dtype=np.float64),
            np.ascontiguousarray(tables.B, dtype=np.float64),
            np.ascontiguousarray(tables.D, dtype=np.float64),
            np.ascontiguousarray(tables.P, dtype=np.float64)]
    W, B, D, P = keep
    d = FormDesc()
    d.kind, d.nq, d.ns, d.nc = kind, W.shape[0], B.shape[1], P.shape[1]
    d.W, d.B, d.D, d.P = _dptr(W), _dptr(B), _dptr(D), _dptr(P)
    cs = list(consts) + [0.0] * (4 - len(consts))
    d.consts = (C.c_double * 4)(*cs)
    d.schedule = schedule
    return d, keep


def schedules(cfg: "fe.Config", tables: "fe.Tables | None" = None,
              schedule: int = SCHED_AUTO) -> list[dict]:
    """The kernels available for a config's form, ranked by the library's cost model
    (femgpu_form_schedules: roofline time on the current device / measured efficiency,
    fastest first; ``chosen`` marks the one ``schedule`` selects)."""
    d, _keep = _desc(cfg.kind, tables or fe.tables(cfg), cfg.consts, schedule)
    out = (ScheduleInfo * 8)()
    n = C.c_int()
    _check(lib().femgpu_form_schedules(C.byref(d), out, 8, C.byref(n)))
    res = []
    for i in range(min(n.value, 8)):
        o = out[i]
        res.append({"kernel": o.kernel_name.decode(), "schedule": SCHEDULE_NAMES[o.schedule],
                    "pipe": "DMMA" if o.pipe else "DFMA", "flops_per_cell": o.flops_per_cell,
                    "bytes_per_cell": o.bytes_per_cell, "peak_flops": o.peak_flops,
                    "peak_bytes": o.peak_bytes, "efficiency": o.efficiency,
                    "predicted_ns_per_cell": o.predicted_ns_per_cell, "chosen": bool(o.chosen)})
    return res


class Form:
    """A femgpu form (element-kernel family) bound to the current CUDA device."""

    def __init__(self, kind: int, tables: "fe.Tables", consts=(), schedule: int = SCHED_AUTO):
        self.kind = kind
        d, self._keep = _desc(kind, tables, consts, schedule)
        self.h = C.c_void_p()
        _check(lib().femgpu_form_create(C.byref(d), C.byref(self.h)))
        inf = FormInfo()
        _check(lib().femgpu_form_get_info(self.h, C.byref(inf)))
        self.n, self.ncoef = inf.n, inf.ncoef
        self.info = {"n": inf.n, "ncoef": inf.ncoef, "schedule": SCHEDULE_NAMES[inf.schedule],
                     "flops_per_cell": inf.flops_per_cell, "bytes_per_cell": inf.bytes_per_cell,
                     "kernels_per_launch": inf.kernels_per_launch,
                     "kernel_name": inf.kernel_name.decode()}

    @classmethod
    def from_config(cls, cfg: "fe.Config", tables: "fe.Tables | None" = None,
                    schedule: int = SCHED_AUTO) -> "Form":
        return cls(cfg.kind, tables or fe.tables(cfg), cfg.consts, schedule)

    def close(self):
        if getattr(self, "h", None):
            lib().femgpu_form_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_io(self, coords, coeffs, out, E, per_out):
        if E < 0:
            return  # the library reports it (FEMGPU_ERR_INVALID_ARG)
        _check_dev(coords, "coords", E, 12)
        if self.ncoef > 0:
            _check_dev(coeffs, "coeffs", E, self.ncoef)
        if out is not None:
            _check_dev(out, "out", E, per_out)

    # -- device path (the hot path) ------------------------------------------
    def assemble(self, coords, coeffs, out, ncells: int | None = None, accumulate: bool = False,
                 stream=None):
        """Element matrices into ``out`` (device tensors; cell-major layouts)."""
        E = int(coords.shape[0]) if ncells is None else int(ncells)
        self._check_io(coords, coeffs, out, E, self.n * self.n)
        s = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        _check(lib().femgpu_assemble(self.h, E, _devptr(coords), _devptr(coeffs), _devptr(out),
                                     int(accumulate), s))

    def assemble_vector(self, coords, coeffs, out, ncells: int | None = None,
                        accumulate: bool = False, stream=None):
        """Element vectors [E][n] of the form's family into ``out`` (device tensors):
        Helmholtz load, St Venant--Kirchhoff / Burgers residual (femgpu_assemble_vector)."""
        E = int(coords.shape[0]) if ncells is None else int(ncells)
        self._check_io(coords, coeffs, out, E, self.n)
        s = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        _check(lib().femgpu_assemble_vector(self.h, E, _devptr(coords), _devptr(coeffs),
                                            _devptr(out), int(accumulate), s))

    def assemble_csr(self, coords, coeffs, pos, vals, ncells: int | None = None, stream=None):
        """Element matrices straight into CSR values: vals[pos] += A_e (device tensors;
        pos from csr_positions).  Fused into the element kernel where it has a
        CSR epilogue (Helmholtz), else kernel + scatter-add."""
        E = int(coords.shape[0]) if ncells is None else int(ncells)
        self._check_io(coords, coeffs, None, E, 0)
        _check_dev(pos, "pos", E, self.n * self.n, "int64")
        _check_dev(vals, "vals", 0, 1)
        s = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        _check(lib().femgpu_assemble_csr(self.h, E, _devptr(coords), _devptr(coeffs),
                                         _devptr(pos), _devptr(vals), s))

    # -- host path (end to end) ----------------------------------------------
    def assemble_host(self, coords: np.ndarray, coeffs: np.ndarray, out: np.ndarray | None = None,
                      accumulate: bool = False) -> np.ndarray:
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        E = coords.shape[0]
        _check_host(coords, "coords", E, 12)
        if self.ncoef > 0:
            _check_host(coeffs, "coeffs", E, self.ncoef)
        if out is None:
            out = np.zeros((E, self.n, self.n))
        _check_host(out, "out", E, self.n * self.n)
        _check(lib().femgpu_assemble_host(self.h, E, _dptr(coords), _dptr(coeffs), _dptr(out),
                                          int(accumulate)))
        return out

    def assemble_host_ptr(self, E: int, coords_ptr: int, coeffs_ptr: int, out_ptr: int,
                          accumulate: bool = False):
        """Same with raw host pointers (pinned torch tensors in bench.py)."""
        dp = C.POINTER(C.c_double)
        _check(lib().femgpu_assemble_host(self.h, E, C.cast(coords_ptr, dp), C.cast(coeffs_ptr, dp),
                                          C.cast(out_ptr, dp), int(accumulate)))

    # -- emitted-C interface (femopt's element kernel signature) ---------------
    def argnames(self):
        out = []
        for group in range(3):
            cnt = C.c_int()
            _check(lib().femgpu_kernel_argc(self.h, group, C.byref(cnt)))
            names = []
            buf = C.create_string_buffer(64)
            for i in range(cnt.value):
                _check(lib().femgpu_kernel_argname(self.h, group, i, buf, 64))
                names.append(buf.value.decode())
            out.append(names)
        return tuple(out)

    def kernel_argv(self, ncells: int, outputs, tables, constants=()):
        """Call like the emitted C: outputs += kernel(tables, constants)."""
        onames, tnames, cnames = self.argnames()
        if len(outputs) != len(onames) or len(tables) != len(tnames) or \
                len(constants) != len(cnames):
            _invalid(f"kernel_argv takes {len(onames)} outputs, {len(tnames)} tables and "
                     f"{len(cnames)} constants; got {len(outputs)}, {len(tables)}, "
                     f"{len(constants)}")
        per = self.n * self.n // len(onames)  # Burgers: nine (ns x ns) blocks
        for o, name in zip(outputs, onames):
            if not isinstance(o, np.ndarray) or o.dtype != np.float64 or \
                    not o.flags.c_contiguous or not o.flags.writeable:
                _invalid(f"output {name}: expected a writeable C-contiguous float64 array "
                         "(updated in place)")
            if o.size < ncells * per:
                _invalid(f"output {name}: {o.size} doubles, needs {ncells} x {per}")
        outs = list(outputs)
        tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in tables]
        for t, name in zip(tabs, tnames):
            is_e = name[0] == "x" or name[:1] in ("f", "u", "w") or name[:2] == "mu" or \
                name[:3] == "lam"
            if is_e and t.size < ncells:
                _invalid(f"table {name}: {t.size} values, needs {ncells} (one per cell)")
        cons = np.ascontiguousarray(list(constants) or [0.0], dtype=np.float64)
        dp = C.POINTER(C.c_double)
        op = (dp * len(outs))(*[_dptr(o) for o in outs])
        tp = (dp * len(tabs))(*[_dptr(t) for t in tabs])
        _check(lib().femgpu_kernel_argv(self.h, ncells, op, tp, _dptr(cons)))


def version() -> str:
    return lib().femgpu_version().decode()


# ----------------------------------------------------------------------------
# either side of the path: gather, symbolic and numeric global assembly
# (device tensors; see include/femgpu.h and mesh.py)
# ----------------------------------------------------------------------------
def _stream(stream):
    return None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)


def gather(V, cells, coef, coef_idx, coords, coeffs, stream=None):
    """coords[e] = V[cells[e]], coeffs[e][s] = coef[coef_idx[e][s]] (int32 index maps)."""
    E, ncoef = int(cells.shape[0]), int(coef_idx.shape[1]) if coef_idx is not None else 0
    _check(lib().femgpu_gather(E, ncoef, _devptr(V), _devptr(cells), _devptr(coef),
                               _devptr(coef_idx), _devptr(coords), _devptr(coeffs),
                               _stream(stream)))


def csr_positions(dof_map, row_ptr, col_idx, pos, stream=None):
    """pos[e][j][k] = CSR position of (dof_map[e][j], dof_map[e][k]) (synchronizes)."""
    E, n = int(dof_map.shape[0]), int(dof_map.shape[1])
    _check(lib().femgpu_csr_positions(E, n, _devptr(dof_map), _devptr(row_ptr), _devptr(col_idx),
                                      _devptr(pos), _stream(stream)))


def scatter_add(A, pos, vals, stream=None):
    """vals[pos[i]] += A[i] over all element-matrix entries."""
    _check(lib().femgpu_scatter_add(int(A.numel()), _devptr(A), _devptr(pos), _devptr(vals),
                                    _stream(stream)))


def csr_row_offsets(dof_map, row_ptr, pos, loc, stream=None):
    """loc[e][j][k] = pos[e][j][k] - row_ptr[dof_map[e][j]] as uint16 (synchronizes)."""
    E, n = int(dof_map.shape[0]), int(dof_map.shape[1])
    _check(lib().femgpu_csr_row_offsets(E, n, _devptr(dof_map), _devptr(row_ptr), _devptr(pos),
                                        _devptr(loc), _stream(stream)))


def csr_gather_rows(row_ptr, inc_ptr, inc, loc, max_row_len, A, vals, accumulate=False,
                    stream=None):
    """Atomic-free numeric assembly: vals[row r] (=|+=) sum of the element-matrix rows
    inc[inc_ptr[r]:inc_ptr[r+1]] placed by loc (one warp per row, fixed order)."""
    nrows, n = int(row_ptr.shape[0]) - 1, int(A.shape[-1])
    _check(lib().femgpu_csr_gather_rows(nrows, n, _devptr(row_ptr), _devptr(inc_ptr), _devptr(inc),
                                        _devptr(loc), int(max_row_len), _devptr(A), _devptr(vals),
                                        int(accumulate), _stream(stream)))
