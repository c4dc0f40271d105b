"""Any femopt kernel IR on the B200 -- Python face of the
C ABI's ``femgpu_ir_*`` entry points (csrc/ir_backend.cpp, include/femgpu.h).

The reference's only backend is ``emit_c`` (/root/reference/proj/src/emit_c.cpp:
108-174): a C function ``fn(double* outputs..., const double* input tables...,
double constants...)`` (each group in name order, :137-140) with pre-evaluated
tables baked in and outputs accumulated with ``+=``.  ``femgpu_ir_create``
generates the GPU counterpart of that function from the same IR -- raw kernels
of ir.py, or femopt's optimized ``to_json`` output -- and compiles it with
NVRTC for sm_100a:

  * the order-free element loop becomes the grid: one thread per cell, or one
    warp per cell with the output rows over the lanes and register
    accumulators (warp whenever the row loop has >= 8 rows: measured faster);
  * expressions are printed exactly as emit_c prints them and compiled without
    FMA contraction, so the results are bit-identical to femopt's emitted C
    (``-ffp-contract=off``) on the same inputs;
  * arity 1 (element vectors) and arity 2 (element matrices) alike.

The hand-written kernels of csrc/ stay the fast path for the BASELINE forms;
this is the generic one.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import femgpu

STRATEGIES = {"auto": 0, "thread": 1, "warp": 2, "gemm": 3}


class IRError(ValueError):
    """The IR is not an emittable femopt kernel (FEMGPU_ERR_NOT_FEM_NEST)."""


class FemgpuIRInfo(C.Structure):
    _fields_ = [("noutputs", C.c_int), ("ninputs", C.c_int), ("nconstants", C.c_int),
                ("per_cell", C.c_int), ("strategy", C.c_int)]


def _lib():
    L = femgpu.lib()
    if not getattr(L, "_ir_ready", False):
        vp = C.c_void_p
        L.femgpu_ir_create.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        L.femgpu_ir_free.argtypes = [vp]
        L.femgpu_ir_free.restype = None
        L.femgpu_ir_get_info.argtypes = [vp, C.POINTER(FemgpuIRInfo)]
        L.femgpu_ir_argname.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.femgpu_ir_arg_size.argtypes = [vp, C.c_int, C.c_int, C.c_long, C.POINTER(C.c_long)]
        L.femgpu_ir_source.argtypes = [vp]
        L.femgpu_ir_source.restype = C.c_char_p
        L.femgpu_ir_launch.argtypes = [vp, C.c_long, C.POINTER(vp), C.POINTER(vp),
                                       C.POINTER(C.c_double), vp]
        L.femgpu_ir_argv.argtypes = [vp, C.c_long, C.POINTER(C.POINTER(C.c_double)),
                                     C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_double)]
        L._ir_ready = True
    return L


def _check(rc: int):
    if rc == 3:  # FEMGPU_ERR_NOT_FEM_NEST
        raise IRError(_lib().femgpu_last_error().decode())
    if rc != 0:
        raise femgpu.FemgpuError(rc, _lib().femgpu_last_error().decode())


class IRKernel:
    """A femopt kernel IR compiled for the B200 (``femgpu_ir_create``)."""

    def __init__(self, ir: dict | str, strategy: str = "auto"):
        text = ir if isinstance(ir, str) else json.dumps(ir)
        L = _lib()
        h = C.c_void_p()
        _check(L.femgpu_ir_create(text.encode(), STRATEGIES[strategy], C.byref(h)))
        self.h = h
        inf = FemgpuIRInfo()
        _check(L.femgpu_ir_get_info(h, C.byref(inf)))
        self.per_cell = bool(inf.per_cell)
        self.strategy = {1: "thread", 2: "warp", 3: "gemm"}[inf.strategy]
        self.outputs = [self._name(0, i) for i in range(inf.noutputs)]
        self.inputs = [self._name(1, i) for i in range(inf.ninputs)]
        self.constants = [self._name(2, i) for i in range(inf.nconstants)]

    def _name(self, group, i):
        buf = C.create_string_buffer(256)
        _check(_lib().femgpu_ir_argname(self.h, group, i, buf, 256))
        return buf.value.decode()

    def close(self):
        if getattr(self, "h", None):
            _lib().femgpu_ir_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def source(self) -> str:
        return _lib().femgpu_ir_source(self.h).decode()

    def size(self, group: int, name: str, ncells: int) -> int:
        names = self.outputs if group == 0 else self.inputs
        n = C.c_long()
        _check(_lib().femgpu_ir_arg_size(self.h, group, names.index(name), int(ncells),
                                         C.byref(n)))
        return n.value

    # -- device ---------------------------------------------------------------
    def run(self, outputs: dict, inputs: dict, constants: dict | None, ncells: int,
            stream=None) -> None:
        """Device tensors by name (float64, contiguous); outputs accumulate (+=)."""
        constants = constants or {}
        for group, names, arrs in ((0, self.outputs, outputs), (1, self.inputs, inputs)):
            for n in names:
                t = arrs[n]
                if t.numel() != self.size(group, n, ncells):
                    raise ValueError(f"{n}: {t.numel()} values, need {self.size(group, n, ncells)}")
        o = (C.c_void_p * max(1, len(self.outputs)))(*[outputs[n].data_ptr() for n in self.outputs])
        i = (C.c_void_p * max(1, len(self.inputs)))(*[inputs[n].data_ptr() for n in self.inputs])
        c = (C.c_double * max(1, len(self.constants)))(*[float(constants[n])
                                                         for n in self.constants])
        s = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        if s is None:
            import torch

            s = torch.cuda.current_stream().cuda_stream
        _check(_lib().femgpu_ir_launch(self.h, int(ncells), o, i, c, s))

    # -- host (emit_c's argv convention) --------------------------------------
    def argv(self, outputs: list, inputs: list, constants: list | None, ncells: int) -> None:
        outs = [np.ascontiguousarray(a, dtype=np.float64) for a in outputs]
        ins = [np.ascontiguousarray(a, dtype=np.float64) for a in inputs]
        dp = C.POINTER(C.c_double)
        o = (dp * max(1, len(outs)))(*[a.ctypes.data_as(dp) for a in outs])
        t = (dp * max(1, len(ins)))(*[a.ctypes.data_as(dp) for a in ins])
        cv = np.asarray(list(constants or []) or [0.0], dtype=np.float64)
        _check(_lib().femgpu_ir_argv(self.h, int(ncells), o, t, cv.ctypes.data_as(dp)))
        for a, b in zip(outputs, outs):
            if a is not b:
                a.reshape(-1)[:] = b.reshape(-1)

    def run_ir_tables(self, ir: dict | str) -> dict:
        """Run on the tables embedded in the IR (femopt IRs carry their data),
        outputs starting from zero; returns numpy arrays by name."""
        d = json.loads(ir) if isinstance(ir, str) else ir
        E = int(d["indices"].get("e", 1)) if self.per_cell else 1
        tabs = d.get("tables", {})
        outs = [np.zeros(self.size(0, n, E)) for n in self.outputs]
        ins = [np.asarray(tabs[n]["values"], dtype=np.float64) for n in self.inputs]
        consts = [float(d["constants"][n]) for n in self.constants]
        self.argv(outs, ins, consts, E)
        return dict(zip(self.outputs, outs))
