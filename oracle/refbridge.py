"""ctypes bridge to the reference femopt built in oracle/_ref/ -- TEST INFRASTRUCTURE.

Only tests/, oracle/ scripts and bench.py's reference arm may import this.
It drives the reference's own C API (/root/reference/proj/include/femopt.h:44-76,
implemented in proj/src/capi.cpp:67-153) plus the one-function shim
oracle/ref_shim.cpp that exposes ``interpret`` (proj/src/interp.cpp:125-154).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "libfemopt_ref.so")


class FemoptOptions(C.Structure):
    # femopt.h:35-40
    _fields_ = [("memory_limit", C.c_size_t), ("enable_preeval", C.c_int),
                ("enable_zero_skip", C.c_int), ("trace", C.c_int)]


class FemoptError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"femopt error {code}: {msg}")
        self.code = code


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref`")
        L = C.CDLL(LIB_PATH)
        vp, cp = C.c_void_p, C.c_char_p
        L.femopt_options_init.argtypes = [C.POINTER(FemoptOptions)]
        L.femopt_kernel_parse.argtypes = [cp, C.POINTER(vp)]
        L.femopt_kernel_free.argtypes = [vp]
        L.femopt_kernel_flops.argtypes = [vp, C.POINTER(C.c_ulonglong)]
        L.femopt_optimize.argtypes = [vp, C.POINTER(FemoptOptions), C.POINTER(vp), C.POINTER(vp)]
        L.femopt_kernel_to_json.argtypes = [vp, C.POINTER(vp)]
        L.femopt_emit_c.argtypes = [vp, cp, C.POINTER(vp)]
        L.femopt_last_error.restype = cp
        L.femopt_string_free.argtypes = [vp]
        L.refshim_interpret.argtypes = [cp, cp, C.POINTER(C.c_double), C.c_long]
        L.refshim_interpret.restype = C.c_long
        L.refshim_last_error.restype = cp
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise FemoptError(rc, lib().femopt_last_error().decode())


def _take_string(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().femopt_string_free(p)
    return s


class Kernel:
    """Owning handle over a parsed femopt kernel (femopt.h:47-50)."""

    def __init__(self, json_text: str | None = None, _handle=None):
        self.h = C.c_void_p()
        if _handle is not None:
            self.h = _handle
        else:
            _check(lib().femopt_kernel_parse(json_text.encode(), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.femopt_kernel_free(self.h)
            self.h = None

    def flops(self) -> int:
        out = C.c_ulonglong()
        _check(lib().femopt_kernel_flops(self.h, C.byref(out)))
        return out.value

    def optimize(self, memory_limit=262144, preeval=True, zero_skip=False, trace=False):
        opt = FemoptOptions()
        lib().femopt_options_init(C.byref(opt))
        opt.memory_limit, opt.enable_preeval = memory_limit, int(preeval)
        opt.enable_zero_skip, opt.trace = int(zero_skip), int(trace)
        out, rep = C.c_void_p(), C.c_void_p()
        _check(lib().femopt_optimize(self.h, C.byref(opt), C.byref(out), C.byref(rep)))
        import json
        return Kernel(_handle=out), json.loads(_take_string(rep))

    def to_json(self) -> str:
        p = C.c_void_p()
        _check(lib().femopt_kernel_to_json(self.h, C.byref(p)))
        return _take_string(p)

    def emit_c(self, fn="kernel") -> str:
        p = C.c_void_p()
        _check(lib().femopt_emit_c(self.h, fn.encode(), C.byref(p)))
        return _take_string(p)


def interpret(json_text: str, output: str) -> np.ndarray:
    """The reference interpreter's value of ``output`` (interp.cpp:125-154)."""
    L = lib()
    n = L.refshim_interpret(json_text.encode(), output.encode(), None, 0)
    if n < 0:
        raise FemoptError(11, L.refshim_last_error().decode())
    out = np.zeros(n)
    L.refshim_interpret(json_text.encode(), output.encode(),
                        out.ctypes.data_as(C.POINTER(C.c_double)), n)
    return out


# ----------------------------------------------------------------------------
# Emitted C: compile and run (mirrors proj/tests/test_backend.cpp:53-105)
# ----------------------------------------------------------------------------


def argv_wrapper(fn: str, nout: int, ntab: int, nconst: int) -> str:
    """Uniform entry point, as test_backend.cpp:62-73 generates it."""
    args = [f"o[{i}]" for i in range(nout)] + [f"t[{i}]" for i in range(ntab)] + \
        [f"c[{i}]" for i in range(nconst)]
    return (f"\nvoid {fn}_argv(double* const* o, const double* const* t, const double* c) {{\n"
            f"  {fn}({', '.join(args)});\n}}\n")


def compile_c(src: str, so_path: str, flags=("-O3", "-march=native", "-ffp-contract=off")):
    with tempfile.NamedTemporaryFile("w", suffix=".c", delete=False) as f:
        f.write(src)
        cpath = f.name
    try:
        subprocess.run(["cc", *flags, "-shared", "-fPIC", "-o", so_path, cpath, "-lm"],
                       check=True, capture_output=True, text=True)
    finally:
        os.unlink(cpath)
    return so_path
