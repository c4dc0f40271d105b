"""The C-ABI library loads and exports every symbol include/femgpu.h declares.

CPU only: no compute calls.  Also checks the error contract without a GPU
(femopt conventions: int codes, thread-local message, no crash).
"""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1604_05872_b200 import femgpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "femgpu.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(femgpu_[a-z_]+)\s*\(", src)))


def test_library_exists_and_loads():
    assert os.path.exists(femgpu.LIB_PATH), "run __graft_entry__.build()"
    femgpu.lib()


def test_exports_every_declared_symbol():
    names = declared()
    assert set(names) == set(femgpu.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", femgpu.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (femgpu_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", femgpu.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_error_contract_without_device():
    L = femgpu.lib()
    assert femgpu.version().startswith("femgpu")
    # null descriptor -> INVALID_ARG with a message, no crash
    h = C.c_void_p()
    assert L.femgpu_form_create(None, C.byref(h)) == 9
    assert b"null" in L.femgpu_last_error()
    assert L.femgpu_form_create(None, None) == 9
    # bad kind
    d = femgpu.FormDesc()
    d.kind = 99
    assert L.femgpu_form_create(C.byref(d), C.byref(h)) == 9
    # null form to every entry point
    assert L.femgpu_assemble(None, 1, None, None, None, 0, None) == 9
    assert L.femgpu_assemble_host(None, 1, None, None, None, 0) == 9
    assert L.femgpu_kernel_argv(None, 1, None, None, None) == 9
    assert L.femgpu_form_get_info(None, None) == 9
    L.femgpu_form_free(None)  # no-op


def test_form_create_reports_device_errors_cleanly():
    """Valid tables on a box without a GPU: a CUDA/NO_DEVICE code, never a crash."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1604_05872_b200 import fe

    with pytest.raises(femgpu.FemgpuError) as e:
        femgpu.Form.from_config(fe.CONFIGS["c1"])
    assert e.value.code in (12, 13)
