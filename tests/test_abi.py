"""The C-ABI library loads and exports every symbol include/wagma_b200.h declares.

CPU only: no device compute is called here (the schedule generator is host
code); the context entry points are only resolved, plus argument validation
that fails before touching CUDA.
"""

import ctypes
import os
import re
import subprocess

from conftest import ROOT
from paper_2005_00124_b200 import _build, _lib


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "wagma_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|char\s*\*|const char\s*\*)\s*\*?\s*(wg_\w+)\s*\(",
                                 src, flags=re.M)))


def test_header_declares_the_bound_symbols():
    decl = declared_symbols()
    assert len(decl) >= 20
    assert sorted(_lib.SIGNATURES) == decl


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_build.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (wg_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_strings_and_validation_without_gpu():
    lib = _lib.load()
    assert lib.wg_strerror(_lib.WG_ESTALE).decode().startswith("stale")
    assert lib.wg_strerror(_lib.WG_ESYNC).decode() == "mismatched sync points"
    assert lib.wg_strerror(_lib.WG_EDIVERGE).decode().startswith("non-finite")
    # every code the header defines has a message and a Python constant
    import os
    hdr = open(os.path.join(os.path.dirname(_build.HERE), "include", "wagma_b200.h")).read()
    for name, val in re.findall(r"#define (WG_E[A-Z]+) (\d+)", hdr):
        assert getattr(_lib, name) == int(val), name
        assert lib.wg_strerror(int(val)).decode() != "unknown error", name
    # invalid configs are rejected before any CUDA call
    cfg = _lib.WgConfig()
    cfg.P, cfg.S, cfg.n_gpus, cfg.n = 6, 2, 1, 10
    h = ctypes.c_void_p()
    assert lib.wg_ctx_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.WG_EINVAL
    cfg.P, cfg.S, cfg.n_gpus = 8, 16, 1
    assert lib.wg_ctx_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.WG_EINVAL
    cfg.P, cfg.S, cfg.n_gpus = 8, 4, 3
    assert lib.wg_ctx_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.WG_EINVAL
    assert lib.wg_launch(None, None, 0, None, None, 0, None) == _lib.WG_EINVAL
