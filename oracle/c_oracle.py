"""Oracle (TEST INFRASTRUCTURE): ctypes wrapper of oracle/wagma_oracle.c.

Used by tests/ (checked bit-exact against wagma_oracle.py) and by bench.py's
CPU-baseline leg only -- see oracle/__init__.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle_wagma.so")

_lib: Optional[ctypes.CDLL] = None


def build() -> str:
    """Compile the C oracle with its Makefile (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        for suffix, ct in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            fn = getattr(lib, f"oracle_wagma_iteration_{suffix}")
            pp = ctypes.POINTER(ctypes.c_void_p)
            fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                           ctypes.c_longlong, ct, ct, ctypes.c_int, pp, pp, pp, pp, pp,
                           ctypes.POINTER(ctypes.c_int), ctypes.c_int]
            fn.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(load().oracle_max_threads())


def _ptrs(arrs: Optional[Sequence[Optional[np.ndarray]]], P: int):
    arr = (ctypes.c_void_p * P)()
    if arrs is None:
        return arr
    for i, a in enumerate(arrs):
        arr[i] = None if a is None else a.ctypes.data
    return arr


def wagma_iteration(W: Sequence[np.ndarray], m: Optional[Sequence[np.ndarray]], g: Sequence[np.ndarray],
                    wprime: Sequence[np.ndarray], masks: Sequence[int], divisor: int, eta: float,
                    beta: float, momentum: bool, contrib: Optional[Sequence[Optional[np.ndarray]]] = None,
                    timely: Optional[Sequence[bool]] = None, nthreads: int = 0) -> None:
    """One iteration for P ranks, in place on W (and m), W' into `wprime`.

    contrib[q] (optional) is rank q's send-buffer snapshot for this version
    (None = its fresh W'); timely[q] selects acc/S versus (acc+W')/(S+1).
    """
    P = len(W)
    dt = W[0].dtype
    for arrs in (W, g, wprime) + ((m,) if momentum else ()):
        for a in arrs:
            assert a.dtype == dt and a.flags.c_contiguous
    lib = load()
    fn = lib.oracle_wagma_iteration_f32 if dt == np.float32 else lib.oracle_wagma_iteration_f64
    cmasks = (ctypes.c_int * max(1, len(masks)))(*masks)
    ctimely = None
    if timely is not None:
        ctimely = (ctypes.c_int * P)(*[1 if x else 0 for x in timely])
    rc = fn(P, divisor, cmasks, len(masks), W[0].size, eta, beta, 1 if momentum else 0,
            _ptrs(W, P), _ptrs(m if momentum else None, P), _ptrs(g, P), _ptrs(wprime, P),
            _ptrs(contrib, P) if contrib is not None else None, ctimely,
            nthreads if nthreads > 0 else max_threads())
    if rc != 0:
        raise RuntimeError(f"oracle_wagma_iteration failed rc={rc}")
