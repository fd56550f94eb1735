"""ctypes front-end of ``certify.c`` -- the e_float certificate.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

``relu_err`` is the quantity of Eq. (comp:error-approx).  The paper prints
2 x that value under Tables 1-2 (reading R3), so
``paper_convention`` returns max|x s(x) - |x|| = 2 relu_err.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "certify.c")
_LIB = os.path.join(_HERE, "_certify.so")
_lib = None


def build():
    """Compile certify.c (gcc, -O2 -fopenmp, no fast-math) if stale."""
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.certify_relu_err.restype = ctypes.c_double
        lib.certify_relu_err.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)]
        lib.certify_sign_err.restype = ctypes.c_double
        lib.certify_sign_err.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
        lib.certify_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _pack(stages, kappas):
    ncoef = np.array([len(c) for c in stages], dtype=np.int32)
    coeffs = np.array([v for c in stages for v in c], dtype=np.float64)
    k = None if kappas is None else np.array(kappas, dtype=np.float64)
    return ncoef, coeffs, k


def relu_err(stages, kappas=None):
    """(max_{x in S_float} |1/2 x (1+s(x)) - relu(x)|, argmax |x|, |S_float|)."""
    lib = _load()
    ncoef, coeffs, k = _pack(stages, kappas)
    am = ctypes.c_double()
    cnt = ctypes.c_longlong()
    e = lib.certify_relu_err(len(stages), ncoef.ctypes.data, coeffs.ctypes.data,
                             None if k is None else k.ctypes.data, ctypes.byref(am), ctypes.byref(cnt))
    return e, am.value, cnt.value


def paper_convention(stages, kappas=None):
    """The value Tables 1-2 print: max|x s(x) - |x|| = 2 relu_err (reading R3)."""
    return 2.0 * relu_err(stages, kappas)[0]


def sign_err(stages, eps, kappas=None):
    """max over float32 x in [eps, 1] of |s(x) - 1|."""
    lib = _load()
    ncoef, coeffs, k = _pack(stages, kappas)
    am = ctypes.c_double()
    e = lib.certify_sign_err(len(stages), ncoef.ctypes.data, coeffs.ctypes.data,
                             None if k is None else k.ctypes.data, float(eps), ctypes.byref(am))
    return e, am.value


def num_threads():
    return _load().certify_num_threads()
