"""ctypes binding of the CPU oracle (liboracle.so) -- TEST INFRASTRUCTURE ONLY.

Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg as the checker; never by the product path.  See the
header of fftmech_oracle.cpp for what is restated and how it is pinned.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OrReport(C.Structure):
    _fields_ = [("n_passes", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("pad_", C.c_int32), ("err_node", C.c_int64), ("err_value", C.c_double),
                ("eq_rel", C.c_double), ("drift", C.c_double), ("wall", C.c_double),
                ("cg_it", C.c_int32 * 64), ("cg_rel", C.c_double * 64),
                ("rel_update", C.c_double * 64)]

    def as_dict(self):
        n = self.n_passes
        return {"passes": n, "converged": bool(self.converged), "status": self.status,
                "cg_it": list(self.cg_it[:n]), "cg_rel": list(self.cg_rel[:n]),
                "rel_update": list(self.rel_update[:n]), "eq_rel": self.eq_rel,
                "drift": self.drift, "wall": self.wall, "err_node": self.err_node}


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "fftmech_oracle.cpp"))):
            build()
        L = C.CDLL(_LIB_PATH)
        L.or_apply_projection.argtypes = [C.c_int, _ip, _dp, C.c_int, C.c_int, _dp, _dp,
                                          C.POINTER(C.c_double)]
        L.or_ghat.argtypes = [C.c_int, _ip, _dp, C.c_int, C.c_int, _dp]
        L.or_apply_projected_tangent.argtypes = [C.c_int, _ip, _dp, C.c_int, C.c_int, _dp, _dp, _dp]
        L.or_fft.argtypes = [C.c_int, _ip, C.c_int, C.c_int, _dp]
        L.or_hyper_evaluate.argtypes = [C.c_int64, C.c_int, _dp, _dp, _dp, _dp, C.c_void_p,
                                        C.POINTER(C.c_int64)]
        L.or_equivalent_stress.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_void_p, _dp, _dp,
                                           C.POINTER(C.c_int64)]
        L.or_simo_evaluate.argtypes = [C.c_int64] + [_dp] * 8 + [_dp, C.c_void_p, _dp, _dp,
                                                                  C.POINTER(C.c_int64),
                                                                  C.POINTER(C.c_double)]
        L.or_sym_eig3.argtypes = [_dp, _dp, _dp]
        L.or_cg_solve.argtypes = [C.c_int, _ip, _dp, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                  C.c_int, _dp, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.or_run_program.argtypes = [C.c_int, _ip, _dp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp,
                                     _dp, C.c_int, _dp, C.c_double, C.c_double, C.c_int, C.c_int,
                                     _dp, _dp, C.c_void_p, C.POINTER(OrReport)]
        L.or_time_projected_tangent.argtypes = [C.c_int, _ip, _dp, C.c_int, _dp, _dp, _dp, C.c_int]
        L.or_time_projected_tangent.restype = C.c_double
        L.or_set_threads.argtypes = [C.c_int]
        L.or_set_threads.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n=None):
    """Worker threads of the oracle's parallel loops (None = all host cores).
    Output is bit-identical for every thread count: only independent lines,
    nodes and vector entries are split, all reductions stay sequential."""
    return lib().or_set_threads(int(n) if n else (os.cpu_count() or 1))


def _grid(points, lengths=None):
    dim = len(points)
    pts = np.ones(3, dtype=np.int32)
    pts[:dim] = points
    ln = np.ones(3)
    if lengths is not None:
        ln[:dim] = lengths
    return dim, pts, ln


def apply_projection(points, tdim, A, mode=0, lengths=None):
    """Returns (G*A, status, residue)."""
    dim, pts, ln = _grid(points, lengths)
    A = np.ascontiguousarray(A, dtype=np.float64).reshape(-1)
    out = np.empty_like(A)
    res = C.c_double(0.0)
    st = lib().or_apply_projection(dim, pts, ln, tdim, mode, A, out, C.byref(res))
    return out, st, res.value


def ghat(points, tdim, mode=0, lengths=None):
    dim, pts, ln = _grid(points, lengths)
    out = np.empty(tdim * tdim * int(np.prod(points)))
    lib().or_ghat(dim, pts, ln, tdim, mode, out)
    return out


def apply_projected_tangent(points, tdim, K, dF, mode=0, lengths=None):
    dim, pts, ln = _grid(points, lengths)
    K = np.ascontiguousarray(K, dtype=np.float64).reshape(-1)
    dF = np.ascontiguousarray(dF, dtype=np.float64).reshape(-1)
    out = np.empty_like(dF)
    st = lib().or_apply_projected_tangent(dim, pts, ln, tdim, mode, K, dF, out)
    return out, st


def fft(points, data, sign=-1):
    """Unnormalised c2c over all axes of each leading slab; data complex (h, n)."""
    data = np.ascontiguousarray(data, dtype=np.complex128)
    h = data.shape[0] if data.ndim > 1 else 1
    dim, pts, _ = _grid(points)
    buf = data.view(np.float64).reshape(-1).copy()
    lib().or_fft(dim, pts, h, sign, buf)
    return buf.view(np.complex128).reshape(data.shape)


def hyper_evaluate(F, lam, mu, tdim=3, want_K=True):
    n = lam.size
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1)
    P = np.empty(tdim * tdim * n)
    K = np.empty(tdim ** 4 * n) if want_K else None
    bad = C.c_int64(-1)
    st = lib().or_hyper_evaluate(n, tdim, F, np.ascontiguousarray(lam, dtype=np.float64),
                                 np.ascontiguousarray(mu, dtype=np.float64), P,
                                 K.ctypes.data if K is not None else None, C.byref(bad))
    return P, K, st, bad.value


def equivalent_stress(F, P, n, tdim=3, kind=0):
    """kind 0: of P; 1: of F^-1 P (hyperelastic); 2: of P F^T (Simo).
    Returns (eq, status, bad_node)."""
    out = np.empty(n)
    bad = C.c_int64(-1)
    Fp = np.ascontiguousarray(F, dtype=np.float64).reshape(-1) if F is not None else None
    st = lib().or_equivalent_stress(n, tdim, kind, Fp.ctypes.data if Fp is not None else None,
                                    np.ascontiguousarray(P, dtype=np.float64).reshape(-1), out, C.byref(bad))
    return out, st, bad.value


def simo_evaluate(F, Fold, be, epsp, lam, mu, ty0, hard, want_K=True):
    n = lam.size
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    P = np.empty(9 * n)
    K = np.empty(81 * n) if want_K else None
    be_t = np.empty(9 * n)
    ep_t = np.empty(n)
    bad = C.c_int64(-1)
    bv = C.c_double(0.0)
    st = lib().or_simo_evaluate(n, f(F), f(Fold), f(be), f(epsp), f(lam), f(mu), f(ty0), f(hard),
                                P, K.ctypes.data if K is not None else None, be_t, ep_t,
                                C.byref(bad), C.byref(bv))
    return {"P": P, "K": K, "be": be_t, "epsp": ep_t, "status": st, "bad": bad.value,
            "bad_value": bv.value}


def sym_eig3(A):
    lam = np.empty(3)
    V = np.empty(9)
    lib().or_sym_eig3(np.ascontiguousarray(A, dtype=np.float64).reshape(-1), lam, V)
    return lam, V.reshape(3, 3)


def cg_solve(points, tdim, K, rhs, eta_cg=1e-8, max_cg=0, mode=0, lengths=None):
    dim, pts, ln = _grid(points, lengths)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64).reshape(-1)
    x = np.empty_like(rhs)
    it = C.c_int(0)
    rel = C.c_double(0)
    st = lib().or_cg_solve(dim, pts, ln, tdim, mode, np.ascontiguousarray(K).reshape(-1), rhs,
                           eta_cg, max_cg, x, C.byref(it), C.byref(rel))
    return x, it.value, rel.value, st


def run_program(points, tdim, kind, lam, mu, fbars, ty0=None, hard=None, F0=None,
                eta_newton=1e-5, eta_cg=1e-8, max_newton=30, max_cg=0, mode=0, lengths=None):
    """Runs increments; returns (F, P, reports(list of dict), status, epsp)."""
    dim, pts, ln = _grid(points, lengths)
    n = int(np.prod(points))
    if F0 is None:
        F = np.zeros(tdim * tdim * n)
        for i in range(tdim):
            F[(i * tdim + i) * n:(i * tdim + i + 1) * n] = 1.0
    else:
        F = np.ascontiguousarray(F0, dtype=np.float64).reshape(-1).copy()
    P = np.zeros_like(F)
    fb = np.ascontiguousarray(fbars, dtype=np.float64).reshape(-1)
    ninc = fb.size // (tdim * tdim)
    reps = (OrReport * max(ninc, 1))()
    z = np.zeros(n)
    epsp = np.zeros(n)
    st = lib().or_run_program(dim, pts, ln, tdim, mode, kind, np.ascontiguousarray(lam, dtype=np.float64),
                              np.ascontiguousarray(mu, dtype=np.float64),
                              z if ty0 is None else np.ascontiguousarray(ty0, dtype=np.float64),
                              z if hard is None else np.ascontiguousarray(hard, dtype=np.float64),
                              ninc, fb, eta_newton, eta_cg, max_newton, max_cg, F, P,
                              epsp.ctypes.data, reps)
    return F, P, [reps[i].as_dict() for i in range(ninc)], st, epsp


def time_projected_tangent(points, K, dF, reps=1):
    dim, pts, ln = _grid(points)
    out = np.empty_like(dF)
    return lib().or_time_projected_tangent(dim, pts, ln, 3, K, dF, out, reps)
