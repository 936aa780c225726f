"""ctypes binding of libfftmech_b200.so (the C ABI in include/fftmech_b200.h).

This is the Python face of the drop-in boundary: tests, bench.py and
__graft_entry__ drive the sm_100a kernels through exactly the entry points a
C/C++/FFI caller would bind.  There is no fallback: if the library is missing
or no CUDA device is visible, construction fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (FM_LIB: another build of the same library, for A/B runs of compile-time variants)
LIB_PATH = os.environ.get("FM_LIB") or os.path.join(_HERE, "lib", "libfftmech_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "fftmech_b200.h")

FM_OK = 0
STATUS_NAMES = {
    0: "FM_OK", 1: "FM_E_INVALID", 2: "FM_E_CUDA", 3: "FM_E_OOM", 4: "FM_E_INVERTED",
    5: "FM_E_NOT_SPD", 6: "FM_E_SINGULAR", 7: "FM_E_CG_STALLED", 8: "FM_E_COMPLEX_RESIDUE",
    9: "FM_E_NEWTON_DIVERGED", 10: "FM_E_NCCL", 11: "FM_E_UNSUPPORTED",
}
MAX_PASSES = 64


class FmError(RuntimeError):
    """Raised for a non-zero fm_status; mirrors fftmech::Error (errors.hpp:11-14)."""

    def __init__(self, status, message, info=None):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.info = info or {}


class ErrorInfo(C.Structure):
    _fields_ = [("status", C.c_int32), ("cg_iterations", C.c_int32), ("node", C.c_int64),
                ("value", C.c_double)]


class SolverParams(C.Structure):
    _fields_ = [("eta_newton", C.c_double), ("eta_cg", C.c_double), ("max_newton", C.c_int32),
                ("max_cg", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("n_passes", C.c_int32), ("converged", C.c_int32),
                ("cg_iterations", C.c_int32 * MAX_PASSES),
                ("cg_rel_residual", C.c_double * MAX_PASSES),
                ("rel_update", C.c_double * MAX_PASSES),
                ("equilibrium_rel_residual", C.c_double), ("max_mean_drift", C.c_double),
                ("wall_seconds", C.c_double), ("matvecs", C.c_int64)]

    def as_dict(self):
        n = min(self.n_passes, MAX_PASSES)  # per-pass records exist for the first MAX_PASSES passes
        return {"passes": self.n_passes, "converged": bool(self.converged),
                "cg_it": list(self.cg_iterations[:n]), "cg_rel": list(self.cg_rel_residual[:n]),
                "rel_update": list(self.rel_update[:n]),
                "eq_rel": self.equilibrium_rel_residual, "drift": self.max_mean_drift,
                "wall": self.wall_seconds, "matvecs": self.matvecs}


_lib = None
_P = C.c_void_p
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")

_SIGS = {
    "fm_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int, C.c_int,
                                C.c_int, C.POINTER(_P)]),
    "fm_ctx_destroy": (C.c_int, [_P]),
    "fm_last_error": (C.c_char_p, [_P]),
    "fm_last_error_info": (C.c_int, [_P, C.POINTER(ErrorInfo)]),
    "fm_ctx_nodes": (C.c_int64, [_P]),
    "fm_ctx_tdim": (C.c_int, [_P]),
    "fm_ctx_synchronize": (C.c_int, [_P]),
    "fm_ctx_stream": (_P, [_P]),
    "fm_ctx_launch_count": (C.c_int64, [_P]),
    "fm_ctx_profile": (C.c_int, [_P, C.c_int]),
    "fm_ctx_kernel_names": (C.c_int, [_P, C.c_char_p, C.c_int]),
    "fm_ctx_profile_read": (C.c_int, [_P, _dp, C.POINTER(C.c_int64)]),
    "fm_field_alloc": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "fm_field_free": (C.c_int, [_P, _P]),
    "fm_field_device_ptr": (_P, [_P]),
    "fm_field_upload": (C.c_int, [_P, _P, _dp, C.c_int64]),
    "fm_field_download": (C.c_int, [_P, _P, _dp, C.c_int64]),
    "fm_field_fill": (C.c_int, [_P, _P, C.c_double]),
    "fm_field_copy": (C.c_int, [_P, _P, _P]),
    "fm_projection_apply": (C.c_int, [_P, _P, _P]),
    "fm_projected_tangent_apply": (C.c_int, [_P, _P, _P, _P]),
    "fm_hyper_evaluate": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "fm_simo_evaluate": (C.c_int, [_P] + [_P] * 12),
    "fm_equivalent_stress": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "fm_dot": (C.c_int, [_P, _P, _P, C.POINTER(C.c_double)]),
    "fm_norm": (C.c_int, [_P, _P, C.POINTER(C.c_double)]),
    "fm_mean": (C.c_int, [_P, _P, _dp]),
    "fm_axpy": (C.c_int, [_P, C.c_double, _P, _P]),
    "fm_scale": (C.c_int, [_P, _P, C.c_double]),
    "fm_add": (C.c_int, [_P, _P, _P, C.c_double]),
    "fm_add_uniform": (C.c_int, [_P, _P, _dp]),
    "fm_cg_solve": (C.c_int, [_P, _P, _P, C.c_double, C.c_int64, _P, C.POINTER(C.c_int32),
                              C.POINTER(C.c_double)]),
    "fm_model_create_hyper": (C.c_int, [_P, _dp, _dp, C.c_int, C.POINTER(_P)]),
    "fm_model_create_simo": (C.c_int, [_P, _dp, _dp, _dp, _dp, C.POINTER(_P)]),
    "fm_model_destroy": (C.c_int, [_P, _P]),
    "fm_model_evaluate": (C.c_int, [_P, _P, _P, _P]),
    "fm_model_commit": (C.c_int, [_P, _P, _P]),
    "fm_model_tangent": (_P, [_P]),
    "fm_model_get_history": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "fm_model_set_history": (C.c_int, [_P, _P, _P, _P, _P]),
    "fm_model_apply": (C.c_int, [_P, _P, _P, _P]),
    "fm_solve_increment": (C.c_int, [_P, _P, _P, _dp, C.POINTER(SolverParams), C.POINTER(Report), _P]),
    "fm_ctx_create_dist": (C.c_int, [C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_P)]),
    "fm_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_int]),
    "fm_model_set_tangent_form": (C.c_int, [_P, _P, C.c_int]),
    "fm_ctx_set_virtual_ranks": (C.c_int, [_P, C.c_int]),
    "fm_ctx_set_transpose": (C.c_int, [_P, C.c_int]),
    "fm_ctx_set_debug": (C.c_int, [_P, C.c_int]),
    "fm_ctx_ranks": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "fm_dist_route": (C.c_int, [C.c_int] * 11 + [C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
}


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it and shares it, e.g. via torch.distributed)."""
    buf = C.create_string_buffer(128)
    st = lib().fm_nccl_unique_id(buf, 128)
    if st != FM_OK:
        raise FmError(st, "ncclGetUniqueId failed")
    return buf.raw


def dist_route(P, Nx, Ny, nzh, ncomp, direction, src, comp, i0, i1, kz):
    """Route of the fused slab transpose (host only), the function the kernels
    evaluate: (destination rank, complex-element index in its buffer).
    direction +1: forward y pass of x-slab `src`, element (comp, xl=i0, y=i1, kz);
    direction -1: x pass of y-slab `src`, element (comp, x=i0, yl=i1, kz)."""
    d, o = C.c_int32(), C.c_int64()
    st = lib().fm_dist_route(P, Nx, Ny, nzh, ncomp, direction, src, comp, i0, i1, kz, C.byref(d), C.byref(o))
    if st != FM_OK:
        raise FmError(st, "fm_dist_route")
    return d.value, o.value


def declared_symbols():
    """Function names declared in include/fftmech_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*\s]+?)\b(fm_\w+)\s*\(", text, re.M)))


def lib():
    """Loads the shared library (no GPU needed to load; calls need one)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FmError(2, f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _grid(points, lengths):
    dim = len(points)
    pts = (C.c_int32 * 3)(*(list(points) + [1] * (3 - dim)))
    ln = (C.c_double * 3)(*((list(lengths) if lengths is not None else [1.0] * dim) + [1.0] * (3 - dim)))
    return dim, pts, ln


class Context:
    """fm_ctx: grid + FFT plans + workspace on one device (replaces
    ProjectionOperator / build_projection, projection.hpp:40-66)."""

    def __init__(self, points, tdim=None, lengths=None, nyquist_mode=0, device=0, dist=None):
        """dist = (nranks, rank, nccl_unique_id): one slab rank per device; fields
        then hold this rank's x-slab (Nx/nranks planes)."""
        L = lib()
        dim, pts, ln = _grid(points, lengths)
        self.points = tuple(points)
        self.tdim = tdim if tdim is not None else dim
        self.ncomp = self.tdim * self.tdim
        h = _P()
        if dist is None:
            st = L.fm_ctx_create(dim, pts, ln, self.tdim, nyquist_mode, device, C.byref(h))
        else:
            nranks, rank, uid = dist
            st = L.fm_ctx_create_dist(dim, pts, ln, self.tdim, nyquist_mode, device, nranks, rank, uid, C.byref(h))
        if st != FM_OK:
            raise FmError(st, "fm_ctx_create failed (is a CUDA device visible?)")
        self.h = h
        self.n = int(L.fm_ctx_nodes(h))  # nodes held here (the local slab when distributed)
        self._fields = []

    def set_virtual_ranks(self, P):
        """Run the slab-decomposed projection with P ranks emulated on this device."""
        self.check(lib().fm_ctx_set_virtual_ranks(self.h, P))

    def set_debug(self, residue_check=True):
        """Imaginary-residue check of every projection (projection.cpp:157-169)."""
        self.check(lib().fm_ctx_set_debug(self.h, 1 if residue_check else 0))

    def last_info(self):
        info = ErrorInfo()
        lib().fm_last_error_info(self.h, C.byref(info))
        return {"status": info.status, "cg_iterations": info.cg_iterations, "node": info.node, "value": info.value}

    def set_transpose(self, mode):
        """0: slab transposes fused into passes 2 and 3 as peer stores; 1: staged all-to-all."""
        self.check(lib().fm_ctx_set_transpose(self.h, mode))

    def ranks(self):
        nr, r, v = C.c_int(), C.c_int(), C.c_int()
        self.check(lib().fm_ctx_ranks(self.h, C.byref(nr), C.byref(r), C.byref(v)))
        return nr.value, r.value, bool(v.value)

    def close(self):
        if getattr(self, "h", None):
            for f in self._fields:
                if f.h:
                    lib().fm_field_free(self.h, f.h)
                    f.h = None
            lib().fm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- error handling
    def check(self, st):
        if st != FM_OK:
            info = ErrorInfo()
            lib().fm_last_error_info(self.h, C.byref(info))
            msg = lib().fm_last_error(self.h).decode()
            raise FmError(st, msg, {"node": info.node, "value": info.value,
                                    "cg_iterations": info.cg_iterations})

    def sync(self):
        self.check(lib().fm_ctx_synchronize(self.h))

    @property
    def stream(self):
        return lib().fm_ctx_stream(self.h)

    def profile(self, enable=True):
        self.check(lib().fm_ctx_profile(self.h, int(enable)))

    def profile_read(self):
        ms = np.zeros(5)
        calls = C.c_int64()
        self.check(lib().fm_ctx_profile_read(self.h, ms, C.byref(calls)))
        return ms, calls.value

    @property
    def launches(self):
        return lib().fm_ctx_launch_count(self.h)

    @property
    def kernel_names(self):
        """Distinct names of this library's kernels launched on the context."""
        buf = C.create_string_buffer(4096)
        lib().fm_ctx_kernel_names(self.h, buf, 4096)
        return [k for k in buf.value.decode().split(",") if k]

    # -- fields
    def field(self, ncomp=None, data=None):
        ncomp = self.ncomp if ncomp is None else ncomp
        h = _P()
        self.check(lib().fm_field_alloc(self.h, ncomp, C.byref(h)))
        f = Field(self, h, ncomp)
        self._fields.append(f)
        if data is not None:
            f.upload(data)
        return f

    def projection(self, A, out=None):
        out = out or self.field()
        self.check(lib().fm_projection_apply(self.h, A.h, out.h))
        return out

    def projected_tangent(self, K, dF, out=None):
        out = out or self.field()
        self.check(lib().fm_projected_tangent_apply(self.h, K.h, dF.h, out.h))
        return out

    def dot(self, a, b):
        r = C.c_double()
        self.check(lib().fm_dot(self.h, a.h, b.h, C.byref(r)))
        return r.value

    def norm(self, a):
        r = C.c_double()
        self.check(lib().fm_norm(self.h, a.h, C.byref(r)))
        return r.value

    def axpy(self, a, x, y):
        """y += a x (device)."""
        self.check(lib().fm_axpy(self.h, C.c_double(a), x.h, y.h))
        return y

    def mean(self, a):
        out = np.zeros(a.ncomp)
        self.check(lib().fm_mean(self.h, a.h, out))
        return out

    def cg_solve(self, K, rhs, eta_cg=1e-8, max_cg=0, x=None):
        x = x or self.field()
        it = C.c_int32()
        rel = C.c_double()
        self.check(lib().fm_cg_solve(self.h, K.h, rhs.h, eta_cg, max_cg, x.h, C.byref(it), C.byref(rel)))
        return x, it.value, rel.value

    EQ_TENSOR, EQ_PK2, EQ_KIRCHHOFF = 0, 1, 2

    def equivalent_stress(self, F, P, kind, out=None):
        """von Mises equivalent (material.cpp:14-31) of P (EQ_TENSOR),
        F^-1 P (EQ_PK2, hyperelastic) or P F^T (EQ_KIRCHHOFF, Simo)."""
        out = out or self.field(1)
        self.check(lib().fm_equivalent_stress(self.h, F.h if F is not None else None, P.h, kind, out.h))
        return out

    def hyper_evaluate(self, F, lam, mu, want_K=True):
        P = self.field()
        K = self.field(self.ncomp * self.ncomp) if want_K else None
        lf = self.field(1, lam)
        mf = self.field(1, mu)
        self.check(lib().fm_hyper_evaluate(self.h, F.h, lf.h, mf.h, P.h, K.h if K else None))
        return P, K

    def simo_evaluate(self, F, Fold, be, epsp, lam, mu, ty0, hard, want_K=True):
        fs = [self.field(1, a) for a in (epsp, lam, mu, ty0, hard)]
        bef = self.field(9, be)
        P, K = self.field(), (self.field(81) if want_K else None)
        be_t, ep_t = self.field(9), self.field(1)
        self.check(lib().fm_simo_evaluate(self.h, F.h, Fold.h, bef.h, fs[0].h, fs[1].h, fs[2].h,
                                          fs[3].h, fs[4].h, P.h, K.h if K else None, be_t.h, ep_t.h))
        return P, K, be_t, ep_t


class Field:
    """fm_field: ncomp component-major slabs of n doubles in HBM."""

    def __init__(self, ctx, h, ncomp):
        self.ctx, self.h, self.ncomp = ctx, h, ncomp

    @property
    def size(self):
        return self.ncomp * self.ctx.n

    @property
    def ptr(self):
        return lib().fm_field_device_ptr(self.h)

    def upload(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        self.ctx.check(lib().fm_field_upload(self.ctx.h, self.h, a, a.size))
        return self

    def download(self, out=None):
        out = np.empty(self.size) if out is None else out
        self.ctx.check(lib().fm_field_download(self.ctx.h, self.h, out, out.size))
        return out

    @property
    def __cuda_array_interface__(self):
        """Zero-copy view of the device slabs ([ncomp * n] fp64) for callers that
        fill or check huge fields on the device (e.g. torch.as_tensor(field,
        device="cuda")); the library's stream must be synchronised around it."""
        return {"shape": (self.size,), "typestr": "<f8", "data": (int(self.ptr), False), "version": 3,
                "strides": None}

    def free(self):
        if self.h:
            lib().fm_field_free(self.ctx.h, self.h)
            self.h = None


class Model:
    """fm_model: MaterialModel (material.hpp:45-65) resident on the device."""

    def __init__(self, ctx, kind, lam, mu, ty0=None, hard=None, matrix_free=False, compact=False):
        self.ctx = ctx
        h = _P()
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        if kind == "hyper":
            ctx.check(lib().fm_model_create_hyper(ctx.h, f(lam), f(mu), int(matrix_free), C.byref(h)))
        else:
            ctx.check(lib().fm_model_create_simo(ctx.h, f(lam), f(mu), f(ty0), f(hard), C.byref(h)))
            if compact:
                ctx.check(lib().fm_model_set_tangent_form(ctx.h, h, 1))
        self.h = h
        self.kind = kind

    def close(self):
        if self.h and self.ctx.h:
            lib().fm_model_destroy(self.ctx.h, self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def evaluate(self, F, P):
        self.ctx.check(lib().fm_model_evaluate(self.ctx.h, self.h, F.h, P.h))

    def commit(self, F):
        self.ctx.check(lib().fm_model_commit(self.ctx.h, self.h, F.h))

    def apply(self, dF, out):
        self.ctx.check(lib().fm_model_apply(self.ctx.h, self.h, dF.h, out.h))
        return out

    def tangent(self):
        """The model-owned K4 field (not owned by the caller), or None when the
        model is matrix-free / compact."""
        h = lib().fm_model_tangent(self.h)
        if not h:
            return None
        nc = self.ctx.ncomp
        return Field(self.ctx, h, nc * nc)

    def history(self, which=0):
        n = self.ctx.n
        be = np.empty(9 * n)
        ep = np.empty(n)
        self.ctx.check(lib().fm_model_get_history(self.ctx.h, self.h, which, be.ctypes.data, ep.ctypes.data))
        return be, ep

    def set_history(self, be=None, epsp=None, f_old=None):
        conv = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        be, epsp, f_old = conv(be), conv(epsp), conv(f_old)
        self.ctx.check(lib().fm_model_set_history(
            self.ctx.h, self.h, None if be is None else be.ctypes.data,
            None if epsp is None else epsp.ctypes.data, None if f_old is None else f_old.ctypes.data))

    def solve_increment(self, F, fbar, eta_newton=1e-5, eta_cg=1e-8, max_newton=30, max_cg=0, P_out=None):
        prm = SolverParams(eta_newton, eta_cg, max_newton, max_cg)
        rep = Report()
        fb = np.ascontiguousarray(fbar, dtype=np.float64).reshape(-1)
        st = lib().fm_solve_increment(self.ctx.h, self.h, F.h, fb, C.byref(prm), C.byref(rep),
                                      P_out.h if P_out is not None else None)
        if st != FM_OK:
            try:
                self.ctx.check(st)
            except FmError as e:
                e.report = rep.as_dict()
                raise
        return rep.as_dict()


def run_program(model, F, fbars, P_out=None, sink=None, **params):
    """run_program (solver.cpp:162-169): increments in order, history committed
    at each convergence (inside solve_increment), reports streamed to `sink`.
    Raises on the first failed increment after notifying the sink of the
    completed ones.  Returns the list of reports."""
    reports = []
    P_out = P_out if P_out is not None else model.ctx.field()
    for idx, fbar in enumerate(fbars):
        rep = model.solve_increment(F, fbar, P_out=P_out, **params)
        reports.append(rep)
        if sink is not None:
            sink(idx, fbar, rep, F, P_out, model)
    return reports


def identity_field(points, tdim):
    n = int(np.prod(points))
    F = np.zeros(tdim * tdim * n)
    for i in range(tdim):
        F[(i * tdim + i) * n:(i * tdim + i + 1) * n] = 1.0
    return F
