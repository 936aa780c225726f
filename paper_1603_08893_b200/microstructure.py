"""Host-side setup: phase grids, per-node parameter binding and load ramps.

This is the (untimed, O(n) once) setup layer around the hot path.  It mirrors
the reference's `microstructure.cpp` / `run_config.cpp` semantics where they
exist and defines the BASELINE.json config generators that do not exist in the
reference:

* `make_cubic_inclusion`   -- microstructure.cpp:19-49 (centred cube)
* `make_laminate`          -- microstructure.cpp:51-88 (largest remainder)
* `bind_parameters`        -- microstructure.cpp:176-203
* `simple_shear_program`   -- run_config.cpp:357-363 (expand_loading)
* `corner_cube`, `bernoulli`, `random_spheres` -- configs 0/1, 2, 3
* `uniform_field`          -- config 4 (seeded U(-1,1), slab by slab)

Random numbers come from `MT19937_64` (std::mt19937_64, whose output sequence
the C++ standard fixes) with u = (x >> 11) * 2^-53 computed explicitly, so the
inputs are identical for the oracle, the GPU path and any C++ consumer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "ElasticParams", "PlasticParams", "PhaseGrid", "MT19937_64",
    "make_cubic_inclusion", "make_laminate", "corner_cube", "bernoulli",
    "random_spheres", "bind_parameters", "simple_shear_program", "uniform_field",
    "node_coords",
]


@dataclass(frozen=True)
class ElasticParams:
    """material.hpp:12-20 -- (E, nu) stored, Lame pair derived."""
    youngs: float = 1.0
    poisson: float = 0.3

    @property
    def lame_lambda(self) -> float:
        return self.youngs * self.poisson / ((1.0 + self.poisson) * (1.0 - 2.0 * self.poisson))

    @property
    def lame_mu(self) -> float:
        return self.youngs / (2.0 * (1.0 + self.poisson))


@dataclass(frozen=True)
class PlasticParams:
    """material.hpp:23-27 -- tau_y = tau_y0 + H eps_p."""
    elastic: ElasticParams = ElasticParams()
    tau_y0: float = 1.0
    hardening: float = 0.0


@dataclass
class PhaseGrid:
    """microstructure.hpp: labels in node order (last axis fastest)."""
    points: tuple
    labels: np.ndarray  # int32, node order
    phase_count: int

    @property
    def dim(self) -> int:
        return len(self.points)


class MT19937_64:
    """std::mt19937_64, vectorised over the 312-word state."""
    _N, _M = 312, 156
    _MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    _UM = np.uint64(0xFFFFFFFF80000000)
    _LM = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int = 5489):
        mt = np.zeros(self._N, dtype=np.uint64)
        x = seed & 0xFFFFFFFFFFFFFFFF
        mt[0] = x
        for i in range(1, self._N):
            x = (6364136223846793005 * (x ^ (x >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            mt[i] = x
        self._mt = mt
        self._buf = np.zeros(0, dtype=np.uint64)

    def _twist(self) -> None:
        mt, N, M = self._mt, self._N, self._M
        one = np.uint64(1)
        new = mt.copy()
        # i in [0, N-M): uses old mt[i+1], old mt[i+M]
        y = (mt[0:N - M] & self._UM) | (mt[1:N - M + 1] & self._LM)
        new[0:N - M] = mt[M:N] ^ (y >> one) ^ np.where((y & one) != 0, self._MATRIX_A, np.uint64(0))
        # i in [N-M, N-1): uses old mt[i+1], new mt[i+M-N]
        y = (mt[N - M:N - 1] & self._UM) | (mt[N - M + 1:N] & self._LM)
        new[N - M:N - 1] = new[0:M - 1] ^ (y >> one) ^ np.where((y & one) != 0, self._MATRIX_A, np.uint64(0))
        y = (mt[N - 1] & self._UM) | (new[0] & self._LM)
        new[N - 1] = new[M - 1] ^ (y >> one) ^ (self._MATRIX_A if int(y) & 1 else np.uint64(0))
        self._mt = new

    @staticmethod
    def _temper(x: np.ndarray) -> np.ndarray:
        x = x ^ ((x >> np.uint64(29)) & np.uint64(0x5555555555555555))
        x = x ^ ((x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
        x = x ^ ((x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
        return x ^ (x >> np.uint64(43))

    def raw(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        got = 0
        while got < count:
            if self._buf.size == 0:
                self._twist()
                self._buf = self._temper(self._mt.copy())
            take = min(count - got, self._buf.size)
            out[got:got + take] = self._buf[:take]
            self._buf = self._buf[take:]
            got += take
        return out

    def uniform(self, count: int) -> np.ndarray:
        """u = (x >> 11) * 2^-53 in [0, 1)."""
        return (self.raw(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def node_coords(points) -> np.ndarray:
    """All node coordinates in node order (grid.hpp:32-39); shape (n, dim)."""
    grids = np.meshgrid(*[np.arange(p) for p in points], indexing="ij")
    return np.stack([g.reshape(-1) for g in grids], axis=1)


def make_cubic_inclusion(points, volume_fraction: float) -> PhaseGrid:
    """microstructure.cpp:19-49 -- centred cube, side = round(f^(1/d) N)."""
    d = len(points)
    if not (0.0 < volume_fraction < 1.0):
        raise ValueError("volume fraction must be in (0,1)")
    side_ratio = volume_fraction ** (1.0 / d)
    inside = np.ones(int(np.prod(points)), dtype=bool)
    xyz = node_coords(points)
    for a in range(d):
        na = points[a]
        side = int(math.floor(side_ratio * na + 0.5))  # std::lround, positive args
        if side <= 0 or side >= na:
            raise ValueError(f"inclusion side rounds to {side} of {na} nodes on axis {a}")
        start = (na - side) // 2
        inside &= (xyz[:, a] >= start) & (xyz[:, a] < start + side)
    return PhaseGrid(tuple(points), inside.astype(np.int32), 2)


def make_laminate(points, fractions) -> PhaseGrid:
    """microstructure.cpp:51-88 -- layers along axis 0, largest remainder."""
    if abs(sum(fractions) - 1.0) > 1e-9:
        raise ValueError("layer fractions must sum to 1")
    n0 = points[0]
    counts, rem, assigned = [], [], 0
    for p, f in enumerate(fractions):
        exact = f * n0
        c = int(math.floor(exact))
        counts.append(c)
        assigned += c
        rem.append((exact - math.floor(exact), p))
    rem.sort(key=lambda t: -t[0])  # std::sort by remainder, descending
    for r in range(n0 - assigned):
        counts[rem[r % len(rem)][1]] += 1
    if any(c == 0 for c in counts):
        raise ValueError("a laminate layer gets zero nodes")
    layer_of = np.concatenate([np.full(c, p, dtype=np.int32) for p, c in enumerate(counts)])
    xyz = node_coords(points)
    return PhaseGrid(tuple(points), layer_of[xyz[:, 0]], len(fractions))


def corner_cube(points, side: int) -> PhaseGrid:
    """Configs 0/1: label 1 iff every coordinate < side."""
    xyz = node_coords(points)
    return PhaseGrid(tuple(points), np.all(xyz < side, axis=1).astype(np.int32), 2)


def bernoulli(points, p: float, seed: int) -> PhaseGrid:
    """Config 2: label 1 iff u < p, u drawn in node order from mt19937_64(seed)."""
    n = int(np.prod(points))
    u = MT19937_64(seed).uniform(n)
    return PhaseGrid(tuple(points), (u < p).astype(np.int32), 2)


def random_spheres(N: int, radius: int, fraction: float, seed: int):
    """Config 3: periodic spheres (min-image distance^2 <= r^2) with centres
    c = N*(u,u,u) added until the labelled fraction reaches `fraction`.
    Returns (PhaseGrid, achieved_fraction, sphere_count)."""
    rng = MT19937_64(seed)
    labels = np.zeros((N, N, N), dtype=np.int32)
    r2 = radius * radius
    offs = np.arange(-radius - 1, radius + 2)
    count = 0
    total = N ** 3
    filled = 0
    while filled < fraction * total:
        c = N * rng.uniform(3)
        # voxels v with min-image |v - c|^2 <= r^2; candidates near floor(c)
        base = np.floor(c).astype(np.int64)
        ax = []
        for a in range(3):
            v = base[a] + offs
            dv = v - c[a]  # v - c, then min image over the period N
            dv = dv - N * np.round(dv / N)
            ax.append((np.mod(v, N), dv * dv))
        d2 = ax[0][1][:, None, None] + ax[1][1][None, :, None] + ax[2][1][None, None, :]
        mask = d2 <= r2
        ix = np.ix_(ax[0][0], ax[1][0], ax[2][0])
        sub = labels[ix]
        newly = mask & (sub == 0)
        filled += int(newly.sum())
        sub[mask] = 1
        labels[ix] = sub
        count += 1
    return PhaseGrid((N, N, N), labels.reshape(-1), 2), filled / total, count


def bind_parameters(pg: PhaseGrid, per_phase):
    """microstructure.cpp:176-203 -> (lambda, mu, tau_y0, hardening) arrays."""
    if len(per_phase) != pg.phase_count:
        raise ValueError(f"got {len(per_phase)} parameter sets for {pg.phase_count} phases")
    pp = [p if isinstance(p, PlasticParams) else PlasticParams(p, 0.0, 0.0) for p in per_phase]
    lab = pg.labels
    lam = np.array([p.elastic.lame_lambda for p in pp])[lab]
    mu = np.array([p.elastic.lame_mu for p in pp])[lab]
    ty = np.array([p.tau_y0 for p in pp])[lab]
    h = np.array([p.hardening for p in pp])[lab]
    return lam, mu, ty, h


def simple_shear_program(gamma: float, increments: int, tdim: int) -> np.ndarray:
    """run_config.cpp:357-363: F_t = I + gamma*t/T e_x (x) e_y; (T, tdim, tdim)."""
    out = np.zeros((increments, tdim, tdim))
    for t in range(1, increments + 1):
        out[t - 1] = np.eye(tdim)
        out[t - 1, 0, 1] = gamma * float(t) / increments
    return out


def _host_lib():
    import ctypes
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libfftmech_host.so")
    if not os.path.exists(path):
        return None
    try:
        lib = ctypes.CDLL(path)
    except OSError:
        return None
    lib.fmh_uniform_field.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    lib.fmh_uniform_field.restype = None
    return lib


def uniform_field(points, ncomp: int, seed: int) -> np.ndarray:
    """Config 4: ncomp slabs i.i.d. U(-1,1) = 2u-1, slab by slab in node order.
    Large fields use the host library's std::mt19937_64 (same stream)."""
    n = int(np.prod(points))
    if ncomp * n >= (1 << 20):
        lib = _host_lib()
        if lib is not None:
            out = np.empty(ncomp * n)
            lib.fmh_uniform_field(seed, ncomp * n, out.ctypes.data)
            return out
    return 2.0 * MT19937_64(seed).uniform(ncomp * n) - 1.0
