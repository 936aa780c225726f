"""Host-side logic of the multi-GPU slab decomposition, exercised across real
process boundaries on the CPU (world_size 2 and 4, gloo): every rank runs the
forward y pass on its x-slab and routes every element where the library's
transpose-fused y pass stores it (fm_dist_route, the function the kernels
evaluate), runs the x pass on its y-slab with global-y frequencies, routes
the result back the way the x pass stores it and inverts -- the gathered
result must equal the single-process projection (projection.cpp:123-171
semantics), and every destination element must be written exactly once."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1603_08893_b200 import abi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ghat_apply(S, kx, ky, kz, Nx, Ny, Nz):
    """Bhat_i. = (Ahat_i . xi) xi / |xi|^2 with ZeroCompatible Nyquist (projection.cpp:87-104)."""
    f = lambda k, N: np.where(k < (N + 1) // 2, k, k - N)
    qx, qy, qz = np.meshgrid(f(kx, Nx), f(ky, Ny), f(kz, Nz), indexing="ij")
    nyq = (((Nx % 2 == 0) & (np.meshgrid(kx, ky, kz, indexing="ij")[0] == Nx // 2))
           | ((Ny % 2 == 0) & (np.meshgrid(kx, ky, kz, indexing="ij")[1] == Ny // 2))
           | ((Nz % 2 == 0) & (np.meshgrid(kx, ky, kz, indexing="ij")[2] == Nz // 2)))
    xi = np.stack([qx, qy, qz]).astype(float)
    n2 = (xi ** 2).sum(0)
    safe = np.where(n2 == 0, 1.0, n2)
    T = S.reshape(3, 3, *S.shape[1:])
    s = np.einsum("il...,l...->i...", T, xi)
    out = np.einsum("i...,j...->ij...", s, xi) / safe
    out[:, :, (n2 == 0) | nyq] = 0.0
    return out.reshape(9, *S.shape[1:])


def _reference(A, Nx, Ny, Nz):
    S = np.fft.fftn(A, axes=(1, 2, 3))
    k = lambda N: np.arange(N)
    return np.real(np.fft.ifftn(_ghat_apply(S, k(Nx), k(Ny), k(Nz), Nx, Ny, Nz), axes=(1, 2, 3)))


def _route_all(P, Nx, Ny, nzh, direction, src, shape):
    """Destination (rank, index) of every element of a [9][i0][i1][kz] block."""
    n0, n1 = shape
    ranks = np.empty((9, n0, n1, nzh), dtype=np.int64)
    idx = np.empty((9, n0, n1, nzh), dtype=np.int64)
    for c in range(9):
        for a in range(n0):
            for b in range(n1):
                for k in range(nzh):
                    ranks[c, a, b, k], idx[c, a, b, k] = abi.dist_route(P, Nx, Ny, nzh, 9, direction, src,
                                                                        c, a, b, k)
    return ranks.reshape(-1), idx.reshape(-1)


def _exchange(P, rank, values, ranks, idx, size):
    """Deliver values[e] to rank ranks[e] at index idx[e] (what the peer stores do)."""
    outgoing = [(idx[ranks == d], values[ranks == d]) for d in range(P)]
    everyone = [None] * P
    dist.all_gather_object(everyone, outgoing)
    buf = np.zeros(size, dtype=complex)
    hits = np.zeros(size, dtype=int)
    for src in range(P):
        i, v = everyone[src][rank]
        buf[i] = v
        np.add.at(hits, i, 1)
    assert np.all(hits == 1), "route is not a bijection onto the destination buffer"
    return buf


def _worker(rank, P, port, pts, A, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    Nx, Ny, Nz = pts
    Xl, Yl, nzh = Nx // P, Ny // P, Nz // 2
    size = 9 * Xl * Ny * nzh  # = 9 * Nx * Yl * nzh: A and B of one rank
    # passes 1-2 on the x-slab [c][xl][y][kz]; the y pass stores into the x-pass inputs B_d
    slab = A[:, rank * Xl:(rank + 1) * Xl]
    S = np.fft.fft(np.fft.rfft(slab, axis=3)[..., :nzh], axis=2)  # Nyquist kz dropped (ZeroCompatible)
    rk, ix = _route_all(P, Nx, Ny, nzh, +1, rank, (Xl, Ny))
    B = _exchange(P, rank, S.reshape(-1), rk, ix, size)
    # pass 3 on the y-slab [c][x][yl][kz]: all x, y in [rank Yl, (rank+1) Yl)
    T = B.reshape(9, Nx, Yl, nzh)
    T = np.fft.fft(T, axis=1)
    T = _ghat_apply(T, np.arange(Nx), rank * Yl + np.arange(Yl), np.arange(nzh), Nx, Ny, Nz)
    T = np.fft.ifft(T, axis=1)
    rk, ix = _route_all(P, Nx, Ny, nzh, -1, rank, (Nx, Yl))
    A2 = _exchange(P, rank, T.reshape(-1), rk, ix, size)
    # passes 4-5 in place on the x-slab spectrum: inverse y, c2r z
    S2 = np.fft.ifft(A2.reshape(9, Xl, Ny, nzh), axis=2)
    S2 = np.concatenate([S2, np.zeros((9, Xl, Ny, 1))], axis=3)
    out = np.fft.irfft(S2, n=Nz, axis=3)
    gathered = [torch.empty(9 * Xl * Ny * Nz, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(out).reshape(-1)))
    if rank == 0:
        full = np.concatenate([g.numpy().reshape(9, Xl, Ny, Nz) for g in gathered], axis=1)
        q.put(full)
    dist.destroy_process_group()


@pytest.mark.parametrize("P,pts", [(2, (8, 6, 10)), (4, (8, 12, 6))])
def test_slab_transpose_routes_across_processes(P, pts):
    rng = np.random.default_rng(7)
    A = rng.uniform(-1, 1, (9, *pts))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, pts, A, q)) for r in range(P)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _reference(A, *pts)
    assert np.max(np.abs(full - ref)) < 1e-12


def test_routes_are_mutually_inverse_permutations():
    """Forward then backward route returns every element to its own place."""
    P, Nx, Ny, nzh = 4, 8, 12, 3
    Xl, Yl = Nx // P, Ny // P
    for s in range(P):
        for c in (0, 4, 8):
            for xl in range(Xl):
                for y in range(Ny):
                    for kz in range(nzh):
                        d, o = abi.dist_route(P, Nx, Ny, nzh, 9, +1, s, c, xl, y, kz)
                        # unravel the B_d index [c][x][yl][kz]
                        cc, rest = divmod(o, Nx * Yl * nzh)
                        x, rest = divmod(rest, Yl * nzh)
                        yl, k = divmod(rest, nzh)
                        assert (cc, x, k, d * Yl + yl) == (c, s * Xl + xl, kz, y)
                        s2, o2 = abi.dist_route(P, Nx, Ny, nzh, 9, -1, d, cc, x, yl, k)
                        assert s2 == s and o2 == ((c * Xl + xl) * Ny + y) * nzh + kz
    with pytest.raises(abi.FmError):
        abi.dist_route(3, 8, 12, 3, 9, +1, 0, 0, 0, 0, 0)  # Nx not divisible
    with pytest.raises(abi.FmError):
        abi.dist_route(2, 8, 12, 3, 9, +1, 0, 0, 4, 0, 0)  # xl outside the slab
