"""Host-side logic of the multi-GPU slab decomposition, exercised across real
process boundaries on the CPU (world_size 2 and 4, gloo): every rank builds
its packed spectrum exactly as pass 2 lays it out, exchanges the chunks the
library's transpose plan (fm_dist_chunk, the offsets the NCCL path uses)
names with point-to-point send/recv, runs the x pass with its global-y
frequencies, exchanges back and inverts -- the gathered result must equal
the single-process projection (projection.cpp:123-171 semantics)."""
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


def _worker(rank, P, port, pts, A, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    Nx, Ny, Nz = pts
    Xl, Yl, nzh = Nx // P, Ny // P, Nz // 2
    # passes 1-2 on the x-slab; pass 2 writes the packed layout [dst][c][xl][yl][kz]
    slab = A[:, rank * Xl:(rank + 1) * Xl]
    S = np.fft.fft(np.fft.rfft(slab, axis=3)[..., :nzh], axis=2)  # Nyquist kz dropped (ZeroCompatible)
    B = np.ascontiguousarray(S.reshape(9, Xl, P, Yl, nzh).transpose(2, 0, 1, 3, 4)).reshape(-1)
    Abuf = np.zeros(9 * Nx * Yl * nzh, dtype=complex)

    def exchange(src_buf, dst_buf, forward):
        reqs, recvd = [], []
        for peer in range(P):
            for c in range(9):
                if forward:   # my B chunk for `peer` -> peer's A; peer's B chunk for me -> my A
                    so, _, cnt = abi.dist_chunk(P, Nx, Ny, nzh, 9, rank, peer, c)
                    _, ro, _ = abi.dist_chunk(P, Nx, Ny, nzh, 9, peer, rank, c)
                else:         # my A chunk of source `peer` -> its B; my B chunk from `peer`
                    _, so, cnt = abi.dist_chunk(P, Nx, Ny, nzh, 9, peer, rank, c)
                    ro, _, _ = abi.dist_chunk(P, Nx, Ny, nzh, 9, rank, peer, c)
                send = torch.from_numpy(src_buf[so:so + cnt].view(np.float64).copy())
                if peer == rank:
                    dst_buf[ro:ro + cnt] = src_buf[so:so + cnt]
                    continue
                recv = torch.empty(2 * cnt, dtype=torch.float64)
                tag = c
                reqs.append(dist.isend(send, peer, tag=tag))
                reqs.append(dist.irecv(recv, peer, tag=tag))
                recvd.append((ro, cnt, recv))
        for r in reqs:
            r.wait()
        for ro, cnt, recv in recvd:
            dst_buf[ro:ro + cnt] = recv.numpy().view(complex)

    exchange(B, Abuf, True)
    # pass 3 on the y-slab: all x, y in [rank Yl, (rank+1) Yl)
    T = Abuf.reshape(9, Nx, Yl, nzh)
    T = np.fft.fft(T, axis=1)
    T = _ghat_apply(T, np.arange(Nx), rank * Yl + np.arange(Yl), np.arange(nzh), Nx, Ny, Nz)
    T = np.fft.ifft(T, axis=1)
    B2 = np.zeros_like(B)
    exchange(np.ascontiguousarray(T).reshape(-1), B2, False)
    # passes 4-5: unpack, inverse y, c2r z
    S2 = B2.reshape(P, 9, Xl, Yl, nzh).transpose(1, 2, 0, 3, 4).reshape(9, Xl, Ny, nzh)
    S2 = np.fft.ifft(S2, axis=2)
    S2 = np.concatenate([S2, np.zeros((9, Xl, Ny, 1))], axis=3)
    out = np.fft.irfft(S2, n=Nz, axis=3)
    gathered = [torch.empty(9 * Xl * Ny * Nz, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(out).reshape(-1)))
    if rank == 0:
        full = np.concatenate([g.numpy().reshape(9, Xl, Ny, Nz) for g in gathered], axis=1)
        q.put(full)
    dist.destroy_process_group()


@pytest.mark.parametrize("P,pts", [(2, (8, 6, 10)), (4, (8, 12, 6))])
def test_slab_transpose_plan_across_processes(P, pts):
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


def test_chunk_plan_covers_every_element_once():
    P, Nx, Ny, nzh, NC = 4, 8, 12, 3, 9
    rank_elems = NC * (Nx // P) * Ny * nzh
    for dst in range(P):
        seen = np.zeros(rank_elems, dtype=int)
        for src in range(P):
            for c in range(NC):
                b, a, cnt = abi.dist_chunk(P, Nx, Ny, nzh, NC, src, dst, c)
                assert cnt == (Nx // P) * (Ny // P) * nzh
                seen[a:a + cnt] += 1
        assert np.all(seen == 1)
    with pytest.raises(abi.FmError):
        abi.dist_chunk(3, 8, 12, 3, 9, 0, 0, 0)  # Nx not divisible
