"""Known-answer fields for the projection at any grid size (SURVEY.md §8(d),
config 4): a sum of real Fourier modes whose projection is analytic.

For A_ij(r) = sum_k a_k,ij cos(2 pi q_k.r / N + phi_k) the reference G
(projection.cpp:87-104, 139-152, ZeroCompatible Nyquist) gives
B_ij(r) = sum_k (sum_l a_k,il xi_l) xi_j / |xi|^2 cos(...), xi = q_k / L,
and 0 for the q = 0 mode and for modes on a Nyquist plane.  Fields are built
and checked on the device through torch (test infrastructure), plane chunk by
plane chunk, so a 1024^3 field (77 GB) never leaves HBM."""
import numpy as np
import torch


def modes(N, seed=11):
    """(q [K,3] ints, amplitudes [K,9], phases [K]): random interior modes plus
    the mean and a Nyquist mode (both projected to zero)."""
    rng = np.random.default_rng(seed)
    q = [rng.integers(-N // 2 + 1, N // 2, size=3) for _ in range(5)]
    q.append(np.array([0, 0, 0]))
    q.append(np.array([N // 2, 3, -2]))  # Nyquist plane in x: ZeroCompatible -> 0
    q = np.array(q, dtype=np.int64)
    a = rng.uniform(-1, 1, (len(q), 9))
    phi = rng.uniform(0, 2 * np.pi, len(q))
    return q, a, phi


def projected_amplitudes(N, q, a):
    """Per-mode amplitudes of G A (analytic)."""
    out = np.zeros_like(a)
    for k in range(len(q)):
        if not q[k].any() or (N % 2 == 0 and np.any(np.abs(q[k]) == N // 2)):
            continue
        xi = q[k].astype(float)
        A = a[k].reshape(3, 3)
        out[k] = (np.outer(A @ xi, xi) / (xi @ xi)).reshape(9)
    return out


def _chunk_phase(N, q, phi, x0, x1, dev):
    x = torch.arange(x0, x1, device=dev, dtype=torch.int64).view(-1, 1, 1)
    y = torch.arange(N, device=dev, dtype=torch.int64).view(1, -1, 1)
    z = torch.arange(N, device=dev, dtype=torch.int64).view(1, 1, -1)
    out = []
    for k in range(len(q)):
        m = torch.remainder(int(q[k, 0]) * x + int(q[k, 1]) * y + int(q[k, 2]) * z, N)  # exact argument mod N
        out.append(torch.cos(m.to(torch.float64) * (2 * np.pi / N) + float(phi[k])))
    return out


def fill(view, N, q, amp, phi, chunk=16):
    """view: flat [9 N^3] device tensor (component-major, z fastest)."""
    dev = view.device
    V = view.view(9, N, N, N)
    for x0 in range(0, N, chunk):
        x1 = min(N, x0 + chunk)
        cs = _chunk_phase(N, q, phi, x0, x1, dev)
        for c in range(9):
            acc = torch.zeros((x1 - x0, N, N), dtype=torch.float64, device=dev)
            for k in range(len(q)):
                if amp[k, c] != 0.0:
                    acc.add_(cs[k], alpha=float(amp[k, c]))
            V[c, x0:x1].copy_(acc)


def max_error(view, N, q, amp, phi, chunk=16):
    """max |view - analytic field| and max |analytic field| over the grid."""
    dev = view.device
    V = view.view(9, N, N, N)
    err, ref = 0.0, 0.0
    for x0 in range(0, N, chunk):
        x1 = min(N, x0 + chunk)
        cs = _chunk_phase(N, q, phi, x0, x1, dev)
        for c in range(9):
            acc = torch.zeros((x1 - x0, N, N), dtype=torch.float64, device=dev)
            for k in range(len(q)):
                if amp[k, c] != 0.0:
                    acc.add_(cs[k], alpha=float(amp[k, c]))
            err = max(err, float((V[c, x0:x1] - acc).abs().max()))
            ref = max(ref, float(acc.abs().max()))
    return err, ref
