"""The known-answer generator of the config-4 large-grid test (fourier_modes.py)
pinned against the CPU oracle's apply_projection (projection.cpp:123-171)."""
import numpy as np
import pytest
import torch

import fourier_modes as FM


@pytest.mark.parametrize("N", [8, 12, 16])
def test_analytic_projection_matches_oracle(N, oracle):
    q, a, phi = FM.modes(N, seed=5)
    b = FM.projected_amplitudes(N, q, a)
    A = torch.zeros(9 * N ** 3, dtype=torch.float64)
    FM.fill(A, N, q, a, phi, chunk=5)
    ref, st, _ = oracle.apply_projection((N, N, N), 3, A.numpy())
    assert st == 0
    err, mx = FM.max_error(torch.from_numpy(ref), N, q, b, phi, chunk=5)
    assert mx > 0.1 and err / mx < 1e-12
