"""Config 4 up to 1024^3 on ONE B200: the projection applied
in place to a sum of Fourier modes must reproduce the analytic projection
(tests/fourier_modes.py) -- an exact known-answer test at any N, checked on
the device -- and stay there when applied again (idempotence, G(G x) = G x).
At 1024^3 the field (77 GB) and the half spectrum (77 GB) fit one B200 when
the output overwrites the input; BASELINE.json places 1024^3 on 8 GPUs."""
import numpy as np
import pytest
import torch

from paper_1603_08893_b200 import abi
import fourier_modes as FM

pytestmark = pytest.mark.gpu


def _run(N, reps=1):
    q, a, phi = FM.modes(N)
    b = FM.projected_amplitudes(N, q, a)
    with abi.Context((N, N, N), 3) as ctx:
        f = ctx.field(9)
        view = torch.as_tensor(f, device="cuda")
        FM.fill(view, N, q, a, phi)
        torch.cuda.synchronize()
        ctx.projection(f, out=f)  # in place: pass 1 consumes the input before pass 5 writes
        ctx.sync()
        e1, r1 = FM.max_error(view, N, q, b, phi)
        torch.cuda.synchronize()
        for _ in range(reps):
            ctx.projection(f, out=f)
        ctx.sync()
        e2, r2 = FM.max_error(view, N, q, b, phi)
    return e1 / r1, e2 / r2


@pytest.mark.parametrize("N", [32, 128, 256])
def test_fourier_modes_known_answer(N):
    e1, e2 = _run(N)
    assert e1 < 1e-12 and e2 < 1e-12, (e1, e2)


def test_fourier_modes_known_answer_1024():
    free, _ = torch.cuda.mem_get_info()
    if free < 160e9:
        pytest.skip(f"1024^3 in place needs ~155 GB of HBM, {free / 1e9:.0f} GB free")
    e1, e2 = _run(1024)
    assert e1 < 1e-11 and e2 < 1e-11, (e1, e2)
