"""Config 4 at 1024^3 on one B200: G applied in place (77 GB field + 77 GB half
spectrum), timed with CUDA events on the library stream, checked against the
analytic projection of a Fourier-mode field (tests/fourier_modes.py)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests"))
import fourier_modes as FM  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
q, a, phi = FM.modes(N)
b = FM.projected_amplitudes(N, q, a)
with abi.Context((N, N, N), 3) as ctx:
    f = ctx.field(9)
    view = torch.as_tensor(f, device="cuda")
    FM.fill(view, N, q, a, phi)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.projection(f, out=f)
    ctx.sync()
    err1, ref = FM.max_error(view, N, q, b, phi)
    torch.cuda.synchronize()
    ctx.profile(True)
    e0.record(st)
    for _ in range(reps):
        ctx.projection(f, out=f)
    e1.record(st)
    e1.synchronize()
    ms, calls = ctx.profile_read()
    ms_g = e0.elapsed_time(e1) / reps
    err2, _ = FM.max_error(view, N, q, b, phi)
n = N ** 3
bg = 2 * 72 + 8 * 144 * (N // 2) / N
print(json.dumps({"grid": N, "in_place": True, "ms": ms_g, "voxel_per_s": n / (ms_g * 1e-3),
                  "bytes_per_voxel": bg, "roofline_frac": bg * n / (ms_g * 1e-3) / 1e9 / hbm,
                  "passes_ms": [m / calls for m in ms], "known_answer_rel_err": err1 / ref,
                  "after_repeats_rel_err": err2 / ref}))
