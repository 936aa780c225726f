"""The distributed data plane on real devices: one process per GPU
(torchrun), fm_ctx_create_dist, both transpose arms, bit for bit against the
single-device result (tests/dist_spawn_run.py).  Needs at least two GPUs with
peer access; skipped otherwise (the virtual-rank tests in test_gpu_dist.py
cover the same kernels and index maps on one device)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("pts,P", [("64x64x64", 2), ("128x64x32", 2), ("512x32x16", 2), ("64x64x64", 4)])
def test_slab_ranks_on_devices_match_single_device(pts, P):
    if _gpus() < P:
        pytest.skip(f"needs {P} GPUs, have {_gpus()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}", "--master-addr",
           "127.0.0.1", "--master-port", "29613", os.path.join(HERE, "dist_spawn_run.py"), pts]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    assert r.stdout.count(": OK") == 2 * P, r.stdout
