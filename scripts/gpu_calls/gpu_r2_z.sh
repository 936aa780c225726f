mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_projection.py tests/test_cli.py tests/test_gpu_debug_residue.py -q -x > gpurun_out/gpu_tests_r2z.log 2>&1; echo rc_tests=$?; tail -12 gpurun_out/gpu_tests_r2z.log
python - <<'PY'
# routed x pass at the 8-rank slab shape of 512^3 (virtual ranks on one device): k_x_warp<RT> vs k_x_stream<RT>
import os, subprocess, sys, json
code = """
import sys, json, os; sys.path.insert(0, '.')
import torch
from paper_1603_08893_b200 import abi
pts=(512,512,512)
with abi.Context(pts,3) as ctx:
    ctx.set_virtual_ranks(8)
    f=ctx.field(9); torch.as_tensor(f, device='cuda').uniform_(-1,1); out=ctx.field(9)
    ctx.projection(f,out=out); ctx.sync(); ctx.profile(True)
    for _ in range(5): ctx.projection(f,out=out)
    ms,calls=ctx.profile_read()
    print(json.dumps({'routed_xw': os.environ.get('FM_XW_ROUTED','1'), 'passes_ms':[round(m/calls,3) for m in ms], 'kernels': ctx.kernel_names}))
"""
for v in ("1", "0"):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, FM_XW_ROUTED=v), capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or r.stderr[-500:])
PY
