"""Compare x-pass variants (FM_XPASS) at N^3: matvec time and output drift."""
import os
import subprocess
import sys

if len(sys.argv) > 2:  # child: one variant
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import time
    import numpy as np
    from paper_1603_08893_b200 import abi
    N = int(sys.argv[1]); n = N ** 3
    ctx = abi.Context((N, N, N), 3)
    rng = np.random.default_rng(0)
    lam = np.where(rng.random(n) < 0.3, 5.769, 0.5769); mu = lam / 1.5
    model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
    F0 = abi.identity_field((N, N, N), 3); F0[n:2 * n] = 0.1
    F = ctx.field(9, F0); P = ctx.field(9)
    model.evaluate(F, P)
    dF = ctx.field(9, rng.uniform(-1, 1, 9 * n)); out = ctx.field(9)
    for _ in range(3):
        model.apply(dF, out)
    ctx.sync()
    reps = 30
    t = time.perf_counter()
    for _ in range(reps):
        model.apply(dF, out)
    ctx.sync()
    dt = (time.perf_counter() - t) / reps
    np.save(f"/tmp/xvar_{sys.argv[2].replace('=', '_')}.npy", out.download())
    print(f"variant {sys.argv[2]} N={N} matvec {dt*1e3:.3f} ms")
else:
    N = sys.argv[1] if len(sys.argv) > 1 else "256"
    import numpy as np
    vs = os.environ.get("VARIANTS", "5 6 7").split()
    for v in vs:  # "6" -> FM_XPASS=6; "FM_ZPIPE=0" -> that variable
        k, val = v.split("=") if "=" in v else ("FM_XPASS", v)
        env = dict(os.environ, **{k: val})
        subprocess.run([sys.executable, __file__, N, v], env=env, check=True)
    ref = np.load(f"/tmp/xvar_{vs[0].replace('=', '_')}.npy")
    for v in vs[1:]:
        o = np.load(f"/tmp/xvar_{v.replace('=', '_')}.npy")
        print(v, "max rel diff vs", vs[0], float(np.abs(o - ref).max() / np.abs(ref).max()))
