"""Config 1 (31^3 J2 corner inclusion), first 3 increments, for kernel timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M
incs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pts = (31, 31, 31)
lam, mu, ty, h = M.bind_parameters(M.corner_cube(pts, 9), [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
                                                          M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)])
with abi.Context(pts, 3) as ctx:
    m = abi.Model(ctx, "simo", lam, mu, ty, h, compact=os.environ.get("CFG1_COMPACT") == "1")
    F = ctx.field(9, abi.identity_field(pts, 3))
    t = time.perf_counter()
    reps = abi.run_program(m, F, M.simple_shear_program(0.1, 20, 3)[:incs])
    ctx.sync()
    print("time", time.perf_counter() - t, [sum(r["cg_it"]) for r in reps])
    import hashlib
    print("F sha1", hashlib.sha1(F.download().tobytes()).hexdigest()[:16])
