"""Time-to-solution of BASELINE.json configs 0, 1 and 2 through the C ABI
(device-resident Newton/CG), for DESIGN.md / bench extras."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M


def run(points, kind, phases, fbars, mf=False, repeat=2):
    out = None
    for _ in range(repeat):
        ctx = abi.Context(points, 3)
        pg = M.corner_cube(points, 9) if points[0] == 31 else M.bernoulli(points, 0.3, 2)
        lam, mu, ty, h = M.bind_parameters(pg, phases)
        model = abi.Model(ctx, kind, lam, mu, ty, h, matrix_free=mf)
        F = ctx.field(9, abi.identity_field(points, 3))
        ctx.sync()
        l0 = ctx.launches
        t = time.perf_counter()
        reps = abi.run_program(model, F, fbars)
        ctx.sync()
        wall = time.perf_counter() - t
        out = {"wall_s": wall, "increments": len(reps), "newton": [r["passes"] for r in reps],
               "cg": [r["cg_it"] for r in reps], "matvecs": sum(r["matvecs"] for r in reps),
               "launches": ctx.launches - l0}
        model.close(); ctx.close()
    return out


if __name__ == "__main__":
    el = [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)]
    pl = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003), M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    res = {}
    which = sys.argv[1:] or ["0", "1", "2"]
    if "0" in which:
        res["config0"] = run((31, 31, 31), "hyper", el, M.simple_shear_program(0.1, 1, 3))
        res["config0_matrix_free"] = run((31, 31, 31), "hyper", el, M.simple_shear_program(0.1, 1, 3), mf=True)
    if "1" in which:
        res["config1"] = run((31, 31, 31), "simo", pl, M.simple_shear_program(0.1, 20, 3), repeat=1)
    if "2" in which:
        res["config2"] = run((256, 256, 256), "hyper", el, M.simple_shear_program(0.1, 1, 3), repeat=1)
        res["config2_matrix_free"] = run((256, 256, 256), "hyper", el, M.simple_shear_program(0.1, 1, 3), mf=True, repeat=1)
    print(json.dumps(res))
