"""BASELINE.json config 3: N^3 finite-strain J2, seeded random periodic spheres
(radius 12 at 512^3, volume fraction 0.25, seed 3), inclusion parameters 2x the
matrix, simple shear to gamma = 0.05 in 10 increments.  Device-resident Newton /
CG with the compact J2 tangent (fits 512^3 on one B200).
usage: python scripts/run_config3.py [N] [radius] [increments_to_run]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
radius = int(sys.argv[2]) if len(sys.argv) > 2 else 12
run_incs = int(sys.argv[3]) if len(sys.argv) > 3 else 10
t0 = time.time()
pg, frac, count = M.random_spheres(N, radius, 0.25, 3)
phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
          M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
lam, mu, ty, h = M.bind_parameters(pg, phases)
setup = time.time() - t0
ctx = abi.Context((N, N, N), 3)
model = abi.Model(ctx, "simo", lam, mu, ty, h, compact=True)
F = ctx.field(9, abi.identity_field((N, N, N), 3))
out = {"grid": N, "radius": radius, "fraction": frac, "spheres": count, "setup_s": setup, "increments": []}
prog = M.simple_shear_program(0.05, 10, 3)[:run_incs]
t = time.time()
for k, fb in enumerate(prog):
    ti = time.time()
    rep = model.solve_increment(F, fb)
    out["increments"].append({"newton": rep["passes"], "cg": rep["cg_it"], "matvecs": rep["matvecs"],
                              "rel_update": rep["rel_update"][-1], "eq_rel": rep["eq_rel"],
                              "wall_s": time.time() - ti})
    print(json.dumps(out["increments"][-1]), flush=True)
out["solve_s"] = time.time() - t
out["matvecs"] = sum(i["matvecs"] for i in out["increments"])
out["ms_per_matvec"] = 1e3 * out["solve_s"] / out["matvecs"]
out["epsp_max"] = float(model.history(0)[1].max())
print(json.dumps(out))
