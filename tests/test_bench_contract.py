"""bench.py's reference arm (`--impl reference`): the JSON line the driver reads, on host cores only.

The arm times the oracle's `apply_projected_tangent` (the restated reference,
proj/core/src/projection.cpp:173-194) on the config-2 generator; here on a
32^3 grid so it runs in the CPU suite.  Under torchrun only rank 0 works."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(extra_env, *args):
    env = dict(os.environ, **extra_env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_line(oracle):
    r = run_bench({}, "--impl", "reference", "--grid", "32", "--steps", "2", "--warmup", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "fp64 CG matvec voxels/s (G:K4:dF)" and line["unit"] == "voxel/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1
    assert line["dtype"] == "f64" and line["data"] == "synthetic"
    assert line["config"]["workload"].startswith("config2: 32^3")
    cb = line["cpu_baseline"]
    assert cb["value"] == line["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "voxel/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly(oracle):
    # torchrun N=2: rank 1 does no work, prints nothing and needs no process group or GPU
    r = run_bench({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}, "--impl", "reference", "--grid", "32",
                  "--gpus", "2", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""
    r0 = run_bench({"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}, "--impl", "reference", "--grid", "32",
                   "--gpus", "2", "--steps", "1", "--warmup", "0")
    assert r0.returncode == 0, r0.stderr[-2000:]
    assert json.loads(r0.stdout.strip().splitlines()[-1])["n_gpus"] == 2
