# config 1 (31^3 J2) persistent CG loop: phase timing and checksums (a fused y-x-y phase, 48 (kz, row) items per
# iteration, measured 100 us against 33 us for the three phases: too little parallelism per item; removed)
mkdir -p gpurun_out
for v in 0 1; do
  echo "== FM_CG_YXY=$v"
  FM_CG_YXY=$v FM_CG_SMALL_TIMING=1 python scripts/cfg1_short.py 2 2>&1 | tail -3 | cut -c1-250
  FM_CG_YXY=$v python scripts/cfg1_short.py 20 2>&1 | tail -2
  FM_CG_YXY=$v CFG1_COMPACT=1 python scripts/cfg1_short.py 20 2>&1 | tail -2
  FM_CG_YXY=$v python scripts/solve_cfg0.py 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_acceptance.py -q -x 2>&1 | tail -2
