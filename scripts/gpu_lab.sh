# phase-label SVK pass 1: per-pass times and config-2 solve with labels (4 / 3 CTAs/SM) and without
mkdir -p gpurun_out
for v in "FM_PHASE_LABELS=0" "FM_PHASE_LABELS=1" "FM_PIPE_LAB_MINB3=1"; do
  echo "== $v"; env $v python scripts/pass_times.py 256 512 | python -c "import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['N'], d['mv_svk_passes_ms'], d['mv_svk_ms'])"
  env $v timeout 300 python scripts/solve_cfg2.py 256 mf 2>&1 | tail -2
done
