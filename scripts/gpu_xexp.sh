# SVK pass 1 A/B (double-buffered staging measured 0.72 vs 0.69 ms at 256^3 and removed)
for v in "FM_PIPE_DB=0" "FM_PIPE_DB=1" "FM_PHASE_LABELS=0"; do env $v python scripts/svk_check.py 256; done
for v in "FM_PIPE_DB=0" "FM_PIPE_DB=1"; do env $v python scripts/svk_check.py 256; done
