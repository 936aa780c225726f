# A/B of a warp-specialised SVK-label pass 1 (FM_ZWS, measured and dropped in v12: DESIGN §3)
for i in 1 2; do
  for v in 0 1 2; do FM_ZWS=$v timeout 120 python scripts/svk_check.py 256 svk; echo "rc=$? FM_ZWS=$v"; done
done 2>&1 | tee gpurun_out/ws_check.log
for v in 0 1 2; do FM_ZWS=$v timeout 120 python scripts/svk_check.py 128 svk; done 2>&1 | tee -a gpurun_out/ws_check.log
