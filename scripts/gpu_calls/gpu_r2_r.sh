mkdir -p gpurun_out
timeout 300 python scripts/x_ab.py 512 7 > gpurun_out/x_ab_512_r2r.jsonl 2>&1; echo rc=$?; cut -c1-300 gpurun_out/x_ab_512_r2r.jsonl
FM_XW_TMA_STORE=1 timeout 300 python scripts/x_ab.py 512 7 2>&1 | cut -c1-300
for d in 16 17; do FM_XDIRECT=7 FM_X_DBG=$d timeout 120 python scripts/x_stride.py 512x512x512 3 2>&1 | tail -2 | cut -c1-260; done > gpurun_out/x_prof_r2r.txt 2>&1; cat gpurun_out/x_prof_r2r.txt
