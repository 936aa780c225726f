mkdir -p gpurun_out
timeout 300 python scripts/x_ab.py 512 7 > gpurun_out/x_ab_512_r2v.jsonl 2>&1; echo rc=$?; cut -c1-300 gpurun_out/x_ab_512_r2v.jsonl
FM_XDIRECT=7 FM_X_DBG=16 timeout 120 python scripts/x_stride.py 512x512x512 3 2>&1 | tail -2 | cut -c1-260
