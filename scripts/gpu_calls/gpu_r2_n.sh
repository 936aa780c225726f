mkdir -p gpurun_out
timeout 300 python scripts/x_ab.py 512 4,7 > gpurun_out/x_ab_512_r2n.jsonl 2>&1; echo rc=$?; cat gpurun_out/x_ab_512_r2n.jsonl | cut -c1-400
FM_XDIRECT=7 FM_X_DBG=1 timeout 120 python scripts/x_stride.py 512x512x512 5 > gpurun_out/x_dbg_r2n.jsonl 2>&1; cat gpurun_out/x_dbg_r2n.jsonl | cut -c1-300
FM_XDIRECT=7 timeout 300 python scripts/x_stride.py 512x64x512,512x128x128,512x256x256 5 >> gpurun_out/x_dbg_r2n.jsonl 2>&1; tail -3 gpurun_out/x_dbg_r2n.jsonl | cut -c1-300
