mkdir -p gpurun_out
for p in 0 1 0 1; do FM_XW_PARK=$p FM_XDIRECT=7 FM_X_DBG=16 timeout 120 python scripts/x_stride.py 512x512x512 5 2>&1 | tail -2 | cut -c1-200; done > gpurun_out/x_park_r2y.txt 2>&1; cat gpurun_out/x_park_r2y.txt
FM_XW_PARK=1 timeout 300 python scripts/x_ab.py 512 7 2>&1 | cut -c1-300
