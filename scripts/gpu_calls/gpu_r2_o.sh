mkdir -p gpurun_out
timeout 300 python scripts/x_ab.py 512 4,7 > gpurun_out/x_ab_512_r2o.jsonl 2>&1; echo rc=$?; cat gpurun_out/x_ab_512_r2o.jsonl | cut -c1-300
for d in 16 17; do FM_XDIRECT=7 FM_X_DBG=$d timeout 120 python scripts/x_stride.py 512x512x512 3 2>&1 | cut -c1-260; done > gpurun_out/x_prof_r2o.txt 2>&1; cat gpurun_out/x_prof_r2o.txt
