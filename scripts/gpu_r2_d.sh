mkdir -p gpurun_out
timeout 600 python scripts/x_ab.py 512 2,4,5 > gpurun_out/x_ab_512_r2d.jsonl 2>&1; echo rc_xab=$?; cat gpurun_out/x_ab_512_r2d.jsonl
timeout 600 python -m pytest tests/test_gpu_projection.py -q -x -k "512" > gpurun_out/gpu_tests_r2d.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/gpu_tests_r2d.log
for m in 2 4; do
FM_XDIRECT=$m python scripts/prof_G.py 512 2 > /dev/null 2>&1 && FM_XDIRECT=$m timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_x_stream" -s 1 -c 1 -o gpurun_out/prof_xs512_m$m python scripts/prof_G.py 512 2 > gpurun_out/ncu_xs_m$m.log 2>&1; echo rc_ncu_$m=$?
done
