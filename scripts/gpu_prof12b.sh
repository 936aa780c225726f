# round-1 v12: ncu --set full of the fused-CG kernels of the config-2 Newton solve (the e2e path):
# pass 1 with the direction / x update and curvature partials, pass 5 with r -= alpha Ap and <r,r> partials
mkdir -p gpurun_out
timeout 300 python scripts/solve_cfg2.py 256 mf > gpurun_out/solve12.log 2>&1; echo rc_solve=$?; tail -2 gpurun_out/solve12.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_zf_pipe<.int.128, .int.2, .bool.1|k_zi_reg<.int.128, .int.16, .int.16, .int.4, .bool.1' -s 6 -c 2 -o gpurun_out/prof_r1v12_cg \
  python scripts/solve_cfg2.py 256 mf > gpurun_out/ncu12c.log 2>&1; echo rc_ncu=$?; tail -3 gpurun_out/ncu12c.log
python scripts/ncu_summary.py gpurun_out/prof_r1v12_cg.ncu-rep > gpurun_out/r1_cg256_fused_v12.md 2>&1
ncu -i gpurun_out/prof_r1v12_cg.ncu-rep --page source --csv --print-source sass > gpurun_out/src_cg.csv 2>/dev/null; python scripts/ncu_stalls.py gpurun_out/src_cg.csv 20 > gpurun_out/stalls_cg_v12.txt 2>&1
ncu -i gpurun_out/prof_r1v12_cg.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/cg_traffic_v12.csv 2>&1
rm -f gpurun_out/src_cg.csv gpurun_out/prof_r1v12_cg.ncu-rep
echo done
