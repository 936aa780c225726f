# round-1 v12 evidence: smoke, ncu --set full of the compact-J2 pass 1 (config-3 operator) at 256^3,
# and the bench's launch list (gpu__time_duration, cold-cache serialised)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke12.log 2>&1; echo rc_smoke=$?
timeout 300 python scripts/svk_check.py 256 j2c > gpurun_out/j2c12.json 2>&1; echo rc_j2c=$?; cat gpurun_out/j2c12.json | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast" -s 1 -c 1 -o gpurun_out/prof_r1v12_j2c python scripts/svk_check.py 256 j2c > gpurun_out/ncu12a.log 2>&1; echo rc_ncu=$?
python scripts/ncu_summary.py gpurun_out/prof_r1v12_j2c.ncu-rep > gpurun_out/r1_matvec256_j2c_v12.md 2>&1
ncu -i gpurun_out/prof_r1v12_j2c.ncu-rep --page source --csv --print-source sass > gpurun_out/src_j2c.csv 2>/dev/null; python scripts/ncu_stalls.py gpurun_out/src_j2c.csv 25 > gpurun_out/stalls_j2c_v12.txt 2>&1; rm -f gpurun_out/src_j2c.csv gpurun_out/prof_r1v12_j2c.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_v12.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu12b.log 2>&1; echo rc_ncu_bench=$?
echo done
