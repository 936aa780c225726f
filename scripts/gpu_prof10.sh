# round-1 v10 evidence: GPU tests, bench (both arms), smoke, ncu launch list and --set full captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rcref=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc_smoke=$?
python scripts/pass_times.py 128 256 512 > gpurun_out/pt10.json 2>&1
python scripts/prof_matvec.py 256 2 mf > /dev/null 2>&1 && python scripts/prof_matvec.py 256 2 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1v10.csv python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu10c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf|k_y_fast|k_x_fast|k_zi_reg" -s 5 -c 5 -o gpurun_out/prof_r1v10_mf python scripts/prof_matvec.py 256 2 mf > gpurun_out/ncu10a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast" -s 1 -c 1 -o gpurun_out/prof_r1v10_k4 python scripts/prof_matvec.py 256 2 > gpurun_out/ncu10b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_x_direct" -s 1 -c 1 -o gpurun_out/prof_r1v10_x512 python scripts/prof_G.py 512 2 > gpurun_out/ncu10d.log 2>&1

# summaries on the box (gpurun_out/ must stay under 64 MiB to come back)
python scripts/ncu_summary.py gpurun_out/prof_r1v10_mf.ncu-rep gpurun_out/launches_r1v10.csv > gpurun_out/r1_matvec256_mf_v10.md 2>&1
python scripts/ncu_summary.py gpurun_out/prof_r1v10_k4.ncu-rep > gpurun_out/r1_matvec256_k4_v10.md 2>&1
python scripts/ncu_summary.py gpurun_out/prof_r1v10_x512.ncu-rep > gpurun_out/r1_x512_v10.md 2>&1
for r in mf k4 x512; do ncu -i gpurun_out/prof_r1v10_$r.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$r.csv 2>/dev/null; python scripts/ncu_stalls.py gpurun_out/src_$r.csv 25 > gpurun_out/stalls_$r.txt 2>&1; rm -f gpurun_out/src_$r.csv; done
rm -f gpurun_out/prof_r1v10_*.ncu-rep
du -sh gpurun_out
echo done
