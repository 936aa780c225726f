# round-1 v11 evidence: GPU tests, bench (both arms), smoke, pass times, ncu of the K4 pass 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rcref=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc_smoke=$?
python scripts/pass_times.py 128 256 512 > gpurun_out/pt11.json 2>&1
python scripts/svk_check.py 256 k4 > gpurun_out/k4_11.json 2>&1; python scripts/svk_check.py 512 >> gpurun_out/k4_11.json 2>&1
python scripts/prof_matvec.py 256 2 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast" -s 1 -c 1 -o gpurun_out/prof_r1v11_k4 python scripts/prof_matvec.py 256 2 > gpurun_out/ncu11b.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_r1v11_k4.ncu-rep > gpurun_out/r1_matvec256_k4_v11.md 2>&1
ncu -i gpurun_out/prof_r1v11_k4.ncu-rep --page source --csv --print-source sass > gpurun_out/src_k4.csv 2>/dev/null; python scripts/ncu_stalls.py gpurun_out/src_k4.csv 25 > gpurun_out/stalls_k4_v11.txt 2>&1; rm -f gpurun_out/src_k4.csv gpurun_out/prof_r1v11_k4.ncu-rep
echo done
