# round 2, call A: smoke (hot-path kernels), full GPU suite incl. the new
# SVK / K4 pass-1 oracle tests, constitutive timings + ncu of k_hyper / k_simo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2a.log 2>&1; echo rc_smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/gpu_tests_r2a.log 2>&1; echo rc_tests=$?
tail -5 gpurun_out/gpu_tests_r2a.log
python scripts/prof_constitutive.py 256 5 > gpurun_out/const_r2a.json 2>&1; echo rc_const=$?; cat gpurun_out/const_r2a.json
python scripts/prof_constitutive.py 256 1 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hyper|k_simo" -c 8 -o gpurun_out/prof_const_r2a python scripts/prof_constitutive.py 256 1 > gpurun_out/ncu_const_r2a.log 2>&1; echo rc_ncu=$?
