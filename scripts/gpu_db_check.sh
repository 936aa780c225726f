# A/B of a double-buffered in-place SVK-label pass 1 (FM_ZPIPE_DB, measured and dropped in v12: DESIGN §3)
for i in 1 2; do
  FM_ZPIPE_DB=0 timeout 300 python scripts/svk_check.py 256 svk
  FM_ZPIPE_DB=1 timeout 300 python scripts/svk_check.py 256 svk
done 2>&1 | tee gpurun_out/db_check.log
FM_ZPIPE_DB=0 timeout 300 python scripts/svk_check.py 128 svk 2>&1 | tee -a gpurun_out/db_check.log
FM_ZPIPE_DB=1 timeout 300 python scripts/svk_check.py 128 svk 2>&1 | tee -a gpurun_out/db_check.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_db.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/gpu_tests_db.log
tail -2 gpurun_out/gpu_tests_db.log
timeout 600 python bench.py > gpurun_out/bench_db.json 2> gpurun_out/bench_db.err; echo "BENCH EXIT $?"
