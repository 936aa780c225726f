mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -i "model name\|^CPU(s)" >> gpurun_out/nproc.txt
bash scripts/ncu_box.sh mf256 "k_zf_pipe|k_y_fast|k_x_|k_zi_reg" 5 5 python scripts/svk_check.py 256
( time python bench.py > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err ) 2> gpurun_out/bench_r2h.time; echo rc_bench=$?; tail -3 gpurun_out/bench_r2h.err; cat gpurun_out/bench_r2h.time
( time python bench.py --impl reference > gpurun_out/bench_ref_r2h.json 2> gpurun_out/bench_ref_r2h.err ) 2> gpurun_out/bench_ref_r2h.time; echo rc_ref=$?; cat gpurun_out/bench_ref_r2h.json; cat gpurun_out/bench_ref_r2h.time
