# round 2, call AF: bench + reference arm on HEAD, ncu of the three 512-point passes that changed
mkdir -p gpurun_out
( time python bench.py > gpurun_out/bench_r2af.json 2> gpurun_out/bench_r2af.err ) 2> gpurun_out/bench_r2af.time; echo rc_bench=$?; tail -2 gpurun_out/bench_r2af.err
( time python bench.py --impl reference > gpurun_out/bench_ref_r2af.json 2> gpurun_out/bench_ref_r2af.err ) 2> gpurun_out/bench_ref_r2af.time; echo rc_ref=$?
bash scripts/ncu_box2.sh g512 "k_x_warp|k_y_fast|k_zf_reg|k_zi_reg" 5 5 python scripts/prof_G.py 512 2
