mkdir -p gpurun_out
python scripts/pass_times.py 512 > gpurun_out/pt512.json 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_x_fast4" -s 1 -c 1 -o gpurun_out/prof_x512 python scripts/prof_G.py 512 2 > gpurun_out/ncux512.log 2>&1; echo rcn=$?
