# ncu --set full of the 512^3 x pass (k_x_direct) with source attribution
mkdir -p gpurun_out
python scripts/prof_G.py 512 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_x_direct" -s 1 -c 1 -o gpurun_out/prof_x512d python scripts/prof_G.py 512 2 > gpurun_out/ncux512d.log 2>&1; echo rcn=$?
