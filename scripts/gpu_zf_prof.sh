python scripts/prof_matvec.py 256 2 mf > gpurun_out/zfp_plain.log 2>&1 || exit 1
FM_ZPIPE=0 ncu --set full --clock-control none --import-source on -k regex:"k_zf" -s 1 -c 1 -o gpurun_out/zf_fast python scripts/prof_matvec.py 256 2 mf > gpurun_out/zfp_a.log 2>&1
FM_ZPIPE=3 ncu --set full --clock-control none --import-source on -k regex:"k_zf" -s 1 -c 1 -o gpurun_out/zf_pipe python scripts/prof_matvec.py 256 2 mf > gpurun_out/zfp_b.log 2>&1
echo done
