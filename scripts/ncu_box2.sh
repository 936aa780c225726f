# like ncu_box.sh, plus the per-opcode stall table and a longer per-line table
tag=$1; rx=$2; skip=$3; cnt=$4; shift 4
mkdir -p gpurun_out
"$@" > gpurun_out/ncu_plain_$tag.log 2>&1 || { echo "plain run failed: $tag"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt -o /tmp/prof_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1 || { echo "ncu failed: $tag"; tail -5 gpurun_out/ncu_$tag.log; exit 1; }
python scripts/ncu_summary.py /tmp/prof_$tag.ncu-rep > gpurun_out/prof_$tag.md 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass > /tmp/src_$tag.csv 2>/dev/null
python scripts/ncu_stalls.py /tmp/src_$tag.csv 60 >> gpurun_out/prof_$tag.md 2>&1
python scripts/ncu_stalls_by_op.py /tmp/src_$tag.csv >> gpurun_out/prof_$tag.md 2>&1
rm -f /tmp/prof_$tag.ncu-rep /tmp/src_$tag.csv
echo "ncu ok: $tag"
