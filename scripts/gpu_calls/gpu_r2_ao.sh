for d in 0 1 2 4 3 5 6 7; do FM_LIB=$PWD/paper_1603_08893_b200/lib/libfftmech_b200_v.so FM_X4_DBG=$d timeout 120 python scripts/x_stride.py 256x256x256 10 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(json.dumps({'dbg':$d,'x_ms':r['passes_ms'][2],'x_frac':r['pass_frac'][2]}))"; done
timeout 120 python scripts/x_stride.py 256x256x256 10 2>&1 | cut -c1-150
