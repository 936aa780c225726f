mkdir -p gpurun_out
for d in 0 1 5 9 4 6 8; do FM_X_DBG=$d python scripts/x_stride.py 512x512x512 5 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(json.dumps({'dbg':$d,'x_ms':r['passes_ms'][2],'x_frac':r['pass_frac'][2]}))"
done > gpurun_out/x_dbg_r2m.jsonl 2>&1; cat gpurun_out/x_dbg_r2m.jsonl
