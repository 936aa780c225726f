mkdir -p gpurun_out
for p in 0 1 2 3; do FM_TMA_PROMO=$p FM_XDIRECT=7 timeout 120 python scripts/x_stride.py 512x512x512 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(json.dumps({'promo':$p,'x_ms':r['passes_ms'][2],'x_frac':r['pass_frac'][2]}))"; done > gpurun_out/x_promo_r2q.jsonl 2>&1; cat gpurun_out/x_promo_r2q.jsonl
