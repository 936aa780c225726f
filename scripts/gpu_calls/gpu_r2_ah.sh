mkdir -p gpurun_out
for d in 0 1 2 3 4 8 12 14 15 7; do FM_ZP_DBG=$d timeout 120 python scripts/svk_check.py 256 2>&1 | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    try:
        r=json.loads(l); print(json.dumps({'dbg':$d,'pass1_ms':r.get('passes_ms',r.get('pass_ms',[None]))[0]}))
    except Exception as e: print('dbg $d:', l[:200])"; done > gpurun_out/zp_dbg_r2ah.jsonl 2>&1; cat gpurun_out/zp_dbg_r2ah.jsonl
