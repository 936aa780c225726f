# 512-point x pass: streaming (evict-first) loads/stores so spills stay in L2 (FM_XCS A/B)
for v in 0 1 0 1; do FM_XCS=$v python scripts/pass_times.py 512 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('xcs=$v', d['G_passes_ms'])"; done
