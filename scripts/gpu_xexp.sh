# 512-point x pass variants: FM_XSPLIT 0 (k_x_direct), 1..3 (k_x_split shapes)
mkdir -p gpurun_out
for m in 0 1 2 3; do FM_XSPLIT=$m timeout 300 python scripts/xdirect_check.py > gpurun_out/xs$m.json 2>&1; echo "xsplit=$m rc=$?"; python -c "import json;d=json.load(open('gpurun_out/xs$m.json'));print(d['G_passes_ms'],d['virtual_P4_bitwise'],d['(512, 8, 16)'], d['idempotence_512'])"; done
