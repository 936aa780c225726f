mkdir -p gpurun_out
for rep in 1 2; do
for lib in libfftmech_b200.so libfftmech_b200_ef16.so; do FM_LIB=$PWD/paper_1603_08893_b200/lib/$lib timeout 120 python scripts/svk_check.py 256 2>&1 | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$lib', r['sha1'], r['passes_ms'], r['ms'])"; done; done
FM_LIB=$PWD/paper_1603_08893_b200/lib/libfftmech_b200_ef16.so timeout 900 python -m pytest tests/test_gpu_svk_oracle.py tests/test_gpu_solver.py -q -x 2>&1 | tail -3
