make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
for cl in 4; do echo "== CL $cl"; ZI_SK_CL=$cl timeout 600 python -m pytest tests/test_gemm_sk_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3; done
for cl in 4 2; do echo "== CL $cl"; ZI_SK_CL=$cl timeout 600 python scripts/bench_gemm_sk.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if 'site' in d: print(d['site'], 'sk', d['sk_tflops'], 'whole', d['whole_tflops'], 'cublas', d['cublas_tflops'], 'zi', d['zi_tflops'])
    else: print(d)
"; done
python - <<'P'
import ctypes, torch, sys
sys.path.insert(0, '.')
torch.cuda.init()
P
