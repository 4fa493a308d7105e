make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python -m pytest tests/test_gemm_sk_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
run() { env $2 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-offload > gpurun_out/bench_ab.log 2>&1
python - "$1" <<'P'
import json,sys
d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])
P
}
run zi-cl2 "ZI_GEMM_SELECT=zi ZI_SK_CL=2"; run zi-cl4 "ZI_GEMM_SELECT=zi ZI_SK_CL=4"; run cublas "ZI_GEMM_SELECT=cublas"
run zi-cl2 "ZI_GEMM_SELECT=zi ZI_SK_CL=2"; run zi-cl4 "ZI_GEMM_SELECT=zi ZI_SK_CL=4"; run cublas "ZI_GEMM_SELECT=cublas"
