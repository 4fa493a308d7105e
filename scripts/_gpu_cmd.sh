make -j8 >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpt_gpu.py tests/test_fused_gpu.py -q -x 2>&1 | tail -2
for f in auto cublas; do ZI_GEMM_SELECT=$f timeout 600 python bench.py --no-cpu --no-offload > gpurun_out/bf$f.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bf$f.json').read().strip().splitlines()[-1]);print('gemm_select=$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"; done
