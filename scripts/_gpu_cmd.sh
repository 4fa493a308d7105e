make -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpt_gpu.py tests/test_fullsize_gpu.py -m gpu -q 2>&1 | tail -2
for ov in 1 0; do ZI_EAGER_ADAM=$ov timeout 600 python bench.py --no-cpu --no-offload > gpurun_out/b$ov.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b$ov.json').read().strip().splitlines()[-1]);print('eager', $ov, d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['share_of_step'], d['roofline']['bytes_per_launch'], d['clocks']['sm_mhz'])"; done
