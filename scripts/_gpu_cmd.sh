make -j8 >/dev/null 2>&1
for rep in 1 2; do for ov in 1 0; do
ZI_OVERLAP_OPT=$ov timeout 600 python bench.py --no-cpu --no-offload > gpurun_out/b$ov.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b$ov.json').read().strip().splitlines()[-1]);print('overlap=$ov', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['share_of_step'], d['clocks']['sm_mhz'])"
done; done
timeout 600 python -m pytest tests/test_gpt_gpu.py tests/test_fullsize_gpu.py -q -m gpu 2>&1 | tail -2
