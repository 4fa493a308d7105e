L=paper_2104_07857_b200/libzinf.so
cp $L /tmp/new.so
for rep in 1 2; do
cp build_ab/libzinf_old.so $L; echo old; timeout 300 python scripts/bench_fused.py 2>&1 | grep -i "softmax"
cp /tmp/new.so $L; echo new; timeout 300 python scripts/bench_fused.py 2>&1 | grep -i "softmax"
done
timeout 600 python -m pytest tests/test_fused_gpu.py tests/test_gpt_gpu.py -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-offload > gpurun_out/b.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
