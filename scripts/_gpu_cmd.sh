make -j8 >/dev/null 2>&1
timeout 600 python bench.py --no-cpu --no-offload > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(d['value'], d['collectives'])"; tail -2 gpurun_out/b.err
