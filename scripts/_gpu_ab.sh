# same-box interleaved A/B of an env knob on the graphed N=1 step: bash scripts/_gpu_ab.sh VAR "A B" [rounds]
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
VAR=$1; VALS=$2; R=${3:-2}
for r in $(seq $R); do for v in $VALS; do env $VAR=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['gpu_launches'])"; done; done
