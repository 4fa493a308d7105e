# run-to-run spread of the main bench arm: 5 back-to-back runs of the same command on one box
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-offload --no-nvme --no-cpu --no-config3 > gpurun_out/noise_$i.log 2> gpurun_out/noise_$i.err
  python - "$i" <<'P'
import json, sys
d = json.loads(open(f"gpurun_out/noise_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"],
      d["roofline"]["frac"], d["roofline"]["achieved"])
P
done
