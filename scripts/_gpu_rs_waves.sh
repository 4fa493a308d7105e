# fused RS + Adam grid of one resident wave (default) vs two (ZI_RS_WAVES=2, the old 8 CTAs / SM)
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_fused_gpu.py tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for w in 1 2; do echo "waves $w: $(ZI_RS_WAVES=$w timeout 300 python scripts/bench_rs_adam.py 2>&1 | head -1)"; done; done
for r in 1 2; do for w in 1 2; do
  ZI_RS_WAVES=$w timeout 600 python bench.py --no-offload --no-nvme --no-cpu --no-config3 > gpurun_out/rsw_${w}_$r.log 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/rsw_${w}_$r.log').read().strip().splitlines()[-1]); print('step waves $w', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline_hbm']['achieved'], d['roofline_hbm']['frac'])"
done; done
