make -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpt_gpu.py tests/test_multiproc_gpu.py -m gpu -q 2>&1 | tail -3
for i in 1 2; do timeout 600 python scripts/offload_equiv.py --batch 32 --params-host 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print({k:d[k] for k in ('ms_per_step_hbm','ms_per_step_offload','hidden_fraction','host_bytes_per_step','transfer_ms_at_duplex_peak','param_reuse_cache_blocks')})"; done
