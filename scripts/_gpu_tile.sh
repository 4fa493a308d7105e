make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_tiling_gpu.py tests/test_fullsize_gpu.py tests/test_harness_gpu.py tests/test_spec_dist_gpu.py -m gpu -q -p no:cacheprovider -x -k "tiling or tiled or config4 or tile or spec or ac9" 2>&1 | tail -2
timeout 600 python -c "
import sys, json; sys.argv=['bench.py']
import bench
print(json.dumps(bench.tiling_leg()))
"
cat > /tmp/tile1.py <<'P'
import torch, sys
sys.path.insert(0, ".")
from paper_2104_07857_b200 import kernels
x = torch.randn(8192, 16384, device="cuda").bfloat16()
W = (torch.randn(8192, 16384, device="cuda") * 16384 ** -0.5).bfloat16()
b = torch.randn(8192, device="cuda").bfloat16()
y = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    kernels.linear_fwd(x, W, b, y)
torch.cuda.synchronize()
P
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"gemm" -s 1 -c 2 python /tmp/tile1.py 2>/dev/null | grep -E "gemm|dram__bytes|duration|tensor" | head -20
