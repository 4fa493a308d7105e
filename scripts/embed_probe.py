import torch, sys
sys.path.insert(0, ".")
from paper_2104_07857_b200 import kernels
T, V, hd = 8192, 50304, 2048
tok = torch.randint(0, V, (T,), device="cuda")
dx = torch.randn(T, hd, device="cuda").bfloat16()
acc = torch.randn(V, hd, device="cuda")
work = torch.empty(2 * V + 1 + T, dtype=torch.int32, device="cuda")
out = torch.empty(V, hd, dtype=torch.bfloat16, device="cuda")
for _ in range(3): kernels.embed_grad(tok, dx, acc, out, work)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): kernels.embed_grad(tok, dx, acc, out, work)
b.record(); torch.cuda.synchronize()
print("embed_grad us", a.elapsed_time(b) / 20 * 1e3)
