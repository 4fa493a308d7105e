import torch, sys
sys.path.insert(0, '.')
from paper_2104_07857_b200 import kernels
torch.manual_seed(8192 + 2048)
for (T, din, dout) in [(8192, 2048, 6144), (2048, 2048, 6144), (8192, 256, 256)]:
    x = torch.randn(T, din, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(T, dout, device="cuda", dtype=torch.bfloat16)
    ref = dy.float().t() @ x.float()
    for odt in (torch.bfloat16, torch.float32):
        dW = torch.empty(dout, din, device="cuda", dtype=odt)
        kernels.gemm(dy.t(), x.t(), dW)
        err = (dW.float() - ref).abs()
        tol = ref.abs() * 2 ** -7 + 1e-3 * (T ** 0.5) * 2 ** -8
        bad = err > tol
        print(T, din, dout, odt, "max err", err.max().item(), "bad", bad.sum().item())
        if bad.any():
            idx = bad.nonzero()
            print(" rows", idx[:, 0].unique()[:10].tolist(), "nrows", idx[:, 0].unique().numel(), "ncols", idx[:, 1].unique().numel())
            for r, c in idx[:5].tolist():
                print("  ", r, c, dW[r, c].item(), ref[r, c].item())
