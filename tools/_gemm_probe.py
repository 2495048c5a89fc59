import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
n=10000
K = torch.randn(n, n+16, dtype=torch.float64, device='cuda')[:, :n]
Ks = K.contiguous()
for k in (16, 24, 40):
    V = torch.randn(n, k, dtype=torch.float64, device='cuda')
    for name, A in (("strided", K), ("contig", Ks)):
        for _ in range(3): Y = A @ V
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): Y = A @ V
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)/10
        print(f"k={k} {name}: {ms*1e3:.1f} us  {8*n*n/ms/1e6:.0f} GB/s  {2*n*n*k/ms/1e9:.1f} TFLOP/s")
