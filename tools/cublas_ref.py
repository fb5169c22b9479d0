"""Library baseline (context only): cuBLAS DGEMM (torch.matmul, float64) on the FD mode-product shapes."""
import torch

for n in (131, 256, 512):
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    X = torch.randn(n, n * n, dtype=torch.float64, device="cuda")  # mode-3 product: (n x n) @ (n x n^2)
    Y = torch.empty_like(X)
    for _ in range(3):
        torch.matmul(A, X, out=Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(A, X, out=Y)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cuBLAS DGEMM {n}x{n}x{n * n}: {ms:.4f} ms, {2 * n ** 4 / ms / 1e9:.2f} TFLOP/s", flush=True)
    Xt = X.t().contiguous()  # mode-1 style: (n^2 x n) @ (n x n)^T
    for _ in range(3):
        torch.matmul(Xt, A.t(), out=Y.view(n * n, n))
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        torch.matmul(Xt, A.t(), out=Y.view(n * n, n))
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cuBLAS DGEMM {n * n}x{n}x{n} (NT): {ms:.4f} ms, {2 * n ** 4 / ms / 1e9:.2f} TFLOP/s", flush=True)
