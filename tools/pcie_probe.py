import torch, time
N = 16777216
h_in = torch.randn(N, dtype=torch.float64).pin_memory()
h_out = torch.empty(N, dtype=torch.float64).pin_memory()
d_a = torch.empty(N, dtype=torch.float64, device='cuda'); d_b = torch.randn(N, dtype=torch.float64, device='cuda')
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
s = [torch.cuda.Stream() for _ in range(4)]
def h2d(k):
    def f():
        ch = N // k
        for i in range(k):
            with torch.cuda.stream(s[i]): d_a[i*ch:(i+1)*ch].copy_(h_in[i*ch:(i+1)*ch], non_blocking=True)
    return f
def d2h(k):
    def f():
        ch = N // k
        for i in range(k):
            with torch.cuda.stream(s[i]): h_out[i*ch:(i+1)*ch].copy_(d_b[i*ch:(i+1)*ch], non_blocking=True)
    return f
def both(k):
    def f():
        ch = N // k
        for i in range(k):
            with torch.cuda.stream(s[i]): d_a[i*ch:(i+1)*ch].copy_(h_in[i*ch:(i+1)*ch], non_blocking=True)
        for i in range(k):
            with torch.cuda.stream(s[(i+2)%4]): h_out[i*ch:(i+1)*ch].copy_(d_b[i*ch:(i+1)*ch], non_blocking=True)
    return f
for k in (1, 2, 4):
    a, b, c = t(h2d(k)), t(d2h(k)), t(both(k))
    print(f"chunks {k}: H2D {a:.2f} ms ({N*8/a/1e6:.1f} GB/s)  D2H {b:.2f} ms ({N*8/b/1e6:.1f} GB/s)  both {c:.2f} ms")
