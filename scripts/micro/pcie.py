import torch, time
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(name, f"{n/dt/1e9:.1f} GB/s")
# chunked D2H on 3 streams
sts = [torch.cuda.Stream() for _ in range(3)]
torch.cuda.synchronize(); t0 = time.perf_counter()
for it in range(5):
    for k in range(8):
        with torch.cuda.stream(sts[k % 3]):
            a = k * (n // 8)
            h[a:a + n // 8].copy_(d[a:a + n // 8], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print("D2H 8 parts / 3 streams", f"{n/dt/1e9:.1f} GB/s")
