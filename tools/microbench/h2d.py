import torch, time
n = 1744651260 // 4
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        chunk = (n + k - 1) // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"streams {k}: {n*4/dt/1e9:.1f} GB/s")
# chunked on one stream
s = torch.cuda.Stream()
for ch in (8<<20, 64<<20):
    torch.cuda.synchronize(); t=time.perf_counter()
    with torch.cuda.stream(s):
        for i in range(0, n, ch):
            d[i:i+ch].copy_(h[i:i+ch], non_blocking=True)
    torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"chunk {ch*4>>20} MB: {n*4/dt/1e9:.1f} GB/s")
