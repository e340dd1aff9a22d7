import torch, time
N = 4 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
def run(nstreams, chunk=64 << 20):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    off = 0; i = 0
    while off < N:
        c = min(chunk, N - off)
        with torch.cuda.stream(ss[i % nstreams]):
            d[off:off+c].copy_(h[off:off+c], non_blocking=True)
        off += c; i += 1
    torch.cuda.synchronize()
    return N / (time.perf_counter() - t0) / 1e9
for ns in (1, 2, 4, 1, 2, 4):
    for ch in (16 << 20, 64 << 20, 256 << 20):
        print(ns, ch >> 20, round(run(ns, ch), 2))
