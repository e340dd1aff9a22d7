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

# bidirectional: H2D and D2H of 2 GB each on two streams at once (the TSM2L host pipeline's case)
M = 2 << 30
hA = torch.empty(M, dtype=torch.uint8, pin_memory=True)
hC = torch.empty(M, dtype=torch.uint8, pin_memory=True)
dA = torch.empty(M, dtype=torch.uint8, device="cuda")
dC = torch.empty(M, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        dA.copy_(hA, non_blocking=True)
    with torch.cuda.stream(s2):
        hC.copy_(dC, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print("bidirectional 2+2 GB:", round(t * 1e3, 1), "ms,", round(2 * M / t / 1e9, 1), "GB/s total")
t0 = time.perf_counter(); hC.copy_(dC); torch.cuda.synchronize(); t = time.perf_counter() - t0
print("D2H alone:", round(M / t / 1e9, 1), "GB/s")
