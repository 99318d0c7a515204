import torch, time
N = 256 << 20
h = torch.empty(N, dtype=torch.uint8).pin_memory(); h.fill_(1)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
def run(nstreams, reps=5):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    part = N // nstreams
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*part:(i+1)*part].copy_(h[i*part:(i+1)*part], non_blocking=True)
    torch.cuda.synchronize()
    return reps * N / (time.perf_counter() - t0) / 1e9
for k in (1, 2, 4): run(k, 1); print("streams", k, "H2D GB/s", round(run(k), 1))
ho = torch.empty(N, dtype=torch.uint8).pin_memory()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): ho.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("D2H GB/s", round(5 * N / (time.perf_counter() - t0) / 1e9, 1))
