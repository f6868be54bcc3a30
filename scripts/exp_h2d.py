import torch, time
n = 730 * 1024 * 1024 // 2
hs = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
ds = [torch.empty(n, dtype=torch.bfloat16, device='cuda') for _ in range(4)]
streams = [torch.cuda.Stream() for _ in range(4)]
def run(k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(4):
        s = streams[i % k]
        with torch.cuda.stream(s):
            ds[i].copy_(hs[i], non_blocking=True)
    torch.cuda.synchronize()
    return 4 * n * 2 / (time.perf_counter() - t0) / 1e9
for k in (1, 2, 4, 1, 2, 4):
    print(k, "streams", round(run(k), 1), "GB/s")
# bidirectional
ho = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(streams[0]):
    for i in range(4): ds[i].copy_(hs[i], non_blocking=True)
with torch.cuda.stream(streams[1]):
    for i in range(2): ho[i].copy_(ds[i], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("H2D 4x + D2H 2x concurrently:", round(6 * n * 2 / dt / 1e9, 1), "GB/s aggregate", round(dt * 1e3, 1), "ms")
