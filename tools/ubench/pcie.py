import torch, time
n = 15_204_352  # one 512^2x58 field
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(6)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(6)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(streams, direction):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i in range(6):
        s = streams[i % len(streams)]
        with torch.cuda.stream(s):
            if direction == "h2d": d[i].copy_(h[i], non_blocking=True)
            else: h[i].copy_(d[i], non_blocking=True)
    torch.cuda.synchronize(); return 6 * n * 8 / (time.perf_counter() - t0) / 1e9
for direction in ("h2d", "d2h"):
    for streams in ([s1], [s1, s2]):
        r = [run(streams, direction) for _ in range(5)]
        print(direction, len(streams), "streams:", round(max(r), 1), "GB/s")
# both directions at once
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(6):
    with torch.cuda.stream(s1): d[i].copy_(h[i], non_blocking=True)
    with torch.cuda.stream(s2): h[(i+3)%6].copy_(d[(i+3)%6], non_blocking=True)
torch.cuda.synchronize(); print("duplex", round(12*n*8/(time.perf_counter()-t0)/1e9, 1), "GB/s total")
