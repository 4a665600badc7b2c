"""Dev probe (run under gpurun): H2D rate of the e2e input pattern (4 grids per chunk, 3 streams) without the kernels."""
import torch, time
N = 512; B = 4096; chunk = 127
hs = [torch.empty((B, N, N), dtype=torch.float32, pin_memory=True) for _ in range(4)]
for h in hs: h.fill_(1.0)
for lanes in (1, 3):
    streams = [torch.cuda.Stream() for _ in range(lanes)]
    dst = [torch.empty((4, chunk, N, N), dtype=torch.float32, device="cuda") for _ in range(lanes)]
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        li = 0
        for off in range(0, B, chunk):
            cnt = min(chunk, B - off)
            s = streams[li]
            with torch.cuda.stream(s):
                for k in range(4):
                    dst[li][k, :cnt].copy_(hs[k][off:off + cnt], non_blocking=True)
            li = (li + 1) % lanes
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print("lanes", lanes, "GB/s", round(4 * B * N * N * 4 / dt / 1e9, 1))
big = torch.empty_like(hs[0], device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); big.copy_(hs[0], non_blocking=True); torch.cuda.synchronize()
print("one 4 GiB copy GB/s", round(B * N * N * 4 / (time.perf_counter() - t0) / 1e9, 1))
