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
# the same copy pattern while the matcher runs on resident inputs on other streams
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00459_b200 as fb
cfg, delta, _ = fb.baseline_config(4)
m = fb.Matcher(cfg, max_batch=512)
f = torch.rand((512, N, N), device="cuda"); g = torch.rand_like(f); mf = torch.rand_like(f); mg = torch.rand_like(f)
m.match_device(f, g, mf, mg, delta=delta); torch.cuda.synchronize()
cs = torch.cuda.Stream(); streams = [torch.cuda.Stream() for _ in range(3)]
dst = [torch.empty((4, chunk, N, N), dtype=torch.float32, device="cuda") for _ in range(3)]
with torch.cuda.stream(cs):
    for _ in range(100):  # ~330 ms of matcher work, about the copies' duration
        m.match_device(f, g, mf, mg, delta=delta, stream=cs.cuda_stream)
t0 = time.perf_counter(); li = 0
for off in range(0, B, chunk):
    cnt = min(chunk, B - off)
    with torch.cuda.stream(streams[li]):
        for k in range(4):
            dst[li][k, :cnt].copy_(hs[k][off:off + cnt], non_blocking=True)
    li = (li + 1) % 3
for s in streams: s.synchronize()
dt = time.perf_counter() - t0
print("lanes 3 with the matcher running GB/s", round(4 * B * N * N * 4 / dt / 1e9, 1), "compute still busy:", not cs.query())
cs.synchronize()
