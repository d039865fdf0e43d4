"""PCIe copy throughput on the box: 268 MB H2D / D2H from pinned memory, one stream vs split over 2 and 4 streams,
and both directions at once (what sffn_forward_host overlaps)."""
import torch, time
n = 268 * 1024 * 1024
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda"); d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
def run(k_h2d, k_d2h, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i in range(k_h2d):
            with torch.cuda.stream(streams[i]):
                a, b = i * n // k_h2d, (i + 1) * n // k_h2d
                d_in[a:b].copy_(h_in[a:b], non_blocking=True)
        for i in range(k_d2h):
            with torch.cuda.stream(streams[4 + i]):
                a, b = i * n // k_d2h, (i + 1) * n // k_d2h
                h_out[a:b].copy_(d_out[a:b], non_blocking=True)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2] * 1e3
for kh, kd in [(1, 0), (2, 0), (4, 0), (0, 1), (0, 2), (1, 1), (2, 2), (4, 4)]:
    ms = run(kh, kd)
    print(f"H2D streams {kh} D2H streams {kd}: {ms:6.2f} ms  ({(n * ((kh > 0) + (kd > 0))) / ms / 1e6:6.1f} GB/s total)")
