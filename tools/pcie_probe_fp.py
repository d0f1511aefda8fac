"""PCIe copy bound of the FloorPlan e2e step: 2^26 rays x 32 B host->device and
2^26 x 24 B device->host, each direction alone and both at once (pinned memory)."""
import torch, time
n_in, n_out = 2147483648, 1610612736
h = torch.empty(n_in, dtype=torch.uint8, pin_memory=True); d = torch.empty(n_in, dtype=torch.uint8, device='cuda')
h2 = torch.empty(n_out, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n_out, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); a=(time.perf_counter()-t)/3
t=time.perf_counter()
for _ in range(3): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); b=(time.perf_counter()-t)/3
t=time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c=(time.perf_counter()-t)/3
print(f"H2D {n_in/a/1e9:.1f} GB/s ({a*1e3:.1f} ms)  D2H {n_out/b/1e9:.1f} GB/s ({b*1e3:.1f} ms)  both {c*1e3:.1f} ms")
