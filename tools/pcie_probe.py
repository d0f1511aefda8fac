import torch, time
n = 671088640
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device='cuda')
h2 = torch.empty(503316480, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(503316480, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); a=(time.perf_counter()-t)/5
t=time.perf_counter()
for _ in range(5): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); b=(time.perf_counter()-t)/5
t=time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c=(time.perf_counter()-t)/5
print(f"H2D {n/a/1e9:.1f} GB/s ({a*1e3:.1f} ms)  D2H {503316480/b/1e9:.1f} GB/s ({b*1e3:.1f} ms)  both {c*1e3:.1f} ms")
