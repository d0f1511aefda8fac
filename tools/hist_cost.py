import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2112_05570_b200.engine import DeviceMesh, new_histogram
d = "fixtures/data/lines1024"
m = DeviceMesh.from_files(f"{d}/scene.txt", f"{d}/mwt.tri")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
h = new_histogram()
def t(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
n = 1 << 24
for _ in range(2):
    print("hist+out %.4f  out only %.4f  hist only %.4f  neither %.4f" % (
        t(lambda: m.trace_generated_device(0, (0, 0, 1, 1), 0, 0, n, True, h)),
        t(lambda: m.trace_generated_device(0, (0, 0, 1, 1), 0, 0, n, True, None)),
        t(lambda: m.trace_generated_device(0, (0, 0, 1, 1), 0, 0, n, False, h)),
        t(lambda: m.trace_generated_device(0, (0, 0, 1, 1), 0, 0, n, False, None))), flush=True)
