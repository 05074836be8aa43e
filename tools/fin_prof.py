import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
n = 1 << 24
x = torch.rand(n, dtype=torch.float64, device="cuda")
for rep in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t1 = time.perf_counter()
    buf.copy_(x, non_blocking=True); torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    a = buf.numpy()
    print(rep, "alloc", round((t1 - t) * 1000, 2), "copy", round((t2 - t1) * 1000, 2))
    del a, buf
import numpy as np
for rep in range(2):
    t = time.perf_counter(); y = x.cpu(); t1 = time.perf_counter()
    print("pageable .cpu()", round((t1 - t) * 1000, 2))
