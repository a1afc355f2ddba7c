import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import synth
from paper_1809_09930_b200 import Index
w = synth.WORKLOADS["expo32"]
D = synth.make(w["gen"], w["count"], w["dims"], seed=0)
host_pts = torch.empty(D.shape, dtype=torch.float64, pin_memory=True); host_pts.numpy()[:] = D
host_out = torch.empty((80_000_000, 2), dtype=torch.int32, pin_memory=True)
s = torch.cuda.Stream()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ix = Index(host_pts.numpy(), w["eps"], w["k"], stream=s.cuda_stream)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    m, nb = ix.self_join_host(host_out, 0, 1, 100_000_000)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ix.free()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"it {it}: index(host) {1e3*(t1-t0):.1f} ms, self_join_host {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms, pairs {m}", flush=True)
