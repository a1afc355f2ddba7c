"""Per-kernel device time of the index build (torch.profiler / CUPTI, warm,
not serialised): python tools/build_profile.py [workload] -> one line per kernel,
mean ms per build over 5 builds, plus the library's own build_ms."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import synth
from paper_1809_09930_b200 import Index

w = dict(synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "expo32"])
D = torch.from_numpy(synth.make(w["gen"], w["count"], w["dims"], seed=0)).cuda()
for _ in range(3):
    Index(D, w["eps"], w["k"]).free()
torch.cuda.synchronize()
R = 5
ms = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(R):
        ix = Index(D, w["eps"], w["k"])
        ms.append(ix.info().build_ms)
        ix.free()
    torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name] += e.device_time_total / 1000.0 if hasattr(e, "device_time_total") else e.cuda_time_total / 1000.0
        cnt[e.name] += 1
s = sum(tot.values()) / R
print(f"kernels+copies {s:.3f} ms per build; library build_ms {sum(ms) / R:.3f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{v / R:8.3f} ms  {cnt[k] / R:5.1f}x  {k[:110]}")
