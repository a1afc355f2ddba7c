"""Per-launch device time of the expo32 join dealt into AB_BATCHES result
batches on one stream (CUDA events around each launch):
python tools/launch_probe.py [n_batches ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1809_09930_b200 import Index

w = dict(synth.WORKLOADS[os.environ.get("AB_WORKLOAD", "expo32")])
D = torch.from_numpy(synth.make(w["gen"], w["count"], w["dims"], seed=0)).cuda()
ix = Index(D, w["eps"], w["k"])
out = torch.empty((ix.estimate(1.0) + 1024, 2), dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for nb in [int(x) for x in sys.argv[1:]] or [3, 24]:
    for rep in range(2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)]
        torch.cuda.synchronize()
        ev[0].record()
        host = []
        for b in range(nb):
            h0 = time.perf_counter()
            ix.self_join_async(out, cnt, b, nb)
            host.append(1e3 * (time.perf_counter() - h0))
            ev[b + 1].record()
        torch.cuda.synchronize()
        t = [ev[b].elapsed_time(ev[b + 1]) for b in range(nb)]
    print(f"nb {nb}: total {sum(t):.1f} ms; per launch " + " ".join(f"{x:.1f}" for x in t), flush=True)
    print(f"   host ms per call " + " ".join(f"{x:.2f}" for x in host), flush=True)
