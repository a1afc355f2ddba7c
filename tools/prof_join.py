"""Run one index build + join of a workload (for ncu / nsight captures):
python tools/prof_join.py --workload expo32 --count 300000 [--reps 2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1809_09930_b200 import Index  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="expo32")
p.add_argument("--count", type=int, default=None)
p.add_argument("--eps", type=float, default=None)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--filter", type=int, default=2)
p.add_argument("--mma-tiles", type=int, default=0)
p.add_argument("--batches", type=int, default=1, help="result batches (bench: 3); batch b = every n_b-th tile")
a = p.parse_args()
w = dict(synth.WORKLOADS[a.workload])
if a.count:
    w["count"] = a.count
if a.eps:
    w["eps"] = a.eps
D = torch.from_numpy(synth.make(w["gen"], w["count"], w["dims"], seed=0)).cuda()
for r in range(a.reps):
    ix = Index(D, w["eps"], w["k"], filter=a.filter, mma_tiles=a.mma_tiles)
    est = ix.estimate(1.0)
    out = torch.empty((est + 1024, 2), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for b in range(a.batches):
        ix.self_join_async(out, cnt, b, a.batches)
    e.record()
    torch.cuda.synchronize()
    print(f"rep {r}: filter={ix.info().filter} tile_q={ix.info().tile_queries} pairs={int(cnt.item())} join_ms={s.elapsed_time(e):.2f} "
          f"build_ms={ix.info().build_ms:.2f} margin={ix.info().filter_margin:.3g}",
          flush=True)
    ix.free()
