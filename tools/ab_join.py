"""A/B timing of builds of the package (copies under ab/<v>/ from tools/ab_prep.sh):
python tools/ab_join.py ab/A [reps]  -- AB_BATCHES (3) result batches of the expo32 join, CUDA events"""
import os, sys
pkg = os.path.abspath(sys.argv[1])
sys.path.insert(0, pkg)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1809_09930_b200 import Index
w = dict(synth.WORKLOADS[os.environ.get("AB_WORKLOAD", "expo32")])
if os.environ.get("AB_COUNT"):
    w["count"] = int(os.environ["AB_COUNT"])
D = torch.from_numpy(synth.make(w["gen"], w["count"], w["dims"], seed=0)).cuda()
import paper_1809_09930_b200 as P
assert P.__file__.startswith(pkg), P.__file__
ts = []
for r in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    ix = Index(D, w["eps"], w["k"])
    est = ix.estimate(1.0)
    out = torch.empty((est + 1024, 2), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    nb = int(os.environ.get("AB_BATCHES", "3"))   # result batches (all on the current stream)
    for b in range(nb):
        ix.self_join_async(out, cnt, b, nb)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
    ix.free()
print(os.path.basename(os.path.dirname(pkg + "/")), "pairs", int(cnt.item()), "join ms", " ".join("%.1f" % t for t in ts))
