"""Phase breakdown of the tcgen05 join (experiment build with -DGJ_UMMA_EXPERIMENT=64):
python tools/umma_prof.py <package dir> -- prints per-block cycles of each role's phases."""
import ctypes, os, sys
pkg = os.path.abspath(sys.argv[1])
sys.path.insert(0, pkg)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1809_09930_b200 import Index, gpujoin
w = dict(synth.WORKLOADS[os.environ.get("AB_WORKLOAD", "expo32")])
D = torch.from_numpy(synth.make(w["gen"], w["count"], w["dims"], seed=0)).cuda()
L = gpujoin.lib()
buf = (ctypes.c_ulonglong * 16)()
ix = Index(D, w["eps"], w["k"])
out = torch.empty((ix.estimate(1.0) + 1024, 2), dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
L.gj_debug_umma_prof(buf)   # reset (estimator launches)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for b in range(3):
    ix.self_join_async(out, cnt, b, 3)
e.record()
torch.cuda.synchronize()
L.gj_debug_umma_prof(buf)
v = list(buf)
blocks = v[10]
warp_blocks = blocks * 8
print(f"join ms {s.elapsed_time(e):.1f} pairs {int(cnt.item())} blocks {blocks}")
names = ["wait accf", "ld+release", "fast path", "rare path (incl decide)", "decide"]
for k, nm in enumerate(names):
    print(f"  epilogue {nm:28s}: {v[k] / warp_blocks:8.1f} cyc per warp-block")
print(f"  rare warp-blocks: {v[5] / warp_blocks * 100:.2f} %   decides: {v[6]}  ({v[4] / max(1, v[6]):.0f} cyc each)")
print(f"  MMA wait acce {v[8] / blocks:.1f}  wait full {v[9] / blocks:.1f}  mma issue {v[12] / blocks:.1f}  "
      f"commits {v[13] / blocks:.1f}  total/block {v[11] / blocks:.1f} cyc")
