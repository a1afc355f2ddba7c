"""Phase breakdown of the tcgen05 join (experiment build: tools/ab_prep.sh prof 64):
python tools/experiments/umma_prof.py ab/prof -- per-block cycles of each role's phases."""
import ctypes, os, sys
pkg = os.path.abspath(sys.argv[1])
sys.path.insert(0, pkg)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
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
blocks = v[12]
wb = v[3]
print(f"join ms {s.elapsed_time(e):.1f} pairs {int(cnt.item())} blocks {blocks} warp-blocks {wb}")
print(f"  epilogue per warp-block: wait accf {v[0] / wb:.1f}  TMEM reads -> release {v[1] / wb:.1f}  "
      f"after release {v[2] / wb:.1f} cyc;  rare {v[5] / wb * 100:.2f} % of warp-blocks, {v[4] / max(1, v[5]):.0f} cyc each")
print(f"  MMA issuer per block: wait release {v[8] / blocks:.1f}  wait loads {v[9] / blocks:.1f}  "
      f"issue {v[10] / blocks:.1f}  commits {v[11] / blocks:.1f} cyc")
