"""Phase breakdown of the persistent tcgen05 join (experiment build with
-DGJ_WS_PROF=1: GJ_NVCC_EXTRA="-DGJ_WS_PROF=1" tools/ab_prep.sh wsprof):
python tools/experiments/ws_prof.py ab/wsprof -- cycles per role and phase."""
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
buf = (ctypes.c_ulonglong * 32)()
ix = Index(D, w["eps"], w["k"])
out = torch.empty((ix.estimate(1.0) + 1024, 2), dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
L.gj_debug_ws_prof(buf)   # reset (estimator launches)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for b in range(3):
    ix.self_join_async(out, cnt, b, 3)
e.record()
torch.cuda.synchronize()
L.gj_debug_ws_prof(buf)
v = [float(x) for x in buf]
ctas = max(v[27], 1)
blocks = max(v[4], 1)
wb = max(v[18], 1)
print(f"join ms {s.elapsed_time(e):.1f} pairs {int(cnt.item())} CTAs {int(ctas)} cycles/CTA {v[26] / ctas:.3g} "
      f"blocks {int(blocks)} fills {int(v[5])} windows {int(v[11])}")
print(f"  MMA per block: wait itf {v[0] / blocks:.1f} wait acce {v[1] / blocks:.1f} wait full {v[2] / blocks:.1f} "
      f"issue+commit {v[3] / blocks:.1f}")
print(f"  producer per block: wait empty {v[6] / blocks:.1f} wait itf {v[7] / blocks:.1f}")
print(f"  setup per CTA: wait ite {v[8] / ctas:.3g} busy {v[9] / ctas:.3g} fills {v[10] / ctas:.1f} "
      f"(busy per fill {v[9] / max(v[10], 1):.0f})")
print(f"  epilogue per warp-block: wait itf {v[12] / wb:.1f} wait accf {v[13] / wb:.1f} ld->release {v[14] / wb:.1f} "
      f"sign+rest {v[15] / wb:.1f} push {v[16] / wb:.1f}; chunks pushed {int(v[19])} ({v[19] / wb * 100:.2f} per 100 warp-blocks)")
ent = max(v[24], 1)
print(f"  decider per CTA: idle {v[20] / ctas:.3g} read pairs {v[21] / ctas:.3g} FP64 {v[23] / ctas:.3g}; "
      f"pairs {int(v[24])} passes {int(v[25])} ({v[24] / max(v[25], 1):.1f} pairs per pass, "
      f"{v[23] / max(v[25], 1):.0f} cyc FP64 per pass)")
