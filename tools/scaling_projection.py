"""Per-rank device time of one bench step for world = 1, 2, 4, 8, every rank's
share run one after another on ONE GPU (index build, estimator, join of the
rank's tiles), to project entity-partitioned scaling before 8 GPUs are
available: python tools/scaling_projection.py [--workload expo32]
Each rank's phase times are the MEDIAN of --reps runs; the projected step is
max over ranks of (build + estimate + join) plus, for world > 1, the two
collectives of the step modelled from the measured NVLink figures of
B200_PROFILING.md: the NCCL broadcast of D (|D| n 8 bytes at the 8-rank
725 GB/s bus bandwidth) and the 8-byte count all-reduce (~0.03 ms)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1809_09930_b200 import Index, num_batches  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="expo32")
p.add_argument("--reps", type=int, default=5)
p.add_argument("--bus-gbs", type=float, default=725.0, help="NVLink bus bandwidth for the broadcast model")
p.add_argument("--worlds", default="1,2,4,8")
a = p.parse_args()
w = synth.WORKLOADS[a.workload]
D = torch.from_numpy(synth.make(w["gen"], w["count"], w["dims"], seed=0)).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
batch_streams = [torch.cuda.Stream() for _ in range(3)]   # as bench.py: three batch streams
res = {}
for world in [int(x) for x in a.worlds.split(",")]:
    per_rank = []
    for rank in range(world):
        runs = []
        for _ in range(a.reps):
            ev[0].record()
            ix = Index(D, w["eps"], w["k"])
            ev[1].record()
            est = ix.estimate(0.01, rank, world)
            ev[2].record()
            nb = num_batches(est, 0)
            cap = est * 2 + (1 << 20)
            out = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            start = torch.cuda.Event()
            start.record()
            for bs in batch_streams:
                bs.wait_event(start)
            for b in range(nb):
                ix.self_join_async(out, cnt, b, nb, rank, world, stream=batch_streams[b % 3].cuda_stream)
            for bs in batch_streams:
                done = torch.cuda.Event()
                done.record(bs)
                torch.cuda.current_stream().wait_event(done)
            ev[3].record()
            torch.cuda.synchronize()
            t = [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
            ix.free()
            del out
            runs.append(t)
        runs.sort(key=sum)
        per_rank.append(runs[len(runs) // 2])   # median step
    coll = 0.0 if world == 1 else w["count"] * w["dims"] * 8 / (a.bus_gbs * 1e9) * 1e3 + 0.03
    step = max(sum(t) for t in per_rank) + coll
    res[world] = {"step_ms": step, "collectives_ms": coll, "per_rank_ms": per_rank}
    eff = res[1]["step_ms"] / (world * step)
    res[world]["efficiency"] = eff
    print(f"world {world}: max-over-ranks step {step:.1f} ms (build {per_rank[0][0]:.1f}, estimate {per_rank[0][1]:.1f}, "
          f"join {max(t[2] for t in per_rank):.1f} max / {min(t[2] for t in per_rank):.1f} min, collectives "
          f"{coll:.2f}) -> efficiency {eff:.2f}", flush=True)
print(json.dumps({"workload": a.workload, "projection": res}))
