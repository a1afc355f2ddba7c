#!/usr/bin/env python
"""Benchmark of the B200 epsilon self-join (arxiv 1809.09930 GPU-Join).

One "step" = the whole hot path over one synthetic dataset: [N>1: NCCL
broadcast of D from rank 0] -> constructIndex (REORDER, grid over k dims,
device radix sort, adjacent-cell CSR, tiles) -> result-size estimator ->
n_b = max(3, ceil(est/b_s)) selfJoinKernel batches into an HBM result
buffer -> [N>1: all-reduce of the pair count].  Entity partitioning (§6.2):
rank r joins the query tiles at positions j = r mod N of the heaviest-first
tile order against the full replicated dataset.

value = result pairs (all ranks) / max-over-ranks device time of a step.
e2e   = the same through the C ABI with HOST buffers: pinned points H2D,
        build, Fig. 4 pipeline with batched D2H of all pairs into pinned host
        memory.

Usage: python bench.py [--gpus N --steps K --warmup W --workload expo32
                        --impl {gpu,reference}]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP64 FMA lanes per SM on B200 (GB100 SM: 64 FP64 units) -> derived FP64 peak
FP64_LANES_PER_SM = 64
N_SMS = 148


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    p.add_argument("--workload", default="expo32", choices=sorted(synth.WORKLOADS))
    p.add_argument("--eps", type=float, default=None)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--count", type=int, default=None)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-reorder", action="store_true")
    p.add_argument("--no-sortidu", action="store_true")
    p.add_argument("--no-shortc", action="store_true")
    p.add_argument("--no-symmetric", action="store_true")
    p.add_argument("--filter", type=int, default=2, choices=[0, 1, 2, 3],
                   help="0 FP64 scan, 1 FP32 certified prefilter, 2 tcgen05 certified bound, 3 mma.sync bound")
    p.add_argument("--mma-tiles", type=int, default=0, choices=[0, 1, 2],
                   help="filter 2: 128-query accumulator tiles per tcgen05 CTA (0 = library default, 1)")
    p.add_argument("--batch-size", type=int, default=0,
                   help="result batch size b_s in pairs (0 = sized against free HBM, R15; the paper used 1e8)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-stats", action="store_true",
                   help="skip the FP64 work-counter pass (roofline = null); for large sweep workloads")
    p.add_argument("--cpu-sample", type=int, default=96,
                   help="oracle query sample for cpu_baseline (~13 s on expo32; the reference arm uses a quarter per step)")
    p.add_argument("--profile", action="store_true", help="short run for ncu: no e2e/cpu baseline/clocks")
    p.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo lets several ranks share one GPU "
                   "to exercise the multi-rank path on a 1-GPU box")
    return p.parse_args()


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        s = [x for x in self.samples if len(x) >= 9 and x[1].replace(".", "").isdigit()]
        if not s:
            return None
        sm = [float(x[1]) for x in s]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for x in s:
            for nm, v in zip(names, x[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(s[0][2]), "samples": len(s),
                "reasons": sorted(reasons)}


def workload(args):
    w = dict(synth.WORKLOADS[args.workload])
    if args.eps is not None:
        w["eps"] = args.eps
    if args.k is not None:
        w["k"] = args.k
    if args.count is not None:
        w["count"] = args.count
    return w


def cpu_baseline(D, eps, m, seed):
    """The oracle as it stands (oracle/brute.neighbors_of), timed on a bounded
    sample of m query points against the full dataset on the host."""
    from oracle import brute
    q = synth.query_sample(D.shape[0], m, seed=seed + 1)
    t = time.perf_counter()
    res = brute.neighbors_of(D, eps, q)
    dt = time.perf_counter() - t
    pairs = sum(len(s) + len(a) for s, a in res)
    return {"value": pairs / dt, "unit": "pairs/s", "cores": 1, "kind": "oracle",
            "sample": f"{len(q)} query points x all {D.shape[0]} points (brute force, numpy einsum, 1 thread)",
            "seconds": dt, "pairs": pairs}


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(args)
    D = synth.make(w["gen"], w["count"], w["dims"], seed=args.seed)
    times, pairs = [], 0
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(D, w["eps"], max(1, args.cpu_sample // 4), args.seed + i)
        if i >= args.warmup:
            times.append(cb["seconds"])
            pairs += cb["pairs"]
    val = pairs / sum(times)
    line = {"impl": "reference", "metric": "self-join result pairs/s", "value": val, "unit": "pairs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * float(np.mean(times)), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, **{k: w[k] for k in ("count", "dims", "eps", "k")}},
            "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": 1, "kind": "oracle",
                             "sample": f"{max(1, args.cpu_sample // 4)} query points per step x all points"},
            "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_1809_09930_b200 import Index, gpujoin, num_batches

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    w = workload(args)
    flags = dict(reorder=not args.no_reorder, sortidu=not args.no_sortidu, shortc=not args.no_shortc,
                 symmetric=not args.no_symmetric, filter=args.filter, mma_tiles=args.mma_tiles)

    # ---- data: generated on rank 0's host; other ranks receive it over NCCL
    N, n = w["count"], w["dims"]
    if rank == 0:
        D_host = synth.make(w["gen"], N, n, seed=args.seed)
    else:
        D_host = None
    D_dev = torch.empty((N, n), dtype=torch.float64, device=dev)
    if rank == 0:
        D_dev.copy_(torch.from_numpy(D_host))

    def bcast(t):
        """NCCL broadcast over NVLink; with --dist-backend gloo staged through host memory."""
        if args.dist_backend == "nccl":
            dist.broadcast(t, src=0)
        else:
            h = t.cpu()
            dist.broadcast(h, src=0)
            t.copy_(h)

    def allreduce(t, op=None):
        op = op or dist.ReduceOp.SUM
        if args.dist_backend == "nccl":
            dist.all_reduce(t, op=op)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)

    def barrier():
        if world > 1:
            if args.dist_backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    batch_streams = [torch.cuda.Stream() for _ in range(3)]
    batch_done = [torch.cuda.Event() for _ in range(3)]

    def one_step(out, cnt, ev_join, ev_phase=None):
        """The timed hot path; returns (index, n_b).  ev_join brackets the join
        kernels; ev_phase (optional) = [after broadcast, after build, after estimate]."""
        if world > 1:
            bcast(D_dev)
        if ev_phase:
            ev_phase[0].record(stream)
        ix = Index(D_dev, w["eps"], w["k"], stream=stream.cuda_stream, **flags)
        if ev_phase:
            ev_phase[1].record(stream)
        est = ix.estimate(0.01, rank, world)
        if ev_phase:
            ev_phase[2].record(stream)
        nb = num_batches(est, args.batch_size)
        cnt.zero_()
        ev_join[0].record(stream)
        # Fig. 4: batches on three streams, so one batch's tail overlaps the next
        for i, bs in enumerate(batch_streams):
            bs.wait_event(ev_join[0])
        for b in range(nb):
            ix.self_join_async(out, cnt, b, nb, rank, world, stream=batch_streams[b % 3].cuda_stream)
        for bs, be in zip(batch_streams, batch_done):
            be.record(bs)
            stream.wait_event(be)
        ev_join[1].record(stream)
        if world > 1:
            tot = cnt.clone()
            allreduce(tot)
        return ix, nb

    # ---- capacity: exact count of this rank's share (outside any timed region)
    if world > 1:
        bcast(D_dev)
    ix0 = Index(D_dev, w["eps"], w["k"], stream=stream.cuda_stream, **flags)
    info = ix0.info()
    exact = ix0.estimate(1.0, rank, world)
    # work counters for the roofline: the tensor-core filters' unit is the
    # evaluated test (gj_join_counts, no distance work); the SHORTC scans need the
    # per-dimension counts of the FP64 stats scan (gj_join_stats)
    stats = None
    if not (args.profile or args.no_stats):
        stats = ix0.counts(rank, world) if info.filter in (2, 3) else ix0.stats(rank, world)
    ix0.free()
    cap = int(exact * 1.02) + 65536
    out = torch.empty((cap, 2), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    # L2 hygiene: the point array (N*n*8 bytes) and the index are re-built every
    # step; an extra 256 MB flush buffer is written between timed steps.
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    for _ in range(args.warmup):
        ix, nb = one_step(out, cnt, ev[2:4])
        torch.cuda.synchronize()
        ix.free()
    launches0 = gpujoin.launch_count()
    clocks = Clocks(local).start() if not args.profile else None
    step_ms, join_ms, phase_ms, pairs = [], [], [], 0
    for _ in range(args.steps):
        flush.fill_(1)
        barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        ix, nb = one_step(out, cnt, ev[2:4], ev[4:7])
        ev[1].record(stream)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(ev[0].elapsed_time(ev[1]))
        join_ms.append(ev[2].elapsed_time(ev[3]))
        phase_ms.append([ev[0].elapsed_time(ev[4]), ev[4].elapsed_time(ev[5]), ev[5].elapsed_time(ev[6]),
                         ev[6].elapsed_time(ev[2])])
        got = int(cnt.item())
        if got > cap:
            raise RuntimeError(f"result buffer overflow {got} > {cap}")
        pairs = got
        ix.free()
    launches = (gpujoin.launch_count() - launches0) // max(1, args.steps)
    clk = clocks.stop() if clocks else None

    ms = float(np.mean(step_ms))
    jms = float(np.mean(join_ms))
    if world > 1:
        t = torch.tensor([ms, jms, float(pairs)], dtype=torch.float64, device=dev)
        tmax = t.clone()
        allreduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        allreduce(tsum)
        ms, jms, total_pairs = float(tmax[0]), float(tmax[1]), int(tsum[2])
    else:
        total_pairs = pairs
    value = total_pairs / (ms / 1000.0)

    # ---- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not args.profile:
        host_pts = torch.empty((N, n), dtype=torch.float64, pin_memory=True)
        if rank == 0:
            host_pts.numpy()[:] = D_host
        if world > 1:
            # non-zero ranks receive D over NCCL, then stage it to host like a user would
            D_dev2 = D_dev.clone()
            host_pts.copy_(D_dev2)
        host_out = torch.empty((cap, 2), dtype=torch.int32, pin_memory=True)
        e2e_s = []
        n_e2e_warm = max(3, args.warmup)   # first host builds grow the library's memory pool
        for i in range(n_e2e_warm + max(7, args.steps)):   # median of >= 7: robust to host-side outliers
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ixh = Index(host_pts.numpy(), w["eps"], w["k"], stream=stream.cuda_stream, **flags)
            t1 = time.perf_counter()
            m, nbh = ixh.self_join_host(host_out, rank, world, args.batch_size)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            ixh.free()
            if rank == 0:
                print(f"[bench] e2e step {i}: index from host {1e3 * (t1 - t0):.1f} ms, "
                      f"self_join_host {1e3 * (dt - (t1 - t0)):.1f} ms", file=sys.stderr, flush=True)
            if i >= n_e2e_warm:
                e2e_s.append(dt)
        e2e_t = float(np.median(e2e_s))   # host-side outliers (page faults, pool growth) are rare but large
        e2e_mean = float(np.mean(e2e_s))
        if world > 1:
            t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
            allreduce(t, op=dist.ReduceOp.MAX)
            e2e_t = float(t[0])
        e2e = {"value": total_pairs / e2e_t, "unit": "pairs/s", "seconds": e2e_t, "stat": "median",
               "mean_seconds": e2e_mean, "steps": len(e2e_s),
               "h2d_bytes_per_step": int(N * n * 8), "d2h_bytes_per_step": int(pairs * 8 + 8 * 3 * 8),
               "api": "gj_build_index(host ptr) + gj_self_join_host(pinned host buffer)", "n_batches": nbh}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the join)
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    clk_max = peaks.get("sm_max_mhz", 1965.0) * 1e6
    filt = info.filter
    roof = None
    if stats is not None:
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            tj = json.load(open(tfile)).get(args.workload, {})
            traffic = tj.get(f"filter{filt}")
        scale = world if world > 1 else 1
        if filt in (2, 3):
            # certified tensor-core bound: one n-dim dot product (2n flops) per
            # evaluated (unordered) candidate pair, on fp16 operands
            alg = 2.0 * n * stats["tests_evaluated"]
            # sustained figure: the join kernels run inside a ~200 ms step under the power cap
            peak = peaks.get("bf16_tflops_sustained", 1400.0)
            bound = "tensor"
            kern = ("k_join_umma (tcgen05/TMEM fp16 bound + FP64 decision)" if filt == 2
                    else "k_join_tc (mma.sync fp16 bound + FP64 decision)")
            pnote = ("measured cuBLAS bf16 sustained, MEASURED_PEAKS.json" if "bf16_tflops_sustained" in peaks
                     else "fallback (B200_PROFILING.md): bf16 sustained ~1.4 PFLOP/s under the power cap") + \
                    "; fp16 has the same nominal dense rate"
        else:
            # SHORTC scan: 3 flops per dimension evaluated (§4.4 "3n")
            alg = 3.0 * stats["dims_evaluated"]
            lanes = 128 if filt == 1 else FP64_LANES_PER_SM
            peak = lanes * 2 * N_SMS * clk_max / 1e12
            bound = "alu"
            kern = "k_join32 (FP32 SHORTC prefilter + FP64 decision)" if filt == 1 else "k_join (FP64 SHORTC)"
            pnote = f"derived {'FP32' if filt == 1 else 'FP64'}: {lanes} FMA lanes x 2 flop x {N_SMS} SMs x max clock"
        achieved = alg * scale / (jms / 1000.0) / 1e12
        roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kern, "peak_note": pnote,
                "alg": {"tests_evaluated": stats["tests_evaluated"], "dims_evaluated": stats.get("dims_evaluated"),
                        "paper_tests": stats["tests"], "paper_dims": stats.get("dims"), "cells": stats["cells"],
                        "alg_tflop_per_join": alg * scale / 1e12},
                "join_ms": jms, "join_share_of_step": jms / ms,
                "filter_margin": info.filter_margin}
    line = {
        "metric": "self-join result pairs/s", "value": value, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": {3: "f16 MMA (f32 acc) bound + f64 decision", 2: "f16 MMA (f32 acc) bound + f64 decision",
                  1: "f32 bound + f64 decision", 0: "f64"}[filt],
        "data": "synthetic",
        "config": {"workload": args.workload, "generator": w["gen"], "count": N, "dims": n, "eps": w["eps"],
                   "k": w["k"], **flags, "batch_size": args.batch_size, "n_batches": nb,
                   "parallelism": f"entity-partitioned dp{world}",
                   "l2": "point set (%.0f MB) + index rebuilt every step; 256 MB flush written between steps"
                         % (N * n * 8 / 1e6)},
        "join_time_s": ms / 1000.0, "pairs": total_pairs, "selectivity": (total_pairs - N) / N,
        "index": {"n_cells": info.n_cells, "n_adjacent": info.n_adjacent, "n_tiles": info.n_tiles,
                  "tile_queries": info.tile_queries,
                  "est_candidates": info.est_candidates},
        "phases_ms": dict(zip(["broadcast", "build_index", "estimate", "plan", "join"],
                              [float(np.mean([p[i] for p in phase_ms])) for i in range(4)] + [jms])),
        "gpu_launches": int(launches), "e2e": e2e, "roofline": roof, "clocks": clk,
    }
    if not args.no_cpu_baseline and not args.profile:
        line["cpu_baseline"] = cpu_baseline(D_host, w["eps"], args.cpu_sample, args.seed)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
