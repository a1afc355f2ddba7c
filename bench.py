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
    p.add_argument("--filter", type=int, default=2, choices=[0, 1, 2],
                   help="0 FP64 scan, 1 FP32 certified prefilter, 2 tcgen05 certified bound")
    p.add_argument("--mma-tiles", type=int, default=0, choices=[0, 1, 2],
                   help="filter 2: 128-query accumulator tiles per tcgen05 CTA (0 = library default, 1)")
    p.add_argument("--batch-size", type=int, default=0,
                   help="result batch size b_s in pairs (0 = sized against free HBM, R15; the paper used 1e8)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-stats", action="store_true",
                   help="skip the FP64 work-counter pass (roofline = null); for large sweep workloads")
    p.add_argument("--cpu-sample", type=int, default=None,
                   help="oracle query sample for cpu_baseline / each reference-arm step (default 96: about "
                        "14 s of CPU work on expo32, spread over all host cores)")
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


_POOL_D = None


def _oracle_chunk(args):
    """Worker: the oracle (oracle/brute.neighbors_of, unchanged) on a chunk of
    query ids against the full dataset inherited from the parent (fork)."""
    from oracle import brute
    eps, q = args
    t = time.perf_counter()
    res = brute.neighbors_of(_POOL_D, eps, q)
    return sum(len(s) + len(a) for s, a in res), time.perf_counter() - t


def cpu_baseline(D, eps, m, seed):
    """The oracle as it stands (oracle/brute.neighbors_of), timed on a bounded
    sample of m query points against the full dataset on ALL host cores: the
    queries are split over one forked worker per core (numpy single-threaded
    in each), wall-clock timed around the whole pool."""
    import multiprocessing as mp
    global _POOL_D
    q = synth.query_sample(D.shape[0], m, seed=seed + 1)
    cores = max(1, min(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count(), len(q)))
    chunks = [q[i::cores] for i in range(cores)]
    _POOL_D = D
    env_threads = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env_threads:
        os.environ[k] = "1"
    try:
        ctx = mp.get_context("fork")
        t = time.perf_counter()
        with ctx.Pool(cores) as pool:
            res = pool.map(_oracle_chunk, [(eps, c) for c in chunks])
        dt = time.perf_counter() - t
    finally:
        _POOL_D = None
        for k, v in env_threads.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    pairs = sum(r[0] for r in res)
    return {"value": pairs / dt, "unit": "pairs/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(q)} query points x all {D.shape[0]} points (brute force, numpy einsum; "
                      f"queries split over {cores} forked workers, one per core)",
            "seconds": dt, "cpu_seconds": float(sum(r[1] for r in res)), "pairs": pairs}


def traffic_record(workload, filt):
    """The newest profiles/*_join_traffic_<workload>.json (tools/ncu_join_traffic.py)
    for the kernel of this filter, or None."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_join_traffic_{workload}.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        if d.get("filter", 2) == filt:
            d["source"] = os.path.relpath(f, ROOT)
            best = d
    return best


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(args)
    D = synth.make(w["gen"], w["count"], w["dims"], seed=args.seed)
    times, pairs, cores = [], 0, 1
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(D, w["eps"], args.cpu_sample, args.seed + i)
        cores = cb["cores"]
        if i >= args.warmup:
            times.append(cb["seconds"])
            pairs += cb["pairs"]
    val = pairs / sum(times)
    line = {"impl": "reference", "metric": "self-join result pairs/s", "value": val, "unit": "pairs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * float(np.mean(times)), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, **{k: w[k] for k in ("count", "dims", "eps", "k")}},
            "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                             "sample": f"{args.cpu_sample} query points per step x all points, over {cores} cores"},
            "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.cpu_sample is None:
        args.cpu_sample = 96
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_1809_09930_b200 import Index, gpujoin
    from paper_1809_09930_b200.distributed import Comm, EntityPartitionedJoin

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
    comm = Comm(device=dev)
    assert (comm.rank, comm.world) == (rank, world)
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

    # ---- capacity: exact count of this rank's share (outside any timed region)
    comm.broadcast(D_dev)
    ix0 = Index(D_dev, w["eps"], w["k"], stream=stream.cuda_stream, **flags)
    info = ix0.info()
    exact = ix0.estimate(1.0, rank, world)
    # work counters for the roofline: the tensor-core filters' unit is the
    # evaluated test (gj_join_counts, no distance work); the SHORTC scans need the
    # per-dimension counts of the FP64 stats scan (gj_join_stats)
    stats, mma_tests = None, None
    if not (args.profile or args.no_stats):
        stats = ix0.counts(rank, world) if info.filter == 2 else ix0.stats(rank, world)
        if info.filter == 2:
            mma_tests = ix0.mma_tests(rank, world) * (world if world > 1 else 1)
    info_k16 = info.mma_depth or None
    ix0.free()
    cap = int(exact * 1.02) + 65536
    out = torch.empty((cap, 2), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    job = EntityPartitionedJoin(comm, D_dev, w["eps"], w["k"], out, cnt, args.batch_size, stream, **flags)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    # L2 hygiene: the point array (N*n*8 bytes) and the index are re-built every
    # step; an extra 256 MB flush buffer is written between timed steps.
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    for _ in range(args.warmup):
        ix, nb, _ = job.step(ev[2:4])
        torch.cuda.synchronize()
        ix.free()
    launches0 = gpujoin.launch_count()
    clocks = Clocks(local).start() if not args.profile else None
    step_ms, join_ms, phase_ms, pairs = [], [], [], 0
    for _ in range(args.steps):
        flush.fill_(1)
        comm.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        ix, nb, _ = job.step(ev[2:4], ev[4:7])
        ev[1].record(stream)
        torch.cuda.synchronize()
        comm.barrier()
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
    # max over ranks of the device times; pairs summed over ranks
    t = torch.tensor([ms, jms], dtype=torch.float64, device=dev)
    comm.all_reduce(t, "max")
    ms, jms = float(t[0]), float(t[1])
    total_pairs = int(comm.all_reduce(torch.tensor([pairs], dtype=torch.int64, device=dev))[0])
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
            comm.barrier()
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
        e2e_t = float(comm.all_reduce(torch.tensor([e2e_t], dtype=torch.float64, device=dev), "max")[0])
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
        scale = world if world > 1 else 1
        if filt == 2:
            # certified tensor-core bound: one n-dim dot product (2n flops) per
            # evaluated (unordered) candidate pair, on fp16 operands
            alg = 2.0 * n * stats["tests_evaluated"]
            # sustained figure: the join kernels run inside a ~100-200 ms step under the power cap
            peak = peaks.get("bf16_tflops_sustained", 1400.0)
            bound = "tensor"
            kern = "k_join_umma (tcgen05/TMEM fp16 bound + FP64 decision)"
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
        # DRAM traffic per join and pipe utilisations: one ncu capture of every
        # join launch of a step of this workload (tools/ncu_join_traffic.py)
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        tj = traffic_record(args.workload, filt)
        traffic = tj.get("dram_bytes_per_join") if tj else None
        roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kern, "peak_note": pnote,
                "alg": {"tests_evaluated": stats["tests_evaluated"], "dims_evaluated": stats.get("dims_evaluated"),
                        "paper_tests": stats["tests"], "paper_dims": stats.get("dims"), "cells": stats["cells"],
                        "alg_tflop_per_join": alg * scale / 1e12},
                "join_ms": jms, "join_share_of_step": jms / ms,
                "filter_margin": info.filter_margin,
                # HBM view (the north_star's metric): measured DRAM bytes of one join over the
                # bench's join time, against the measured copy bandwidth
                "hbm": {"traffic_bytes_per_join": traffic,
                        "achieved_gbs": traffic / (jms / 1000.0) / 1e9 if traffic else None,
                        "peak_gbs": hbm_peak,
                        "frac": traffic / (jms / 1000.0) / 1e9 / hbm_peak if traffic else None,
                        "peak_note": "measured copy bandwidth, MEASURED_PEAKS.json" if "hbm_gbs" in peaks
                                     else "fallback 6.65 TB/s (B200_PROFILING.md)",
                        "note": "the tcgen05 bound makes the join tensor/TMEM-bound; HBM is not its roofline"},
                "ncu": ({k: tj.get(k) for k in ("tensor_pipe_pct", "fp64_pipe_pct", "fp64_inst_pct", "alu_pipe_pct",
                                                "issue_pct", "l2_hit_pct", "dram_pct", "launches", "source")}
                        if tj else None)}
        if mma_tests is not None and mma_tests > 0:
            # executed accumulator entries (128 x 128 blocks incl. padding) per evaluated test,
            # and the executed MMA depth K over the useful n: executed / useful tensor work
            roof["mma_waste"] = {"mma_tests": mma_tests, "tests_evaluated": stats["tests_evaluated"],
                                 "block_ratio": mma_tests / max(1, stats["tests_evaluated"]),
                                 "k_executed": info_k16, "k_useful": n,
                                 "flop_ratio": mma_tests * 2.0 * info_k16 / max(1.0, alg)}
    line = {
        "metric": "self-join result pairs/s", "value": value, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": {2: "f16 MMA (f32 acc) bound + f64 decision",
                  1: "f32 bound + f64 decision", 0: "f64"}[filt],
        "data": "synthetic",
        "config": {"workload": args.workload, "generator": w["gen"], "count": N, "dims": n, "eps": w["eps"],
                   "k": w["k"], **flags,
                   # SHORTC exists in the SIMT scans only (filters 0/1); the tcgen05 bound
                   # evaluates all MMA dims, survivors get a full FP64 test
                   "shortc": bool(flags["shortc"] and filt in (0, 1)), "shortc_requested": flags["shortc"],
                   "filter": filt, "filter_requested": args.filter,
                   "batch_size": args.batch_size, "n_batches": nb,
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
