"""Per-join DRAM traffic and pipe utilisation from ONE ncu capture of every
join launch of one bench step (all result batches):

    ncu --set full --clock-control none -k regex:k_join -s <warm-up launches> -c <batches> \
        -o gpurun_out/join python bench.py --profile --steps 1 --warmup 1 ...
    python tools/ncu_join_traffic.py gpurun_out/join.ncu-rep expo32 [filter] > profiles/r2_join_traffic_expo32.json

Sums dram__bytes_{read,write} and the kernel durations over the launches and
time-weights the per-launch utilisations (tensor pipe, FP64 pipe, issue, L2
hit).  bench.py reads the JSON (profiles/<round>_join_traffic_<workload>.json)
for its roofline block: traffic = DRAM bytes per join, hbm_frac = traffic /
join time / measured HBM peak.  ncu replays are cold-cache and serialised, so
the durations here are not bench times; the bytes and utilisations are the
evidence."""
import csv
import io
import json
import subprocess
import sys

rep, workload = sys.argv[1], sys.argv[2]
filt = int(sys.argv[3]) if len(sys.argv) > 3 else 2
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, rows = r[0], r[1], r[2:]


def col(name):
    return h.index(name) if name in h else None


def num(row, name, scale_units=True):
    i = col(name)
    if i is None or not row[i]:
        return None
    try:
        v = float(row[i].replace(",", ""))
    except ValueError:
        return None
    if v != v:   # nan: metric not collected for this launch
        return None
    if scale_units:
        u = units[i].lower()
        v *= {"gbyte": 1e9, "mbyte": 1e6, "kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
              "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0, "second": 1.0}.get(u, 1.0)
    return v


UTIL = {
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_inst_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}
launches = []
for row in rows:
    name = row[col("Kernel Name")]
    d = num(row, "gpu__time_duration.sum")
    rd = num(row, "dram__bytes_read.sum")
    wr = num(row, "dram__bytes_write.sum")
    launches.append({"kernel": name[:80], "duration_s": d, "dram_read": rd, "dram_write": wr,
                     **{k: num(row, m, False) for k, m in UTIL.items()}})
T = sum(l["duration_s"] for l in launches) or 1.0
ok = [l for l in launches if l["dram_read"] is not None and l["dram_write"] is not None]
# launches whose DRAM counters were not collected are scaled in by duration
scale = T / sum(l["duration_s"] for l in ok) if ok else None
out = {"workload": workload, "filter": filt, "report": rep, "launches": len(launches),
       "launches_with_dram": len(ok),
       "dram_bytes_per_join": sum(l["dram_read"] + l["dram_write"] for l in ok) * scale if ok else None,
       "dram_read_bytes": sum(l["dram_read"] for l in ok) * scale if ok else None,
       "dram_write_bytes": sum(l["dram_write"] for l in ok) * scale if ok else None,
       "ncu_duration_s": T}
for k in UTIL:
    vals = [(l[k], l["duration_s"]) for l in launches if l[k] is not None]
    out[k] = sum(v * d for v, d in vals) / sum(d for _, d in vals) if vals else None
out["per_launch"] = launches
print(json.dumps(out, indent=1))
