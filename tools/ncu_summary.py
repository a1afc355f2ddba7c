"""Summarise an ncu report (raw metrics + top stall sites): python tools/ncu_summary.py rep.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "smsp__cycles_active.avg"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w} = {v[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r)
hh = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hh)]   # first kernel section
iS, iSrc, iE = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source"), hh.index("Instructions Executed")
def fnum(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


tot = sum(fnum(x[iS]) for x in data) or 1.0
cols = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(fnum(x[hh.index(c)]) for x in data) for c in cols}
print("# warp stall reasons (share of samples)")
for c, s in sorted(agg.items(), key=lambda t: -t[1])[:8]:
    print(f"{c} = {100 * s / tot:.1f} %")
print(f"# top {ntop} SASS sites by stall samples")
for x in sorted(data, key=lambda x: -fnum(x[iS]))[:ntop]:
    st = sorted(((fnum(x[hh.index(c)]), c) for c in cols), reverse=True)[:2]
    print(f"{100 * fnum(x[iS]) / tot:5.1f}% {x[iSrc][:58]:58s} exec={x[iE]} {st[0][1]}/{st[1][1]}")
