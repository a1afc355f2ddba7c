"""Per-kernel share of device time from an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launch_summary.py launches.csv "<command line>" > summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[h + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    u = r[iu].strip().lower()
    v = v / 1e6 if u in ("nsecond", "ns") else (v / 1e3 if u in ("usecond", "us") else v)   # -> ms
    tot[r[ik]] += v
    cnt[r[ik]] += 1
T = sum(tot.values())
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({sys.argv[2] if len(sys.argv) > 2 else ''}), "
      f"cold-cache serialised launches")
print(f"# {sum(cnt.values())} launches, total {T:.1f} ms; share of device time per kernel:")
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    print(f"{100 * v / T:6.2f}% {v:11.3f} ms {cnt[k]:6d} launches  {k}")
