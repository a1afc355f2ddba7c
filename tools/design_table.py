"""Regenerate DESIGN.md's measured table from a bench line + sweep file:
python tools/design_table.py profiles/r1_bench_v8_expo32.json profiles/r1_sweep_v8.jsonl"""
import json
import sys

txt = open(sys.argv[1]).read().strip()
try:
    b = json.loads(txt)
except json.JSONDecodeError:
    b = json.loads(txt.splitlines()[-1])
rows = [json.loads(l) for l in open(sys.argv[2]) if l.strip()]
names = {0: "FP64 scan", 1: "FP32 bound", 2: "tcgen05 bound"}


def row(d):
    c = d["config"]
    r = d.get("roofline") or {}
    flags = [f for f, on in (("no REORDER", not c["reorder"]), ("no SORTIDU", not c["sortidu"])) if on]
    filt = names[c["filter"]]
    if c.get("filter_requested", c["filter"]) == 2 and c["filter"] != 2:
        filt += " (fp16 bound not certifiable)"
    frac = ("%.3f %s" % (r["frac"], r["bound"])) if r.get("frac") else "-"
    return (f'| {c["workload"]} | {c["eps"]} | {c["k"]} | {", ".join(flags) or "-"} | {filt} | {c["n_batches"]} | '
            f'{d["pairs"]:,} | {d["selectivity"]:.1f} | {d["phases_ms"]["join"]:.1f} | {d["ms_per_step"]:.1f} | '
            f'{d["value"] / 1e6:.0f} M | {1000 * d["e2e"]["seconds"]:.0f} | {frac} |')


out = [f"## Measured (1 B200, round 2; `{sys.argv[1]}`, `{sys.argv[2]}`)", "",
       "`bench.py --steps 3 --warmup 3` per line (the bench default line: 5 steps; expo64_10m: 2); step = index build + estimator + "
       "batched join, inputs resident in HBM; join = the join kernels of all result batches (CUDA events); e2e = the "
       "same through the C ABI from host memory (median step).  Roofline fraction: tensor = 2n x evaluated tests / "
       "join time / the bf16 sustained peak (bench `roofline.peak`, `peak_note`); alu = 3 flops x SHORTC dims / join time / derived FP32 or "
       "FP64 peak (DESIGN §Roofline).", "",
       "| workload | eps | k | flags | filter | n_b | pairs | S_D | join ms | step ms | pairs/s | e2e ms | roofline frac |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|---|", row(b)] + [row(d) for d in rows]
out += ["", f'Oracle (numpy brute force, all host cores) on the bench sample: {b["cpu_baseline"]["value"]:.0f} pairs/s '
        f'({b["cpu_baseline"]["sample"]}).' if "cpu_baseline" in b else "", ""]
s = open("DESIGN.md").read()
i, j = s.index("## Measured"), s.index("## Multi-GPU")
open("DESIGN.md", "w").write(s[:i] + "\n".join(out) + "\n" + s[j:])
