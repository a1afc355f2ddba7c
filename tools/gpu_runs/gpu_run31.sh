cd $GRAFT_REPO_ROOT
B="timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
o=gpurun_out/sweep_r31.jsonl; : > $o
for e in 0.50 0.55 0.60; do $B --workload uniform16 --eps $e >> $o 2>/dev/null; done
$B --workload expo32 --no-reorder >> $o 2>/dev/null
$B --workload expo32 --no-sortidu >> $o 2>/dev/null
for k in 4 5 6 7 8; do $B --workload songs90 --k $k --no-stats >> $o 2>/dev/null; done
$B --workload songs90 --eps 0.01 --no-stats >> $o 2>/dev/null
$B --workload expo16 >> $o 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload expo64_10m --no-stats >> $o 2>gpurun_out/sweep_r31_10m.err
python - <<'PY'
import json
for l in open("gpurun_out/sweep_r31.jsonl"):
    d = json.loads(l); c = d["config"]; r = d.get("roofline") or {}
    print(c["workload"], "eps", c["eps"], "k", c["k"], "reorder", c["reorder"], "sortidu", c["sortidu"], "filter", d["dtype"][:6],
          "join_ms %.1f" % d["phases_ms"]["join"], "step_ms %.1f" % d["ms_per_step"], "pairs", d["pairs"], "S_D %.2f" % d["selectivity"],
          "Mpairs/s %.1f" % (d["value"] / 1e6), "frac", r.get("frac"))
PY
tail -3 gpurun_out/sweep_r31_10m.err
