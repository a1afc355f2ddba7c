cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
B="timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
o=gpurun_out/sweep_r40.jsonl; : > $o
for e in 0.50 0.55 0.60; do $B --workload uniform16 --eps $e >> $o 2>/dev/null; done
$B --workload expo32 --no-reorder >> $o 2>/dev/null
$B --workload expo32 --no-sortidu >> $o 2>/dev/null
for k in 4 5 6 7 8; do $B --workload songs90 --k $k >> $o 2>/dev/null; done
$B --workload songs90 --eps 0.01 >> $o 2>/dev/null
$B --workload expo16 >> $o 2>/dev/null
$B --workload expo64_10m >> $o 2>gpurun_out/sweep_r40_10m.err
timeout 900 python bench.py > gpurun_out/bench_r40.json 2>/dev/null
python - <<'PY'
import json
for l in list(open("gpurun_out/sweep_r40.jsonl")) + list(open("gpurun_out/bench_r40.json")):
    d = json.loads(l); c = d["config"]; r = d.get("roofline") or {}
    print(c["workload"], "eps", c["eps"], "k", c["k"], "nb", c["n_batches"], "join_ms %.1f" % d["phases_ms"]["join"], "step_ms %.1f" % d["ms_per_step"], "pairs", d["pairs"],
          "Mpairs/s %.1f" % (d["value"] / 1e6), "frac %.3f" % (r.get("frac") or 0), "e2e_ms %.1f" % (1000 * d["e2e"]["seconds"]))
PY
