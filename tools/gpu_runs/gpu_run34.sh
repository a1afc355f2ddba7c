cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "counts or counters" 2>&1 | tail -2
B="timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
o=gpurun_out/sweep_r34.jsonl; : > $o
$B --workload songs90 --k 6 >> $o 2> gpurun_out/songs6.err; tail -3 gpurun_out/songs6.err
$B --workload expo64_10m >> $o 2>/dev/null
$B >> $o 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/sweep_r34.jsonl"):
    d = json.loads(l); c = d["config"]; r = d.get("roofline") or {}
    print(c["workload"], "k", c["k"], "join_ms %.1f" % d["phases_ms"]["join"], "step %.1f" % d["ms_per_step"], "pairs", d["pairs"], "frac", r.get("frac"), "e2e_s", d["e2e"]["seconds"])
PY
