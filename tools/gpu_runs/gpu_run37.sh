cd $GRAFT_REPO_ROOT
for e in 0.005 0.01; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload songs90 --eps $e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['eps'], 'join', d['phases_ms']['join'], 'pairs', d['pairs'], 'frac', r['frac'], r['achieved'], r['peak'], r['alg'])"; done
