cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/prof_join.py --workload songs90 --reps 2 --filter 1 2>&1 | tail -1
timeout 600 python tools/prof_join.py --workload songs90 --eps 0.01 --reps 2 --filter 1 2>&1 | tail -1
for e in 0.005 0.01; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload songs90 --eps $e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['eps'], 'join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'e2e', d['e2e']['seconds'], 'frac', r['frac'])"; done
