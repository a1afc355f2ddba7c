cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for e in 0.005 0.01; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload songs90 --eps $e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['eps'], 'join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'pairs', d['pairs'], 'frac', r['frac'])"; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('expo32 join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'e2e', d['e2e']['seconds'], 'frac', r['frac'])"
