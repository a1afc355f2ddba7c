cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -k "filt or boundary or flag" 2>&1 | tail -2
for e in 0.005 0.01; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload songs90 --eps $e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['eps'], 'join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'e2e', d['e2e']['seconds'], 'pairs', d['pairs'], 'frac', r['frac'])"; done
