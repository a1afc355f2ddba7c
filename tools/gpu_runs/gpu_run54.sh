cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('expo32 join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'e2e', d['e2e']['seconds'], 'frac', r['frac'], d['clocks'])"
for w in uniform16 expo16; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $w 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], 'join', d['phases_ms']['join'], 'frac', r['frac'])"; done
