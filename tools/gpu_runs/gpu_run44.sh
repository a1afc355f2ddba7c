cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
for i in 1 2; do timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('expo32 join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'e2e', d['e2e']['seconds'], 'frac', r['frac'], d['clocks'])"; done
