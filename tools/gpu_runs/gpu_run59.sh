cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "fullsize or batches or partition" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('expo32 join', d['phases_ms']['join'], 'step', d['ms_per_step'], 'e2e', d['e2e']['seconds'], 'frac', r['frac'], d['clocks'])"
timeout 900 python tools/scaling_projection.py 2>&1 | grep "^world"
