cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r75.json 2> gpurun_out/bench_r75.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r75.json')); r=d['roofline']; print('%.1f Mpairs/s'%(d['value']/1e6), 'step %.1f'%d['ms_per_step'], {k: round(v,2) for k,v in d['phases_ms'].items()}, 'e2e %.1f'%(1000*d['e2e']['seconds']), 'frac %.3f'%r['frac'], d['index'])"
timeout 900 python tools/scaling_projection.py 2>&1 | grep "^world"
