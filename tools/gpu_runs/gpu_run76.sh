cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r76.json 2> gpurun_out/bench_r76.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r76.json')); r=d['roofline']; print('%.1f Mpairs/s'%(d['value']/1e6), 'step %.1f'%d['ms_per_step'], 'join %.1f'%d['phases_ms']['join'], 'e2e %.1f (mean %.1f)'%(1000*d['e2e']['seconds'], 1000*d['e2e']['mean_seconds']), 'frac %.3f'%r['frac'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/bench_r76_ref.json 2>/dev/null; cut -c1-160 gpurun_out/bench_r76_ref.json
