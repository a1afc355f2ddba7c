cd $GRAFT_REPO_ROOT
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r69.json 2> gpurun_out/bench_r69.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r69.json')); r=d['roofline']; print('%.1f Mpairs/s'%(d['value']/1e6), 'step %.1f'%d['ms_per_step'], 'join %.1f'%d['phases_ms']['join'], 'e2e %.1f'%(1000*d['e2e']['seconds']), 'frac %.3f'%r['frac'], r['peak'], r['peak_note'], d['clocks'], d['gpu_launches'], d['cpu_baseline']['value'])"
