cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 900 python bench.py > gpurun_out/bench_r66_$i.json 2> gpurun_out/bench_r66_$i.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r66_$i.json')); print(d['value']/1e6, d['ms_per_step'], d['phases_ms'], d['clocks'], d['e2e']['seconds'], d['roofline']['frac'])"; done
