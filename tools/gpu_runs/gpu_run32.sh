cd $GRAFT_REPO_ROOT
timeout 600 python tools/e2e_probe.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "batches or neighbor or estimator or partition or degenerate" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r32.json 2> gpurun_out/bench_r32.err; tail -2 gpurun_out/bench_r32.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r32.json')); print('ms/step', d['ms_per_step'], d['phases_ms'], 'e2e', d['e2e']['seconds'], d['e2e']['value']/1e6, 'Mpairs/s', d['clocks'])"
