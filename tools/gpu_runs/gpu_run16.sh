cd $GRAFT_REPO_ROOT
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms/step %.1f'%d['ms_per_step'], {k: round(v,1) for k,v in d['phases_ms'].items()}, 'e2e s %.3f'%d['e2e']['seconds'])"; }
for i in 1; do
echo old; (cd old_r18 && timeout 600 python bench.py --no-cpu-baseline 2>../gpurun_out/old.err | summ)
echo new-mt1; timeout 600 python bench.py --no-cpu-baseline --mma-tiles 1 2>/dev/null | summ
echo new-mt2; timeout 600 python bench.py --no-cpu-baseline --mma-tiles 2 2>/dev/null | summ
done
