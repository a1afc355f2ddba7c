cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,utilization.gpu --format=csv
for mt in 1 2 1 2; do timeout 600 python bench.py --no-cpu-baseline --mma-tiles $mt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MT', d['config']['mma_tiles'], 'ms/step %.1f'%d['ms_per_step'], d['phases_ms'], 'e2e s %.3f'%d['e2e']['seconds'])"; done
