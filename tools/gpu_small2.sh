timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for k in 2 1; do for m in 4 2 8; do for w in "--workload c1 --substeps 1000" "--workload c2 --substeps 1000" "--workload p1000 --substeps 1000" "--workload p2000 --substeps 500"; do
 SW2D_STEP_KERNEL=$k SW2D_MIN_ROWS=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kind $k minrows $m $w', round(d['value']/1e9,2), 'Gcell/s', round(d['ms_per_step']/d['config']['substeps_per_step']*1000,2), 'us/step')"
done; done; done
