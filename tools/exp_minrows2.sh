for m in 8 6 4 3 2; do for w in "--workload c2 --substeps 1000" "--workload p1000 --substeps 1000" "--workload c1 --substeps 1000"; do
  SW2D_MIN_ROWS2=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minrows2 $m $w', '%.3e'%d['value'], 'us/step %.3f'%(d['ms_per_step']), d['roofline']['plan'][:50])"
done; done
