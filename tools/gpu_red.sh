for r in 0 1 2; do for w in "--workload c3" "--workload c5 --reduce none" "--workload p2000 --substeps 200" "--workload c2 --substeps 1000"; do
SW2D_MIN_RED=$r python bench.py $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minred $r $w', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done
