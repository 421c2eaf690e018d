# sweep CTAs/SM for c3/c5 without reductions
for b in 1 2; do for w in "--workload c3 --reduce none" "--workload c5 --reduce none" "--workload c5"; do
 SW2D_CTAS_PER_SM=$b timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bps $b $w', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
