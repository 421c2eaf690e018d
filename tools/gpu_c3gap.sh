for T in 10 100 1000; do
python bench.py --workload c3 --substeps $T --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 T=$T', round(d['value']/1e9,2), 'Gcell/s', round(d['ms_per_step']/$T*1000,1), 'us/step', d['clocks']['sm_mhz'])"
python bench.py --workload c3 --reduce volume --substeps $T --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 red1 T=$T', round(d['value']/1e9,2), 'Gcell/s', round(d['ms_per_step']/$T*1000,1), 'us/step', d['clocks']['sm_mhz'])"
done
SW2D_CTAS_PER_SM=1 SW2D_MIN_ROWS=1024 python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c 60-110
