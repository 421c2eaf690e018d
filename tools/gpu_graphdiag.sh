mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_all_tests.log 2>&1; tail -3 gpurun_out/gpu_all_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
for w in "--workload c2 --substeps 1000 --reduce none" "--workload c2 --substeps 1000 --reduce volume" "--workload c2 --substeps 1000 --reduce all" "--workload c1 --substeps 1000 --reduce all" "--workload c5"; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '%.3e'%d['value'], 'ms/step', round(d['ms_per_step'],3), d['gpu_launches'])"
done
