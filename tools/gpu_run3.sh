mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_tests.log 2>&1
for w in "--workload c5" "--workload c5 --reduce none" "--workload c5 --reduce all" "--workload c3" "--workload c2 --substeps 1000"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value']/1e9, 'Gcell/s', d['roofline']['achieved'], 'GB/s', d['roofline']['frac'], d['clocks'])" >> gpurun_out/bench3.log 2>&1
done
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench3.log
