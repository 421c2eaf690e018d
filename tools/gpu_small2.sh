mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_all_tests.log 2>&1; tail -3 gpurun_out/gpu_all_tests.log
for w in "--workload c2 --substeps 1000" "--workload c2 --substeps 1000 --reduce volume" "--workload c2 --substeps 1000 --reduce all" "--workload c1 --substeps 1000" "--workload p1000 --substeps 1000"; do
  for lib in libsw2d_prev.so libsw2d.so; do
  SW2D_LIBRARY=paper_1711_04471_b200/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $w', '%.3e'%d['value'], 'us/step', round(d['ms_per_step']*1000/1000,3), d['roofline']['plan'][:60])"
  done
done
