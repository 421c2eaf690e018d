# one iteration: parity tests, bench variants, ncu of the C5 step kernel
# usage: bash tools/gpu_iter.sh <label>
label=${1:-iter}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_tests_$label.log 2>&1
tail -2 gpurun_out/gpu_tests_$label.log
rm -f gpurun_out/bench_$label.log
for w in "--workload c5" "--workload c5 --reduce none" "--workload c3" "--workload c2 --substeps 1000"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['frac'],4), d['clocks'])" >> gpurun_out/bench_$label.log 2>&1
done
cat gpurun_out/bench_$label.log
if [ "$2" = "prof" ]; then bash tools/gpu_prof.sh $label | tail -40; fi
