# A/B of step-kernel kinds: bash tools/gpu_ab.sh <label> [prof]
label=${1:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_tests_$label.log 2>&1
tail -2 gpurun_out/gpu_tests_$label.log
SW2D_STEP_KERNEL=0 timeout 900 python -m pytest tests -m gpu -q -rf -x -k "virtual or ragged or c1" > gpurun_out/gpu_tests0_$label.log 2>&1
tail -1 gpurun_out/gpu_tests0_$label.log
rm -f gpurun_out/bench_$label.log
for k in 1; do
for w in "--workload c5" "--workload c1 --substeps 1000" "--workload c2 --substeps 1000" "--workload p1000 --substeps 1000" "--workload p2000 --substeps 500"; do
  SW2D_STEP_KERNEL=$k timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kind $k $w', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/bench_$label.log 2>&1
done; done
cat gpurun_out/bench_$label.log
if [ "$2" = "prof" ]; then bash tools/gpu_prof.sh $label | tail -40; fi
