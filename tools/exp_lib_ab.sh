# A/B of two library builds on the bench lines: bash tools/exp_lib_ab.sh <label> <libB> [tests]
label=${1:-ab}; libB=${2:-paper_1711_04471_b200/libsw2d_u2.so}
mkdir -p gpurun_out
if [ "$3" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_tests_$label.log 2>&1
  tail -2 gpurun_out/gpu_tests_$label.log
fi
out=gpurun_out/ab_$label.log; rm -f $out
for rep in 1 2; do
for lib in paper_1711_04471_b200/libsw2d.so $libB; do
for w in "--workload c5" "--workload c3" "--workload c5 --reduce all" "--workload p1000 --substeps 1000"; do
  SW2D_LIBRARY=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib) $w', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $out 2>&1
done; done; done
cat $out
