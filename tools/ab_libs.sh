# A/B of library builds on bench lines:
#   bash tools/ab_libs.sh <label> "<lib1> <lib2> ..." "<workload args 1>|<workload args 2>|..." [reps]
# every (rep, lib, workload) runs bench.py once (no e2e, no cpu baseline); one
# summary line each in gpurun_out/ab_<label>.log
label=$1; libs=$2; wls=$3; reps=${4:-2}
out=gpurun_out/ab_$label.log; rm -f $out; mkdir -p gpurun_out
IFS='|' read -ra W <<< "$wls"
for rep in $(seq $reps); do
for lib in $libs; do
for w in "${W[@]}"; do
  SW2D_LIBRARY=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib) | $w |', round(d['value']/1e9,2), 'Gcell/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $out 2>&1
done; done; done
cat $out
