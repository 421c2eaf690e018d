# A/B of environment settings on bench lines:
#   bash tools/ab_env.sh <label> "<env1>;<env2>;..." "<workload args 1>|<workload args 2>|..." [reps]
# (an env entry is space-separated VAR=val pairs; "-" for none)
label=$1; envs=$2; wls=$3; reps=${4:-1}
out=gpurun_out/ab_$label.log; rm -f $out; mkdir -p gpurun_out
IFS=';' read -ra EV <<< "$envs"
IFS='|' read -ra W <<< "$wls"
for rep in $(seq $reps); do
for e in "${EV[@]}"; do
for w in "${W[@]}"; do
  ee=$e; [ "$e" = "-" ] && ee="SW2D_AB=1"
  env $ee timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e | $w |', round(d['value']/1e9,2), 'Gcell/s', round(d['ms_per_step']*1e3/d['config']['substeps_per_step'],3), 'us/step', round(d['roofline']['frac'],4), d['roofline'].get('plan','')[:60], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $out 2>&1
done; done; done
cat $out
