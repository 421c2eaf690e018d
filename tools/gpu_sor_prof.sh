# ncu --set full of one sor_iter launch per config (after a plain run exits 0)
# usage: bash tools/gpu_sor_prof.sh <label> [kz] [cache-control: all|none] [configs]
label=${1:-sor}; kz=${2:-0}; cc=${3:-all}; cfgs=${4:-"sor1024 sor300"}
mkdir -p gpurun_out
for c in $cfgs; do
  Q="python tools/sor_time.py $c --kz $kz --iters 5"
  timeout 600 $Q > gpurun_out/sor_plain_${label}_$c.log 2>&1 && \
    timeout 900 ncu --set full --cache-control $cc --clock-control none --import-source on -k regex:sor_iter -s 8 -c 1 \
      -o gpurun_out/sorprof_${label}_$c $Q > gpurun_out/sor_ncu_${label}_$c.log 2>&1
  python tools/ncu_summary.py gpurun_out/sorprof_${label}_$c.ncu-rep ${label}_$c > gpurun_out/sor_summary_${label}_$c.json 2>&1
  cat gpurun_out/sor_plain_${label}_$c.log; head -60 gpurun_out/sor_summary_${label}_$c.json
done
