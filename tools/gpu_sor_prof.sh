# ncu --set full of one SOR launch (after the same command exits 0 without ncu)
# usage: gpu_sor_prof.sh <label> <config> <every> [env...]
label=$1; c=$2; every=$3; shift 3
mkdir -p gpurun_out
Q="python tools/sor_time.py $c --kz 0 --iters 5 --every $every"
env "$@" timeout 300 $Q > gpurun_out/sor_plain_${label}.log 2>&1 && \
  env "$@" timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:sor_ -s 8 -c 1 \
    -o gpurun_out/sorprof_${label} $Q > gpurun_out/sor_ncu_${label}.log 2>&1
python tools/ncu_summary.py gpurun_out/sorprof_${label}.ncu-rep ${label} > gpurun_out/sor_summary_${label}.json 2>&1
cat gpurun_out/sor_plain_${label}.log; head -45 gpurun_out/sor_summary_${label}.json
