# usage: bash tools/gpu_prof.sh <label> [bench args...]
# plain run, then ncu --set full of one step-kernel launch, then the summary
label=$1; shift
mkdir -p gpurun_out
Q="python bench.py --profile --steps 1 --warmup 3 --substeps 4 $*"
timeout 600 $Q > gpurun_out/plain_$label.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o gpurun_out/prof_$label $Q > gpurun_out/ncu_$label.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_$label.ncu-rep $label > gpurun_out/summary_$label.json 2>&1
tail -c 400 gpurun_out/plain_$label.log; head -40 gpurun_out/summary_$label.json
