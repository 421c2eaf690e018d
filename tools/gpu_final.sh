# round evidence: full bench line, ncu launch list of a bench command, ncu --set full of the step kernel
label=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$label.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_$label.jsonl 2> gpurun_out/bench_$label.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$label.jsonl 2> gpurun_out/bench_ref_$label.err; echo "ref rc=$?"
C="python bench.py --steps 2 --warmup 3 --substeps 20"
timeout 900 $C > gpurun_out/plain_launch_$label.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$label.csv $C > gpurun_out/ncu_launch_$label.log 2>&1
echo "launch list rc=$?"
bash tools/gpu_prof.sh $label > /dev/null 2>&1; echo "prof rc=$?"
cat gpurun_out/bench_$label.jsonl gpurun_out/bench_ref_$label.jsonl
