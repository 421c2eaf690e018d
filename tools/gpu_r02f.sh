# r02f evidence: default bench line, ncu launch list of the default command,
# ncu --set full of the C5 (RED=1) and C3 (RED=0) two-step launches
set -x
python bench.py > gpurun_out/r02f_bench.jsonl 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r02f_bench.jsonl
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02f_plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_launch.log 2>&1
echo "launch list rc=$?"
bash tools/gpu_prof.sh r02f_c5 --workload c5
bash tools/gpu_prof.sh r02f_c3 --workload c3
