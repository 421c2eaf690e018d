# NEXT-4 evidence: parity tests, bench lines, launch list, ncu --set full
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sor.py -q -rf -x > gpurun_out/sor_final_tests.log 2>&1; tail -2 gpurun_out/sor_final_tests.log
timeout 300 python bench.py --workload sor300 --steps 10 --warmup 3 > gpurun_out/bench_sor300.json 2> gpurun_out/bench_sor300.err
timeout 300 python bench.py --workload sor1024 --steps 5 --warmup 3 > gpurun_out/bench_sor1024.json 2> gpurun_out/bench_sor1024.err
tail -c 1500 gpurun_out/bench_sor300.json; echo; tail -c 600 gpurun_out/bench_sor1024.json; echo
timeout 300 python bench.py --workload sor300 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_sor300.csv \
    python bench.py --workload sor300 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_sor300.log 2>&1
bash tools/gpu_sor_prof.sh sor300_res sor300 1 | tail -40
bash tools/gpu_sor_prof.sh sor1024_res sor1024 1 | tail -40
