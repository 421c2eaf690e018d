# correctness + bench + ncu launch list + ncu full of the step kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
P="python bench.py --profile --steps 2 --warmup 3 --substeps 10"
timeout 600 $P > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu1.log 2>&1
Q="python bench.py --profile --steps 1 --warmup 3 --substeps 4"
timeout 600 $Q > gpurun_out/plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o gpurun_out/prof_step $Q > gpurun_out/ncu2.log 2>&1
tail -5 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log; tail -c 2500 gpurun_out/bench.log; tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
