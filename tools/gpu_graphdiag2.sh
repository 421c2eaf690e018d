mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_all_tests.log 2>&1; tail -3 gpurun_out/gpu_all_tests.log
bash tools/exp_ab_multi.sh "--workload c5" libsw2d_prev.so libsw2d.so
bash tools/exp_ab_multi.sh "--workload c2 --substeps 1000 --reduce volume" libsw2d_prev.so libsw2d.so
