set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02i_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02i_gpu_tests.log
tail -3 gpurun_out/r02i_gpu_tests.log
grep -q "rc=0" gpurun_out/r02i_gpu_tests.log || exit 1
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; tail -3 gpurun_out/r02i_smoke.log
bash tools/ab_env.sh r02i "-;SW2D_PERSIST=0;SW2D_PERSIST=1" "--workload c2|--workload c2 --reduce volume|--workload c1 --substeps 1000|--workload c1 --substeps 1000 --reduce volume|--workload c1 --substeps 1000 --reduce all|--workload c2 --reduce all" 1
