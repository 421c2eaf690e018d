set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k persistent > gpurun_out/r02g_persist_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_persist_tests.log
tail -3 gpurun_out/r02g_persist_tests.log
grep -q "rc=0" gpurun_out/r02g_persist_tests.log || exit 1
bash tools/ab_env.sh r02g "SW2D_PERSIST=0;SW2D_PERSIST=1;SW2D_PERSIST=1 SW2D_PERSIST_RW=1;SW2D_PERSIST=1 SW2D_PERSIST_RW=2;SW2D_PERSIST=1 SW2D_PERSIST_K=1;SW2D_PERSIST=1 SW2D_PERSIST_K=1 SW2D_PERSIST_RW=1;SW2D_PERSIST=1 SW2D_PERSIST_K=1 SW2D_PERSIST_RW=2" "--workload c2|--workload c1 --substeps 1000|--workload p1000 --substeps 1000|--workload c2 --reduce volume" 1
