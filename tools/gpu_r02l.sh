set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k persistent > gpurun_out/r02l_persist_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02l_persist_tests.log
tail -2 gpurun_out/r02l_persist_tests.log
bash tools/ab_env.sh r02l "-;SW2D_PERSIST=0" "--workload c2|--workload c1 --substeps 1000|--workload c2 --reduce volume" 1
timeout 300 python tools/xfer_probe.py > gpurun_out/r02l_xfer.json 2> gpurun_out/r02l_xfer.err; cat gpurun_out/r02l_xfer.json; tail -3 gpurun_out/r02l_xfer.err
