set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k persistent > gpurun_out/r02k_persist_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02k_persist_tests.log
tail -3 gpurun_out/r02k_persist_tests.log
grep -q "rc=0" gpurun_out/r02k_persist_tests.log || exit 1
bash tools/ab_env.sh r02k "-;SW2D_PERSIST=0;SW2D_PERSIST_SHAPE=0;SW2D_PERSIST_SHAPE=2;SW2D_PERSIST_SHAPE=3;SW2D_PERSIST_SHAPE=4;SW2D_PERSIST_SHAPE=5" "--workload c2|--workload c1 --substeps 1000" 1
timeout 300 python tools/xfer_probe.py > gpurun_out/r02k_xfer.json 2> gpurun_out/r02k_xfer.err; cat gpurun_out/r02k_xfer.json; tail -3 gpurun_out/r02k_xfer.err
