set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 400 python -m pytest tests/test_gpu_p2p_procs.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r02a_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/r02a_p2p.log
tail -5 gpurun_out/r02a_p2p.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02a_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02a_gpu_tests.log
tail -15 gpurun_out/r02a_gpu_tests.log
