set -x
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02j_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_gpu_tests.log
tail -3 gpurun_out/r02j_gpu_tests.log
SW2D_LIBRARY=$PWD/paper_1711_04471_b200/libsw2d_dbg.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02j_gpu_tests_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_gpu_tests_dbg.log
tail -3 gpurun_out/r02j_gpu_tests_dbg.log
