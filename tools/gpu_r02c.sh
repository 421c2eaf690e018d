set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02c_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_gpu_tests.log
tail -5 gpurun_out/r02c_gpu_tests.log
P=paper_1711_04471_b200
bash tools/ab_libs.sh r02c "$P/libsw2d_base.so $P/libsw2d.so $P/libsw2d_red0p.so" "--workload c5|--workload c3|--workload c5 --reduce none|--workload c5 --reduce all|--workload p2000" 2
