set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k persistent > gpurun_out/r02e_persist_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_persist_tests.log
tail -3 gpurun_out/r02e_persist_tests.log
P=paper_1711_04471_b200
bash tools/ab_libs.sh r02e "$P/libsw2d.so $P/libsw2d_nowait.so" "--workload c2|--workload c1 --substeps 1000" 1
bash tools/ab_env.sh r02e_th "SW2D_PERSIST_TH=4;SW2D_PERSIST_TH=8;SW2D_PERSIST_TH=16;SW2D_PERSIST_TH=32;SW2D_PERSIST_K=1 SW2D_PERSIST_TH=8" "--workload c2|--workload c1 --substeps 1000" 1
