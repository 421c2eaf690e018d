set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k persistent > gpurun_out/r02d_persist_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_persist_tests.log
tail -5 gpurun_out/r02d_persist_tests.log
grep -q "rc=0" gpurun_out/r02d_persist_tests.log || exit 1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02d_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_gpu_tests.log
tail -5 gpurun_out/r02d_gpu_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; tail -3 gpurun_out/r02d_smoke.log
P=paper_1711_04471_b200
bash tools/ab_libs.sh r02d "$P/libsw2d_base.so $P/libsw2d.so $P/libsw2d_p1.so $P/libsw2d_p0.so" "--workload c5|--workload c5 --reduce none|--workload c3|--workload c5 --reduce all" 1
bash tools/ab_env.sh r02d_small "-;SW2D_PERSIST=0;SW2D_PERSIST_K=1;SW2D_PERSIST_TH=8;SW2D_PERSIST_TH=16;SW2D_PERSIST_TH=24;SW2D_PERSIST_TH=32" "--workload c2|--workload c1 --substeps 1000|--workload p1000 --substeps 1000|--workload c2 --reduce volume" 1
