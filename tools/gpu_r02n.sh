set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02n_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02n_gpu_tests.log
tail -2 gpurun_out/r02n_gpu_tests.log
grep -q "rc=0" gpurun_out/r02n_gpu_tests.log || exit 1
python bench.py > gpurun_out/r02n_bench.jsonl 2> gpurun_out/r02n_bench.err; echo "bench rc=$?"
P=paper_1711_04471_b200
bash tools/ab_libs.sh r02n "$P/libsw2d_sor0.so $P/libsw2d.so" "--workload sor300|--workload sor300 --sor-residual-every 0|--workload sor1024 --steps 5" 2
