# r02b: timed-path parity + no-transfer test, even split with real ranks,
# the default bench line (new roofline / e2e fields), forced-NCCL single rank A/B
set -x
timeout 900 python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "timed or transfer or even_split or nccl_machinery" > gpurun_out/r02b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_tests.log
tail -20 gpurun_out/r02b_tests.log
python bench.py > gpurun_out/r02b_bench.jsonl 2> gpurun_out/r02b_bench.err; echo "rc=$?"
tail -3 gpurun_out/r02b_bench.err
SW2D_FORCE_NCCL=1 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r02b_bench_forcenccl.jsonl 2>> gpurun_out/r02b_bench.err; echo "rc=$?"
SW2D_FORCE_NCCL=1 python bench.py --no-e2e --no-cpu-baseline --halo p2p > gpurun_out/r02b_bench_forcep2p.jsonl 2>> gpurun_out/r02b_bench.err; echo "rc=$?"
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r02b_bench_repeat.jsonl 2>> gpurun_out/r02b_bench.err; echo "rc=$?"
