set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02m_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02m_gpu_tests.log
tail -2 gpurun_out/r02m_gpu_tests.log
grep -q "rc=0" gpurun_out/r02m_gpu_tests.log || exit 1
python bench.py > gpurun_out/r02m_bench.jsonl 2> gpurun_out/r02m_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02m_bench.jsonl
timeout 300 python tools/xfer_probe.py > gpurun_out/r02m_xfer.json 2> gpurun_out/r02m_xfer.err; head -c 1200 gpurun_out/r02m_xfer.json
