# warp-specialised two-step kernel: parity (all GPU tests with it on) + A/B
mkdir -p gpurun_out
SW2D_TWO_STEP_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x > gpurun_out/ws_tests.log 2>&1; tail -3 gpurun_out/ws_tests.log
for w in "--workload c5" "--workload c3" "--workload c5 --reduce none"; do
  for v in 0 1; do
    SW2D_TWO_STEP_WS=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $w 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ws=$v $w', '%.4e'%d['value'], d['clocks']['sm_mhz'])"
  done
done
