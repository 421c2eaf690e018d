# NEXT-4 SOR: GPU parity tests + timing sweep over z-chunks
# usage: bash tools/gpu_sor.sh <label> [kz-list]
label=${1:-sor}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sor.py -q -rf -x > gpurun_out/sor_tests_$label.log 2>&1
tail -15 gpurun_out/sor_tests_$label.log
timeout 200 python tools/sor_time.py sor300 sor1024 --kz ${2:-0,13,29,45} > gpurun_out/sor_time_$label.log 2>&1
echo "--- residual every iteration" >> gpurun_out/sor_time_$label.log
timeout 200 python tools/sor_time.py sor300 sor1024 --kz 0 --every 1 >> gpurun_out/sor_time_$label.log 2>&1
echo "--- no L2 hints" >> gpurun_out/sor_time_$label.log
SOR3D_HINT=0 timeout 200 python tools/sor_time.py sor300 --kz 0 >> gpurun_out/sor_time_$label.log 2>&1
cat gpurun_out/sor_time_$label.log
