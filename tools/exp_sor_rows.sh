timeout 300 python -m pytest tests/test_gpu_sor.py -q -rf -x 2>&1 | tail -3
for r in 32 16; do
  SOR3D_ROWS=$r timeout 120 python tools/sor_time.py sor300 sor1024 --kz 0
  SOR3D_ROWS=$r timeout 120 python tools/sor_time.py sor300 --kz 0 --every 1
done
