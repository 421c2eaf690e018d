SOR3D_KERNEL=1 timeout 300 python -m pytest tests/test_gpu_sor.py -q -x 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_sor.py -q -x -k rows 2>&1 | tail -1
for k in 0 1; do for r in 32 16; do
  echo "== kernel $k rows $r"
  SOR3D_KERNEL=$k SOR3D_ROWS=$r timeout 120 python tools/sor_time.py sor300 sor1024 --kz 0 | grep iters
  SOR3D_KERNEL=$k SOR3D_ROWS=$r timeout 120 python tools/sor_time.py sor300 sor1024 --kz 0 --every 1 | grep iters
done; done
