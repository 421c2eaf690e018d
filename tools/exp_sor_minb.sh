timeout 300 python -m pytest tests/test_gpu_sor.py -q -rf -x 2>&1 | tail -2
for lib in libsw2d.so libsw2d_v1.so libsw2d_v2.so; do
  for r in 32 16; do
    echo "== $lib rows=$r"
    SW2D_LIBRARY=paper_1711_04471_b200/$lib SOR3D_ROWS=$r timeout 120 python tools/sor_time.py sor300 sor1024 --kz 0 | grep iters
    SW2D_LIBRARY=paper_1711_04471_b200/$lib SOR3D_ROWS=$r timeout 120 python tools/sor_time.py sor300 --kz 0 --every 1 | grep iters
  done
done
