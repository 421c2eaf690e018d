# A/B of SOR kernel builds: bash tools/exp_sor_ab.sh lib1 lib2 ...
timeout 300 python -m pytest tests/test_gpu_sor.py -q -x 2>&1 | tail -1
for lib in "$@"; do
  echo "== $lib"
  SW2D_LIBRARY=paper_1711_04471_b200/$lib timeout 120 python tools/sor_time.py sor300 sor1024 --kz 0 | grep iters
  SW2D_LIBRARY=paper_1711_04471_b200/$lib timeout 120 python tools/sor_time.py sor300 sor1024 --kz 0 --every 1 | grep iters
done
