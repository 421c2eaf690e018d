# run the GPU parity suite against the device-bounds-checked build
# (compute-sanitizer is closed on this pool)
python -m paper_1711_04471_b200._build --debug > /dev/null
SW2D_LIBRARY=$PWD/paper_1711_04471_b200/libsw2d_dbg.so timeout 1200 python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "bounds|passed|failed" | head -5
