# repeat the GPU suite (flakiness), then the bounds-checked debug build
mkdir -p gpurun_out
for r in 1 2 3; do timeout 600 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -1; done
python -m paper_1711_04471_b200._build --debug > /dev/null 2>&1
SW2D_LIBRARY=paper_1711_04471_b200/libsw2d_dbg.so timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
