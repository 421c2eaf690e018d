mkdir -p gpurun_out
Q="python bench.py --profile --steps 1 --warmup 3 --substeps 4"
SW2D_TWO_STEP_WS=1 timeout 600 $Q > gpurun_out/ws_plain.log 2>&1 && \
  SW2D_TWO_STEP_WS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o gpurun_out/prof_ws $Q > gpurun_out/ncu_ws.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_ws.ncu-rep ws --cells 268435456 2>&1 | head -45
