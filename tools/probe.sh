#!/bin/bash
# tools/probe.sh [RED] [extra nvcc flags...]: SASS loop counts of sw2d_step_cta2<RED, 0>
RED=${1:-1}; shift
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  --fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xptxas -v -DPROBE_RED=$RED "$@" \
  -I include -I paper_1711_04471_b200/csrc -cubin -o /tmp/probe.cubin tools/cta2_probe.cu 2>&1 \
  | grep -E "registers|spill" | head -4
python tools/sass_loop.py /tmp/probe.cubin step_cta2 | awk '{ if ($0 ~ /loop/ && $3+0 > 500) print; else if ($0 !~ /loop/) print }'
