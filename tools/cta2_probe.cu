// tools/cta2_probe.cu — compile one instantiation of the two-step kernel for
// SASS studies without the rest of the library (seconds, not a minute):
//   nvcc <library flags> -DSW2D_PROBE -DPROBE_RED=1 -I include -I csrc -cubin \
//        tools/cta2_probe.cu && python tools/sass_loop.py probe.cubin cta2
#define SW2D_PROBE 1
#include "sw2d_kernels.cu"
#ifndef PROBE_RED
#define PROBE_RED 1
#endif
namespace sw2d_dev {
namespace {
template __global__ void sw2d_step_cta2<PROBE_RED, false>(const StepArgs);
}
}
