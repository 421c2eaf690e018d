// paper_1711_04471_b200/csrc/sw2d_cta2_r1.cu — the two-step kernel
// (sw2d_kernels.cu) with diagnostics level RED = 1, in a translation unit of
// its own so that the library's TUs compile in parallel (each instance of the
// kernel, with its three row-loop copies, takes minutes in ptxas).
#define SW2D_PROBE 1   // the device code of sw2d_kernels.cu without its launchers
#include "sw2d_kernels.cu"

namespace sw2d_dev {
void launch_step2_r1(const StepArgs& a, void* stream, bool remote) {
  cudaStream_t s = (cudaStream_t)stream;
  if (remote)
    launch_two<1, true>(a, s);
  else
    launch_two<1, false>(a, s);
}
}  // namespace sw2d_dev
