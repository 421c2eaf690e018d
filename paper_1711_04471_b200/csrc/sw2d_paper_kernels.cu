// paper_1711_04471_b200/csrc/sw2d_paper_kernels.cu — the paper-shaped,
// unfused step (SW2D_VARIANT_PAPER).
//
// The paper's compiler turns the 2DSW time loop into "three map-style
// kernels".  This variant keeps that shape to measure what
// fusion buys: three plain one-thread-per-cell map kernels per step, with h
// and the wet flags stored in HBM between steps as the textbook's update does:
//   K1 dyn/momentum:  un, vn        <- eta, u, v, wet          (21 B/cell)
//   K2 dyn/continuity: etan          <- eta, un, vn, h          (20 B/cell)
//   K3 shapiro+update: eta, h, wet', u, v <- etan, wet, hzero, un, vn (34 B/cell)
// = 75 B/cell-step against the fused pass's 28.  The wet flags are double
// buffered (K3 reads the start-of-step flags of its neighbours and writes the
// new ones; reading R17).  Arithmetic is operation for operation the oracle's.
#include <cuda_runtime.h>

#include <cstdint>

#include "sw2d_internal.cuh"

namespace sw2d_dev {

namespace {

__device__ __forceinline__ float flux_exact(float s, float hl, float hr) {
  return s > 0.0f ? __fmul_rn(s, hl) : (s < 0.0f ? __fmul_rn(s, hr) : 0.0f);
}

__device__ __forceinline__ bool flows(bool wc, bool wn, float d) {
  return wc ? (wn || d > 0.0f) : (wn && d < 0.0f);
}

struct Cell {
  int k;          // 1-based column
  long long r;    // storage row
  long long o;    // element offset
  long long jg;   // global 1-based row
  bool ok;
};

__device__ __forceinline__ Cell cell_of(const PaperArgs& a) {
  Cell c;
  c.k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const long long jl = (long long)blockIdx.y * blockDim.y + threadIdx.y;  // 0-based local row
  c.r = jl + kHaloRows;
  c.o = c.r * a.pitch + c.k + kColOff;
  c.jg = a.jbase + c.r;
  c.ok = c.k <= a.nx && jl < a.nrows;
  return c;
}

__global__ void paper_momentum(const PaperArgs a) {
  const Cell c = cell_of(a);
  if (!c.ok) return;
  const float e = a.E[c.o];
  const bool wc = a.wet_in[c.o];
  float un = 0.0f, vn = 0.0f;
  if (c.k != a.nx) {
    const float du = __fmul_rn(a.c.cgx, __fsub_rn(a.E[c.o + 1], e));
    if (flows(wc, a.wet_in[c.o + 1], du)) un = __fadd_rn(a.U[c.o], du);
  }
  if (c.jg != a.ny) {
    const float dv = __fmul_rn(a.c.cgy, __fsub_rn(a.E[c.o + a.pitch], e));
    if (flows(wc, a.wet_in[c.o + a.pitch], dv)) vn = __fadd_rn(a.V[c.o], dv);
  }
  a.un[c.o] = un;
  a.vn[c.o] = vn;
}

__global__ void paper_continuity(const PaperArgs a) {
  const Cell c = cell_of(a);
  if (!c.ok) return;
  const long long o = c.o, p = a.pitch;
  const float hc = a.h[o];
  const float fe = flux_exact(a.un[o], hc, a.h[o + 1]);
  const float fw = flux_exact(a.un[o - 1], a.h[o - 1], hc);
  const float fn = flux_exact(a.vn[o], hc, a.h[o + p]);
  const float fs = flux_exact(a.vn[o - p], a.h[o - p], hc);
  a.etan[o] = __fsub_rn(__fsub_rn(a.E[o], __fmul_rn(a.c.cx, __fsub_rn(fe, fw))),
                        __fmul_rn(a.c.cy, __fsub_rn(fn, fs)));
}

__global__ void paper_shapiro_update(const PaperArgs a) {
  const Cell c = cell_of(a);
  if (!c.ok) return;
  const long long o = c.o, p = a.pitch;
  const float en = a.etan[o];
  float e = en;
  if (a.wet_in[o]) {
    const bool wE = a.wet_in[o + 1], wW = a.wet_in[o - 1];
    const bool wN = a.wet_in[o + p], wS = a.wet_in[o - p];
    const float s = (float)((int)wE + (int)wW + (int)wN + (int)wS);
    const float q = a.c.q;
    const float t1 = __fmul_rn(__fsub_rn(1.0f, __fmul_rn(q, s)), en);
    const float t2 = __fmul_rn(q, __fadd_rn(wE ? a.etan[o + 1] : 0.0f, wW ? a.etan[o - 1] : 0.0f));
    const float t3 = __fmul_rn(q, __fadd_rn(wN ? a.etan[o + p] : 0.0f, wS ? a.etan[o - p] : 0.0f));
    e = __fadd_rn(__fadd_rn(t1, t2), t3);
  }
  // update: eta, h, wet, and "updating the velocity"
  const float h = __fadd_rn(a.H0[o], e);
  a.Eo[o] = e;
  a.h[o] = h;
  a.wet_out[o] = (h < a.c.hmin) ? 0 : 1;
  a.Uo[o] = a.un[o];
  a.Vo[o] = a.vn[o];
}

__global__ void paper_init(const PaperArgs a) {
  const Cell c = cell_of(a);
  if (!c.ok) return;
  const float h = __fadd_rn(a.H0[c.o], a.E[c.o]);
  a.h[c.o] = h;
  a.wet_out[c.o] = (h < a.c.hmin) ? 0 : 1;
}

dim3 grid_of(const PaperArgs& a, dim3 blk) {
  return dim3((unsigned)((a.nx + blk.x - 1) / blk.x), (unsigned)((a.nrows + blk.y - 1) / blk.y));
}

}  // namespace

void launch_paper_step(const PaperArgs& a, void* stream) {
  const dim3 blk(128, 2);
  const dim3 g = grid_of(a, blk);
  cudaStream_t s = (cudaStream_t)stream;
  paper_momentum<<<g, blk, 0, s>>>(a);
  paper_continuity<<<g, blk, 0, s>>>(a);
  paper_shapiro_update<<<g, blk, 0, s>>>(a);
}

void launch_paper_init(const PaperArgs& a, void* stream) {
  const dim3 blk(128, 2);
  paper_init<<<grid_of(a, blk), blk, 0, (cudaStream_t)stream>>>(a);
}

}  // namespace sw2d_dev
