// paper_1711_04471_b200/csrc/sw2d_kernels.cu — sm_100a kernels of the 2DSW
// time step (arXiv 1711.04471 §6.2).
//
// The paper's compiler emits the step as three map kernels (dyn, shapiro,
// update) that each stream the grid through memory.  Here the
// whole step — momentum predictor, sea-level predictor, Shapiro filter, state
// commit and (optionally) the diagnostics — is ONE pass: 16 B read (eta, u,
// v, hzero) + 12 B written (eta', u', v') per cell-step, the minimum for the
// state.  h, wet, un, vn and etan live in registers.
//
// Work decomposition:
//  * a warp owns a strip of 128 storage columns (32 lanes x float4) and
//    marches down a segment of rows; lanes 1..30 produce the strip's 120
//    output columns, lanes 0 and 31 are halo lanes that recompute the
//    neighbouring strip's edge so every horizontal neighbour comes from a warp
//    shuffle (the step's dependency cone is 2 cells wide);
//  * per loaded row L the warp computes wet(L), un(L), vn(L-1), the fluxes and
//    etan(L-1), and the Shapiro filter of row L-2, keeping a rolling window of
//    rows in registers, so each input element is loaded once (plus the 4-row
//    overlap between vertically adjacent segments);
//  * every floating-point operation is an explicit round-to-nearest intrinsic
//    (__fadd_rn/__fsub_rn/__fmul_rn: never contracted into an FMA) in the
//    order of DESIGN.md "Oracle step", and every branch of the scheme is a
//    select, so results are bitwise those of the sequential definition.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <type_traits>

#include "sw2d_internal.cuh"

namespace sw2d_dev {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void st4(float* p, float a, float b, float c,
                                    float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

struct Acc {
  double sum_eta;
  double wet;
  float max_eta, neg_min_eta, max_u, max_v;
  int wet_i;   // wet cells counted in the row loop (exact; added to wet before the fold)
  __device__ void init() {
    sum_eta = 0.0;
    wet = 0.0;
    wet_i = 0;
    max_eta = __int_as_float(0xff800000);  // -inf
    neg_min_eta = __int_as_float(0xff800000);
    max_u = 0.0f;
    max_v = 0.0f;
  }
};

__device__ __forceinline__ double shfl_xor_d(double x, int m) {
  return __shfl_xor_sync(kFull, x, m);
}

// Block reduction of Acc -> one partial per CTA, then the last CTA of the
// step (over all launches sharing the counter) folds the partials in a fixed
// order (deterministic) and writes the 7-double record.
template <int LEVEL, int NW>
__device__ void block_reduce_and_finalize(Acc acc, const RedArgs& r) {
  acc.wet += (double)acc.wet_i;
  __shared__ Acc sh[NW];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // sh / last may still be read by a previous call
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    acc.sum_eta += shfl_xor_d(acc.sum_eta, m);
    if (LEVEL >= 2) {
      acc.wet += shfl_xor_d(acc.wet, m);
      acc.max_eta = fmaxf(acc.max_eta, __shfl_xor_sync(kFull, acc.max_eta, m));
      acc.neg_min_eta =
          fmaxf(acc.neg_min_eta, __shfl_xor_sync(kFull, acc.neg_min_eta, m));
      acc.max_u = fmaxf(acc.max_u, __shfl_xor_sync(kFull, acc.max_u, m));
      acc.max_v = fmaxf(acc.max_v, __shfl_xor_sync(kFull, acc.max_v, m));
    }
  }
  if (lane == 0) sh[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = sh[0];
    for (int w = 1; w < NW; ++w) {
      t.sum_eta += sh[w].sum_eta;
      t.wet += sh[w].wet;
      t.max_eta = fmaxf(t.max_eta, sh[w].max_eta);
      t.neg_min_eta = fmaxf(t.neg_min_eta, sh[w].neg_min_eta);
      t.max_u = fmaxf(t.max_u, sh[w].max_u);
      t.max_v = fmaxf(t.max_v, sh[w].max_v);
    }
    RedPartial p;
    p.sum_eta = t.sum_eta;
    p.wet = t.wet;
    p.max_eta = t.max_eta;
    p.neg_min_eta = t.neg_min_eta;
    p.max_u = t.max_u;
    p.max_v = t.max_v;
    r.partials[r.part_base + blockIdx.x] = p;
    __threadfence();
    const unsigned ticket = atomicAdd(r.counter, 1u);
    last = (ticket == (unsigned)(r.expected - 1));
  }
  __syncthreads();
  if (last) {  // block-uniform
    __threadfence();
    // Fixed-order fold: thread t takes slots t, t+32*NW, ... in order, then a
    // fixed tree over threads.
    Acc t;
    t.init();
    for (int i = threadIdx.x; i < r.expected; i += 32 * NW) {
      const volatile RedPartial* p = r.partials + i;
      t.sum_eta += p->sum_eta;
      t.wet += p->wet;
      t.max_eta = fmaxf(t.max_eta, p->max_eta);
      t.neg_min_eta = fmaxf(t.neg_min_eta, p->neg_min_eta);
      t.max_u = fmaxf(t.max_u, p->max_u);
      t.max_v = fmaxf(t.max_v, p->max_v);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      t.sum_eta += shfl_xor_d(t.sum_eta, m);
      t.wet += shfl_xor_d(t.wet, m);
      t.max_eta = fmaxf(t.max_eta, __shfl_xor_sync(kFull, t.max_eta, m));
      t.neg_min_eta = fmaxf(t.neg_min_eta, __shfl_xor_sync(kFull, t.neg_min_eta, m));
      t.max_u = fmaxf(t.max_u, __shfl_xor_sync(kFull, t.max_u, m));
      t.max_v = fmaxf(t.max_v, __shfl_xor_sync(kFull, t.max_v, m));
    }
    __syncthreads();
    if (lane == 0) sh[warp] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      Acc f = sh[0];
      for (int w = 1; w < NW; ++w) {
        f.sum_eta += sh[w].sum_eta;
        f.wet += sh[w].wet;
        f.max_eta = fmaxf(f.max_eta, sh[w].max_eta);
        f.neg_min_eta = fmaxf(f.neg_min_eta, sh[w].neg_min_eta);
        f.max_u = fmaxf(f.max_u, sh[w].max_u);
        f.max_v = fmaxf(f.max_v, sh[w].max_v);
      }
      r.rec[kRecVol] = r.dxdy * (*r.h0sum + f.sum_eta);
      r.rec[kRecSumEta] = f.sum_eta;
      r.rec[kRecWet] = f.wet;
      r.rec[kRecMaxEta] = f.max_eta;
      r.rec[kRecNegMinEta] = f.neg_min_eta;
      r.rec[kRecMaxU] = f.max_u;
      r.rec[kRecMaxV] = f.max_v;
      *r.counter = 0u;  // ready for the next step (stream-ordered)
    }
  }
}

// Deferred form (replayed graphs on small grids): the CTA's partial only; the
// steps' records are folded later by fold_steps, off the launch's critical
// path (no ticket, no last-CTA tail).
template <int LEVEL, int NW>
__device__ void block_reduce_to_partial(Acc acc, RedPartial* dst) {
  acc.wet += (double)acc.wet_i;
  __shared__ Acc sh[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // sh may still be read by a previous call
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    acc.sum_eta += shfl_xor_d(acc.sum_eta, m);
    if (LEVEL >= 2) {
      acc.wet += shfl_xor_d(acc.wet, m);
      acc.max_eta = fmaxf(acc.max_eta, __shfl_xor_sync(kFull, acc.max_eta, m));
      acc.neg_min_eta = fmaxf(acc.neg_min_eta, __shfl_xor_sync(kFull, acc.neg_min_eta, m));
      acc.max_u = fmaxf(acc.max_u, __shfl_xor_sync(kFull, acc.max_u, m));
      acc.max_v = fmaxf(acc.max_v, __shfl_xor_sync(kFull, acc.max_v, m));
    }
  }
  if (lane == 0) sh[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = sh[0];
    for (int w = 1; w < NW; ++w) {
      t.sum_eta += sh[w].sum_eta;
      t.wet += sh[w].wet;
      t.max_eta = fmaxf(t.max_eta, sh[w].max_eta);
      t.neg_min_eta = fmaxf(t.neg_min_eta, sh[w].neg_min_eta);
      t.max_u = fmaxf(t.max_u, sh[w].max_u);
      t.max_v = fmaxf(t.max_v, sh[w].max_v);
    }
    RedPartial p;
    p.sum_eta = t.sum_eta;
    p.wet = t.wet;
    p.max_eta = t.max_eta;
    p.neg_min_eta = t.neg_min_eta;
    p.max_u = t.max_u;
    p.max_v = t.max_v;
    dst[blockIdx.x] = p;
  }
}

// CTA s folds step s's `blocks` partials (fixed order) into its record, history
// slot (*dstep + s) % len.  The caller sets *dstep before the steps run.
constexpr int kFoldThreads = 128;
__global__ void __launch_bounds__(kFoldThreads)
    fold_steps(const RedPartial* partials, int blocks, double* hist, int len,
               const unsigned long long* dstep, const double* h0sum, double dxdy) {
  __shared__ Acc sh[kFoldThreads / 32];
  // a step whose slot a later step of this batch overwrites is not folded
  // (the CTAs run in any order)
  if ((int)blockIdx.x + len < (int)gridDim.x) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const RedPartial* p0 = partials + (size_t)blockIdx.x * blocks;
  Acc t;
  t.init();
  for (int i = threadIdx.x; i < blocks; i += kFoldThreads) {
    const RedPartial& p = p0[i];
    t.sum_eta += p.sum_eta;
    t.wet += p.wet;
    t.max_eta = fmaxf(t.max_eta, p.max_eta);
    t.neg_min_eta = fmaxf(t.neg_min_eta, p.neg_min_eta);
    t.max_u = fmaxf(t.max_u, p.max_u);
    t.max_v = fmaxf(t.max_v, p.max_v);
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    t.sum_eta += shfl_xor_d(t.sum_eta, m);
    t.wet += shfl_xor_d(t.wet, m);
    t.max_eta = fmaxf(t.max_eta, __shfl_xor_sync(kFull, t.max_eta, m));
    t.neg_min_eta = fmaxf(t.neg_min_eta, __shfl_xor_sync(kFull, t.neg_min_eta, m));
    t.max_u = fmaxf(t.max_u, __shfl_xor_sync(kFull, t.max_u, m));
    t.max_v = fmaxf(t.max_v, __shfl_xor_sync(kFull, t.max_v, m));
  }
  if (lane == 0) sh[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc f = sh[0];
    for (int w = 1; w < kFoldThreads / 32; ++w) {
      f.sum_eta += sh[w].sum_eta;
      f.wet += sh[w].wet;
      f.max_eta = fmaxf(f.max_eta, sh[w].max_eta);
      f.neg_min_eta = fmaxf(f.neg_min_eta, sh[w].neg_min_eta);
      f.max_u = fmaxf(f.max_u, sh[w].max_u);
      f.max_v = fmaxf(f.max_v, sh[w].max_v);
    }
    double* rec = hist + (size_t)((*dstep + blockIdx.x) % (unsigned long long)len) * kRecN;
    rec[kRecVol] = dxdy * (*h0sum + f.sum_eta);
    rec[kRecSumEta] = f.sum_eta;
    rec[kRecWet] = f.wet;
    rec[kRecMaxEta] = f.max_eta;
    rec[kRecNegMinEta] = f.neg_min_eta;
    rec[kRecMaxU] = f.max_u;
    rec[kRecMaxV] = f.max_v;
  }
}

// ---------------------------------------------------------------------------
// The fused step.
//
// Per lane: 4 consecutive columns k0..k0+3 (one float4 of each field).  Wet
// flags travel as bit masks (bit c = column k0+c) so one shuffle moves a
// lane's four flags.  The Shapiro filter of row r is split in two halves:
// when etan(r) is known (iteration r+1) the part that needs rows r-1 and r
// is formed, A = t1 + t2 and sS = sel(wS, etan(r-1)); when etan(r+1) is known
// (iteration r+2) the north term completes E'(r) = A + q*(sel(wN, etan(r+1))
// + sS) — the same operations, in the same order, as the sequential scheme
// (fadd is commutative), so the window is two rows deep everywhere.
// ---------------------------------------------------------------------------

// rolling window carried from row L-1 into row L (C columns per lane)
template <int C>
struct WinT {
  float e[C];      // eta(L-1)
  float h[C];      // h(L-1)
  float un[C];     // un(L-1)
  float v[C];      // V(L-1), old
  float fy[C];     // y-flux through the north face of row L-2
  float A[C];      // Shapiro of row L-2: t1 + t2
  float sS[C];     // Shapiro of row L-2: sel(wS, etan(L-3))
  float etC[C];    // etan(L-2)
  float h0P[C];    // hzero(L-1)   (diagnostics level 2)
  float h0PP[C];   // hzero(L-2)   (diagnostics level 2)
  float w1[C];     // wet flags (1.0 / 0.0) of row L-1
  float w2[C];     // wet flags of row L-2
  float w1W, w1E;  // wet flags of row L-1 at columns k0-1 and k0+C
  float hR;        // h(L-1, k0+C)
  __device__ void zero() {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      e[c] = h[c] = un[c] = v[c] = fy[c] = 0.0f;
      A[c] = sS[c] = etC[c] = h0P[c] = h0PP[c] = 0.0f;
      w1[c] = w2[c] = 0.0f;
    }
    w1W = w1E = 0.0f;
    hR = 0.0f;
  }
};
using Win = WinT<4>;

struct Ctx {
  float cgx, cgy, cx, cy, q, hmin;
  float nz;          // -0.0f, opaque to ptxas (Coef::nz; see vmul2)
  unsigned colmask;  // columns 1..nx of this lane's four
  unsigned umask;    // columns 1..nx-1 (faces that are not the east wall)
  float cmf[4];      // colmask as 1.0 / 0.0 per column
  float umf[4];      // umask as 1.0 / 0.0 per column
  float cgxc[4];     // cgx on faces that are not walls (umask), 0 on wall / outside faces
  float hminc[4];    // hmin on columns 1..nx, +inf outside (those cells are dry)
  int ny, ra, rb;    // global rows (1-based): grid rows, this segment's output rows
  bool out_lane;
  int col;                 // storage column of this lane's element 0 (REMOTE only)
  long long pitch;         // (REMOTE only)
  const Remote* rem;       // (REMOTE only)
#ifdef SW2D_DEBUG_BOUNDS
  const float* dU;         // field bases and size for the bounds checks
  const float* dV;
  const float* dE;
  long long nelem;
#endif
};

// P2P halo: mirror an output row into the neighbour slabs that need it
// (the CTA kernel, 4 columns per lane)
__device__ __forceinline__ void remote_store(const Ctx& x, int field, int row, float a, float b,
                                             float c, float d) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const Remote& m = x.rem[r];
    if (row >= m.lo && row <= m.hi) {
      float* base = field == 0 ? m.En : (field == 1 ? m.Un : m.Vn);
      SW2D_CHECK(row - m.jbase >= 0 && (row - m.jbase) * x.pitch + x.col + 4 <= m.nelem);
      st4(base + (long long)(row - m.jbase) * x.pitch + x.col, a, b, c, d);
    }
  }
}

__device__ __forceinline__ bool bit(unsigned m, int i) { return (m >> i) & 1u; }

// rows r with lo <= r <= hi (requires lo <= hi)
__device__ __forceinline__ bool in_rows(int r, int lo, int hi) {
  return (unsigned)(r - lo) <= (unsigned)(hi - lo);
}

// Upwind flux s > 0 ? s*hL : (s < 0 ? s*hR : 0) is computed as
// s * (s > 0 ? hL : hR): equal in value for finite depths (s = 0 gives a zero
// either way).
// Wet/dry face rule (reading R4): the face between a cell with wet flag wc
// and its east/north neighbour (wn) carries flow iff
// wc ? (wn || d > 0) : (wn && d < 0); a blocked face gets 0.  The row step
// evaluates it as exact arithmetic, wc*wn + (wc - wn)*d > 0 (R26,
// SW2D_FACE_ARITH); the A/B form below is the predicate program the rule is
// (two compares with a predicate combine, one 3-input predicate op, one
// select; ptxas otherwise if-converts the C++ into a chain of selects).
#ifndef SW2D_INTERIOR_SELECT2
#define SW2D_INTERIOR_SELECT2 1  // the select form for all seven diagnostics too (A/B: 0)
#endif
#ifndef SW2D_INTERIOR_SELECT
#define SW2D_INTERIOR_SELECT 1  // interior commits without a lane branch (A/B: 0)
#endif
#ifndef SW2D_FACE_ARITH
#define SW2D_FACE_ARITH 1   // 0: the predicate program below (A/B)
#endif
#if !SW2D_FACE_ARITH
__device__ __forceinline__ float face_sel(float wc, float wn, float d, float s) {
  float r;
  asm("{\n\t.reg .pred pc, pn, pa, pb;\n\t"
      "setp.ne.f32 pc, %1, 0f00000000;\n\t"
      "setp.ne.f32 pn, %2, 0f00000000;\n\t"
      "setp.gt.or.f32 pa, %3, 0f00000000, pn;\n\t"
      "setp.lt.and.f32 pb, %3, 0f00000000, pn;\n\t"
      "and.pred pa, pa, pc;\n\t"
      "or.pred pa, pa, pb;\n\t"
      "selp.f32 %0, %4, 0f00000000, pa;\n\t}"
      : "=f"(r)
      : "f"(wc), "f"(wn), "f"(d), "f"(s));
  return r;
}
#endif


// Column-parallel FP32 arithmetic on C-column arrays.  sm_100a issues the
// packed add/sub/mul.rn.f32x2 (SASS FADD2 / FMUL2) at the scalar instruction
// rate (tools/f32x2_probe.cu: 3.7 warp-instructions/clk/SM either way), so a
// pair of columns costs one issue slot.  Each element is rounded to nearest
// exactly like __fadd_rn / __fsub_rn / __fmul_rn (no FTZ): bitwise the same
// results.  SW2D_F32X2=0 builds the scalar form (A/B).
//
// ptxas (CUDA 12.9) contracts a packed mul.rn.f32x2 feeding a packed add or
// subtract into FFMA2 even under --fmad=false (one rounding instead of two;
// also when the add is written as an FMA with a unit multiplier).  A scalar
// FMUL feeding a packed add, or a packed FMUL feeding a scalar add, is left
// alone, so only the adds and subtracts are packed (17 of the 31 FP32
// operations per cell and step); the products stay scalar (vmul).
#ifndef SW2D_F32X2
#define SW2D_F32X2 1
#endif
// the step kernels pack only in the instantiations with diagnostics RED >=
// SW2D_F32X2_MIN_RED (without diagnostics the packed form
// measured slower on C3 and p2000)
#ifndef SW2D_F32X2_MIN_RED
#define SW2D_F32X2_MIN_RED 0
#endif
#ifndef SW2D_F32X2_SHIFTED
#define SW2D_F32X2_SHIFTED 0
#endif
#define SW2D_PAIR_ASM(PTXOP)                                                                 \
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t" PTXOP      \
      " rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"                                                 \
      : "=f"(d0), "=f"(d1)                                                                   \
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1))
__device__ __forceinline__ void vadd2(float& d0, float& d1, float a0, float a1, float b0,
                                      float b1) {
  SW2D_PAIR_ASM("add.rn.f32x2");
}
__device__ __forceinline__ void vsub2(float& d0, float& d1, float a0, float a1, float b0,
                                      float b1) {
  SW2D_PAIR_ASM("sub.rn.f32x2");
}
// Packed products as fma.rn.f32x2 with a -0 addend: a*b + (-0) rounds once
// exactly like mul.rn (the sign of a zero product included).  The -0 comes
// from a kernel parameter (Coef::nz) so ptxas cannot fold the FMA back into a
// multiply — it contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under
// --fmad=false (one rounding instead of two), and it does the same to an FMA
// whose addend it knows is -0.  An FMA is never fused with the add that
// consumes it.  SW2D_PACKED_MUL=0 keeps the products scalar.
#ifndef SW2D_PACKED_MUL
#define SW2D_PACKED_MUL 1
#endif
__device__ __forceinline__ void vmul2(float& d0, float& d1, float a0, float a1, float b0,
                                      float b1, float nz) {
#if SW2D_PACKED_MUL && SW2D_F32X2
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%6};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(nz));
#else
  d0 = __fmul_rn(a0, b0);
  d1 = __fmul_rn(a1, b1);
#endif
}
template <int C, bool P = true>
__device__ __forceinline__ void vmul(float (&d)[C], const float (&a)[C], const float (&b)[C],
                                     float nz) {
#pragma unroll
  for (int c = 0; c < C; c += ((SW2D_F32X2 && P) ? 2 : 1)) {
    if (SW2D_F32X2 && P && c + 1 < C)
      vmul2(d[c], d[c + 1], a[c], a[c + 1], b[c], b[c + 1], nz);
    else
      d[c] = __fmul_rn(a[c], b[c]);
  }
}
template <int C, bool P = true>
__device__ __forceinline__ void vmul(float (&d)[C], const float a, const float (&b)[C],
                                     float nz) {
  float aa[C];
#pragma unroll
  for (int c = 0; c < C; ++c) aa[c] = a;
  vmul<C, P>(d, aa, b, nz);
}
#undef SW2D_PAIR_ASM

// sel(w, x) + y with a wet flag w in {0, 1}: the product w * x is exact (x or
// a zero), so the fused multiply-add rounds once exactly where the oracle's
// select-then-add rounds once: bitwise the same value (R24).  Only
// these flag products are ever fused; SW2D_EXACT_FMA=0 builds mul + add.
#ifndef SW2D_EXACT_FMA
#define SW2D_EXACT_FMA 1
#endif
__device__ __forceinline__ float selfma(float w, float x, float y) {
#if SW2D_EXACT_FMA
  return __fmaf_rn(w, x, y);
#else
  return __fadd_rn(__fmul_rn(w, x), y);
#endif
}
// packed pair form (fma.rn.f32x2 -> FFMA2), same exactness argument per element
__device__ __forceinline__ void selfma2(float& d0, float& d1, float w0, float w1, float x0,
                                        float x1, float y0, float y1) {
#if SW2D_EXACT_FMA && SW2D_F32X2
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(w0), "f"(w1), "f"(x0), "f"(x1), "f"(y0), "f"(y1));
#else
  d0 = selfma(w0, x0, y0);
  d1 = selfma(w1, x1, y1);
#endif
}
template <int C, bool P = true>
__device__ __forceinline__ void vselfma(float (&d)[C], const float (&w)[C], const float (&x)[C],
                                        const float (&y)[C]) {
#pragma unroll
  for (int c = 0; c < C; c += (P ? 2 : 1)) {
    if (P && c + 1 < C)
      selfma2(d[c], d[c + 1], w[c], w[c + 1], x[c], x[c + 1], y[c], y[c + 1]);
    else
      d[c] = selfma(w[c], x[c], y[c]);
  }
}
#define SW2D_PAIR_OP(NAME, SCALAR)                                                          \
  template <int C, bool P = true>                                                            \
  __device__ __forceinline__ void NAME(float (&d)[C], const float (&a)[C],                   \
                                       const float (&b)[C]) {                                \
    _Pragma("unroll") for (int c = 0; c < C; c += ((SW2D_F32X2 && P) ? 2 : 1)) {             \
      if (SW2D_F32X2 && P && c + 1 < C) {                                                    \
        NAME##2(d[c], d[c + 1], a[c], a[c + 1], b[c], b[c + 1]);                             \
      } else {                                                                               \
        d[c] = SCALAR(a[c], b[c]);                                                           \
      }                                                                                      \
    }                                                                                        \
  }                                                                                          \
  template <int C, bool P = true>                                                            \
  __device__ __forceinline__ void NAME(float (&d)[C], const float a, const float (&b)[C]) {  \
    float aa[C];                                                                             \
    _Pragma("unroll") for (int c = 0; c < C; ++c) aa[c] = a;                                 \
    NAME<C, P>(d, aa, b);                                                                    \
  }
SW2D_PAIR_OP(vadd, __fadd_rn)
SW2D_PAIR_OP(vsub, __fsub_rn)
#undef SW2D_PAIR_OP

// One loaded row L: reads the window `w` (rows L-1, L-2), writes `o`.
// C consecutive floats of a row (C = 4: float4, C = 2: float2)
template <int C>
__device__ __forceinline__ void stC(float* p, const float (&v)[C]) {
  if constexpr (C == 4) {
    st4(p, v[0], v[1], v[2], v[3]);
  } else if constexpr (C == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) p[c] = v[c];
  }
}

// the new-state values one row_stepC produces: u'(L), v'(L-1), eta'(L-2)
template <int C>
struct RowOut {
  float un[C], vn[C], En[C];
};

// STORE: write the outputs of this segment's rows to global memory; else
// return them in `out` (the first step of a two-step pass keeps its state in
// registers).  The diagnostics of the segment's rows are accumulated either way.
// EDGE = false: the caller guarantees that rows L-2 .. L are output rows of
// the segment inside 1..ny (and L-1 is not a wall row): no row tests.
template <int RED, bool REMOTE, int C, bool STORE = true, bool EDGE = true>
__device__ __forceinline__ void row_stepC(const WinT<C>& w, WinT<C>& o, const float (&eL)[C],
                                         const float (&h0L)[C], const float (&uL)[C],
                                         const float (&vL)[C], const int L, const Ctx& x,
                                         Acc& acc, float* pU, float* pV, float* pE,
                                         RowOut<C>* out = nullptr) {
  // Wet flags are carried as 1.0f / 0.0f: a select sel(w, x) = w ? x : 0 is
  // then the product w * x, equal in value for finite x (x * 0 is a zero of
  // either sign; signed zeros never change a later non-zero value or a
  // comparison here), and s = wE + wW + wN + wS is the exact integer count.

  // a1: h and wet flags of row L (rows outside 1..ny and columns outside
  // 1..nx are dry)
  constexpr bool kPack = RED >= SW2D_F32X2_MIN_RED;
  // the pairs with a neighbour-shifted operand (they need IMAD.MOV to align)
  constexpr bool kPackS = kPack && SW2D_F32X2_SHIFTED;
  const bool rowok = !EDGE || in_rows(L, 1, x.ny);
  float hL[C], wL[C];
  vadd<C, kPack>(hL, h0L, eL);
#pragma unroll
  for (int c = 0; c < C; ++c)   // hminc: hmin on columns 1..nx, +inf outside (never <= finite h)
    wL[c] = (rowok && !(hL[c] < x.hminc[c])) ? 1.0f : 0.0f;
  const float eR = __shfl_down_sync(kFull, eL[0], 1);
  const float hR = __shfl_down_sync(kFull, hL[0], 1);
  const float wR = __shfl_down_sync(kFull, wL[0], 1);
  const float wLf = __shfl_up_sync(kFull, wL[C - 1], 1);

  // a2: un(L) on the east faces of row L; vn(L-1) on the north faces of L-1.
  // East/west wall faces (and faces outside the grid) must come out 0: their
  // pressure-gradient coefficient is taken as 0 (cgxc, per column), so the
  // face rule reduces to wc && wn, and such a face always has a dry cell (the
  // halo) on one side: blocked -> 0, with no per-cell mask multiply.  Every
  // other face keeps cgx and the arithmetic of §4.  (The same trick per row
  // for the north/south walls made ptxas emit more selects: the row select
  // stays.)
  const bool vrow = !EDGE || ((L - 1 >= 1) && (L - 1 < x.ny));  // not the north / south wall
  // (the arithmetic below is column-parallel: vadd / vsub / vmul, same
  // operations and operand order as the scalar form)
  float en[C], du[C], dv[C], su[C], sv[C], un[C], vn[C];
#pragma unroll
  for (int c = 0; c < C; ++c) en[c] = (c < C - 1) ? eL[c + 1] : eR;
  vsub<C, kPackS>(du, en, eL);
  float cg[C];
#pragma unroll
  for (int c = 0; c < C; ++c) cg[c] = x.cgxc[c];
  vmul<C, kPack>(du, cg, du, x.nz);
  vsub<C, kPack>(dv, eL, w.e);
#if SW2D_FACE_ARITH
  // north / south wall rows: coefficient 0, so dv = 0 and the face rule
  // below blocks the face (one side is outside the grid, dry)
  vmul<C, kPack>(dv, vrow ? x.cgy : 0.0f, dv, x.nz);
#else
  vmul<C, kPack>(dv, x.cgy, dv, x.nz);
#endif
  vadd<C, kPack>(su, uL, du);
  vadd<C, kPack>(sv, w.v, dv);
#if SW2D_FACE_ARITH
  // The face rule as exact arithmetic (R26): with wet flags wc, wn in {0, 1},
  // f = wc*wn + (wc - wn)*d is exactly 1 (both wet), d (only wc), -d (only wn)
  // or a zero (neither), so the face carries flow iff f > 0 — the rule of
  // R4 — and every operation here is exact (no rounding): packed pairs, one
  // compare and one select per face instead of a predicate program.
  float wnE[C], fu[C], fv[C], tq[C];
#pragma unroll
  for (int c = 0; c < C; ++c) wnE[c] = (c < C - 1) ? wL[c + 1] : wR;
  vsub<C, kPackS>(tq, wL, wnE);
  vmul<C, kPack>(tq, tq, du, x.nz);
  vselfma<C, kPackS>(fu, wL, wnE, tq);
  vsub<C, kPack>(tq, w.w1, wL);
  vmul<C, kPack>(tq, tq, dv, x.nz);
  vselfma<C, kPack>(fv, w.w1, wL, tq);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    un[c] = fu[c] > 0.0f ? su[c] : 0.0f;
    vn[c] = fv[c] > 0.0f ? sv[c] : 0.0f;
  }
#else
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float wn = (c < C - 1) ? wL[c + 1] : wR;
    un[c] = face_sel(wL[c], wn, du[c], su[c]);
    vn[c] = vrow ? face_sel(w.w1[c], wL[c], dv[c], sv[c]) : 0.0f;
  }
#endif

  // a3: fluxes of row L-1 and etan(L-1)
  float hx[C], hy[C], fx[C], fy[C], et[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    hx[c] = w.un[c] > 0.0f ? w.h[c] : ((c < C - 1) ? w.h[c + 1] : w.hR);
    hy[c] = vn[c] > 0.0f ? w.h[c] : hL[c];
  }
  vmul<C, kPack>(fx, w.un, hx, x.nz);
  vmul<C, kPack>(fy, vn, hy, x.nz);
  const float fxw = __shfl_up_sync(kFull, fx[C - 1], 1);
  float fw[C], t[C], t2[C];
#pragma unroll
  for (int c = 0; c < C; ++c) fw[c] = (c > 0) ? fx[c - 1] : fxw;
  vsub<C, kPackS>(t, fx, fw);
  vmul<C, kPack>(t, x.cx, t, x.nz);
  vsub<C, kPack>(t, w.e, t);
  vsub<C, kPack>(t2, fy, w.fy);
  vmul<C, kPack>(t2, x.cy, t2, x.nz);
  vsub<C, kPack>(et, t, t2);

  // a4 (second half): E'(L-2) = wet ? A + q*(sel(wN, etan(L-1)) + sS) : etan(L-2)
  float En[C], t3[C];
  vselfma<C, kPack>(t3, w.w1, et, w.sS);   // sel(wN, etan(L-1)) + sS
  vmul<C, kPack>(t3, x.q, t3, x.nz);
  vadd<C, kPack>(t3, w.A, t3);
#pragma unroll
  for (int c = 0; c < C; ++c) En[c] = (w.w2[c] != 0.0f) ? t3[c] : w.etC[c];

  // a4 (first half) for row L-1: s, t1, t2, sS
  const float etW = __shfl_up_sync(kFull, et[C - 1], 1);
  const float etE = __shfl_down_sync(kFull, et[0], 1);
  float wE[C], wW[C], eE[C], eW[C], sc[C], t1[C], xE[C], xW[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    wE[c] = (c < C - 1) ? w.w1[c + 1] : w.w1E;
    wW[c] = (c > 0) ? w.w1[c - 1] : w.w1W;
    eE[c] = (c < C - 1) ? et[c + 1] : etE;
    eW[c] = (c > 0) ? et[c - 1] : etW;
  }
  vadd<C, kPackS>(sc, wE, wW);
  vadd<C, kPack>(sc, sc, wL);
  vadd<C, kPack>(sc, sc, w.w2);
  vmul<C, kPack>(sc, x.q, sc, x.nz);
  vsub<C, kPack>(sc, 1.0f, sc);
  vmul<C, kPack>(t1, sc, et, x.nz);
  vmul<C, kPack>(xW, wW, eW, x.nz);
  vselfma<C, kPackS>(xE, wE, eE, xW);      // sel(wE, etanE) + sel(wW, etanW)
  vmul<C, kPack>(xE, x.q, xE, x.nz);
  vadd<C, kPack>(o.A, t1, xE);
  vmul<C, kPack>(o.sS, w.w2, w.etC, x.nz);

  // a5: commit (lanes 1..30, rows of this segment)
#if SW2D_INTERIOR_SELECT
  if constexpr (!EDGE && C == 4 && (RED <= 1 || SW2D_INTERIOR_SELECT2)) {
    // interior rows: the stores predicated on the lane, the volume sum
    // folded through a select (a halo lane adds +0): no divergent branch in
    // the loop (C5 with VOLUME per step +5%; with all seven diagnostics the
    // selects cost as much as the branch saves and spill the P2P variant, so
    // RED = 2 keeps the branch)
    if (x.out_lane) {
      if constexpr (STORE) {
        stC<C>(pU, un);
        stC<C>(pV, vn);
        stC<C>(pE, En);
      }
      if constexpr (REMOTE) {
        remote_store(x, 1, L, un[0], un[1], un[2], un[3]);
        remote_store(x, 2, L - 1, vn[0], vn[1], vn[2], vn[3]);
        remote_store(x, 0, L - 2, En[0], En[1], En[2], En[3]);
      }
    }
    if (RED >= 1) {
      const float quad = __fadd_rn(__fadd_rn(En[0], En[1]), __fadd_rn(En[2], En[3]));
      acc.sum_eta += (double)(x.out_lane ? quad : 0.0f);
    }
    if (RED >= 2) {   // (neutral values on halo lanes and outside columns)
      const float ninf = __int_as_float(0xff800000);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const bool ok = x.out_lane && bit(x.colmask, c);
        acc.max_u = fmaxf(acc.max_u, x.out_lane ? fabsf(un[c]) : 0.0f);
        acc.max_v = fmaxf(acc.max_v, x.out_lane ? fabsf(vn[c]) : 0.0f);
        acc.max_eta = fmaxf(acc.max_eta, ok ? En[c] : ninf);
        acc.neg_min_eta = fmaxf(acc.neg_min_eta, ok ? -En[c] : ninf);
        acc.wet_i += (ok && !(__fadd_rn(w.h0PP[c], En[c]) < x.hmin)) ? 1 : 0;
      }
    }
  } else
#endif
  if (x.out_lane) {
    if (!EDGE || in_rows(L, x.ra, x.rb)) {
#ifdef SW2D_DEBUG_BOUNDS
      if constexpr (STORE) SW2D_CHECK(pU >= x.dU && pU + C <= x.dU + x.nelem);
#endif
      if constexpr (STORE) stC<C>(pU, un);
      if constexpr (REMOTE && C == 4) remote_store(x, 1, L, un[0], un[1], un[2], un[3]);
      if (RED >= 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc.max_u = fmaxf(acc.max_u, fabsf(un[c]));
      }
    }
    if (!EDGE || in_rows(L - 1, x.ra, x.rb)) {
#ifdef SW2D_DEBUG_BOUNDS
      if constexpr (STORE) SW2D_CHECK(pV >= x.dV && pV + C <= x.dV + x.nelem);
#endif
      if constexpr (STORE) stC<C>(pV, vn);
      if constexpr (REMOTE && C == 4) remote_store(x, 2, L - 1, vn[0], vn[1], vn[2], vn[3]);
      if (RED >= 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc.max_v = fmaxf(acc.max_v, fabsf(vn[c]));
      }
    }
    if (!EDGE || in_rows(L - 2, x.ra, x.rb)) {
#ifdef SW2D_DEBUG_BOUNDS
      if constexpr (STORE) SW2D_CHECK(pE >= x.dE && pE + C <= x.dE + x.nelem);
#endif
      if constexpr (STORE) stC<C>(pE, En);
      if constexpr (REMOTE && C == 4) remote_store(x, 0, L - 2, En[0], En[1], En[2], En[3]);
      if (RED >= 1) {
        // columns outside 1..nx hold exactly 0 (their etan is 0)
        if constexpr (C == 4) {
          // the quad's sum in fp32 (relative error <= 2^-23 of the quad), one
          // conversion and one fp64 add: -1 F2F/DADD pair per cell, +3.8% on
          // C5; the sums stay far inside the 1e-5 tolerance (R16)
          acc.sum_eta += (double)__fadd_rn(__fadd_rn(En[0], En[1]), __fadd_rn(En[2], En[3]));
        } else if constexpr (C == 2) {
          acc.sum_eta += (double)__fadd_rn(En[0], En[1]);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) acc.sum_eta += (double)En[c];
        }
      }
      if (RED >= 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if (bit(x.colmask, c)) {
            acc.max_eta = fmaxf(acc.max_eta, En[c]);
            acc.neg_min_eta = fmaxf(acc.neg_min_eta, -En[c]);
            acc.wet_i += (__fadd_rn(w.h0PP[c], En[c]) < x.hmin) ? 0 : 1;
          }
        }
      }
    }
  }

  if constexpr (!STORE) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      out->un[c] = un[c];
      out->vn[c] = vn[c];
      out->En[c] = En[c];
    }
  }

  // the window for row L+1
#pragma unroll
  for (int c = 0; c < C; ++c) {
    o.e[c] = eL[c];
    o.h[c] = hL[c];
    o.un[c] = un[c];
    o.v[c] = vL[c];
    o.fy[c] = fy[c];
    o.etC[c] = et[c];
    o.w1[c] = wL[c];
    o.w2[c] = w.w1[c];
    if (RED >= 2) {
      o.h0PP[c] = w.h0P[c];
      o.h0P[c] = h0L[c];
    }
  }
  o.w1W = wLf;
  o.w1E = wR;
  o.hR = hR;
}

// float4 adapter (the TMA kernels: 4 columns per lane)
template <int RED, bool REMOTE>
__device__ __forceinline__ void row_step(const Win& w, Win& o, const float4 E4, const float4 H4,
                                         const float4 U4, const float4 V4, const int L,
                                         const Ctx& x, Acc& acc, float* pU, float* pV,
                                         float* pE) {
  const float eL[4] = {E4.x, E4.y, E4.z, E4.w};
  const float h0L[4] = {H4.x, H4.y, H4.z, H4.w};
  const float uL[4] = {U4.x, U4.y, U4.z, U4.w};
  const float vL[4] = {V4.x, V4.y, V4.z, V4.w};
  row_stepC<RED, REMOTE, 4>(w, o, eL, h0L, uL, vL, L, x, acc, pU, pV, pE);
}

// --- TMA bulk copies and mbarriers (the CTA row rings below) ----------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const float* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --- CTA-shared row ring with a producer warp (kind 1, the default) --------
// A CTA owns kCtaStrips adjacent warp strips of one row segment.  Warp
// kCtaStrips is the producer: it streams one contiguous window of
// 120 * (active strips) + 8 columns per field and row (the strips' 8-column
// halo overlaps are fetched once per CTA) through a ring of kCtaStages
// stages with cp.async.bulk (TMA), one full/empty mbarrier pair per stage.
// The compute warps wait on `full`, copy their float4 of each field out of
// the stage and release it on `empty` (one arrival per compute warp).
constexpr int kCtaStrips = 8;
#ifndef SW2D_CTA_EXIT_BARRIER
#define SW2D_CTA_EXIT_BARRIER 1
#endif
constexpr bool kCtaBarrierAtExit = SW2D_CTA_EXIT_BARRIER;
#ifndef SW2D_CTA_STAGES
#define SW2D_CTA_STAGES 6
#endif
constexpr int kCtaStages = SW2D_CTA_STAGES;   // ring rows of the CTA kernels
constexpr int kCtaWinBytes = (kCtaStrips * kColsPerStrip + 8) * 4;   // one field, one row
constexpr int kCtaStageBytes = 4 * kCtaWinBytes;
constexpr int kCtaThreads = 32 * (kCtaStrips + 1);
constexpr int kCtaSmem = kCtaStages * kCtaStageBytes + 2 * 8 * kCtaStages;

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int RED, bool REMOTE>
__global__ void __launch_bounds__(kCtaThreads, 1)
    sw2d_step_cta(const StepArgs a) {
  extern __shared__ __align__(128) unsigned char dsm[];
  unsigned char* ring = dsm;
  const uint32_t sring = smem_u32(ring);
  const uint32_t sfull = sring + kCtaStages * kCtaStageBytes;
  const uint32_t sempty = sfull + 8 * kCtaStages;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // the strips are spread evenly over the ncc CTA columns (7 or 8 each)
  const int ncc = (a.nstrips + kCtaStrips - 1) / kCtaStrips;
  const int cc = blockIdx.x % ncc;
  const int seg = blockIdx.x / ncc;
  const int strip0 = (cc * a.nstrips) / ncc;
  const int nact = ((cc + 1) * a.nstrips) / ncc - strip0;   // active compute warps

  Acc acc;
  acc.init();

  const int ra = (int)a.row_lo + seg * a.rows_per_seg;
  const int rb = min((int)a.row_hi, ra + a.rows_per_seg - 1);
  const int first = ra - 2;        // first loaded row
  const int n = rb + 2 - first + 1; // rows streamed
  const long long pitch = a.s.pitch;
  const long long off0 =
      (long long)(first - (int)a.s.jbase) * pitch + strip0 * kColsPerStrip + kStripBase;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < kCtaStages; ++st) {
      mbar_init(sfull + 8 * st, 1);
      mbar_init(sempty + 8 * st, nact);
    }
    fence_proxy_async();
  }
  __syncthreads();

  if (warp == kCtaStrips) {
    // producer warp: one elected lane streams the rows
    if (lane == 0) {
      const uint32_t wb = (uint32_t)(nact * kColsPerStrip + 8) * 4u;
      for (int r = 0; r < n; ++r) {
        const int st = r % kCtaStages;
        if (r >= kCtaStages) {
          const uint32_t ph = (uint32_t)(r / kCtaStages - 1) & 1u;
          while (!mbar_try_wait(sempty + 8 * st, ph)) {
          }
        }
        const long long o = off0 + (long long)r * pitch;
        SW2D_CHECK(o >= 0 && o + wb / 4 <= a.s.nelem);
        const uint32_t d = sring + st * kCtaStageBytes, b = sfull + 8 * st;
        mbar_expect_tx(b, 4u * wb);
        bulk_g2s(d, a.s.E + o, wb, b);
        bulk_g2s(d + kCtaWinBytes, a.s.H0 + o, wb, b);
        bulk_g2s(d + 2 * kCtaWinBytes, a.s.U + o, wb, b);
        bulk_g2s(d + 3 * kCtaWinBytes, a.s.V + o, wb, b);
      }
    }
  } else if (warp < nact) {
    Ctx x;
    x.ra = ra;
    x.rb = rb;
    const int c0 = (strip0 + warp) * kColsPerStrip + kStripBase + lane * 4;
    const int k0 = c0 - kColOff;
    x.colmask = 0;
    x.umask = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      x.colmask |= (k0 + c >= 1 && k0 + c <= a.nx) ? (1u << c) : 0u;
      x.umask |= (k0 + c >= 1 && k0 + c <= a.nx - 1) ? (1u << c) : 0u;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      x.cmf[c] = (x.colmask >> c) & 1u ? 1.0f : 0.0f;
      x.umf[c] = (x.umask >> c) & 1u ? 1.0f : 0.0f;
    }
    x.cgx = a.c.cgx; x.cgy = a.c.cgy; x.cx = a.c.cx; x.cy = a.c.cy;
    for (int c = 0; c < 4; ++c) x.cgxc[c] = x.umf[c] != 0.0f ? x.cgx : 0.0f;
    for (int c = 0; c < 4; ++c) x.hminc[c] = x.cmf[c] != 0.0f ? a.c.hmin : __int_as_float(0x7f800000);
    x.q = a.c.q; x.hmin = a.c.hmin; x.nz = a.c.nz;
    x.ny = (int)a.ny;
    x.out_lane = (lane >= 1) && (lane <= kOutLanes);
#ifdef SW2D_DEBUG_BOUNDS
    x.dU = a.s.Un;
    x.dV = a.s.Vn;
    x.dE = a.s.En;
    x.nelem = a.s.nelem;
#endif
    x.col = c0;
    x.pitch = pitch;
    x.rem = a.rem;

    Win wa, wb;
    wa.zero();

    float* __restrict__ En = a.s.En;
    float* __restrict__ Un = a.s.Un;
    float* __restrict__ Vn = a.s.Vn;
    const long long lo = off0 + warp * kColsPerStrip + lane * 4;
    const int sl = (warp * kColsPerStrip + lane * 4) * 4;

    auto fetch = [&](int i, float4& E4, float4& H4, float4& U4, float4& V4) {
      const int st = i % kCtaStages;
      const uint32_t ph = (uint32_t)(i / kCtaStages) & 1u;
      while (!mbar_try_wait(sfull + 8 * st, ph)) {
      }
      const unsigned char* base = ring + st * kCtaStageBytes + sl;
      E4 = *reinterpret_cast<const float4*>(base);
      H4 = *reinterpret_cast<const float4*>(base + kCtaWinBytes);
      U4 = *reinterpret_cast<const float4*>(base + 2 * kCtaWinBytes);
      V4 = *reinterpret_cast<const float4*>(base + 3 * kCtaWinBytes);
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + 8 * st);
    };

    int i = 0;
    for (; i + 1 < n; i += 2) {
      float4 E4, H4, U4, V4;
      const long long o = lo + (long long)i * pitch;
      fetch(i, E4, H4, U4, V4);
      row_step<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc, Un + o, Vn + o - pitch,
                    En + o - 2 * pitch);
      fetch(i + 1, E4, H4, U4, V4);
      row_step<RED, REMOTE>(wb, wa, E4, H4, U4, V4, first + i + 1, x, acc, Un + o + pitch, Vn + o,
                    En + o - pitch);
    }
    if (i < n) {
      float4 E4, H4, U4, V4;
      const long long o = lo + (long long)i * pitch;
      fetch(i, E4, H4, U4, V4);
      row_step<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc, Un + o, Vn + o - pitch,
                    En + o - 2 * pitch);
    }
  }
  if (RED >= 1) {
    block_reduce_and_finalize<RED, kCtaStrips + 1>(acc, a.red);
  } else if (kCtaBarrierAtExit) {
    __syncthreads();  // keep the producer warp resident until the compute warps finish
  }
}

// --- Two steps per pass (the CTA ring kernel, single slab) ------------------
#ifndef SW2D_CTA2_PIPE
#define SW2D_CTA2_PIPE 2      // second march one row behind (A/B builds: 0, 1)
#endif
#ifndef SW2D_CTA2_INTERIOR
#define SW2D_CTA2_INTERIOR 1  // a row loop without row tests between the segment's edges
#endif
#ifndef SW2D_CTA2_PIPE_ALL
#define SW2D_CTA2_PIPE_ALL 1  // the pipelined pair without diagnostics too (A/B: 0)
#endif
#ifndef SW2D_CTA2_UNROLL3
#define SW2D_CTA2_UNROLL3 1   // (without PIPE) 0: the two-row loop
#endif
// A second row march, fed from registers, advances the first march's output
// by one more step before anything is written: state n is read once and
// state n+2 written once, 28 B per two cell-steps.  The second march runs two
// rows behind the first (its input row m = L-2 needs eta(n+1) of row L-2,
// which the first march completes when it loads row L), so a segment of R
// output rows streams R + 8 input rows.  The 4-column halo lanes cover the two
// steps' cone (2 columns each).  Both steps keep the oracle's arithmetic
// (bitwise), and both steps' diagnostics are folded (two records).
template <int C>
struct Win2 {
  WinT<C> s1, s2;  // the two marches' windows
  __device__ void zero() {
    s1.zero();
    s2.zero();
  }
};

// The state n+1 of row L-2 that the second march consumes is assembled from
// slots updated in place (no shifting): uS / hS hold u(n+1) and hzero of the
// row two iterations back (the caller alternates two slots), vS holds v(n+1)
// of the row one iteration back.
template <int RED, bool REMOTE, int C>
__device__ __forceinline__ void row_step2C(const Win2<C>& w, Win2<C>& o, const float (&eL)[C],
                                           const float (&h0L)[C], const float (&uL)[C],
                                           const float (&vL)[C], const int L, const Ctx& x,
                                           Acc& acc1, Acc& acc2, float* pU, float* pV, float* pE,
                                           const float (&uIn)[C], const float (&hIn)[C],
                                           const float (&vS)[C], float (&uOut)[C],
                                           float (&hOut)[C], float (&vOut)[C]) {
  RowOut<C> r1;
  row_stepC<RED, false, C, false>(w.s1, o.s1, eL, h0L, uL, vL, L, x, acc1, nullptr, nullptr,
                                  nullptr, &r1);
  // state n+1 of row L-2: eta from this iteration, u from two, v from one back
  row_stepC<RED, REMOTE, C, true>(w.s2, o.s2, r1.En, hIn, uIn, vS, L - 2, x, acc2, pU, pV, pE);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    uOut[c] = r1.un[c];
    hOut[c] = h0L[c];
    vOut[c] = r1.vn[c];
  }
}

// in place: the slots uS / hS are read, then overwritten
template <int RED, bool REMOTE, int C>
__device__ __forceinline__ void row_step2C(const Win2<C>& w, Win2<C>& o, const float (&eL)[C],
                                           const float (&h0L)[C], const float (&uL)[C],
                                           const float (&vL)[C], const int L, const Ctx& x,
                                           Acc& acc1, Acc& acc2, float* pU, float* pV, float* pE,
                                           float (&uS)[C], float (&hS)[C], const float (&vS)[C],
                                           float (&vOut)[C]) {
  row_step2C<RED, REMOTE, C>(w, o, eL, h0L, uL, vL, L, x, acc1, acc2, pU, pV, pE, uS, hS, vS, uS,
                             hS, vOut);
}

// Software-pipelined pair: the second march runs one loaded row further
// behind (row L-3), on state n+1 the first march completed in earlier
// iterations, so within one iteration the two marches are independent and
// their dependency chains interleave (each march alone leaves the warp waiting
// on fixed-latency results: the kernel's time follows rows, not instructions).
//   eta(n+1) of row L-3: the first march of the previous row (slot En1, read
//     by march 2, then overwritten with this row's),
//   u(n+1), hzero of row L-3: three rows back (slot uS/hS, read, then
//     overwritten), v(n+1) of row L-3: two rows back (vIn); this row's: vOut.
template <int RED, bool REMOTE, int C>
__device__ __forceinline__ void row_step2P(const Win2<C>& w, Win2<C>& o, const float (&eL)[C],
                                           const float (&h0L)[C], const float (&uL)[C],
                                           const float (&vL)[C], const int L, const Ctx& x,
                                           Acc& acc1, Acc& acc2, float* pU, float* pV, float* pE,
                                           float (&uS)[C], float (&hS)[C], const float (&vIn)[C],
                                           float (&vOut)[C], float (&En1)[C]) {
  row_stepC<RED, REMOTE, C, true>(w.s2, o.s2, En1, hS, uS, vIn, L - 3, x, acc2, pU, pV, pE);
  RowOut<C> r1;
  row_stepC<RED, false, C, false>(w.s1, o.s1, eL, h0L, uL, vL, L, x, acc1, nullptr, nullptr,
                                  nullptr, &r1);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    uS[c] = r1.un[c];
    hS[c] = h0L[c];
    vOut[c] = r1.vn[c];
    En1[c] = r1.En[c];
  }
}

template <int RED, bool REMOTE>
__device__ __forceinline__ void row_step2p(const Win2<4>& w, Win2<4>& o, const float4 E4,
                                           const float4 H4, const float4 U4, const float4 V4,
                                           const int L, const Ctx& x, Acc& acc1, Acc& acc2,
                                           float* pU, float* pV, float* pE, float (&uS)[4],
                                           float (&hS)[4], const float (&vIn)[4],
                                           float (&vOut)[4], float (&En1)[4]) {
  const float eL[4] = {E4.x, E4.y, E4.z, E4.w};
  const float h0L[4] = {H4.x, H4.y, H4.z, H4.w};
  const float uL[4] = {U4.x, U4.y, U4.z, U4.w};
  const float vL[4] = {V4.x, V4.y, V4.z, V4.w};
  row_step2P<RED, REMOTE, 4>(w, o, eL, h0L, uL, vL, L, x, acc1, acc2, pU, pV, pE, uS, hS, vIn,
                             vOut, En1);
}

template <int RED, bool REMOTE>
__device__ __forceinline__ void row_step2(const Win2<4>& w, Win2<4>& o, const float4 E4,
                                          const float4 H4, const float4 U4, const float4 V4,
                                          const int L, const Ctx& x, Acc& acc1, Acc& acc2,
                                          float* pU, float* pV, float* pE,
                                          const float (&uIn)[4], const float (&hIn)[4],
                                          const float (&vS)[4], float (&uOut)[4],
                                          float (&hOut)[4], float (&vOut)[4]) {
  const float eL[4] = {E4.x, E4.y, E4.z, E4.w};
  const float h0L[4] = {H4.x, H4.y, H4.z, H4.w};
  const float uL[4] = {U4.x, U4.y, U4.z, U4.w};
  const float vL[4] = {V4.x, V4.y, V4.z, V4.w};
  row_step2C<RED, REMOTE, 4>(w, o, eL, h0L, uL, vL, L, x, acc1, acc2, pU, pV, pE, uIn, hIn, vS,
                             uOut, hOut, vOut);
}

// 7 compute warps + the producer: 8 warps (2 per scheduler) can use up to 255
// registers per thread; the two marches' windows need ~200.
constexpr int kCta2Strips = 7;
constexpr int kCta2Threads = 32 * (kCta2Strips + 1);
constexpr int kCta2WinBytes = (kCta2Strips * kColsPerStrip + 8) * 4;
constexpr int kCta2StageBytes = 4 * kCta2WinBytes;
[[maybe_unused]] constexpr int kCta2Smem = kCtaStages * kCta2StageBytes + 2 * 8 * kCtaStages;

template <int RED, bool REMOTE>
__global__ void __launch_bounds__(kCta2Threads, 1)
    sw2d_step_cta2(const StepArgs a) {
  // the pipelined pair (C5 VOLUME +1%, all seven +0.5%; without diagnostics
  // +0.7% since the face rule became arithmetic, -2% before)
  constexpr bool kPipe = SW2D_CTA2_PIPE && (RED >= 1 || SW2D_CTA2_PIPE_ALL);
  extern __shared__ __align__(128) unsigned char dsm[];
  unsigned char* ring = dsm;
  const uint32_t sring = smem_u32(ring);
  const uint32_t sfull = sring + kCtaStages * kCta2StageBytes;
  const uint32_t sempty = sfull + 8 * kCtaStages;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int ncc = (a.nstrips + kCta2Strips - 1) / kCta2Strips;
  // column group g holds strips [g*nstrips/ncc, (g+1)*nstrips/ncc) (6 or 7)
  auto gstrip = [&](int g) { return (int)(((long long)g * a.nstrips) / ncc); };

  // This CTA's work: one or two pieces (column group, output rows [ra, rb]).
  // sk_ctas == 0: CTA b is group b % ncc, row segment b / ncc.  Otherwise the
  // launch's group-rows are split evenly over sk_ctas CTAs (a CTA's time
  // follows its rows: its warps march side by side), so every SM gets the same
  // rows whatever the number of column groups; a CTA whose share crosses the
  // end of a group continues at the top of the next (a second piece).
  int pg[2] = {0, 0}, pra[2] = {0, 0}, prb[2] = {-1, -1};
  int npc = 0;
  if (a.sk_ctas == 0) {
    const int seg = blockIdx.x / ncc;
    pg[0] = blockIdx.x % ncc;
    pra[0] = (int)a.row_lo + seg * a.rows_per_seg;
    prb[0] = min((int)a.row_hi, pra[0] + a.rows_per_seg - 1);
    npc = 1;
  } else {
    // rows of all groups, group-major; CTA b takes units [b*W/sk, (b+1)*W/sk)
    const long long R = a.row_hi - a.row_lo + 1;
    const long long W = (long long)ncc * R;
    const long long beg = (long long)blockIdx.x * W / a.sk_ctas;
    const long long end = ((long long)blockIdx.x + 1) * W / a.sk_ctas;
    if (end > beg) {
      const int g = (int)(beg / R);
      const long long r0 = beg - (long long)g * R;
      const long long e0 = min(end - (long long)g * R, R);
      pg[0] = g;
      pra[0] = (int)(a.row_lo + r0);
      prb[0] = (int)(a.row_lo + e0 - 1);
      npc = 1;
      if (end > (long long)(g + 1) * R) {
        pg[1] = g + 1;
        pra[1] = (int)a.row_lo;
        prb[1] = (int)(a.row_lo + end - (long long)(g + 1) * R - 1);
        npc = 2;
      }
    }
  }

  Acc acc1, acc2;
  acc1.init();
  acc2.init();

  const long long pitch = a.s.pitch;
  const int srows = (int)(a.s.nelem / pitch);    // storage rows of each field

  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < kCtaStages; ++st) {
      mbar_init(sfull + 8 * st, 1);
      mbar_init(sempty + 8 * st, kCta2Strips);   // every compute warp releases every stage
    }
    fence_proxy_async();
  }
  __syncthreads();

  // the ring's stage and phase follow the CTA's running row count over its pieces
  int rbase = 0;
  for (int pc = 0; pc < npc; ++pc) {
    const int cc = pc ? pg[1] : pg[0];
    const int ra = pc ? pra[1] : pra[0];
    const int rb = pc ? prb[1] : prb[0];
    const int strip0 = gstrip(cc);
    const int nact = gstrip(cc + 1) - strip0;
    const int first = ra - 4;          // first streamed row
    const int n = rb + 4 + (kPipe ? 1 : 0) - first + 1;  // rows streamed (pipelined: one more)
    const int sfirst = first - (int)a.s.jbase;      // storage row of `first` (may be < 0)
    const long long off0 = (long long)sfirst * pitch + strip0 * kColsPerStrip + kStripBase;

    if (warp == kCta2Strips) {
      // the whole producer warp waits; lane 0 issues the copies.  A row outside
      // the stored rows is written as zeros into its stage by the warp (generic
      // stores, then a proxy fence before the stage is next filled by TMA), so
      // the compute warps read every stage unconditionally.
      const uint32_t wb = (uint32_t)(nact * kColsPerStrip + 8) * 4u;
      for (int r = 0; r < n; ++r) {
        const int rg = rbase + r;
        const int st = rg % kCtaStages;
        if (rg >= kCtaStages) {
          const uint32_t ph = (uint32_t)(rg / kCtaStages - 1) & 1u;
          while (!mbar_try_wait(sempty + 8 * st, ph)) {
          }
        }
        const uint32_t d = sring + st * kCta2StageBytes, b = sfull + 8 * st;
        const int sr = sfirst + r;
        if (sr < 0 || sr >= srows) {   // outside the stored rows: zeros
          float4* z = reinterpret_cast<float4*>(ring + st * kCta2StageBytes);
          for (int t = lane; t < kCta2StageBytes / 16; t += 32)
            z[t] = make_float4(0.f, 0.f, 0.f, 0.f);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_expect_tx(b, 0);
          continue;
        }
        if (lane == 0) {
          const long long o = off0 + (long long)r * pitch;
          SW2D_CHECK(o >= 0 && o + wb / 4 <= a.s.nelem);
          mbar_expect_tx(b, 4u * wb);
          bulk_g2s(d, a.s.E + o, wb, b);
          bulk_g2s(d + kCta2WinBytes, a.s.H0 + o, wb, b);
          bulk_g2s(d + 2 * kCta2WinBytes, a.s.U + o, wb, b);
          bulk_g2s(d + 3 * kCta2WinBytes, a.s.V + o, wb, b);
        }
        __syncwarp();
      }
    } else if (warp < nact) {
      Ctx x;
      x.ra = ra;
      x.rb = rb;
      const int c0 = (strip0 + warp) * kColsPerStrip + kStripBase + lane * 4;
      const int k0 = c0 - kColOff;
      x.colmask = 0;
      x.umask = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        x.colmask |= (k0 + c >= 1 && k0 + c <= a.nx) ? (1u << c) : 0u;
        x.umask |= (k0 + c >= 1 && k0 + c <= a.nx - 1) ? (1u << c) : 0u;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        x.cmf[c] = (x.colmask >> c) & 1u ? 1.0f : 0.0f;
        x.umf[c] = (x.umask >> c) & 1u ? 1.0f : 0.0f;
      }
      x.cgx = a.c.cgx; x.cgy = a.c.cgy; x.cx = a.c.cx; x.cy = a.c.cy;
      for (int c = 0; c < 4; ++c) x.cgxc[c] = x.umf[c] != 0.0f ? x.cgx : 0.0f;
      for (int c = 0; c < 4; ++c)
        x.hminc[c] = x.cmf[c] != 0.0f ? a.c.hmin : __int_as_float(0x7f800000);
      x.q = a.c.q; x.hmin = a.c.hmin; x.nz = a.c.nz;
      x.ny = (int)a.ny;
      x.out_lane = (lane >= 1) && (lane <= kOutLanes);
      x.col = c0;
      x.pitch = pitch;
      x.rem = a.rem;
#ifdef SW2D_DEBUG_BOUNDS
      x.dU = a.s.Un;
      x.dV = a.s.Vn;
      x.dE = a.s.En;
      x.nelem = a.s.nelem;
#endif
      Win2<4> wa, wb;
      wa.zero();
      float uA[4] = {0.f, 0.f, 0.f, 0.f}, uB[4] = {0.f, 0.f, 0.f, 0.f};
      float hA[4] = {0.f, 0.f, 0.f, 0.f}, hB[4] = {0.f, 0.f, 0.f, 0.f};
      // v(n+1) of the row one iteration back, alternating slots (no copies)
      float vA[4] = {0.f, 0.f, 0.f, 0.f}, vB[4] = {0.f, 0.f, 0.f, 0.f};
      float* __restrict__ En = a.s.En;
      float* __restrict__ Un = a.s.Un;
      float* __restrict__ Vn = a.s.Vn;
      const long long lo = off0 + warp * kColsPerStrip + lane * 4;
      const int sl = (warp * kColsPerStrip + lane * 4) * 4;

      auto fetch = [&](int i, float4& E4, float4& H4, float4& U4, float4& V4) {
        const int st = (rbase + i) % kCtaStages;
        const uint32_t ph = (uint32_t)((rbase + i) / kCtaStages) & 1u;
        while (!mbar_try_wait(sfull + 8 * st, ph)) {
        }
        const unsigned char* base = ring + st * kCta2StageBytes + sl;
        E4 = *reinterpret_cast<const float4*>(base);
        H4 = *reinterpret_cast<const float4*>(base + kCta2WinBytes);
        U4 = *reinterpret_cast<const float4*>(base + 2 * kCta2WinBytes);
        V4 = *reinterpret_cast<const float4*>(base + 3 * kCta2WinBytes);
        __syncwarp();
        if (lane == 0) mbar_arrive(sempty + 8 * st);
      };
      // the second march's rows L-2, L-3, L-4 (output pointers)
      int i = 0;
      if constexpr (kPipe) {
      // three rows per iteration; slots: u/h in place with period 3 (row k uses
      // slot k % 3), v written to slot k % 3 and read from (k + 1) % 3
      Win2<4> wc;
      float uC[4] = {0.f, 0.f, 0.f, 0.f}, hC[4] = {0.f, 0.f, 0.f, 0.f};
      float vC[4] = {0.f, 0.f, 0.f, 0.f};
      float e1[4] = {0.f, 0.f, 0.f, 0.f};
      // the second march writes u'(L-3), v'(L-4), eta'(L-5)
#if SW2D_CTA2_PIPE == 2
      // per row: march 2 (row L-3, from the slots) first, then the row's
      // fetch straight into the hzero slot it just consumed (no copy; the
      // shared-memory loads run under march 2's arithmetic), then march 1
      // (edge: std::true_type on the segment's first and last rows, whose
      // outputs may fall outside it or the grid; false_type in between)
      auto phase = [&](auto edge, Win2<4>& w, Win2<4>& ow, int ii, long long o, float (&uS)[4],
                       float (&hS)[4], const float (&vIn)[4],
                       float (&vOut)[4]) __attribute__((always_inline)) {
        constexpr bool kEdge = decltype(edge)::value;
        const int L = first + ii;
        row_stepC<RED, REMOTE, 4, true, kEdge>(w.s2, ow.s2, e1, hS, uS, vIn, L - 3, x, acc2,
                                               Un + o, Vn + o - pitch, En + o - 2 * pitch);
        float4 E4, H4, U4, V4;
        fetch(ii, E4, H4, U4, V4);
        const float eL[4] = {E4.x, E4.y, E4.z, E4.w};
        const float uL[4] = {U4.x, U4.y, U4.z, U4.w};
        const float vL[4] = {V4.x, V4.y, V4.z, V4.w};
        hS[0] = H4.x; hS[1] = H4.y; hS[2] = H4.z; hS[3] = H4.w;
        RowOut<4> r1;
        row_stepC<RED, false, 4, false, kEdge>(w.s1, ow.s1, eL, hS, uL, vL, L, x, acc1, nullptr,
                                               nullptr, nullptr, &r1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uS[c] = r1.un[c];
          vOut[c] = r1.vn[c];
          e1[c] = r1.En[c];
        }
      };
      auto three = [&](auto edge) __attribute__((always_inline)) {
        const long long o = lo + (long long)(i - 3) * pitch;   // row first + i - 3
        phase(edge, wa, wb, i, o, uA, hA, vB, vA);
        phase(edge, wb, wc, i + 1, o + pitch, uB, hB, vC, vB);
        phase(edge, wc, wa, i + 2, o + 2 * pitch, uC, hC, vA, vC);
      };
#if SW2D_CTA2_INTERIOR
      // row L = first + i writes u'(L-3), v'(L-4), eta'(L-5) (march 2) and
      // folds rows L .. L-2 of march 1: all of them segment rows (ra = first
      // + 4 .. rb = first + n - 6, inside 1..ny) for 9 <= i <= n - 6
      for (; i + 2 < n && i < 9; i += 3) three(std::true_type{});
      for (; i + 2 < n - 5; i += 3) three(std::false_type{});
#endif
      for (; i + 2 < n; i += 3) three(std::true_type{});
#else
      for (; i + 2 < n; i += 3) {
        float4 E4, H4, U4, V4;
        const long long o = lo + (long long)(i - 3) * pitch;   // row first + i - 3
        fetch(i, E4, H4, U4, V4);
        row_step2p<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc1, acc2, Un + o,
                                Vn + o - pitch, En + o - 2 * pitch, uA, hA, vB, vA, e1);
        fetch(i + 1, E4, H4, U4, V4);
        row_step2p<RED, REMOTE>(wb, wc, E4, H4, U4, V4, first + i + 1, x, acc1, acc2,
                                Un + o + pitch, Vn + o, En + o - pitch, uB, hB, vC, vB, e1);
        fetch(i + 2, E4, H4, U4, V4);
        row_step2p<RED, REMOTE>(wc, wa, E4, H4, U4, V4, first + i + 2, x, acc1, acc2,
                                Un + o + 2 * pitch, Vn + o + pitch, En + o, uC, hC, vA, vC, e1);
      }
#endif
      for (; i < n; ++i) {   // 0..2 remaining rows: shift the slots instead
        float4 E4, H4, U4, V4;
        const long long o = lo + (long long)(i - 3) * pitch;
        fetch(i, E4, H4, U4, V4);
        row_step2p<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc1, acc2, Un + o,
                                Vn + o - pitch, En + o - 2 * pitch, uA, hA, vB, vA, e1);
        wa = wb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float tu = uA[c], th = hA[c], tv = vA[c];
          uA[c] = uB[c]; hA[c] = hB[c]; vA[c] = vB[c];
          uB[c] = uC[c]; hB[c] = hC[c]; vB[c] = vC[c];
          uC[c] = tu; hC[c] = th; vC[c] = tv;
        }
      }
      } else {
#if SW2D_CTA2_UNROLL3
      // three rows per iteration: every value the loop carries (the wet flags of
      // rows L-1 / L-2, u(n+1) and hzero two rows back, v(n+1) one row back)
      // rotates through three register slots, so no copies at the back edge
      Win2<4> wc;
      float uC[4] = {0.f, 0.f, 0.f, 0.f}, hC[4] = {0.f, 0.f, 0.f, 0.f};
      float vC[4] = {0.f, 0.f, 0.f, 0.f};
      // half k reads u/h slot (k+1)%3, writes slot k%3; reads v slot (k-1)%3, writes k%3
      for (; i + 2 < n; i += 3) {
        float4 E4, H4, U4, V4;
        const long long o = lo + (long long)(i - 2) * pitch;   // row first + i - 2
        fetch(i, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc1, acc2, Un + o,
                       Vn + o - pitch, En + o - 2 * pitch, uB, hB, vC, uA, hA, vA);
        fetch(i + 1, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wb, wc, E4, H4, U4, V4, first + i + 1, x, acc1, acc2, Un + o + pitch,
                       Vn + o, En + o - pitch, uC, hC, vA, uB, hB, vB);
        fetch(i + 2, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wc, wa, E4, H4, U4, V4, first + i + 2, x, acc1, acc2,
                       Un + o + 2 * pitch, Vn + o + pitch, En + o, uA, hA, vB, uC, hC, vC);
      }
      for (; i < n; ++i) {   // 0..2 remaining rows: fall back to copies
        float4 E4, H4, U4, V4;
        const long long o = lo + (long long)(i - 2) * pitch;
        fetch(i, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc1, acc2, Un + o,
                       Vn + o - pitch, En + o - 2 * pitch, uB, hB, vC, uA, hA, vA);
        wa = wb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {   // shift the slots by one half
          const float tu = uA[c], th = hA[c], tv = vA[c];
          uA[c] = uB[c]; hA[c] = hB[c]; vA[c] = vB[c];
          uB[c] = uC[c]; hB[c] = hC[c]; vB[c] = vC[c];
          uC[c] = tu; hC[c] = th; vC[c] = tv;
        }
      }
#else
      for (; i + 1 < n; i += 2) {
        float4 E4, H4, U4, V4;
        const long long o = lo + (long long)(i - 2) * pitch;   // row first + i - 2
        fetch(i, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc1, acc2, Un + o,
                       Vn + o - pitch, En + o - 2 * pitch, uA, hA, vB, uA, hA, vA);
        fetch(i + 1, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wb, wa, E4, H4, U4, V4, first + i + 1, x, acc1, acc2, Un + o + pitch,
                       Vn + o, En + o - pitch, uB, hB, vA, uB, hB, vB);
      }
      if (i < n) {
        float4 E4, H4, U4, V4;
        const long long o = lo + (long long)(i - 2) * pitch;
        fetch(i, E4, H4, U4, V4);
        row_step2<RED, REMOTE>(wa, wb, E4, H4, U4, V4, first + i, x, acc1, acc2, Un + o,
                       Vn + o - pitch, En + o - 2 * pitch, uA, hA, vB, uA, hA, vA);
      }
#endif
      }
    } else {
      // a warp without a strip in this piece still releases every stage
      for (int i = 0; i < n; ++i) {
        const int st = (rbase + i) % kCtaStages;
        const uint32_t ph = (uint32_t)((rbase + i) / kCtaStages) & 1u;
        while (!mbar_try_wait(sfull + 8 * st, ph)) {
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(sempty + 8 * st);
      }
    }
    rbase += n;
  }  // pieces
  if (RED >= 1) {
    block_reduce_and_finalize<RED, kCta2Strips + 1>(acc1, a.red);
    block_reduce_and_finalize<RED, kCta2Strips + 1>(acc2, a.red2);
  } else {
    __syncthreads();
  }
}

// --- Small grids: C = 2 columns per lane, plain loads (kind 2) --------------
// The paper's own grids (500^2 .. 2000^2) are L2-resident and latency-bound:
// a warp's row march costs about one dependent chain per row.  This variant
// halves the columns per lane (60 output columns per warp strip), doubling
// the warps that march in parallel, and loads rows with plain 64-bit loads
// (one row prefetched in registers) instead of a TMA ring whose start-up
// latency would not be amortised over a few rows.
constexpr int kSmallC = 2;
constexpr int kSmallWarps = 4;
constexpr int kSmallCols = kOutLanes * kSmallC;   // 60 output columns per strip
constexpr int kSmall2Cols = 28 * kSmallC;         // two-step strips: 56 (2 halo lanes per side)

__device__ __forceinline__ void ldg2(const float* p, float (&v)[2]) {
  const float2 t = __ldg(reinterpret_cast<const float2*>(p));
  v[0] = t.x;
  v[1] = t.y;
}

template <int RED>
__global__ void __launch_bounds__(32 * kSmallWarps)
    sw2d_step_small(const StepArgs a) {
  constexpr int C = kSmallC;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kSmallWarps + (threadIdx.x >> 5);
  const int strip = gw % a.nstrips;
  const int seg = gw / a.nstrips;
  Acc acc;
  acc.init();
  if (seg < a.nsegs) {  // warp-uniform
    Ctx x;
    x.ra = (int)a.row_lo + seg * a.rows_per_seg;
    x.rb = min((int)a.row_hi, x.ra + a.rows_per_seg - 1);
    const int k0 = strip * kSmallCols + C * (lane - 1) + 1;  // 1-based column of element 0
    const int c0 = k0 + kColOff;                              // its storage column
    x.colmask = 0;
    x.umask = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      x.colmask |= (k0 + c >= 1 && k0 + c <= a.nx) ? (1u << c) : 0u;
      x.umask |= (k0 + c >= 1 && k0 + c <= a.nx - 1) ? (1u << c) : 0u;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      x.cmf[c] = (x.colmask >> c) & 1u ? 1.0f : 0.0f;
      x.umf[c] = (x.umask >> c) & 1u ? 1.0f : 0.0f;
    }
    x.cgx = a.c.cgx; x.cgy = a.c.cgy; x.cx = a.c.cx; x.cy = a.c.cy;
    for (int c = 0; c < 4; ++c) x.cgxc[c] = x.umf[c] != 0.0f ? x.cgx : 0.0f;
    for (int c = 0; c < 4; ++c) x.hminc[c] = x.cmf[c] != 0.0f ? a.c.hmin : __int_as_float(0x7f800000);
    x.q = a.c.q; x.hmin = a.c.hmin; x.nz = a.c.nz;
    x.ny = (int)a.ny;
    x.out_lane = (lane >= 1) && (lane <= kOutLanes);
#ifdef SW2D_DEBUG_BOUNDS
    x.dU = a.s.Un;
    x.dV = a.s.Vn;
    x.dE = a.s.En;
    x.nelem = a.s.nelem;
#endif
    const long long pitch = a.s.pitch;
    const int first = x.ra - 2, n = x.rb + 2 - first + 1;
    const long long lo = (long long)(first - (int)a.s.jbase) * pitch + c0;
    const float* __restrict__ E = a.s.E;
    const float* __restrict__ H = a.s.H0;
    const float* __restrict__ U = a.s.U;
    const float* __restrict__ V = a.s.V;
    float* __restrict__ En = a.s.En;
    float* __restrict__ Un = a.s.Un;
    float* __restrict__ Vn = a.s.Vn;
    WinT<C> wa, wb;
    wa.zero();
    float aE[C], aH[C], aU[C], aV[C], bE[C], bH[C], bU[C], bV[C];
    ldg2(E + lo, aE); ldg2(H + lo, aH); ldg2(U + lo, aU); ldg2(V + lo, aV);
    int i = 0;
    for (; i + 1 < n; i += 2) {
      const long long o = lo + (long long)i * pitch, o1 = o + pitch;
      ldg2(E + o1, bE); ldg2(H + o1, bH); ldg2(U + o1, bU); ldg2(V + o1, bV);
      row_stepC<RED, false, C>(wa, wb, aE, aH, aU, aV, first + i, x, acc, Un + o,
                               Vn + o - pitch, En + o - 2 * pitch);
      if (i + 2 < n) {
        const long long o2 = o1 + pitch;
        ldg2(E + o2, aE); ldg2(H + o2, aH); ldg2(U + o2, aU); ldg2(V + o2, aV);
      }
      row_stepC<RED, false, C>(wb, wa, bE, bH, bU, bV, first + i + 1, x, acc, Un + o1, Vn + o,
                               En + o - pitch);
    }
    if (i < n) {
      const long long o = lo + (long long)i * pitch;
      row_stepC<RED, false, C>(wa, wb, aE, aH, aU, aV, first + i, x, acc, Un + o,
                               Vn + o - pitch, En + o - 2 * pitch);
    }
  }
  if (RED >= 1) block_reduce_and_finalize<RED, kSmallWarps>(acc, a.red);
}

// Two steps per launch on the small-grid layout (kind 2): each warp runs the
// two row marches of row_step2C with C = 2 columns per lane and plain loads
// (one row prefetched).  Two steps need a 4-column halo on each side of a
// strip (2 per step), so lanes 0, 1 and 30, 31 are halo lanes and a strip has
// 28 x 2 = 56 output columns.  Rows outside the stored rows read as zeros.
#ifndef SW2D_SMALL2_MINB
#define SW2D_SMALL2_MINB 1
#endif
// DEFER: write the two steps' CTA partials to red.partials / red2.partials
// (+ part_base + CTA) for fold_steps instead of folding them here.
template <int RED, bool DEFER>
__global__ void __launch_bounds__(32 * kSmallWarps, SW2D_SMALL2_MINB)
    sw2d_step_small2(const StepArgs a) {
  constexpr int C = kSmallC;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kSmallWarps + (threadIdx.x >> 5);
  const int strip = gw % a.nstrips;
  const int seg = gw / a.nstrips;
  Acc acc1, acc2;
  acc1.init();
  acc2.init();
  if (seg < a.nsegs) {  // warp-uniform
    Ctx x;
    x.ra = (int)a.row_lo + seg * a.rows_per_seg;
    x.rb = min((int)a.row_hi, x.ra + a.rows_per_seg - 1);
    const int k0 = strip * kSmall2Cols + C * (lane - 2) + 1;  // 1-based column of element 0
    const int c0 = k0 + kColOff;                              // its storage column
    x.colmask = 0;
    x.umask = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      x.colmask |= (k0 + c >= 1 && k0 + c <= a.nx) ? (1u << c) : 0u;
      x.umask |= (k0 + c >= 1 && k0 + c <= a.nx - 1) ? (1u << c) : 0u;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      x.cmf[c] = (x.colmask >> c) & 1u ? 1.0f : 0.0f;
      x.umf[c] = (x.umask >> c) & 1u ? 1.0f : 0.0f;
    }
    x.cgx = a.c.cgx; x.cgy = a.c.cgy; x.cx = a.c.cx; x.cy = a.c.cy;
    for (int c = 0; c < 4; ++c) x.cgxc[c] = x.umf[c] != 0.0f ? x.cgx : 0.0f;
    for (int c = 0; c < 4; ++c) x.hminc[c] = x.cmf[c] != 0.0f ? a.c.hmin : __int_as_float(0x7f800000);
    x.q = a.c.q; x.hmin = a.c.hmin; x.nz = a.c.nz;
    x.ny = (int)a.ny;
    x.out_lane = (lane >= 2) && (lane <= 29);
#ifdef SW2D_DEBUG_BOUNDS
    x.dU = a.s.Un;
    x.dV = a.s.Vn;
    x.dE = a.s.En;
    x.nelem = a.s.nelem;
#endif
    const long long pitch = a.s.pitch;
    const int srows = (int)(a.s.nelem / pitch);   // storage rows of each field
    const int first = x.ra - 4, n = x.rb + 4 - first + 1;
    const int sfirst = first - (int)a.s.jbase;     // storage row of `first` (may be < 0)
    const long long lo = (long long)sfirst * pitch + c0;
    const float* __restrict__ E = a.s.E;
    const float* __restrict__ H = a.s.H0;
    const float* __restrict__ U = a.s.U;
    const float* __restrict__ V = a.s.V;
    float* __restrict__ En = a.s.En;
    float* __restrict__ Un = a.s.Un;
    float* __restrict__ Vn = a.s.Vn;
    auto load = [&](int i, float (&e)[C], float (&hh)[C], float (&u)[C], float (&v)[C]) {
      const int sr = sfirst + i;
      if (sr < 0 || sr >= srows) {
#pragma unroll
        for (int c = 0; c < C; ++c) e[c] = hh[c] = u[c] = v[c] = 0.0f;
      } else {
        const long long o = lo + (long long)i * pitch;
        ldg2(E + o, e); ldg2(H + o, hh); ldg2(U + o, u); ldg2(V + o, v);
      }
    };
    Win2<C> wa, wb;
    wa.zero();
    float uA[C] = {0.f, 0.f}, uB[C] = {0.f, 0.f}, hA[C] = {0.f, 0.f}, hB[C] = {0.f, 0.f};
    float vA[C] = {0.f, 0.f}, vB[C] = {0.f, 0.f};
    float aE[C], aH[C], aU[C], aV[C], bE[C], bH[C], bU[C], bV[C];
    load(0, aE, aH, aU, aV);
    int i = 0;
    for (; i + 1 < n; i += 2) {
      const long long o = lo + (long long)(i - 2) * pitch;   // row first + i - 2
      load(i + 1, bE, bH, bU, bV);
      row_step2C<RED, false, C>(wa, wb, aE, aH, aU, aV, first + i, x, acc1, acc2, Un + o,
                                Vn + o - pitch, En + o - 2 * pitch, uA, hA, vB, vA);
      if (i + 2 < n) load(i + 2, aE, aH, aU, aV);
      row_step2C<RED, false, C>(wb, wa, bE, bH, bU, bV, first + i + 1, x, acc1, acc2,
                                Un + o + pitch, Vn + o, En + o - pitch, uB, hB, vA, vB);
    }
    if (i < n) {
      const long long o = lo + (long long)(i - 2) * pitch;
      row_step2C<RED, false, C>(wa, wb, aE, aH, aU, aV, first + i, x, acc1, acc2, Un + o,
                                Vn + o - pitch, En + o - 2 * pitch, uA, hA, vB, vA);
    }
  }
  if (RED >= 1 && DEFER) {
    block_reduce_to_partial<RED, kSmallWarps>(acc1, a.red.partials + a.red.part_base);
    block_reduce_to_partial<RED, kSmallWarps>(acc2, a.red2.partials + a.red2.part_base);
  } else if (RED >= 1) {
    block_reduce_and_finalize<RED, kSmallWarps>(acc1, a.red);
    block_reduce_and_finalize<RED, kSmallWarps>(acc2, a.red2);
  }
}

// ---------------------------------------------------------------------------
// set_state ingest: finiteness check, wall-face zeroing, sum of hzero.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) sw2d_ingest(const IngestArgs a) {
  Acc acc;
  acc.init();
  const long long n = a.nrows * (long long)a.nx;
  bool bad = false;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads) {
    const long long r = i / a.nx + kHaloRows;
    const int k = (int)(i % a.nx) + 1;
    const long long o = r * a.pitch + k + kColOff;
    const float h0 = a.H0[o], e = a.E[o];
    float u = a.U[o], v = a.V[o];
    if (k == a.nx) { a.U[o] = 0.0f; u = 0.0f; }
    if (a.jbase + r == a.ny) { a.V[o] = 0.0f; v = 0.0f; }
    bad |= !isfinite(h0) || !isfinite(e) || !isfinite(u) || !isfinite(v);
    acc.sum_eta += (double)h0;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.bad, 1);
  // reuse the fold: record[kRecSumEta] = sum(hzero)
  block_reduce_and_finalize<1, kWarpsPerBlock>(acc, a.red);
}

// ---------------------------------------------------------------------------
// Diagnostics of the current state (unfused, 16 B/cell).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) sw2d_reduce_state(const ReduceArgs a) {
  Acc acc;
  acc.init();
  const long long n = a.nrows * (long long)a.nx;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads) {
    const long long r = i / a.nx + kHaloRows;
    const int k = (int)(i % a.nx) + 1;
    const long long o = r * a.pitch + k + kColOff;
    const float e = a.E[o], h0 = a.H0[o];
    acc.sum_eta += (double)e;
    acc.max_eta = fmaxf(acc.max_eta, e);
    acc.neg_min_eta = fmaxf(acc.neg_min_eta, -e);
    acc.max_u = fmaxf(acc.max_u, fabsf(a.U[o]));
    acc.max_v = fmaxf(acc.max_v, fabsf(a.V[o]));
    acc.wet += (__fadd_rn(h0, e) < a.hmin) ? 0.0 : 1.0;
  }
  block_reduce_and_finalize<2, kWarpsPerBlock>(acc, a.red);
}

__global__ void sw2d_wet_mask(const float* E, const float* H0, long long pitch,
                              long long nrows, int nx, float hmin,
                              unsigned char* out) {
  const long long n = nrows * (long long)nx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / nx + kHaloRows;
    const int k = (int)(i % nx) + 1;
    const long long o = r * pitch + k + kColOff;
    out[i] = (__fadd_rn(H0[o], E[o]) < hmin) ? 0 : 1;
  }
}

int grid_stride_blocks(long long n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long b = (n + kThreads - 1) / kThreads;
  const long long cap = 8LL * sms;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

// (instantiated in sw2d_cta2_r0/1/2.cu, one diagnostics level per translation
// unit: the three row-loop copies make each instance take minutes in ptxas)
namespace {
template <int RED, bool REMOTE>
void launch_two(const StepArgs& a, cudaStream_t s) {
  static unsigned long long attr_devices = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_devices >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(sw2d_step_cta2<RED, REMOTE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kCta2Smem);
    cudaFuncSetAttribute(sw2d_step_cta2<RED, REMOTE>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr_devices |= 1ull << (dev & 63);
  }
  const int ncc = (a.nstrips + kCta2Strips - 1) / kCta2Strips;
  const int blocks = a.sk_ctas > 0 ? a.sk_ctas : ncc * a.nsegs;
  sw2d_step_cta2<RED, REMOTE><<<blocks, kCta2Threads, kCta2Smem, s>>>(a);
}
}  // namespace

#ifndef SW2D_PROBE   // tools/cta2_probe.cu: the kernels alone, one instantiation (SASS studies)
int step_strips_per_cta(int kind) {
  return kind == 2 ? kSmallWarps : kCtaStrips;
}

int step_strip_cols(int kind) { return kind == 2 ? kSmallCols : kColsPerStrip; }
int step2_small_strip_cols() { return kSmall2Cols; }

int step_grid(int kind, int nstrips, int nsegs) {
  if (kind == 2) {  // independent warps: (strip, segment) pairs, kSmallWarps per CTA
    const long long warps = (long long)nstrips * nsegs;
    return (int)((warps + kSmallWarps - 1) / kSmallWarps);
  }
  const int per = step_strips_per_cta(kind);
  return ((nstrips + per - 1) / per) * nsegs;
}

namespace {
template <int RED, bool REMOTE>
void cta_attributes() {
  cudaFuncSetAttribute(sw2d_step_cta<RED, REMOTE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kCtaSmem);
  cudaFuncSetAttribute(sw2d_step_cta<RED, REMOTE>,
                       cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

template <int RED, bool REMOTE>
void launch_kind(const StepArgs& a, int kind, cudaStream_t s) {
  const int blocks = step_grid(kind, a.nstrips, a.nsegs);
  if (kind == 2 && !REMOTE) {
    sw2d_step_small<RED><<<blocks, 32 * kSmallWarps, 0, s>>>(a);
    return;
  }
  static unsigned long long attr_devices = 0;  // dynamic smem above 48 KB, per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_devices >> (dev & 63) & 1ull)) {
    cta_attributes<RED, REMOTE>();
    attr_devices |= 1ull << (dev & 63);
  }
  sw2d_step_cta<RED, REMOTE><<<step_grid(1, a.nstrips, a.nsegs), kCtaThreads, kCtaSmem, s>>>(a);
}

template <int RED>
int occupancy_kind(int kind) {
  int n = 0;
  if (kind == 2) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_small<RED>, 32 * kSmallWarps, 0);
  } else {
    cta_attributes<RED, false>();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_cta<RED, false>, kCtaThreads,
                                                  kCtaSmem);
  }
  return n < 1 ? 1 : n;
}
}  // namespace


int step2_strips_per_cta() { return kCta2Strips; }

void launch_step2_small(const StepArgs& a, int red_level, void* stream, bool defer) {
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = step_grid(2, a.nstrips, a.nsegs);
  if (red_level >= 2 && defer)
    sw2d_step_small2<2, true><<<blocks, 32 * kSmallWarps, 0, s>>>(a);
  else if (red_level >= 2)
    sw2d_step_small2<2, false><<<blocks, 32 * kSmallWarps, 0, s>>>(a);
  else if (red_level == 1 && defer)
    sw2d_step_small2<1, true><<<blocks, 32 * kSmallWarps, 0, s>>>(a);
  else if (red_level == 1)
    sw2d_step_small2<1, false><<<blocks, 32 * kSmallWarps, 0, s>>>(a);
  else
    sw2d_step_small2<0, false><<<blocks, 32 * kSmallWarps, 0, s>>>(a);
}

void launch_fold_steps(const RedPartial* partials, int blocks, int nsteps, double* hist, int len,
                       const unsigned long long* dstep, const double* h0sum, double dxdy,
                       void* stream) {
  fold_steps<<<nsteps, kFoldThreads, 0, (cudaStream_t)stream>>>(partials, blocks, hist, len,
                                                               dstep, h0sum, dxdy);
}

int step2_small_occupancy_blocks_per_sm(int red_level) {
  int n = 0;
  if (red_level >= 2)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_small2<2, false>, 32 * kSmallWarps, 0);
  else if (red_level == 1)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_small2<1, false>, 32 * kSmallWarps, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_small2<0, false>, 32 * kSmallWarps, 0);
  return n < 1 ? 1 : n;
}

void launch_step2(const StepArgs& a, int red_level, void* stream, bool remote) {
  if (red_level >= 2)
    launch_step2_r2(a, stream, remote);
  else if (red_level == 1)
    launch_step2_r1(a, stream, remote);
  else
    launch_step2_r0(a, stream, remote);
}

void launch_step(const StepArgs& a, int red_level, int kind, void* stream, bool remote) {
  cudaStream_t s = (cudaStream_t)stream;
  if (remote) {
    if (red_level >= 2)
      launch_kind<2, true>(a, kind, s);
    else if (red_level == 1)
      launch_kind<1, true>(a, kind, s);
    else
      launch_kind<0, true>(a, kind, s);
  } else if (red_level >= 2) {
    launch_kind<2, false>(a, kind, s);
  } else if (red_level == 1) {
    launch_kind<1, false>(a, kind, s);
  } else {
    launch_kind<0, false>(a, kind, s);
  }
}

int step_occupancy_blocks_per_sm(int red_level, int kind) {
  if (red_level >= 2) return occupancy_kind<2>(kind);
  if (red_level == 1) return occupancy_kind<1>(kind);
  return occupancy_kind<0>(kind);
}

int ingest_blocks(const IngestArgs& a) {
  return grid_stride_blocks(a.nrows * (long long)a.nx);
}

void launch_ingest(const IngestArgs& a, void* stream) {
  sw2d_ingest<<<ingest_blocks(a), kThreads, 0, (cudaStream_t)stream>>>(a);
}

int reduce_blocks(const ReduceArgs& a) {
  return grid_stride_blocks(a.nrows * (long long)a.nx);
}

void launch_reduce(const ReduceArgs& a, void* stream) {
  sw2d_reduce_state<<<reduce_blocks(a), kThreads, 0, (cudaStream_t)stream>>>(a);
}

void launch_wet(const float* E, const float* H0, long long pitch,
                long long nrows, int nx, float hmin, unsigned char* out,
                void* stream) {
  const long long n = nrows * (long long)nx;
  const int blocks = grid_stride_blocks(n);
  sw2d_wet_mask<<<blocks, kThreads, 0, (cudaStream_t)stream>>>(E, H0, pitch, nrows,
                                                               nx, hmin, out);
}

#endif  // SW2D_PROBE

}  // namespace sw2d_dev
