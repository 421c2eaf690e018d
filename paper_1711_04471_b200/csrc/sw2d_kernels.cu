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

#include "sw2d_internal.cuh"

namespace sw2d_dev {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ void st4(float* p, float a, float b, float c,
                                    float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

// Upwind volume flux through a face with velocity s (reading R3):
// s > 0 ? s*hL : (s < 0 ? s*hR : 0), both products formed, then selected.
__device__ __forceinline__ float flux(float s, float hl, float hr) {
  const float a = __fmul_rn(s, hl);
  const float b = __fmul_rn(s, hr);
  return s > 0.0f ? a : (s < 0.0f ? b : 0.0f);
}

// Wet/dry face rule of the momentum predictor (reading R4): returns the new
// face velocity old + d if the face carries flow, else 0.
__device__ __forceinline__ float face(bool wc, bool wn, float d, float old,
                                      bool ok) {
  const bool flow = wc ? (wn || d > 0.0f) : (wn && d < 0.0f);
  return (ok && flow) ? __fadd_rn(old, d) : 0.0f;
}

struct Acc {
  double sum_eta;
  double wet;
  float max_eta, neg_min_eta, max_u, max_v;
  __device__ void init() {
    sum_eta = 0.0;
    wet = 0.0;
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
template <int LEVEL>
__device__ void block_reduce_and_finalize(Acc acc, const RedArgs& r) {
  __shared__ Acc sh[kWarpsPerBlock];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    for (int w = 1; w < kWarpsPerBlock; ++w) {
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
  if (!last) return;
  __threadfence();
  // Fixed-order fold: thread t takes slots t, t+128, ... in order, then a
  // fixed tree over threads.
  Acc t;
  t.init();
  for (int i = threadIdx.x; i < r.expected; i += kThreads) {
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
    for (int w = 1; w < kWarpsPerBlock; ++w) {
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

// ---------------------------------------------------------------------------
// The fused step.
// ---------------------------------------------------------------------------
template <int RED>
__global__ void __launch_bounds__(kThreads)
    sw2d_step_fused(const StepArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int strip = gw % a.nstrips;
  const int seg = gw / a.nstrips;

  Acc acc;
  acc.init();

  if (seg < a.nsegs) {  // warp-uniform
    const long long ra = a.row_lo + (long long)seg * a.rows_per_seg;
    const long long rb = min(a.row_hi, ra + a.rows_per_seg - 1);
    const int c0 = strip * kColsPerStrip + lane * 4;  // storage column of element 0
    const int k0 = c0 - kColOff;                      // its 1-based column
    const int nx = a.nx;
    const long long ny = a.ny;
    const bool out_lane = (lane >= 1) && (lane <= kOutLanes);
    bool colok[4], uok[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      colok[c] = (k0 + c >= 1) && (k0 + c <= nx);
      uok[c] = (k0 + c >= 1) && (k0 + c <= nx - 1);
    }
    const float cgx = a.c.cgx, cgy = a.c.cgy, cx = a.c.cx, cy = a.c.cy;
    const float q = a.c.q, hmin = a.c.hmin;
    const long long pitch = a.s.pitch;

    // rolling window (rows relative to the loaded row L)
    float eP[4] = {0.f, 0.f, 0.f, 0.f};    // eta(L-1)
    float hP[4] = {0.f, 0.f, 0.f, 0.f};    // h(L-1)
    float unP[4] = {0.f, 0.f, 0.f, 0.f};   // un(L-1)
    float vP[4] = {0.f, 0.f, 0.f, 0.f};    // V(L-1) (old)
    float fyP[4] = {0.f, 0.f, 0.f, 0.f};   // y-flux through the north face of row L-2
    float etP[4] = {0.f, 0.f, 0.f, 0.f};   // etan(L-2)
    float etPP[4] = {0.f, 0.f, 0.f, 0.f};  // etan(L-3)
    float h0P[4] = {0.f, 0.f, 0.f, 0.f};   // hzero(L-1)  (RED >= 2)
    float h0PP[4] = {0.f, 0.f, 0.f, 0.f};  // hzero(L-2)  (RED >= 2)
    float hRP = 0.f;                       // h(L-1, k0+4)
    unsigned wP = 0, wPP = 0, wPPP = 0;    // wet bits of rows L-1, L-2, L-3

    long long L = ra - 2;
    const long long last = rb + 2;
    long long off = (L - a.s.jbase) * pitch + c0;
    float4 nE = ldg4(a.s.E + off), nH = ldg4(a.s.H0 + off);
    float4 nU = ldg4(a.s.U + off), nV = ldg4(a.s.V + off);

    for (; L <= last; ++L) {
      const float eL[4] = {nE.x, nE.y, nE.z, nE.w};
      const float h0L[4] = {nH.x, nH.y, nH.z, nH.w};
      const float uL[4] = {nU.x, nU.y, nU.z, nU.w};
      const float vL[4] = {nV.x, nV.y, nV.z, nV.w};
      const long long cur = off;
      if (L < last) off += pitch;  // prefetch the next row (re-load the last one)
      nE = ldg4(a.s.E + off);
      nH = ldg4(a.s.H0 + off);
      nU = ldg4(a.s.U + off);
      nV = ldg4(a.s.V + off);

      // a1: h and wet of row L
      const bool rowok = (L >= 1) && (L <= ny);
      float hL[4];
      unsigned wL = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        hL[c] = __fadd_rn(h0L[c], eL[c]);
        wL |= (rowok && colok[c] && !(hL[c] < hmin)) ? (1u << c) : 0u;
      }
      const float eR = __shfl_down_sync(kFull, eL[0], 1);
      const float hR = __shfl_down_sync(kFull, hL[0], 1);
      const unsigned wRb = __shfl_down_sync(kFull, wL, 1);

      // a2: un(L) (east faces) and vn(L-1) (north faces of row L-1)
      float unL[4], vnP[4];
      const bool vrow = (L - 1 >= 1) && (L - 1 <= ny - 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float en = (c < 3) ? eL[c + 1] : eR;
        const bool wn = (c < 3) ? ((wL >> (c + 1)) & 1u) : (wRb & 1u);
        const float du = __fmul_rn(cgx, __fsub_rn(en, eL[c]));
        unL[c] = face((wL >> c) & 1u, wn, du, uL[c], rowok && uok[c]);
        const float dv = __fmul_rn(cgy, __fsub_rn(eL[c], eP[c]));
        vnP[c] = face((wP >> c) & 1u, (wL >> c) & 1u, dv, vP[c],
                      vrow && colok[c]);
      }

      // a3: fluxes and etan(L-1)
      float fx[4], fy[4], et[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float hr = (c < 3) ? hP[c + 1] : hRP;
        fx[c] = flux(unP[c], hP[c], hr);
        fy[c] = flux(vnP[c], hP[c], hL[c]);
      }
      const float fxw = __shfl_up_sync(kFull, fx[3], 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float fw = (c > 0) ? fx[c - 1] : fxw;
        et[c] = __fsub_rn(__fsub_rn(eP[c], __fmul_rn(cx, __fsub_rn(fx[c], fw))),
                          __fmul_rn(cy, __fsub_rn(fy[c], fyP[c])));
      }

      // a4: Shapiro filter of row L-2 (centre etP, north et, south etPP)
      const float etW = __shfl_up_sync(kFull, etP[3], 1);
      const float etE = __shfl_down_sync(kFull, etP[0], 1);
      const unsigned wWb = __shfl_up_sync(kFull, wPP, 1);
      const unsigned wEb = __shfl_down_sync(kFull, wPP, 1);
      float En[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const unsigned wE = (c < 3) ? ((wPP >> (c + 1)) & 1u) : (wEb & 1u);
        const unsigned wW = (c > 0) ? ((wPP >> (c - 1)) & 1u) : ((wWb >> 3) & 1u);
        const unsigned wN = (wP >> c) & 1u;
        const unsigned wS = (wPPP >> c) & 1u;
        const float xE = (c < 3) ? etP[c + 1] : etE;
        const float xW = (c > 0) ? etP[c - 1] : etW;
        const float s = (float)(int)(wE + wW + wN + wS);
        const float t1 = __fmul_rn(__fsub_rn(1.0f, __fmul_rn(q, s)), etP[c]);
        const float t2 = __fmul_rn(q, __fadd_rn(wE ? xE : 0.0f, wW ? xW : 0.0f));
        const float t3 = __fmul_rn(q, __fadd_rn(wN ? et[c] : 0.0f, wS ? etPP[c] : 0.0f));
        const float f = ((wPP >> c) & 1u) ? __fadd_rn(__fadd_rn(t1, t2), t3) : etP[c];
        En[c] = colok[c] ? f : 0.0f;
      }

      // a5: commit (lanes 1..30; rows of this segment only)
      if (out_lane) {
        if (L >= ra && L <= rb) {
          st4(a.s.Un + cur, unL[0], unL[1], unL[2], unL[3]);
          if (RED >= 2) {
#pragma unroll
            for (int c = 0; c < 4; ++c) acc.max_u = fmaxf(acc.max_u, fabsf(unL[c]));
          }
        }
        if (L - 1 >= ra && L - 1 <= rb) {
          st4(a.s.Vn + cur - pitch, vnP[0], vnP[1], vnP[2], vnP[3]);
          if (RED >= 2) {
#pragma unroll
            for (int c = 0; c < 4; ++c) acc.max_v = fmaxf(acc.max_v, fabsf(vnP[c]));
          }
        }
        if (L - 2 >= ra && L - 2 <= rb) {
          st4(a.s.En + cur - 2 * pitch, En[0], En[1], En[2], En[3]);
          if (RED >= 1) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (colok[c]) {
                acc.sum_eta += (double)En[c];
                if (RED >= 2) {
                  acc.max_eta = fmaxf(acc.max_eta, En[c]);
                  acc.neg_min_eta = fmaxf(acc.neg_min_eta, -En[c]);
                  acc.wet += (__fadd_rn(h0PP[c], En[c]) < hmin) ? 0.0 : 1.0;
                }
              }
            }
          }
        }
      }

      // rotate the window
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        etPP[c] = etP[c];
        etP[c] = et[c];
        eP[c] = eL[c];
        hP[c] = hL[c];
        unP[c] = unL[c];
        vP[c] = vL[c];
        fyP[c] = fy[c];
        if (RED >= 2) {
          h0PP[c] = h0P[c];
          h0P[c] = h0L[c];
        }
      }
      hRP = hR;
      wPPP = wPP;
      wPP = wP;
      wP = wL;
    }
  }
  if (RED >= 1) block_reduce_and_finalize<RED>(acc, a.red);
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
  block_reduce_and_finalize<1>(acc, a.red);
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
  block_reduce_and_finalize<2>(acc, a.red);
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

int step_blocks(const StepArgs& a) {
  const long long warps = (long long)a.nstrips * a.nsegs;
  return (int)((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
}

void launch_step(const StepArgs& a, int red_level, void* stream) {
  const int blocks = step_blocks(a);
  cudaStream_t s = (cudaStream_t)stream;
  if (red_level >= 2)
    sw2d_step_fused<2><<<blocks, kThreads, 0, s>>>(a);
  else if (red_level == 1)
    sw2d_step_fused<1><<<blocks, kThreads, 0, s>>>(a);
  else
    sw2d_step_fused<0><<<blocks, kThreads, 0, s>>>(a);
}

int step_occupancy_blocks_per_sm(int red_level) {
  int n = 0;
  if (red_level >= 2)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_fused<2>, kThreads, 0);
  else if (red_level == 1)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_fused<1>, kThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sw2d_step_fused<0>, kThreads, 0);
  return n < 1 ? 1 : n;
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

}  // namespace sw2d_dev
