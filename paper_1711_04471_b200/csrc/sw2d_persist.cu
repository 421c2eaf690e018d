// paper_1711_04471_b200/csrc/sw2d_persist.cu — persistent cooperative kernel
// for the paper's small grids.
//
// The paper times 500^2 .. 2000^2 grids for 10,000 steps.  Their state lives
// in L2 and one step is a few microseconds of work spread over the GPU, so a
// kernel launch (or graph node) per pass and the start-up of a row march
// cost more than the arithmetic.  Here ONE cooperative launch runs many
// steps: every CTA owns a fixed tile of TW x TH cells (TW = 64 - 2A, A = 2K)
// for the whole launch and advances it K steps at a time in shared memory
// (tile + A-cell apron: the dependency cone of K steps is 2K cells), then
//   * stores the tile's exact centre into the next state buffer (L2),
//   * publishes a per-tile step counter (release),
//   * waits until its 8 neighbour tiles have published the same block
//     (acquire) — they have then written the apron it needs and finished
//     reading the buffer it will overwrite next (double buffering),
//   * reloads only its apron ring; the centre stays in shared memory.
// There is no grid-wide barrier and no relaunch.  The blocks wait on one
// another, so the launch is cooperative (all CTAs co-resident, guaranteed by
// the driver) — the one sanctioned form of inter-CTA waiting on one GPU.
//
// Per step and cell the arithmetic is the oracle's, operation for operation,
// in four CTA-synchronised phases (h and wet; face velocities; etan; Shapiro
// + commit), like the oracle's loop nests (oracle/sw2d_ref.c): bitwise parity.
// Cells outside the grid are dry with zero velocity (the closed basin).  The
// apron's outer cells go stale one ring per phase and never reach the centre.
//
// Diagnostics: per step, each CTA folds its centre cells (fp64 sums, exact
// max/min/count) into one partial; fold_steps folds the partials of a launch
// in a fixed order after it (deterministic; the deferred fold of the graphs).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "sw2d_internal.cuh"

namespace sw2d_dev {

namespace {

constexpr int kPX = 64;       // shared tile width (2 columns per lane)
constexpr int kPThreadsY = 8; // blockDim = (32, kPThreadsY)
constexpr int kPThreads = 32 * kPThreadsY;
constexpr int kPFlagStride = 32;        // uints between two tiles' flags (128 B)
constexpr int kPSmemMax = 226 * 1024;   // dynamic shared memory cap (the reduction's static buffer fits beside)

__device__ __forceinline__ float p_flux(float s, float hl, float hr) {
  return s > 0.0f ? __fmul_rn(s, hl) : (s < 0.0f ? __fmul_rn(s, hr) : 0.0f);
}

__device__ __forceinline__ bool p_flows(bool wc, bool wn, float d) {
  return wc ? (wn || d > 0.0f) : (wn && d < 0.0f);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct PAcc {
  double s;
  double wet;
  float mx, nmn, mu, mv;
};

template <int K, int RED>
__global__ void __launch_bounds__(kPThreads)
    sw2d_persist(const PersistArgs a) {
  constexpr int A = 2 * K;            // apron cells per side
  constexpr int TW = kPX - 2 * A;     // tile width
  extern __shared__ __align__(16) float psm[];
  const int TH = a.th, Y = TH + 2 * A, N = Y * kPX;
  float* sE = psm;        // eta (state being advanced)
  float* sH0 = sE + N;    // hzero (static)
  float* sU = sH0 + N;
  float* sV = sU + N;
  float* sh = sV + N;     // h
  float* sw = sh + N;     // wet flags 1/0
  float* sun = sw + N;    // un
  float* svn = sun + N;   // vn
  float* set = svn + N;   // etan

  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int tile = blockIdx.x;
  const int tk = tile % a.ntx, tj = tile / a.ntx;
  const int gk0 = tk * TW + 1 - A;   // global 1-based column of shared column 0
  const int gj0 = tj * TH + 1 - A;   // global 1-based row of shared row 0
  const int nx = a.nx, ny = a.ny;
  const long long pitch = a.pitch;
  const float cgx = a.c.cgx, cgy = a.c.cgy, cx = a.c.cx, cy = a.c.cy, q = a.c.q,
              hmin = a.c.hmin;

  // in-grid masks of this thread's two columns
  const int x0 = 2 * tx;
  const int gka = gk0 + x0, gkb = gka + 1;
  const bool ina = gka >= 1 && gka <= nx, inb = gkb >= 1 && gkb <= nx;

  auto gofs = [&](int y, int x) -> long long {
    return (long long)(gj0 + y - a.jbase) * pitch + (gk0 + x) + kColOff;
  };
  auto in_grid = [&](int y, int x) {
    const int gj = gj0 + y, gk = gk0 + x;
    return gj >= 1 && gj <= ny && gk >= 1 && gk <= nx;
  };

  int b = a.cur;   // buffer holding the current state
  // initial load: the whole apron'd tile (zero outside the grid)
  for (int y = ty; y < Y; y += kPThreadsY) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int x = x0 + c, i = y * kPX + x;
      float e = 0.0f, h0 = 0.0f, u = 0.0f, v = 0.0f;
      if (in_grid(y, x)) {
        const long long o = gofs(y, x);
        e = __ldcg(a.E[b] + o);
        h0 = __ldcg(a.H0 + o);
        u = __ldcg(a.U[b] + o);
        v = __ldcg(a.V[b] + o);
      }
      sE[i] = e;
      sH0[i] = h0;
      sU[i] = u;
      sV[i] = v;
    }
  }
  __syncthreads();

  // neighbour tiles (8-neighbourhood; -1 when outside)
  int nb = -1;
  if (tid < 9 && tid != 4) {
    const int dj = tid / 3 - 1, dk = tid % 3 - 1;
    const int nj = tj + dj, nk = tk + dk;
    if (nj >= 0 && nj < a.nty && nk >= 0 && nk < a.ntx) nb = nj * a.ntx + nk;
  }

  int done = 0;
  while (done < a.nsteps) {
    const int kk = min(K, a.nsteps - done);
    for (int s = 0; s < kk; ++s) {
      const int step = done + s;
      // P1: h and wet
      for (int y = ty; y < Y; y += kPThreadsY) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int x = x0 + c, i = y * kPX + x;
          const float hv = __fadd_rn(sH0[i], sE[i]);
          sh[i] = hv;
          sw[i] = (in_grid(y, x) && !(hv < hmin)) ? 1.0f : 0.0f;
        }
      }
      __syncthreads();
      // P2: face velocities (walls and faces outside the grid: 0)
      for (int y = ty; y < Y; y += kPThreadsY) {
        const int gj = gj0 + y;
        const bool rin = gj >= 1 && gj <= ny;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int x = x0 + c, i = y * kPX + x;
          const int gk = gk0 + x;
          float u = 0.0f, v = 0.0f;
          if (rin && (c ? inb : ina)) {
            if (gk != nx && x + 1 < kPX) {
              const float du = __fmul_rn(cgx, __fsub_rn(sE[i + 1], sE[i]));
              if (p_flows(sw[i] != 0.0f, sw[i + 1] != 0.0f, du)) u = __fadd_rn(sU[i], du);
            }
            if (gj != ny && y + 1 < Y) {
              const float dv = __fmul_rn(cgy, __fsub_rn(sE[i + kPX], sE[i]));
              if (p_flows(sw[i] != 0.0f, sw[i + kPX] != 0.0f, dv)) v = __fadd_rn(sV[i], dv);
            }
          }
          sun[i] = u;
          svn[i] = v;
        }
      }
      __syncthreads();
      // P3: etan (the outermost ring stays stale)
      for (int y = ty; y < Y; y += kPThreadsY) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int x = x0 + c, i = y * kPX + x;
          float e = 0.0f;
          if (x >= 1 && x + 1 < kPX && y >= 1 && y + 1 < Y) {
            const float hc = sh[i];
            const float fe = p_flux(sun[i], hc, sh[i + 1]);
            const float fw = p_flux(sun[i - 1], sh[i - 1], hc);
            const float fn = p_flux(svn[i], hc, sh[i + kPX]);
            const float fs = p_flux(svn[i - kPX], sh[i - kPX], hc);
            e = __fsub_rn(__fsub_rn(sE[i], __fmul_rn(cx, __fsub_rn(fe, fw))),
                          __fmul_rn(cy, __fsub_rn(fn, fs)));
          }
          set[i] = e;
        }
      }
      __syncthreads();
      // P4: Shapiro filter and commit; diagnostics over the exact centre
      PAcc acc;
      acc.s = 0.0;
      acc.wet = 0.0;
      acc.mx = __int_as_float(0xff800000);
      acc.nmn = __int_as_float(0xff800000);
      acc.mu = 0.0f;
      acc.mv = 0.0f;
      for (int y = ty; y < Y; y += kPThreadsY) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int x = x0 + c, i = y * kPX + x;
          float e = 0.0f;
          const bool in = in_grid(y, x);
          if (in) {
            e = set[i];
            if (sw[i] != 0.0f && x >= 1 && x + 1 < kPX && y >= 1 && y + 1 < Y) {
              const bool wE = sw[i + 1] != 0.0f, wW = sw[i - 1] != 0.0f;
              const bool wN = sw[i + kPX] != 0.0f, wS = sw[i - kPX] != 0.0f;
              const float sc = (float)((int)wE + (int)wW + (int)wN + (int)wS);
              const float t1 = __fmul_rn(__fsub_rn(1.0f, __fmul_rn(q, sc)), e);
              const float t2 =
                  __fmul_rn(q, __fadd_rn(wE ? set[i + 1] : 0.0f, wW ? set[i - 1] : 0.0f));
              const float t3 =
                  __fmul_rn(q, __fadd_rn(wN ? set[i + kPX] : 0.0f, wS ? set[i - kPX] : 0.0f));
              e = __fadd_rn(__fadd_rn(t1, t2), t3);
            }
          }
          const float un = sun[i], vn = svn[i];
          if (RED >= 1 && in && y >= A && y < A + TH && x >= A && x < A + TW) {
            acc.s += (double)e;
            if (RED >= 2) {
              acc.mx = fmaxf(acc.mx, e);
              acc.nmn = fmaxf(acc.nmn, -e);
              acc.wet += (__fadd_rn(sH0[i], e) < hmin) ? 0.0 : 1.0;
              acc.mu = fmaxf(acc.mu, fabsf(un));
              acc.mv = fmaxf(acc.mv, fabsf(vn));
            }
          }
          // commit after everyone's reads of this step's et / un / vn: each
          // cell's new E, U, V are written by its own thread only, and no
          // thread reads E, U, V again before the next P1 barrier
          sE[i] = e;
          sU[i] = un;
          sV[i] = vn;
        }
      }
      if (RED >= 1) {   // CTA fold of this step's partial (deferred fold_steps)
        __shared__ PAcc red_sh[kPThreads / 32];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
          acc.s += __shfl_xor_sync(0xffffffffu, acc.s, m);
          if (RED >= 2) {
            acc.wet += __shfl_xor_sync(0xffffffffu, acc.wet, m);
            acc.mx = fmaxf(acc.mx, __shfl_xor_sync(0xffffffffu, acc.mx, m));
            acc.nmn = fmaxf(acc.nmn, __shfl_xor_sync(0xffffffffu, acc.nmn, m));
            acc.mu = fmaxf(acc.mu, __shfl_xor_sync(0xffffffffu, acc.mu, m));
            acc.mv = fmaxf(acc.mv, __shfl_xor_sync(0xffffffffu, acc.mv, m));
          }
        }
        if (tx == 0) red_sh[ty] = acc;
        __syncthreads();
        if (tid == 0) {
          PAcc t = red_sh[0];
          for (int w = 1; w < kPThreadsY; ++w) {
            t.s += red_sh[w].s;
            t.wet += red_sh[w].wet;
            t.mx = fmaxf(t.mx, red_sh[w].mx);
            t.nmn = fmaxf(t.nmn, red_sh[w].nmn);
            t.mu = fmaxf(t.mu, red_sh[w].mu);
            t.mv = fmaxf(t.mv, red_sh[w].mv);
          }
          RedPartial p;
          p.sum_eta = t.s;
          p.wet = t.wet;
          p.max_eta = t.mx;
          p.neg_min_eta = t.nmn;
          p.max_u = t.mu;
          p.max_v = t.mv;
          a.part[(size_t)step * gridDim.x + tile] = p;
        }
      }
      __syncthreads();
    }
    done += kk;
    b ^= 1;
    // publish the exact centre of the new state, then the tile's counter
    for (int y = A + ty; y < A + TH; y += kPThreadsY) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = x0 + c;
        if (x >= A && x < A + TW && in_grid(y, x)) {
          const int i = y * kPX + x;
          const long long o = gofs(y, x);
          __stcg(a.E[b] + o, sE[i]);
          __stcg(a.U[b] + o, sU[i]);
          __stcg(a.V[b] + o, sV[i]);
        }
      }
    }
    if (done >= a.nsteps) break;
    __syncthreads();
    // (the barrier orders the CTA's stores before thread 0's release, which
    // is cumulative at gpu scope)
    if (tid == 0) st_release(a.flags + (size_t)tile * kPFlagStride, a.flag_base + (unsigned)done);
    // wait for the neighbours' same block (they wrote our apron and are done
    // reading the buffer we write next); each flag sits in its own 128-byte
    // line (no hot L2 slice), and the pollers back off
#ifndef SW2D_PERSIST_NOWAIT   // timing experiments only: wrong results without the wait
    if (nb >= 0) {
#else
    if (false) {
#endif
      const unsigned want = a.flag_base + (unsigned)done;
      const unsigned* f = a.flags + (size_t)nb * kPFlagStride;
      while ((int)(ld_acquire(f) - want) < 0) __nanosleep(32);
    }
    __syncthreads();
    // reload the apron ring (the centre is already here)
    for (int y = ty; y < Y; y += kPThreadsY) {
      const bool rowc = y >= A && y < A + TH;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = x0 + c;
        if (rowc && x >= A && x < A + TW) continue;
        const int i = y * kPX + x;
        float e = 0.0f, u = 0.0f, v = 0.0f;
        if (in_grid(y, x)) {
          const long long o = gofs(y, x);
          e = __ldcg(a.E[b] + o);
          u = __ldcg(a.U[b] + o);
          v = __ldcg(a.V[b] + o);
        }
        sE[i] = e;
        sU[i] = u;
        sV[i] = v;
      }
    }
    __syncthreads();
  }
}

template <int K, int RED>
void persist_attr() {
  static unsigned long long attr_devices = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_devices >> (dev & 63) & 1ull)) {
    // (static + dynamic shared memory must stay within 227 KB per CTA)
    cudaFuncSetAttribute(sw2d_persist<K, RED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPSmemMax);
    attr_devices |= 1ull << (dev & 63);
  }
}

template <int K, int RED>
int persist_capacity_k(int th) {
  persist_attr<K, RED>();
  int per_sm = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (persist_smem_bytes(K, th) > (size_t)kPSmemMax) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sw2d_persist<K, RED>, kPThreads,
                                                    persist_smem_bytes(K, th)) != cudaSuccess) {
    cudaGetLastError();   // not sticky: the planner falls back
    return 0;
  }
  return per_sm * sms;
}

template <int K, int RED>
int launch_persist_k(const PersistArgs& a, cudaStream_t s) {
  persist_attr<K, RED>();
  void* args[] = {const_cast<PersistArgs*>(&a)};
  const cudaError_t e = cudaLaunchCooperativeKernel(
      (const void*)sw2d_persist<K, RED>, dim3((unsigned)(a.ntx * a.nty)),
      dim3(32, kPThreadsY), args, persist_smem_bytes(K, a.th), s);
  return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace

size_t persist_smem_bytes(int K, int th) {
  return (size_t)9 * (size_t)(th + 4 * K) * kPX * sizeof(float);
}

int persist_tile_cols(int K) { return kPX - 4 * K; }

size_t persist_flag_words(int ntiles) { return (size_t)ntiles * kPFlagStride; }

int persist_capacity(int K, int red_level, int th) {
  if (K == 1)
    return red_level >= 2 ? persist_capacity_k<1, 2>(th)
                          : red_level ? persist_capacity_k<1, 1>(th) : persist_capacity_k<1, 0>(th);
  return red_level >= 2 ? persist_capacity_k<2, 2>(th)
                        : red_level ? persist_capacity_k<2, 1>(th) : persist_capacity_k<2, 0>(th);
}

int launch_persist(const PersistArgs& a, int K, int red_level, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (K == 1)
    return red_level >= 2 ? launch_persist_k<1, 2>(a, s)
                          : red_level ? launch_persist_k<1, 1>(a, s) : launch_persist_k<1, 0>(a, s);
  return red_level >= 2 ? launch_persist_k<2, 2>(a, s)
                        : red_level ? launch_persist_k<2, 1>(a, s) : launch_persist_k<2, 0>(a, s);
}

}  // namespace sw2d_dev
