// paper_1711_04471_b200/csrc/sw2d_persist.cu — persistent cooperative kernel
// for the paper's small grids.
//
// The paper times 500^2 .. 2000^2 grids for 10,000 steps.  Their state lives
// in L2 and one step is a few microseconds of work spread over the GPU, so a
// kernel launch (or graph node) per pass and the start-up of a row march
// cost more than the arithmetic.  Here ONE cooperative launch runs many
// steps: every CTA owns a fixed tile of (64 - 4K) x (PW RW - 4K) cells for
// the whole launch and advances it K steps at a time in shared memory (tile
// + 2K-cell apron: the dependency cone of K steps), then
//   * stores the outer ring of the tile's exact centre (all of it after the
//     last block) into the next state buffer (L2),
//   * publishes a per-tile step counter (st.release.gpu, own 128-byte line),
//   * waits until its 8 neighbour tiles have published the same block
//     (ld.acquire.gpu, back-off) — they have then written the apron it needs
//     and finished reading the buffer it will overwrite next,
//   * reloads only its apron ring; the centre stays in shared memory.
// There is no grid-wide barrier and no relaunch.  The blocks wait on one
// another, so the launch is cooperative (all CTAs co-resident, guaranteed by
// the driver) — the one sanctioned form of inter-CTA waiting on one GPU.
//
// A step is three phases separated by CTA barriers: (h, wet, u', v'),
// (etan), (Shapiro filter + commit).  Each thread keeps its 2 x RW cells in
// registers across the phases; x neighbours come from warp shuffles (a warp
// owns a 64-column shared row, 2 columns per lane), y neighbours through
// shared memory.  Every operation is the oracle's, in its order
// (oracle/sw2d_ref.c; the face rule and the exact flag FMAs as in the row
// march, R24): bitwise parity.  Cells outside the grid are dry with zero
// velocity (the closed basin); the apron's outer cells go stale two rings
// per step and never reach the centre.
//
// Diagnostics: per step, each warp folds its centre cells (fp64 sums, exact
// max/min/count) into one partial — no CTA barrier for it; fold_steps folds
// the partials of a launch in a fixed order after it (deterministic; the
// deferred fold of the graphs).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "sw2d_internal.cuh"

namespace sw2d_dev {

namespace {

constexpr int kPX = 64;       // shared tile width: 32 lanes x 2 columns
constexpr int kPFlagStride = 32;        // uints between two tiles' flags (128 B)
constexpr int kPSmemMax = 226 * 1024;   // dynamic shared memory cap (static buffers fit beside)
constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Tagged ring words (PersistArgs::ring, plans with one CTA per SM): a value
// and the step count it belongs to in one 8-byte word, stored and loaded as
// single-copy-atomic relaxed accesses at gpu scope: a reader that sees the
// tag it waits for sees that block's value — no counter, fence or CTA
// barrier between a tile's ring stores and its neighbours' reloads.
__device__ __forceinline__ void st_tagged(unsigned long long* p, unsigned tag, float v) {
  const unsigned long long w =
      ((unsigned long long)tag << 32) | (unsigned long long)__float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tagged(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

#ifndef SW2D_PERSIST_FACE_ARITH
#define SW2D_PERSIST_FACE_ARITH 1
#endif
// the face rule (R4) as exact arithmetic (R26, as in the row march): with
// flags wc, wn in {0, 1}, wc*wn + (wc - wn)*d > 0 iff the face carries flow
__device__ __forceinline__ float p_face_arith(float wc, float wn, float d, float s) {
  const float f = __fmaf_rn(wc, wn, __fmul_rn(__fsub_rn(wc, wn), d));
  return f > 0.0f ? s : 0.0f;
}
// the face rule's predicate program: flow ? s : 0
__device__ __forceinline__ float p_face(float wc, float wn, float d, float s) {
#if SW2D_PERSIST_FACE_ARITH
  return p_face_arith(wc, wn, d, s);
#else
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
#endif
}

// upwind flux s * (s > 0 ? hl : hr): equal in value to the oracle's
// F(s, hl, hr) for finite depths (reading R22)
__device__ __forceinline__ float p_flux(float s, float hl, float hr) {
  return __fmul_rn(s, s > 0.0f ? hl : hr);
}

struct PAcc {
  double s;
  double wet;
  float mx, nmn, mu, mv;
};

// K: steps per block; PW: warps per CTA (warp w owns shared rows w, w + PW,
// ...); RW: shared rows per thread (the shared tile is PW RW rows)
// (8 warps x 2 rows: at most 64 registers, so 4 CTAs fit an SM; 16 warps:
// 64, so 2 fit)
template <int K, int PW, int RW, int RED, bool TAG>
__global__ void __launch_bounds__(32 * PW, (PW == 8 && RW == 2) ? 4 : (PW == 16 ? 2 : 1))
    sw2d_persist(const PersistArgs a) {
  constexpr int A = 2 * K;            // apron cells per side
  constexpr int TW = kPX - 2 * A;     // tile width
  constexpr int Y = PW * RW;          // shared tile rows
  constexpr int TH = Y - 2 * A;       // tile rows
  constexpr int N = Y * kPX;
  extern __shared__ __align__(16) float psm[];
  float* sE = psm;        // eta (the state being advanced; U, V, H0 likewise)
  float* sU = sE + N;
  float* sV = sU + N;
  float* sH0 = sV + N;
  float* sh = sH0 + N;    // h of this step
  float* sw = sh + N;     // wet flags 1/0
  float* svn = sw + N;    // vn (read one row up by etan)
  float* set = svn + N;   // etan

  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int tk = tile % a.ntx, tj = tile / a.ntx;
  const int gk0 = tk * TW + 1 - A;   // global 1-based column of shared column 0
  const int gj0 = tj * TH + 1 - A;   // global 1-based row of shared row 0
  const int nx = a.nx, ny = a.ny;
  const long long pitch = a.pitch;
  const float cy = a.c.cy, cx = a.c.cx, q = a.c.q;
  const int c0 = 2 * lane;           // this thread's columns c0, c0 + 1

  // per-thread constants: in-grid column flags, wall-face coefficients
  // (cgx on faces that are neither walls nor outside, 0 there: the face rule
  // then blocks them, as for the row march), hmin or +inf outside
  float hminc[2], cgxc[2];
  bool colin[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int gk = gk0 + c0 + c;
    colin[c] = gk >= 1 && gk <= nx;
    hminc[c] = colin[c] ? a.c.hmin : __int_as_float(0x7f800000);
    cgxc[c] = (gk >= 1 && gk < nx) ? a.c.cgx : 0.0f;
  }
  float cgyr[RW];
  bool rowin[RW], rowin_n[RW];
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const int gj = gj0 + wp + PW * k;
    rowin[k] = gj >= 1 && gj <= ny;
    rowin_n[k] = gj + 1 >= 1 && gj + 1 <= ny;
    cgyr[k] = (gj >= 1 && gj < ny) ? a.c.cgy : 0.0f;
  }
  auto gofs = [&](int y, int x) -> long long {
    return (long long)(gj0 + y - a.jbase) * pitch + (gk0 + x) + kColOff;
  };
  // tagged ring words: [parity][field][ny][nx], field planes ring_plane apart
  auto rofs = [&](int par, int y, int x) -> long long {
    return (long long)par * 3 * a.ring_plane + (long long)(gj0 + y - 1) * nx + (gk0 + x - 1);
  };
  constexpr bool tagged = TAG;   // tagged ring words (a.ring) instead of counters

  int b = a.cur;   // buffer holding the current state
  // initial load: the whole apron'd tile (zero outside the grid)
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const int y = wp + PW * k, i = y * kPX + c0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float e = 0.0f, h0 = 0.0f, u = 0.0f, v = 0.0f;
      if (rowin[k] && colin[c]) {
        const long long o = gofs(y, c0 + c);
        e = __ldcg(a.E[b] + o);
        h0 = __ldcg(a.H0 + o);
        u = __ldcg(a.U[b] + o);
        v = __ldcg(a.V[b] + o);
      }
      sE[i + c] = e;
      sH0[i + c] = h0;
      sU[i + c] = u;
      sV[i + c] = v;
    }
  }
  __syncthreads();

  // neighbour tiles (8-neighbourhood; -1 when outside)
  int nb = -1;
  if (threadIdx.x < 9 && threadIdx.x != 4) {
    const int dj = threadIdx.x / 3 - 1, dk = threadIdx.x % 3 - 1;
    const int nj = tj + dj, nk = tk + dk;
    if (nj >= 0 && nj < a.nty && nk >= 0 && nk < a.ntx) nb = nj * a.ntx + nk;
  }

  int done = 0;
  while (done < a.nsteps) {
    const int kk = min(K, a.nsteps - done);
    for (int s = 0; s < kk; ++s) {
      const int step = done + s;
      // this thread's cells, kept in registers across the phases
      float e[RW][2], u[RW][2], v[RW][2], h0[RW][2], h[RW][2], w[RW][2], un[RW][2],
          vn[RW][2], et[RW][2];
      // P1: h, wet; un (east faces), vn (north faces)
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const int y = wp + PW * k, i = y * kPX + c0;
        const int iN = min(y + 1, Y - 1) * kPX + c0;   // the last row's north is stale anyway
        const float2 e2 = *reinterpret_cast<const float2*>(sE + i);
        const float2 h02 = *reinterpret_cast<const float2*>(sH0 + i);
        const float2 u2 = *reinterpret_cast<const float2*>(sU + i);
        const float2 v2 = *reinterpret_cast<const float2*>(sV + i);
        const float2 eN2 = *reinterpret_cast<const float2*>(sE + iN);
        const float2 h0N2 = *reinterpret_cast<const float2*>(sH0 + iN);
        e[k][0] = e2.x; e[k][1] = e2.y;
        h0[k][0] = h02.x; h0[k][1] = h02.y;
        u[k][0] = u2.x; u[k][1] = u2.y;
        v[k][0] = v2.x; v[k][1] = v2.y;
        const float eN[2] = {eN2.x, eN2.y}, h0N[2] = {h0N2.x, h0N2.y};
        float wN[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          h[k][c] = __fadd_rn(h0[k][c], e[k][c]);
          w[k][c] = (rowin[k] && !(h[k][c] < hminc[c])) ? 1.0f : 0.0f;
          const float hN = __fadd_rn(h0N[c], eN[c]);
          wN[c] = (rowin_n[k] && !(hN < hminc[c])) ? 1.0f : 0.0f;
        }
        // east neighbours: column c0 + 2 is the next lane's first
        const float eE1 = __shfl_down_sync(kFullMask, e[k][0], 1);
        const float wE1 = __shfl_down_sync(kFullMask, w[k][0], 1);
        const float eE[2] = {e[k][1], eE1}, wE[2] = {w[k][1], wE1};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float du = __fmul_rn(cgxc[c], __fsub_rn(eE[c], e[k][c]));
          un[k][c] = p_face(w[k][c], wE[c], du, __fadd_rn(u[k][c], du));
          const float dv = __fmul_rn(cgyr[k], __fsub_rn(eN[c], e[k][c]));
          vn[k][c] = p_face(w[k][c], wN[c], dv, __fadd_rn(v[k][c], dv));
        }
        *reinterpret_cast<float2*>(sh + i) = make_float2(h[k][0], h[k][1]);
        *reinterpret_cast<float2*>(sw + i) = make_float2(w[k][0], w[k][1]);
        *reinterpret_cast<float2*>(svn + i) = make_float2(vn[k][0], vn[k][1]);
      }
      __syncthreads();
      // P2: etan = (E - cx (Fe - Fw)) - cy (Fn - Fs)
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const int y = wp + PW * k;
        const int iN = min(y + 1, Y - 1) * kPX + c0, iS = max(y - 1, 0) * kPX + c0;
        const float2 hN2 = *reinterpret_cast<const float2*>(sh + iN);
        const float2 hS2 = *reinterpret_cast<const float2*>(sh + iS);
        const float2 vS2 = *reinterpret_cast<const float2*>(svn + iS);
        const float hN[2] = {hN2.x, hN2.y}, hS[2] = {hS2.x, hS2.y}, vS[2] = {vS2.x, vS2.y};
        const float hE1 = __shfl_down_sync(kFullMask, h[k][0], 1);
        const float hW0 = __shfl_up_sync(kFullMask, h[k][1], 1);
        const float uW0 = __shfl_up_sync(kFullMask, un[k][1], 1);
        const float hE[2] = {h[k][1], hE1}, hW[2] = {hW0, h[k][0]}, uW[2] = {uW0, un[k][0]};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float fe = p_flux(un[k][c], h[k][c], hE[c]);
          const float fw = p_flux(uW[c], hW[c], h[k][c]);
          const float fn = p_flux(vn[k][c], h[k][c], hN[c]);
          const float fs = p_flux(vS[c], hS[c], h[k][c]);
          et[k][c] = __fsub_rn(__fsub_rn(e[k][c], __fmul_rn(cx, __fsub_rn(fe, fw))),
                               __fmul_rn(cy, __fsub_rn(fn, fs)));
        }
        *reinterpret_cast<float2*>(set + y * kPX + c0) = make_float2(et[k][0], et[k][1]);
      }
      __syncthreads();
      // P3: Shapiro filter (wet cells), commit
      PAcc acc;
      acc.s = 0.0;
      acc.wet = 0.0;
      acc.mx = __int_as_float(0xff800000);
      acc.nmn = __int_as_float(0xff800000);
      acc.mu = 0.0f;
      acc.mv = 0.0f;
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const int y = wp + PW * k, i = y * kPX + c0;
        const int iN = min(y + 1, Y - 1) * kPX + c0, iS = max(y - 1, 0) * kPX + c0;
        const float2 eN2 = *reinterpret_cast<const float2*>(set + iN);
        const float2 eS2 = *reinterpret_cast<const float2*>(set + iS);
        const float2 wN2 = *reinterpret_cast<const float2*>(sw + iN);
        const float2 wS2 = *reinterpret_cast<const float2*>(sw + iS);
        const float etE1 = __shfl_down_sync(kFullMask, et[k][0], 1);
        const float etW0 = __shfl_up_sync(kFullMask, et[k][1], 1);
        const float wE1 = __shfl_down_sync(kFullMask, w[k][0], 1);
        const float wW0 = __shfl_up_sync(kFullMask, w[k][1], 1);
        const float etE[2] = {et[k][1], etE1}, etW[2] = {etW0, et[k][0]};
        const float wE[2] = {w[k][1], wE1}, wW[2] = {wW0, w[k][0]};
        const float etN[2] = {eN2.x, eN2.y}, etS[2] = {eS2.x, eS2.y};
        const float wN[2] = {wN2.x, wN2.y}, wS[2] = {wS2.x, wS2.y};
        float en[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          // E' = ((1 - q s) etan + q (sel(wE, .) + sel(wW, .))) + q (sel(wN, .) + sel(wS, .));
          // a select sel(w, x) + y is the exact fma(w, x, y) (R24)
          const float sc = __fadd_rn(__fadd_rn(__fadd_rn(wE[c], wW[c]), wN[c]), wS[c]);
          const float t1 = __fmul_rn(__fsub_rn(1.0f, __fmul_rn(q, sc)), et[k][c]);
          const float t2 = __fmul_rn(q, __fmaf_rn(wE[c], etE[c], __fmul_rn(wW[c], etW[c])));
          const float t3 = __fmul_rn(q, __fmaf_rn(wN[c], etN[c], __fmul_rn(wS[c], etS[c])));
          en[c] = w[k][c] != 0.0f ? __fadd_rn(__fadd_rn(t1, t2), t3) : et[k][c];
        }
        *reinterpret_cast<float2*>(sE + i) = make_float2(en[0], en[1]);
        *reinterpret_cast<float2*>(sU + i) = make_float2(un[k][0], un[k][1]);
        *reinterpret_cast<float2*>(sV + i) = make_float2(vn[k][0], vn[k][1]);
        if (RED >= 1 && y >= A && y < A + TH && c0 >= A && c0 < A + TW) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (!(rowin[k] && colin[c])) continue;
            acc.s += (double)en[c];
            if (RED >= 2) {
              acc.mx = fmaxf(acc.mx, en[c]);
              acc.nmn = fmaxf(acc.nmn, -en[c]);
              acc.wet += (__fadd_rn(h0[k][c], en[c]) < a.c.hmin) ? 0.0 : 1.0;
              acc.mu = fmaxf(acc.mu, fabsf(un[k][c]));
              acc.mv = fmaxf(acc.mv, fabsf(vn[k][c]));
            }
          }
        }
      }
      if (RED >= 1) {   // this warp's partial of the step (folded by fold_steps)
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
          acc.s += __shfl_xor_sync(kFullMask, acc.s, m);
          if (RED >= 2) {
            acc.wet += __shfl_xor_sync(kFullMask, acc.wet, m);
            acc.mx = fmaxf(acc.mx, __shfl_xor_sync(kFullMask, acc.mx, m));
            acc.nmn = fmaxf(acc.nmn, __shfl_xor_sync(kFullMask, acc.nmn, m));
            acc.mu = fmaxf(acc.mu, __shfl_xor_sync(kFullMask, acc.mu, m));
            acc.mv = fmaxf(acc.mv, __shfl_xor_sync(kFullMask, acc.mv, m));
          }
        }
        if (lane == 0) {
          RedPartial pr;
          pr.sum_eta = acc.s;
          pr.wet = acc.wet;
          pr.max_eta = acc.mx;
          pr.neg_min_eta = acc.nmn;
          pr.max_u = acc.mu;
          pr.max_v = acc.mv;
          a.part[((size_t)step * gridDim.x + tile) * PW + wp] = pr;
        }
      }
      __syncthreads();
    }
    done += kk;
    b ^= 1;
    // publish the exact centre of the new state, then the tile's counter.
    // Between blocks the neighbours read only the centre's outer ring (A
    // cells wide): that much is stored; after the last block all of it.
    const bool last = done >= a.nsteps;
    const unsigned tag = a.flag_base + (unsigned)done;
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const int y = wp + PW * k;
      if (y < A || y >= A + TH || !rowin[k]) continue;
      const bool yring = y < 2 * A || y >= TH;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = c0 + c;
        if (x >= A && x < A + TW && colin[c] && (last || yring || x < 2 * A || x >= TW)) {
          const int i = y * kPX + x;
          if (tagged && !last) {   // the ring as tagged words (parity b), not the state
            unsigned long long* r = a.ring + rofs(b, y, x);
            st_tagged(r, tag, sE[i]);
            st_tagged(r + a.ring_plane, tag, sU[i]);
            st_tagged(r + 2 * a.ring_plane, tag, sV[i]);
            continue;
          }
          const long long o = gofs(y, x);
          __stcg(a.E[b] + o, sE[i]);
          __stcg(a.U[b] + o, sU[i]);
          __stcg(a.V[b] + o, sV[i]);
        }
      }
    }
    if (last) break;
    if constexpr (tagged) {
      // reload the apron straight from the neighbours' tagged words, each
      // awaited by itself.  The words of parity b are rewritten two blocks
      // later, after the neighbour consumed this tile's next ring, which was
      // stored only after these loads returned (their values feed it)
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const int y = wp + PW * k;
        const bool rowc = y >= A && y < A + TH;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int x = c0 + c;
          if (rowc && x >= A && x < A + TW) continue;
          const int i = y * kPX + x;
          float e = 0.0f, u = 0.0f, v = 0.0f;
          if (rowin[k] && colin[c]) {
            const unsigned long long* r = a.ring + rofs(b, y, x);
            unsigned long long we, wu, wv;
            for (;;) {
              we = ld_tagged(r);
              wu = ld_tagged(r + a.ring_plane);
              wv = ld_tagged(r + 2 * a.ring_plane);
              if ((unsigned)(we >> 32) == tag && (unsigned)(wu >> 32) == tag &&
                  (unsigned)(wv >> 32) == tag)
                break;
              __nanosleep(20);
            }
            e = __uint_as_float((unsigned)we);
            u = __uint_as_float((unsigned)wu);
            v = __uint_as_float((unsigned)wv);
          }
          sE[i] = e;
          sU[i] = u;
          sV[i] = v;
        }
      }
      __syncthreads();
      continue;
    }
    __syncthreads();
    // (the barrier orders the CTA's stores before thread 0's release, which
    // is cumulative at gpu scope)
    if (threadIdx.x == 0)
      st_release(a.flags + (size_t)tile * kPFlagStride, a.flag_base + (unsigned)done);
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
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const int y = wp + PW * k;
      const bool rowc = y >= A && y < A + TH;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = c0 + c;
        if (rowc && x >= A && x < A + TW) continue;
        const int i = y * kPX + x;
        float e = 0.0f, u = 0.0f, v = 0.0f;
        if (rowin[k] && colin[c]) {
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

template <int K, int PW, int RW, int RED, bool TAG>
void persist_attr() {
  static unsigned long long attr_devices = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_devices >> (dev & 63) & 1ull)) {
    // (static + dynamic shared memory must stay within 227 KB per CTA)
    cudaFuncSetAttribute(sw2d_persist<K, PW, RW, RED, TAG>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmemMax);
    attr_devices |= 1ull << (dev & 63);
  }
}

constexpr size_t smem_of(int y) { return (size_t)8 * (size_t)y * kPX * sizeof(float); }

template <int K, int PW, int RW, int RED>
int capacity_t() {   // co-resident CTAs of both handshake variants (the smaller)
  persist_attr<K, PW, RW, RED, false>();
  persist_attr<K, PW, RW, RED, true>();
  int per_sm = 0, per_sm_t = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sw2d_persist<K, PW, RW, RED, false>,
                                                    32 * PW, smem_of(PW * RW)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_t, sw2d_persist<K, PW, RW, RED, true>,
                                                    32 * PW, smem_of(PW * RW)) != cudaSuccess) {
    cudaGetLastError();   // not sticky: the planner falls back
    return 0;
  }
  return (per_sm < per_sm_t ? per_sm : per_sm_t) * sms;
}

template <int K, int PW, int RW, int RED>
int launch_t(const PersistArgs& a, cudaStream_t s) {
  void* args[] = {const_cast<PersistArgs*>(&a)};
  const void* fn = a.ring ? (const void*)sw2d_persist<K, PW, RW, RED, true>
                          : (const void*)sw2d_persist<K, PW, RW, RED, false>;
  if (a.ring)
    persist_attr<K, PW, RW, RED, true>();
  else
    persist_attr<K, PW, RW, RED, false>();
  const cudaError_t e = cudaLaunchCooperativeKernel(fn,
                                                    dim3((unsigned)(a.ntx * a.nty)),
                                                    dim3(32 * PW), args, smem_of(PW * RW), s);
  return e == cudaSuccess ? 0 : (int)e;
}

// the (warps, rows per thread) shapes: 0-2: 16 warps x 1-3 rows, 3-5: 8 warps x 2-4 rows
template <int K, int RED>
int capacity_shape(int shape) {
  switch (shape) {
    case 0: return capacity_t<K, 16, 1, RED>();
    case 1: return capacity_t<K, 16, 2, RED>();
    case 2: return capacity_t<K, 16, 3, RED>();
    case 3: return capacity_t<K, 8, 2, RED>();
    case 4: return capacity_t<K, 8, 3, RED>();
    default: return capacity_t<K, 8, 4, RED>();
  }
}
template <int K, int RED>
int launch_shape(const PersistArgs& a, cudaStream_t s) {
  switch (a.shape) {
    case 0: return launch_t<K, 16, 1, RED>(a, s);
    case 1: return launch_t<K, 16, 2, RED>(a, s);
    case 2: return launch_t<K, 16, 3, RED>(a, s);
    case 3: return launch_t<K, 8, 2, RED>(a, s);
    case 4: return launch_t<K, 8, 3, RED>(a, s);
    default: return launch_t<K, 8, 4, RED>(a, s);
  }
}

}  // namespace

int persist_shapes() { return 6; }
int persist_shape_rows(int shape) {   // shared-tile rows (warps x rows per thread)
  static const int y[6] = {16, 32, 48, 16, 24, 32};
  return y[shape];
}
int persist_shape_warps(int shape) { return shape < 3 ? 16 : 8; }
// a tile must be at least as tall as the apron (2K rows), or the apron would
// reach past the neighbour tile whose counter is awaited: 0 = shape unusable
int persist_tile_rows(int K, int shape) {
  const int th = persist_shape_rows(shape) - 4 * K;
  return th >= 2 * K ? th : 0;
}
int persist_tile_cols(int K) { return kPX - 4 * K; }
size_t persist_flag_words(int ntiles) { return (size_t)ntiles * kPFlagStride; }
size_t persist_ring_words(long long nx, long long ny) { return (size_t)6 * (size_t)nx * (size_t)ny; }

// K = 3, 4 need more than 16 shared rows: shapes 0 and 3 have no usable tile
// rows then (the planner skips them: persist_tile_rows <= 0)
template <int K>
int capacity_k(int red_level, int shape) {
  if (persist_tile_rows(K, shape) <= 0) return 0;
  return red_level >= 2 ? capacity_shape<K, 2>(shape)
                        : red_level ? capacity_shape<K, 1>(shape) : capacity_shape<K, 0>(shape);
}
template <int K>
int launch_k(const PersistArgs& a, int red_level, cudaStream_t s) {
  return red_level >= 2 ? launch_shape<K, 2>(a, s)
                        : red_level ? launch_shape<K, 1>(a, s) : launch_shape<K, 0>(a, s);
}

int persist_capacity(int K, int red_level, int shape) {
  switch (K) {
    case 1: return capacity_k<1>(red_level, shape);
    case 3: return capacity_k<3>(red_level, shape);
    case 4: return capacity_k<4>(red_level, shape);
    default: return capacity_k<2>(red_level, shape);
  }
}

int launch_persist(const PersistArgs& a, int K, int red_level, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (persist_tile_rows(K, a.shape) <= 0) return (int)cudaErrorInvalidValue;
  switch (K) {
    case 1: return launch_k<1>(a, red_level, s);
    case 3: return launch_k<3>(a, red_level, s);
    case 4: return launch_k<4>(a, red_level, s);
    default: return launch_k<2>(a, red_level, s);
  }
}

}  // namespace sw2d_dev
