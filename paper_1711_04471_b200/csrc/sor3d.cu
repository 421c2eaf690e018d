// paper_1711_04471_b200/csrc/sor3d.cu — red-black SOR for the Poisson
// equation on sm_100a (include/sor3d.h).
//
// The UFLES "press" solver of arXiv 1711.04471 §6.3 (PAPER.md:399-401, 418,
// 427-428).  One launch = one full red-black iteration, out of place
// (p_in -> p_out, ping-pong), in a single pass over HBM/L2:
//
//   * A CTA owns an output tile of 60 x 28 (x, y) columns and a z-chunk of
//     KZ planes.  It marches up the planes with a 64 x 32 "extended" tile
//     (2-cell apron in x and y).  512 threads: each half-warp is one row of
//     16 lanes and each lane an x-quad (one float4), so a row's x neighbours
//     come from half-warp shuffles and its y neighbours through shared
//     memory; each lane updates two cells of each colour.
//   * Step m of the march: the red cells of plane m are updated over the
//     tile + 1-cell apron from p_in (z neighbours from a register window);
//     the black cells of plane m-1 are updated over the tile from the new red
//     values of planes m-2, m-1, m; plane m-1 is stored.  Red cells of plane
//     m and black cells of plane m-1 sit at the same two lanes of a quad, so
//     each step has one static shape per parity.  The apron recomputes the
//     neighbours' red cells, so no CTA waits for another and the result is
//     exactly the sequential red-then-black sweep (cells of one colour do not
//     depend on each other).  One barrier per step (double-buffered shared
//     planes); the march is unrolled by 4 (the register window's period).
//   * The residual of p_in (the state after the previous iteration) uses the
//     same loads: its neighbour sum is the red update's.  A record is folded
//     per CTA (fp64 sum of r^2, fp32 max |r|) and the last CTA folds the
//     partials in a fixed order (deterministic) into the history ring.
//   * When p and rhs fit in 70% of L2, loads of p_in carry an evict-first
//     and loads of rhs / stores of p_out an evict-last L2 policy.  Measured
//     without effect at 300 x 300 x 90: the 97 MB ping-pong footprint is
//     above what L2 keeps for a streaming pattern.
//
// Every operation is the oracle's (oracle/sor_ref.c), in the same order and
// precision (explicit round-to-nearest intrinsics, built with --fmad=false):
// bitwise parity of p.  Padded storage (zeros) makes every load in-bounds.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sor3d.h"
#include <nvtx3/nvToolsExt.h>

namespace sor3d_dev {

constexpr int kSx = 16;                     // lanes per row (x-quads); rows per CTA: R = 32 or 16
constexpr int kOutX = 4 * kSx - 4;          // 60 output columns per tile
constexpr int kColOff = 1;                  // storage column of interior i is i + 1
constexpr int kRowOff = 1;                  // storage row of interior j is j + 1
constexpr int kPlaneOff = 2;                // storage plane of interior k is k + 2
constexpr unsigned kFull = 0xffffffffu;
static_assert(kSx == 16, "rows are half-warps; a warp holds two rows of equal parity");

struct Part {
  double s;
  float mx;
  float pad;
};

struct Red {
  Part* part;
  unsigned* counter;
  double* rec;  // 2 doubles: L2, Linf
  int expected;
};

struct Args {
  const float* pin;
  float* pout;
  const float* rhs;
  long long pitch, plane;  // elements
  int nx, ny, nz, kz;
  float cx, cy, cz, dd, invd, om, om1;
  float negz;  // -0.0f: the packed products' addend (a parameter: opaque to ptxas)
  Red red;
};

__device__ __forceinline__ float upd(float p, float ns, float rh, const Args& a) {
  // oracle: om1 * p + om * ((nsum - rhs) * invd)
  return __fadd_rn(__fmul_rn(a.om1, p), __fmul_rn(a.om, __fmul_rn(__fsub_rn(ns, rh), a.invd)));
}

// nsum = (cx*(E+W) + cy*(N+S)) + cz*(U+D)
__device__ __forceinline__ float nsum(float e, float w, float n, float s, float u, float d,
                                      const Args& a) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a.cx, __fadd_rn(e, w)), __fmul_rn(a.cy, __fadd_rn(n, s))),
                   __fmul_rn(a.cz, __fadd_rn(u, d)));
}


template <int NT>
__device__ void fold(double s, float mx, const Red& r) {
  __shared__ double shs[NT / 32];
  __shared__ float shm[NT / 32];
  __shared__ bool last;
  constexpr int NW = NT / 32;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    s += __shfl_xor_sync(kFull, s, o);
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if (lane == 0) {
    shs[warp] = s;
    shm[warp] = mx;
  }
  __syncthreads();
  if (t == 0) {
    double bs = shs[0];
    float bm = shm[0];
    for (int w = 1; w < NW; ++w) {
      bs += shs[w];
      bm = fmaxf(bm, shm[w]);
    }
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    r.part[cta].s = bs;
    r.part[cta].mx = bm;
    __threadfence();
    last = atomicAdd(r.counter, 1u) == (unsigned)(r.expected - 1);
  }
  __syncthreads();
  if (!last) return;  // block-uniform
  __threadfence();
  double fs = 0.0;
  float fm = 0.0f;
  for (int i = t; i < r.expected; i += NT) {
    const volatile Part* p = r.part + i;
    fs += p->s;
    fm = fmaxf(fm, p->mx);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    fs += __shfl_xor_sync(kFull, fs, o);
    fm = fmaxf(fm, __shfl_xor_sync(kFull, fm, o));
  }
  __syncthreads();
  if (lane == 0) {
    shs[warp] = fs;
    shm[warp] = fm;
  }
  __syncthreads();
  if (t == 0) {
    double bs = shs[0];
    float bm = shm[0];
    for (int w = 1; w < NW; ++w) {
      bs += shs[w];
      bm = fmaxf(bm, shm[w]);
    }
    r.rec[0] = sqrt(bs);
    r.rec[1] = bm;
    *r.counter = 0u;  // ready for the next record (stream-ordered)
  }
}

// L2 eviction-priority hints (createpolicy + ld/st .L2::cache_hint).  Used
// when p and rhs fit in L2 together: p_in is dead after its last read (the
// next iteration overwrites it), rhs and p_out are read again by the next
// iteration.
template <bool LAST>
__device__ __forceinline__ uint64_t l2pol() {
  uint64_t p;
  if (LAST)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <bool H, bool LAST>
__device__ __forceinline__ float4 ldh(const float* p) {
  if (!H) return __ldg(reinterpret_cast<const float4*>(p));
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(l2pol<LAST>()));
  return v;
}
template <bool H>
__device__ __forceinline__ void sth(float* p, float4 v) {
  if (!H) {
    *reinterpret_cast<float4*>(p) = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(l2pol<true>()) : "memory");
}

// shared-memory quad read (kept as a call site marker for the SASS maps)
__device__ __forceinline__ float4 lds4(const float4* p) { return *p; }

#ifndef SOR_MINB
#define SOR_MINB(R) (64 / (R))  // 1024 threads per SM: at most 64 registers
#endif

// Per-thread state of the z-march: p_in planes m-1 .. m+2, rhs planes
// m-1 .. m+2, new (red-updated) planes m-2, m-1, and the stream pointers.
struct March {
  float4 pz0, pz1, pz2, pf;
  float4 r1, r2, rf1, rf2;
  float4 n0, n1;
  // the three streams: without the residual, one 32-bit element offset of
  // this lane's quad in plane m+3 (p_in and rhs; p_out plane m-1 is ofs - 4
  // planes; sor3d_create keeps arrays below 2^31 elements); with it, three
  // pointers (each form measured best for its variant)
  unsigned ofs;
  const float* pp;  // p_in plane m+3
  const float* rp;  // rhs plane m+3
  float* op;        // p_out plane m-1
  double acc;
  float amx;
};

// Storage slot of cell c (0..3) of an aligned x-quad: the packed layout
// (SOR_PACKED, below) keeps a quad (c0, c1, c2, c3) as (c0, c2, c1, c3).
#ifndef SOR_PACKED
#define SOR_PACKED 1
#endif
__host__ __device__ constexpr int slot(int c) {
  return SOR_PACKED ? (c == 1 ? 2 : (c == 2 ? 1 : c)) : c;
}
__device__ __forceinline__ float& comp(float4& v, int c) {
  const int k = slot(c);
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
__device__ __forceinline__ float compv(const float4& v, int c) {
  const int k = slot(c);
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

struct Lane {
  int m0;        // first plane of the march (k0 - 1)
  int k0, k1;    // output planes
  int nz;
  long long plane;
  int intr;      // bit c: cell c is an interior cell (the red update applies)
  int outm;      // bit c: cell c is an output cell (tile, interior): stored
  bool all4;     // outm == 15
  bool anyout;   // outm != 0
  int tx, ty;
  int yn, ys;
};

// One step of the march at plane m (step index S: compile-time parity; P =
// (i0 + j + m) & 1 is the class of the cells updated in this step: red cells
// of plane m and black cells of plane m-1 both sit at c = P, P + 2).
template <int R, int P, int S, bool RES, bool WRITE, bool H>
__device__ __forceinline__ void step(March& st, const Lane& L, const Args& a, int m,
                                     float4 (*s_in)[R][kSx], float4 (*s_new)[R][kSx]) {
  const int tx = L.tx, ty = L.ty;
  // One barrier per step: s_in and s_new are double-buffered by step parity,
  // so this barrier publishes s_in(m) and s_new(m-1) and retires every read
  // of the buffers the step writes (last read in step m-1).
  s_in[S][ty][tx] = st.pz1;
  __syncthreads();
  const float4 N = lds4(&s_in[S][L.yn][tx]), S4 = lds4(&s_in[S][L.ys][tx]);
  // the x neighbour outside the lane's quad: W of cell 0 (P = 0) or E of cell 3
  const float xo = P == 0 ? __shfl_up_sync(kFull, st.pz1.w, 1, kSx)
                          : __shfl_down_sync(kFull, st.pz1.x, 1, kSx);
  float4 pn = st.pz1;
  const bool mint = m >= 1 && m <= L.nz;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const bool upd_here = (c & 1) == P;
    if (!upd_here && !RES) continue;
    float W, E;
    if (upd_here) {
      W = c == 0 ? xo : compv(st.pz1, c - 1);
      E = c == 3 ? xo : compv(st.pz1, c + 1);
    } else {  // residual only: the other two cells (their x neighbours are in the quad or shuffled)
      W = c == 0 ? __shfl_up_sync(kFull, st.pz1.w, 1, kSx) : compv(st.pz1, c - 1);
      E = c == 3 ? __shfl_down_sync(kFull, st.pz1.x, 1, kSx) : compv(st.pz1, c + 1);
    }
    const float ns = nsum(E, W, compv(N, c), compv(S4, c), compv(st.pz2, c), compv(st.pz0, c), a);
    // red update of interior cells (apron cells outside the box are never read)
    if (upd_here && mint && (L.intr >> c & 1)) comp(pn, c) = upd(compv(st.pz1, c), ns, compv(st.r2, c), a);
    if (RES && m >= L.k0 && m <= L.k1 && (L.outm >> c & 1)) {
      const float r = __fsub_rn(compv(st.r2, c), __fsub_rn(ns, __fmul_rn(a.dd, compv(st.pz1, c))));
      st.acc = fma((double)r, (double)r, st.acc);
      st.amx = fmaxf(st.amx, fabsf(r));
    }
  }
  if (WRITE) {
    s_new[S][ty][tx] = pn;  // read by the black phase of step m+1
    const float4 Nb = lds4(&s_new[S ^ 1][L.yn][tx]), Sb = lds4(&s_new[S ^ 1][L.ys][tx]);
    const float xb = P == 0 ? __shfl_up_sync(kFull, st.n1.w, 1, kSx)
                            : __shfl_down_sync(kFull, st.n1.x, 1, kSx);
    if (m - 1 >= L.k0 && m - 1 <= L.k1) {
      // black cells of plane m-1 (computed everywhere, stored on output cells)
      float4 o = st.n1;
#pragma unroll
      for (int c = P; c < 4; c += 2) {
        const float W = c == 0 ? xb : compv(st.n1, c - 1);
        const float E = c == 3 ? xb : compv(st.n1, c + 1);
        const float ns = nsum(E, W, compv(Nb, c), compv(Sb, c), compv(pn, c), compv(st.n0, c), a);
        comp(o, c) = upd(compv(st.n1, c), ns, compv(st.r1, c), a);
      }
      if constexpr (RES) {
        if (L.outm == 15) {
          sth<H>(st.op, o);
        } else if (L.outm) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (L.outm >> c & 1) st.op[slot(c)] = compv(o, c);
        }
      } else {
        float* op = a.pout + (st.ofs - 4u * (unsigned)L.plane);
        if (L.all4) {
          sth<H>(op, o);
        } else if (L.anyout) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (L.outm >> c & 1) op[slot(c)] = compv(o, c);
        }
      }
    }
  }
  // rotate the z window, prefetch plane m+3
  st.pz0 = st.pz1;
  st.pz1 = st.pz2;
  st.pz2 = st.pf;
  st.pf = ldh<H, false>(RES ? st.pp : a.pin + st.ofs);
  st.r1 = st.r2;
  st.r2 = st.rf1;
  st.rf1 = st.rf2;
  st.rf2 = ldh<H, true>(RES ? st.rp : a.rhs + st.ofs);
  st.n0 = st.n1;
  st.n1 = pn;
  if constexpr (RES) {
    st.pp += L.plane;
    st.rp += L.plane;
    st.op += L.plane;
  } else {
    st.ofs += (unsigned)L.plane;
  }
}

// --- packed form (SOR_PACKED): the storage keeps each aligned x-quad of
// cells (c0, c1, c2, c3) as (c0, c2, c1, c3), so a lane's float4 holds the
// pair of one colour in .x/.y (c0, c2) and the other in .z/.w (c1, c3): the
// two cells of one colour in a step are one register pair and every
// operation of their update is one paired instruction (FADD2, and FFMA2
// with a -0 addend for the products, rounding like mul.rn: the 2DSW
// kernel's R25).  Same operations per cell, same order: bitwise.
struct f2 {
  float a, b;
};
__device__ __forceinline__ f2 add2(f2 x, f2 y) {
  f2 r;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(r.a), "=f"(r.b) : "f"(x.a), "f"(x.b), "f"(y.a), "f"(y.b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 x, f2 y) {
  f2 r;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(r.a), "=f"(r.b) : "f"(x.a), "f"(x.b), "f"(y.a), "f"(y.b));
  return r;
}
// c * x (c broadcast) rounded once: fma(c, x, -0)
__device__ __forceinline__ f2 mul2(float c, f2 x, float nz) {
  f2 r;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%2};\n\tmov.b64 rb, {%3,%4};\n\t"
      "mov.b64 rc, {%5,%5};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(r.a), "=f"(r.b) : "f"(c), "f"(x.a), "f"(x.b), "f"(nz));
  return r;
}
// nsum = (cx (E + W) + cy (N + S)) + cz (U + D), per element as nsum()
__device__ __forceinline__ f2 nsum2(f2 e, f2 w, f2 n, f2 s, f2 u, f2 d, const Args& a) {
  return add2(add2(mul2(a.cx, add2(e, w), a.negz), mul2(a.cy, add2(n, s), a.negz)),
              mul2(a.cz, add2(u, d), a.negz));
}
// om1 p + om ((nsum - rhs) invd), per element as upd()
__device__ __forceinline__ f2 upd2(f2 p, f2 ns, f2 rh, const Args& a) {
  return add2(mul2(a.om1, p, a.negz), mul2(a.om, mul2(a.invd, sub2(ns, rh), a.negz), a.negz));
}
__device__ __forceinline__ f2 lo(const float4& v) { return f2{v.x, v.y}; }   // cells 0, 2
__device__ __forceinline__ f2 hi(const float4& v) { return f2{v.z, v.w}; }   // cells 1, 3
template <int P>
__device__ __forceinline__ f2 cls(const float4& v) { return P ? hi(v) : lo(v); }
template <int P>
__device__ __forceinline__ void set_cls(float4& v, f2 x) {
  if (P) { v.z = x.a; v.w = x.b; } else { v.x = x.a; v.y = x.b; }
}
// x neighbours of the colour-P pair of quad q (cells P, P+2): W, E pairs.
// prev_w: the previous lane's cell 3 (.w), next_x: the next lane's cell 0 (.x)
template <int P>
__device__ __forceinline__ void xnb(const float4& q, float prev_w, float next_x, f2& w, f2& e) {
  if (P == 0) {   // cells 0, 2: W = (c-1, c1), E = (c1, c3)
    w = f2{prev_w, q.z};
    e = hi(q);
  } else {        // cells 1, 3: W = (c0, c2), E = (c2, c4)
    w = lo(q);
    e = f2{q.y, next_x};
  }
}

// One march step in the packed form (see step()): the same schedule, the
// updated class of the step is the register pair cls<P>.
template <int R, int P, int S, bool RES, bool WRITE, bool H>
__device__ __forceinline__ void step_packed(March& st, const Lane& L, const Args& a, int m,
                                            float4 (*s_in)[R][kSx], float4 (*s_new)[R][kSx]) {
  const int tx = L.tx, ty = L.ty;
  s_in[S][ty][tx] = st.pz1;
  __syncthreads();
  const float4 N = lds4(&s_in[S][L.yn][tx]), S4 = lds4(&s_in[S][L.ys][tx]);
  const float pw = __shfl_up_sync(kFull, st.pz1.w, 1, kSx);
  const float nxv = __shfl_down_sync(kFull, st.pz1.x, 1, kSx);
  float4 pn = st.pz1;
  const bool mint = m >= 1 && m <= L.nz;
  {
    f2 w, e;
    xnb<P>(st.pz1, pw, nxv, w, e);
    const f2 ns = nsum2(e, w, cls<P>(N), cls<P>(S4), cls<P>(st.pz2), cls<P>(st.pz0), a);
    const f2 nv = upd2(cls<P>(st.pz1), ns, cls<P>(st.r2), a);
    // red update of interior cells (apron cells outside the box are never read)
    const f2 old = cls<P>(st.pz1);
    const int b0 = L.intr >> P & 1, b1 = L.intr >> (P + 2) & 1;
    set_cls<P>(pn, f2{(mint && b0) ? nv.a : old.a, (mint && b1) ? nv.b : old.b});
    if (RES && m >= L.k0 && m <= L.k1) {
      // residual r = rhs - (nsum - dd p) of all four cells: this class, then the other
      const f2 r1 = sub2(cls<P>(st.r2), sub2(ns, mul2(a.dd, cls<P>(st.pz1), a.negz)));
      f2 w2, e2;
      xnb<P ^ 1>(st.pz1, pw, nxv, w2, e2);
      const f2 ns2 = nsum2(e2, w2, cls<P ^ 1>(N), cls<P ^ 1>(S4), cls<P ^ 1>(st.pz2),
                           cls<P ^ 1>(st.pz0), a);
      const f2 r2 = sub2(cls<P ^ 1>(st.r2), sub2(ns2, mul2(a.dd, cls<P ^ 1>(st.pz1), a.negz)));
      const float rr[4] = {r1.a, r1.b, r2.a, r2.b};
      const int cc[4] = {P, P + 2, P ^ 1, (P ^ 1) + 2};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (L.outm >> cc[t] & 1) {
          st.acc = fma((double)rr[t], (double)rr[t], st.acc);
          st.amx = fmaxf(st.amx, fabsf(rr[t]));
        }
    }
  }
  if (WRITE) {
    s_new[S][ty][tx] = pn;  // read by the black phase of step m+1
    const float4 Nb = lds4(&s_new[S ^ 1][L.yn][tx]), Sb = lds4(&s_new[S ^ 1][L.ys][tx]);
    const float pwb = __shfl_up_sync(kFull, st.n1.w, 1, kSx);
    const float nxb = __shfl_down_sync(kFull, st.n1.x, 1, kSx);
    if (m - 1 >= L.k0 && m - 1 <= L.k1) {
      // black cells of plane m-1 (computed everywhere, stored on output cells)
      float4 o = st.n1;
      f2 w, e;
      xnb<P>(st.n1, pwb, nxb, w, e);
      const f2 ns = nsum2(e, w, cls<P>(Nb), cls<P>(Sb), cls<P>(pn), cls<P>(st.n0), a);
      set_cls<P>(o, upd2(cls<P>(st.n1), ns, cls<P>(st.r1), a));
      float* op = RES ? st.op : a.pout + (st.ofs - 4u * (unsigned)L.plane);
      if (L.all4) {
        sth<H>(op, o);
      } else if (L.anyout) {
        // storage slot k of the quad holds cell (0, 2, 1, 3)[k]
        if (L.outm & 1) op[0] = o.x;
        if (L.outm & 4) op[1] = o.y;
        if (L.outm & 2) op[2] = o.z;
        if (L.outm & 8) op[3] = o.w;
      }
    }
  }
  st.pz0 = st.pz1;
  st.pz1 = st.pz2;
  st.pz2 = st.pf;
  st.pf = ldh<H, false>(RES ? st.pp : a.pin + st.ofs);
  st.r1 = st.r2;
  st.r2 = st.rf1;
  st.rf1 = st.rf2;
  st.rf2 = ldh<H, true>(RES ? st.rp : a.rhs + st.ofs);
  st.n0 = st.n1;
  st.n1 = pn;
  if constexpr (RES) {
    st.pp += L.plane;
    st.rp += L.plane;
    st.op += L.plane;
  } else {
    st.ofs += (unsigned)L.plane;
  }
}

template <int R, int P0, bool RES, bool WRITE, bool H>
__device__ __forceinline__ void march(March& st, const Lane& L, const Args& a, int nsteps,
                                      float4 (*s_in)[R][kSx], float4 (*s_new)[R][kSx]) {
  for (int s = 0; s < nsteps; s += 4) {
    const int m = L.m0 + s;
    // the packed step where it measured faster: without the residual (its
    // extra registers spill the residual variants at 64 per thread), on
    // L2-resident grids (H; sor300 2.46e11 -> 2.78e11, sor1024 slower)
    if constexpr (SOR_PACKED && !RES && H) {
      step_packed<R, P0, 0, RES, WRITE, H>(st, L, a, m, s_in, s_new);
      step_packed<R, P0 ^ 1, 1, RES, WRITE, H>(st, L, a, m + 1, s_in, s_new);
      step_packed<R, P0, 0, RES, WRITE, H>(st, L, a, m + 2, s_in, s_new);
      step_packed<R, P0 ^ 1, 1, RES, WRITE, H>(st, L, a, m + 3, s_in, s_new);
    } else {
      step<R, P0, 0, RES, WRITE, H>(st, L, a, m, s_in, s_new);
      step<R, P0 ^ 1, 1, RES, WRITE, H>(st, L, a, m + 1, s_in, s_new);
      step<R, P0, 0, RES, WRITE, H>(st, L, a, m + 2, s_in, s_new);
      step<R, P0 ^ 1, 1, RES, WRITE, H>(st, L, a, m + 3, s_in, s_new);
    }
  }
}

// RES: fold the residual of p_in; WRITE: perform the iteration (else a
// residual-only pass).  Thread (tx, ty) holds the x-quad x = 4tx .. 4tx+3 of
// row y = ty of the extended 128 x 16 tile.
template <int R, bool RES, bool WRITE, bool H>
__global__ void __launch_bounds__(kSx * R, SOR_MINB(R)) sor_iter(const Args a) {
  __shared__ float4 s_in[2][R][kSx];
  __shared__ float4 s_new[2][R][kSx];
  // Row of the extended tile: a warp holds two rows of equal parity (half-warp
  // h of warp w is row 4 (w / 2) + (w % 2) + 2 h), so the red/black shape of
  // a step is warp-uniform.
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = lane & (kSx - 1);
  const int ty = 4 * (w >> 1) + (w & 1) + 2 * (lane >> 4);
  const int i0 = blockIdx.x * kOutX + 4 * tx - 1;  // 1-based i of cell 0 (odd)
  const int j = blockIdx.y * (R - 4) + ty - 1;     // 1-based j
  Lane L;
  L.k0 = blockIdx.z * a.kz + 1;
  L.k1 = min(L.k0 + a.kz - 1, a.nz);
  L.m0 = L.k0 - 1;
  L.nz = a.nz;
  L.plane = a.plane;
  const bool rowin = j >= 1 && j <= a.ny;
  const bool outy = ty >= 2 && ty <= R - 3;
  L.intr = 0;
  L.outm = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int x = 4 * tx + c, i = i0 + c;
    const bool in = rowin && i >= 1 && i <= a.nx;
    if (in) L.intr |= 1 << c;
    if (in && outy && x >= 2 && x <= 4 * kSx - 3) L.outm |= 1 << c;
  }
  L.all4 = L.outm == 15;
  L.anyout = L.outm != 0;
  L.tx = tx;
  L.ty = ty;
  L.yn = min(ty + 1, R - 1);
  L.ys = max(ty - 1, 0);

  const long long col = (long long)(j + kRowOff) * a.pitch + (i0 + kColOff);
  auto at = [&](int k) { return (long long)(k + kPlaneOff) * a.plane + col; };
  March st;
  st.pz0 = ldh<H, false>(a.pin + at(L.k0 - 2));
  st.pz1 = ldh<H, false>(a.pin + at(L.k0 - 1));
  st.pz2 = ldh<H, false>(a.pin + at(L.k0));
  st.pf = ldh<H, false>(a.pin + at(L.k0 + 1));
  st.r1 = ldh<H, true>(a.rhs + at(L.k0 - 2));
  st.r2 = ldh<H, true>(a.rhs + at(L.k0 - 1));
  st.rf1 = ldh<H, true>(a.rhs + at(L.k0));
  st.rf2 = ldh<H, true>(a.rhs + at(L.k0 + 1));
  st.n0 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  st.n1 = st.n0;
  if constexpr (RES) {
    st.pp = a.pin + at(L.k0 + 2);
    st.rp = a.rhs + at(L.k0 + 2);
    st.op = a.pout + at(L.k0 - 2);
  } else {
    st.ofs = (unsigned)at(L.k0 + 2);
  }
  st.acc = 0.0;
  st.amx = 0.0f;
  const int nsteps = L.k1 - L.k0 + 3;  // m = k0-1 .. k1+1 (rounded up to 4: extra steps store nothing)
  if (((i0 + j + L.m0) & 1) == 0)
    march<R, 0, RES, WRITE, H>(st, L, a, nsteps, s_in, s_new);
  else
    march<R, 1, RES, WRITE, H>(st, L, a, nsteps, s_in, s_new);
  if (RES) fold<kSx * R>(st.acc, st.amx, a.red);
}

}  // namespace sor3d_dev

// ---------------------------------------------------------------------------
// Host runtime (C ABI)
// ---------------------------------------------------------------------------

using namespace sor3d_dev;

struct sor3d {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t nx = 0, ny = 0, nz = 0;
  float cx = 0, cy = 0, cz = 0, dd = 0, invd = 0, om = 0, om1 = 0;
  int gx = 0, gy = 0, gz = 0, kz = 0;
  long long pitch = 0, rows = 0, planes = 0, plane = 0;
  float* p[2] = {nullptr, nullptr};
  float* rhs = nullptr;
  int cur = 0;
  Part* part = nullptr;
  unsigned* counter = nullptr;
  double* hist = nullptr;  // [cap][2]
  double* scratch = nullptr;  // [2] for sor3d_residual
  float* stage = nullptr;     // dense staging buffer for host uploads/downloads (lazy)
  int cap = 0;
  int rows_cta = 32;  // extended tile rows (CTA = 16 x rows_cta threads)
  bool hint = false;  // L2 eviction hints (p and rhs fit in L2)
  int64_t nrec = 0;
  bool have_state = false;
  int64_t nlaunch = 0;
  int sticky = 0;
  std::string err, plan;
};

namespace {

thread_local std::string t_create_err;

struct NvtxRange {  // NVTX range over an API call
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int fail(sor3d* h, int code, const std::string& msg) {
  if (h) {
    h->err = msg;
    if (code == SOR3D_ECUDA) h->sticky = code;
  } else {
    t_create_err = msg;
  }
  return code;
}

#define SOR_TRY(h, call)                                                        \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return fail((h), e_ == cudaErrorMemoryAllocation ? SOR3D_ENOMEM : SOR3D_ECUDA, \
                  std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

#define SOR_ENTER(h)                         \
  do {                                       \
    if (!(h)) return SOR3D_EINVAL;           \
    if ((h)->sticky) return (h)->sticky;     \
    SOR_TRY((h), cudaSetDevice((h)->device)); \
  } while (0)

bool finite_pos(float x) { return std::isfinite(x) && x > 0.0f; }

Args make_args(const sor3d* h) {
  Args a;
  a.pin = h->p[h->cur];
  a.pout = h->p[h->cur ^ 1];
  a.rhs = h->rhs;
  a.pitch = h->pitch;
  a.plane = h->plane;
  a.nx = (int)h->nx;
  a.ny = (int)h->ny;
  a.nz = (int)h->nz;
  a.kz = h->kz;
  a.cx = h->cx;
  a.cy = h->cy;
  a.cz = h->cz;
  a.dd = h->dd;
  a.invd = h->invd;
  a.om = h->om;
  a.om1 = h->om1;
  a.negz = -0.0f;
  a.red.part = h->part;
  a.red.counter = h->counter;
  a.red.rec = nullptr;
  a.red.expected = h->gx * h->gy * h->gz;
  return a;
}

// one launch: WRITE = iterate (and swap), RES = fold the residual of p_in into rec
int launch(sor3d* h, bool write, double* rec) {
  Args a = make_args(h);
  a.red.rec = rec;
  void (*k)(const Args);
  if (h->rows_cta == 16) {
    if (h->hint)
      k = write ? (rec ? sor_iter<16, true, true, true> : sor_iter<16, false, true, true>)
                : sor_iter<16, true, false, true>;
    else
      k = write ? (rec ? sor_iter<16, true, true, false> : sor_iter<16, false, true, false>)
                : sor_iter<16, true, false, false>;
  } else {
    if (h->hint)
      k = write ? (rec ? sor_iter<32, true, true, true> : sor_iter<32, false, true, true>)
                : sor_iter<32, true, false, true>;
    else
      k = write ? (rec ? sor_iter<32, true, true, false> : sor_iter<32, false, true, false>)
                : sor_iter<32, true, false, false>;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)h->gx, (unsigned)h->gy, (unsigned)h->gz);
  cfg.blockDim = dim3(kSx * h->rows_cta);
  cfg.stream = h->stream;
  SOR_TRY(h, cudaLaunchKernelEx(&cfg, k, a));
  ++h->nlaunch;
  SOR_TRY(h, cudaGetLastError());
  if (write) h->cur ^= 1;
  return SOR3D_OK;
}

double* next_record(sor3d* h) {
  double* r = h->hist + 2 * (h->nrec % h->cap);
  ++h->nrec;
  return r;
}

// storage index of a cell at padded position x (rows and planes are whole
// quads): the packed layout keeps quad (c0, c1, c2, c3) as (c0, c2, c1, c3)
__device__ __forceinline__ long long store_slot(long long x) {
#if SOR_PACKED
  const int q = (int)(x & 3);
  return (x & ~3LL) | (q == 1 ? 2 : (q == 2 ? 1 : q));
#else
  return x;
#endif
}

// Dense [nz][ny][nx] <-> padded storage, one grid-stride pass: TO_PAD also
// counts non-finite values (sor3d_set's check).
template <bool TO_PAD>
__global__ void repack(float* pad, const float* din, float* dout, int nx, int ny, long long rows,
                       long long pitch, long long plane, unsigned* bad) {
  unsigned nb = 0;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const long long k = row / ny, j = row % ny;
    const long long po = (k + 1 + kPlaneOff) * plane + (j + 1 + kRowOff) * pitch + 1 + kColOff;
    const long long dofs = row * nx;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      const long long q = store_slot(po + i);
      if (TO_PAD) {
        const float v = din[dofs + i];
        nb += !isfinite(v);
        pad[q] = v;
      } else {
        dout[dofs + i] = pad[q];
      }
    }
  }
  if (TO_PAD && nb) atomicAdd(bad, nb);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void free_all(sor3d* h) {
  cudaFree(h->p[0]);
  cudaFree(h->p[1]);
  cudaFree(h->rhs);
  cudaFree(h->part);
  cudaFree(h->counter);
  cudaFree(h->hist);
  cudaFree(h->scratch);
  cudaFree(h->stage);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
}

// host arrays go through a dense device staging buffer (one contiguous copy)
// and a repack kernel; device arrays are repacked directly
int upload(sor3d* h, float* pad, const float* src, unsigned* bad) {
  const long long n = h->nx * h->ny * h->nz;
  const float* d = src;
  if (!is_device_ptr(src)) {
    if (!h->stage) SOR_TRY(h, cudaMalloc(&h->stage, (size_t)n * sizeof(float)));
    SOR_TRY(h, cudaMemcpyAsync(h->stage, src, (size_t)n * sizeof(float), cudaMemcpyDefault,
                               h->stream));
    d = h->stage;
  }
  const long long rows = h->ny * h->nz;
  repack<true><<<(unsigned)std::min<long long>(rows, 148 * 16), 256, 0, h->stream>>>(
      pad, d, nullptr, (int)h->nx, (int)h->ny, rows, h->pitch, h->plane, bad);
  SOR_TRY(h, cudaGetLastError());
  return SOR3D_OK;
}

}  // namespace

extern "C" {

int sor3d_abi_version(void) { return SOR3D_ABI_VERSION; }

int sor3d_create(const sor3d_params* prm, void* cuda_stream, sor3d** out) {
  if (!out) return fail(nullptr, SOR3D_EINVAL, "out is NULL");
  *out = nullptr;
  if (!prm) return fail(nullptr, SOR3D_EINVAL, "params is NULL");
  const int64_t lim = 1LL << 20;
  if (prm->nx < 1 || prm->ny < 1 || prm->nz < 1 || prm->nx > lim || prm->ny > lim || prm->nz > lim)
    return fail(nullptr, SOR3D_EINVAL, "nx, ny, nz must be in [1, 2^20]");
  if (!finite_pos(prm->dx) || !finite_pos(prm->dy) || !finite_pos(prm->dz))
    return fail(nullptr, SOR3D_EINVAL, "dx, dy, dz must be finite and > 0");
  if (!(prm->omega > 0.0f && prm->omega < 2.0f))
    return fail(nullptr, SOR3D_EINVAL, "omega must be in (0, 2)");
  if (prm->history_len < 0) return fail(nullptr, SOR3D_EINVAL, "history_len must be >= 0");
  sor3d* h = new sor3d();
  auto bail = [&](int rc) {
    t_create_err = h->err;
    free_all(h);
    delete h;
    return rc;
  };
#define CREATE_TRY(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      h->err = std::string(#call) + ": " + cudaGetErrorString(e_);                   \
      return bail(e_ == cudaErrorMemoryAllocation ? SOR3D_ENOMEM : SOR3D_ECUDA);       \
    }                                                                                 \
  } while (0)
  CREATE_TRY(cudaGetDevice(&h->device));
  h->nx = prm->nx;
  h->ny = prm->ny;
  h->nz = prm->nz;
  // coefficients (reading S4): in double, one rounding each
  const double ax = 1.0 / ((double)prm->dx * (double)prm->dx);
  const double ay = 1.0 / ((double)prm->dy * (double)prm->dy);
  const double az = 1.0 / ((double)prm->dz * (double)prm->dz);
  h->cx = (float)ax;
  h->cy = (float)ay;
  h->cz = (float)az;
  h->dd = (float)(2.0 * (ax + ay + az));
  h->invd = (float)(1.0 / (2.0 * (ax + ay + az)));
  h->om = prm->omega;
  h->om1 = (float)(1.0 - (double)prm->omega);
  if (!std::isfinite(h->dd) || !std::isfinite(h->cx) || !std::isfinite(h->cy) ||
      !std::isfinite(h->cz) || h->invd == 0.0f) {
    h->err = "dx, dy, dz give non-finite stencil weights";
    return bail(SOR3D_EINVAL);
  }
  // geometry: tiles of 60 x 12 columns, z-chunks of kz planes; about 4 CTAs
  // per SM (SOR3D_KZ overrides the chunk)
  h->gx = (int)((h->nx + kOutX - 1) / kOutX);
  h->rows_cta = 32;
  if (const char* e = std::getenv("SOR3D_ROWS")) h->rows_cta = std::atoi(e) == 16 ? 16 : 32;
  const int outy = h->rows_cta - 4;
  h->gy = (int)((h->ny + outy - 1) / outy);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  int kz = 0;
  if (const char* e = std::getenv("SOR3D_KZ")) kz = std::atoi(e);
  if (kz <= 0) {
    // z-chunk by a wave model: a CTA marches kz + 3 planes (rounded up to the
    // 4-step unroll); the launch takes ceil(CTAs / resident slots) waves.
    int per_sm = 0;
    if (h->rows_cta == 16)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sor_iter<16, false, true, false>, kSx * 16, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sor_iter<32, false, true, false>, kSx * 32, 0);
    const long long slots = (long long)std::max(per_sm, 1) * sms;
    const long long cols = (long long)h->gx * h->gy;
    double best = 0.0;
    for (int64_t c = h->nz; c >= 1; --c) {
      const int64_t gz = (h->nz + c - 1) / c;
      const double waves = (double)((cols * gz + slots - 1) / slots);
      const double cost = waves * (double)((c + 3 + 3) / 4 * 4);
      if (kz == 0 || cost < best * 0.999) {
        best = cost;
        kz = (int)c;
      }
    }
  }
  h->kz = (int)std::min<int64_t>(kz, h->nz);
  h->gz = (int)((h->nz + h->kz - 1) / h->kz);
  h->pitch = ((long long)h->gx * kOutX + 4 + 7) / 8 * 8;
  h->rows = (long long)h->gy * outy + 4;
  h->planes = (long long)h->gz * h->kz + 12;
  h->plane = h->pitch * h->rows;
  if (h->plane * h->planes >= (1LL << 31)) {  // 32-bit element offsets in the kernel
    h->err = "grid too large (padded arrays must stay below 2^31 elements)";
    return bail(SOR3D_EINVAL);
  }
  const size_t bytes = (size_t)h->plane * (size_t)h->planes * sizeof(float);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device);
  h->hint = 2.0 * (double)bytes <= 0.7 * (double)l2;  // rhs + p_out stay
  if (const char* e = std::getenv("SOR3D_HINT")) h->hint = std::atoi(e) != 0;
  if (cuda_stream) {
    h->stream = (cudaStream_t)cuda_stream;
  } else {
    CREATE_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  for (float** f : {&h->p[0], &h->p[1], &h->rhs}) {
    CREATE_TRY(cudaMalloc(f, bytes));
    CREATE_TRY(cudaMemset(*f, 0, bytes));
  }
  const int nparts = h->gx * h->gy * h->gz;
  h->cap = prm->history_len > 0 ? prm->history_len : 1024;
  CREATE_TRY(cudaMalloc(&h->part, (size_t)nparts * sizeof(Part)));
  CREATE_TRY(cudaMalloc(&h->counter, sizeof(unsigned)));
  CREATE_TRY(cudaMemset(h->counter, 0, sizeof(unsigned)));
  CREATE_TRY(cudaMalloc(&h->hist, (size_t)h->cap * 2 * sizeof(double)));
  CREATE_TRY(cudaMalloc(&h->scratch, 2 * sizeof(double)));
  CREATE_TRY(cudaDeviceSynchronize());
#undef CREATE_TRY
  char buf[256];
  std::snprintf(buf, sizeof(buf),
                "sor_iter: tile %dx%d (x,y) of a 64x%d apron'd block (%d thr, float4, half-warp rows), z-chunk %d, "
                "grid %dx%dx%d = %d CTAs, 1 launch/iteration, ping-pong%s",
                kOutX, outy, h->rows_cta, kSx * h->rows_cta, h->kz, h->gx, h->gy, h->gz, nparts, h->hint ? ", L2 hints" : "");
  h->plan = buf;
  *out = h;
  return SOR3D_OK;
}

int sor3d_set(sor3d* h, const float* p, const float* rhs) {
  NvtxRange nvtx_("sor3d_set");
  SOR_ENTER(h);
  if (!rhs) return fail(h, SOR3D_EINVAL, "rhs is NULL");
  h->have_state = false;
  unsigned* bad = reinterpret_cast<unsigned*>(h->scratch);
  SOR_TRY(h, cudaMemsetAsync(bad, 0, sizeof(unsigned), h->stream));
  int rc = upload(h, h->rhs, rhs, bad);
  if (rc) return rc;
  if (p) {
    rc = upload(h, h->p[0], p, bad);
    if (rc) return rc;
  } else {  // p = 0 (the padding is zero already)
    SOR_TRY(h, cudaMemsetAsync(h->p[0], 0, (size_t)h->plane * (size_t)h->planes * sizeof(float),
                               h->stream));
  }
  unsigned nb = 0;
  SOR_TRY(h, cudaMemcpyAsync(&nb, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
  SOR_TRY(h, cudaStreamSynchronize(h->stream));
  h->cur = 0;
  h->nrec = 0;
  h->have_state = nb == 0;
  if (nb) return fail(h, SOR3D_EINVAL, "p or rhs has non-finite values");
  return SOR3D_OK;
}

int sor3d_iterate(sor3d* h, int64_t n, int64_t every) {
  NvtxRange nvtx_("sor3d_iterate");
  SOR_ENTER(h);
  if (n < 0 || every < 0) return fail(h, SOR3D_EINVAL, "n and residual_every must be >= 0");
  if (!h->have_state) return fail(h, SOR3D_ESTATE, "sor3d_iterate before sor3d_set");
  for (int64_t t = 1; t <= n; ++t) {
    // launch t performs iteration t and folds the residual after iteration t-1
    const bool res = every > 0 && t >= 2 && (t - 1) % every == 0;
    const int rc = launch(h, true, res ? next_record(h) : nullptr);
    if (rc) return rc;
  }
  if (every > 0 && n >= 1) {
    const int rc = launch(h, false, next_record(h));
    if (rc) return rc;
  }
  return SOR3D_OK;
}

int sor3d_residual(sor3d* h, double out[2]) {
  NvtxRange nvtx_("sor3d_residual");
  SOR_ENTER(h);
  if (!out) return fail(h, SOR3D_EINVAL, "out is NULL");
  if (!h->have_state) return fail(h, SOR3D_ESTATE, "sor3d_residual before sor3d_set");
  const int rc = launch(h, false, h->scratch);
  if (rc) return rc;
  SOR_TRY(h, cudaMemcpyAsync(out, h->scratch, 2 * sizeof(double), cudaMemcpyDefault, h->stream));
  SOR_TRY(h, cudaStreamSynchronize(h->stream));
  return SOR3D_OK;
}

int sor3d_residual_history(sor3d* h, double* out, int64_t n) {
  SOR_ENTER(h);
  if (!out || n < 0 || n > h->nrec || n > h->cap)
    return fail(h, SOR3D_EINVAL, "n must be <= min(records, history_len)");
  if (n == 0) return SOR3D_OK;
  // the whole ring in one copy on the handle's stream, then index on the host
  std::vector<double> ring(2 * (size_t)h->cap);
  SOR_TRY(h, cudaMemcpyAsync(ring.data(), h->hist, ring.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, h->stream));
  SOR_TRY(h, cudaStreamSynchronize(h->stream));
  for (int64_t t = 0; t < n; ++t) {
    const int64_t r = (h->nrec - n + t) % h->cap;
    out[2 * t] = ring[2 * r];
    out[2 * t + 1] = ring[2 * r + 1];
  }
  return SOR3D_OK;
}

int64_t sor3d_history_count(const sor3d* h) { return h ? h->nrec : -1; }

int sor3d_get(sor3d* h, float* p) {
  NvtxRange nvtx_("sor3d_get");
  SOR_ENTER(h);
  if (!p) return fail(h, SOR3D_EINVAL, "p is NULL");
  if (!h->have_state) return fail(h, SOR3D_ESTATE, "sor3d_get before sor3d_set");
  const long long n = h->nx * h->ny * h->nz, rows = h->ny * h->nz;
  const bool dev = is_device_ptr(p);
  if (!dev && !h->stage) SOR_TRY(h, cudaMalloc(&h->stage, (size_t)n * sizeof(float)));
  float* d = dev ? p : h->stage;
  repack<false><<<(unsigned)std::min<long long>(rows, 148 * 16), 256, 0, h->stream>>>(
      h->p[h->cur], nullptr, d, (int)h->nx, (int)h->ny, rows, h->pitch, h->plane, nullptr);
  SOR_TRY(h, cudaGetLastError());
  if (!dev)
    SOR_TRY(h, cudaMemcpyAsync(p, d, (size_t)n * sizeof(float), cudaMemcpyDefault, h->stream));
  SOR_TRY(h, cudaStreamSynchronize(h->stream));
  return SOR3D_OK;
}

int sor3d_sync(sor3d* h) {
  SOR_ENTER(h);
  SOR_TRY(h, cudaStreamSynchronize(h->stream));
  return SOR3D_OK;
}

int64_t sor3d_launch_count(const sor3d* h) { return h ? h->nlaunch : -1; }

const char* sor3d_plan(const sor3d* h) { return h ? h->plan.c_str() : ""; }

void sor3d_destroy(sor3d* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  free_all(h);
  delete h;
}

const char* sor3d_last_error(const sor3d* h) { return h ? h->err.c_str() : t_create_err.c_str(); }

}  // extern "C"
