// paper_1711_04471_b200/csrc/sw2d_tb_kernels.cu — temporally blocked steps
// for the paper's small grids.
//
// The paper's 2DSW runs are 500^2 .. 2000^2 grids for 10,000 steps
// (PAPER.md:382-385).  Their whole state fits in L2 and one fused step is a
// few microseconds of work, so per-step launch and pipeline latency, not HBM,
// bound the time.  This kernel advances K steps per launch: each CTA loads a
// tile plus a 2K-cell apron (the step's dependency cone is 2 cells) into
// shared memory, runs K steps there, and writes back the tile's centre, which
// is exact.  Every cell's arithmetic is the oracle's, operation for
// operation (bitwise parity), in four CTA-synchronised phases per step:
//   P1 h, wet  P2 un, vn  P3 etan  P4 Shapiro + commit.
// Cells outside the grid are dry with zero velocity (the closed basin);
// cells within 2s of the apron's outer edge are garbage after s steps and
// never reach the centre.
#include <cuda_runtime.h>

#include <cstdint>

#include "sw2d_internal.cuh"

namespace sw2d_dev {

namespace {

__device__ __forceinline__ float tb_flux(float s, float hl, float hr) {
  return s > 0.0f ? __fmul_rn(s, hl) : (s < 0.0f ? __fmul_rn(s, hr) : 0.0f);
}

__device__ __forceinline__ bool tb_flows(bool wc, bool wn, float d) {
  return wc ? (wn || d > 0.0f) : (wn && d < 0.0f);
}

constexpr int kTbX = 32, kTbY = 16;  // threads

__global__ void __launch_bounds__(kTbX * kTbY)
    sw2d_step_tb(const TbArgs a) {
  extern __shared__ __align__(16) unsigned char tsm[];
  const int X = a.tw + 4 * a.K, Y = a.th + 4 * a.K;  // tile + apron
  const int N = X * Y;
  float* E = reinterpret_cast<float*>(tsm);
  float* H0 = E + N;
  float* h = H0 + N;
  float* U = h + N;
  float* V = U + N;
  float* un = V + N;
  float* vn = un + N;
  float* et = vn + N;
  unsigned char* w = reinterpret_cast<unsigned char*>(et + N);

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tk = blockIdx.x, tj = blockIdx.y;
  const int gk0 = tk * a.tw + 1 - 2 * a.K;  // global 1-based column of apron x = 0
  const int gj0 = tj * a.th + 1 - 2 * a.K;  // global 1-based row of apron y = 0
  const int nx = a.nx, ny = a.ny;
  const long long pitch = a.pitch;

  // load the apron'd tile (zero outside the grid)
  for (int y = ty; y < Y; y += kTbY) {
    const int gj = gj0 + y;
    const bool rin = gj >= 1 && gj <= ny;
    const long long rowoff = (long long)(gj - a.jbase) * pitch + kColOff;
    for (int x = tx; x < X; x += kTbX) {
      const int gk = gk0 + x;
      const int i = y * X + x;
      if (rin && gk >= 1 && gk <= nx) {
        const long long o = rowoff + gk;
        E[i] = a.E[o];
        H0[i] = a.H0[o];
        U[i] = a.U[o];
        V[i] = a.V[o];
      } else {
        E[i] = 0.0f;
        H0[i] = 0.0f;
        U[i] = 0.0f;
        V[i] = 0.0f;
      }
    }
  }
  __syncthreads();

  const float cgx = a.c.cgx, cgy = a.c.cgy, cx = a.c.cx, cy = a.c.cy, q = a.c.q,
              hmin = a.c.hmin;
  for (int s = 0; s < a.K; ++s) {
    // P1: h and wet (dry outside the grid)
    for (int y = ty; y < Y; y += kTbY) {
      const int gj = gj0 + y;
      for (int x = tx; x < X; x += kTbX) {
        const int gk = gk0 + x;
        const int i = y * X + x;
        const float hv = __fadd_rn(H0[i], E[i]);
        h[i] = hv;
        w[i] = (gj >= 1 && gj <= ny && gk >= 1 && gk <= nx && !(hv < hmin)) ? 1 : 0;
      }
    }
    __syncthreads();
    // P2: face velocities (walls and faces outside the grid are 0)
    for (int y = ty; y < Y; y += kTbY) {
      const int gj = gj0 + y;
      for (int x = tx; x < X; x += kTbX) {
        const int gk = gk0 + x;
        const int i = y * X + x;
        float u = 0.0f, v = 0.0f;
        if (gj >= 1 && gj <= ny && gk >= 1 && gk <= nx) {
          if (gk != nx && x + 1 < X) {
            const float du = __fmul_rn(cgx, __fsub_rn(E[i + 1], E[i]));
            if (tb_flows(w[i], w[i + 1], du)) u = __fadd_rn(U[i], du);
          }
          if (gj != ny && y + 1 < Y) {
            const float dv = __fmul_rn(cgy, __fsub_rn(E[i + X], E[i]));
            if (tb_flows(w[i], w[i + X], dv)) v = __fadd_rn(V[i], dv);
          }
        }
        un[i] = u;
        vn[i] = v;
      }
    }
    __syncthreads();
    // P3: etan (the apron's outermost ring is left as garbage-free zero)
    for (int y = ty; y < Y; y += kTbY) {
      for (int x = tx; x < X; x += kTbX) {
        const int i = y * X + x;
        float e = 0.0f;
        if (x >= 1 && x + 1 < X && y >= 1 && y + 1 < Y) {
          const float hc = h[i];
          const float fe = tb_flux(un[i], hc, h[i + 1]);
          const float fw = tb_flux(un[i - 1], h[i - 1], hc);
          const float fn = tb_flux(vn[i], hc, h[i + X]);
          const float fs = tb_flux(vn[i - X], h[i - X], hc);
          e = __fsub_rn(__fsub_rn(E[i], __fmul_rn(cx, __fsub_rn(fe, fw))),
                        __fmul_rn(cy, __fsub_rn(fn, fs)));
        }
        et[i] = e;
      }
    }
    __syncthreads();
    // P4: Shapiro filter and commit (eta in place; u, v <- un, vn)
    for (int y = ty; y < Y; y += kTbY) {
      const int gj = gj0 + y;
      for (int x = tx; x < X; x += kTbX) {
        const int gk = gk0 + x;
        const int i = y * X + x;
        float e = 0.0f;
        if (gj >= 1 && gj <= ny && gk >= 1 && gk <= nx) {
          e = et[i];
          if (w[i] && x >= 1 && x + 1 < X && y >= 1 && y + 1 < Y) {
            const bool wE = w[i + 1], wW = w[i - 1], wN = w[i + X], wS = w[i - X];
            const float sc = (float)((int)wE + (int)wW + (int)wN + (int)wS);
            const float t1 = __fmul_rn(__fsub_rn(1.0f, __fmul_rn(q, sc)), e);
            const float t2 = __fmul_rn(q, __fadd_rn(wE ? et[i + 1] : 0.0f, wW ? et[i - 1] : 0.0f));
            const float t3 = __fmul_rn(q, __fadd_rn(wN ? et[i + X] : 0.0f, wS ? et[i - X] : 0.0f));
            e = __fadd_rn(__fadd_rn(t1, t2), t3);
          }
        }
        E[i] = e;
        U[i] = un[i];
        V[i] = vn[i];
      }
    }
    __syncthreads();
  }

  // write back the tile's centre (inside the grid)
  for (int y = 2 * a.K + ty; y < 2 * a.K + a.th; y += kTbY) {
    const int gj = gj0 + y;
    if (gj > ny) break;
    const long long rowoff = (long long)(gj - a.jbase) * pitch + kColOff;
    for (int x = 2 * a.K + tx; x < 2 * a.K + a.tw; x += kTbX) {
      const int gk = gk0 + x;
      if (gk > nx) break;
      const int i = y * X + x;
      const long long o = rowoff + gk;
      a.En[o] = E[i];
      a.Un[o] = U[i];
      a.Vn[o] = V[i];
    }
  }
}

}  // namespace

size_t tb_smem_bytes(int tw, int th, int K) {
  const size_t n = (size_t)(tw + 4 * K) * (size_t)(th + 4 * K);
  return n * (8 * sizeof(float) + 1) + 16;
}

void launch_tb(const TbArgs& a, void* stream) {
  static unsigned long long attr_devices = 0;  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_devices >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(sw2d_step_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_devices |= 1ull << (dev & 63);
  }
  const dim3 grid((unsigned)((a.nx + a.tw - 1) / a.tw), (unsigned)((a.ny + a.th - 1) / a.th));
  sw2d_step_tb<<<grid, dim3(kTbX, kTbY), tb_smem_bytes(a.tw, a.th, a.K),
                 (cudaStream_t)stream>>>(a);
}

}  // namespace sw2d_dev
