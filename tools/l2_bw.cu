// tools/l2_bw.cu — L2 bandwidth probe (the small-grid roofline's peak,
// bench.py `roofline` for grids whose state fits in L2).
//
// Reads (ld.global.cg: L1 bypassed) and copies an L2-resident buffer of
// 8..64 MB many times over with a grid of 148 x 8 CTAs x 512 threads, float4
// per access, and reports bytes moved / time (CUDA events, best of 5).  An
// HBM-sized buffer (1 GB) is measured the same way for comparison.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_bw tools/l2_bw.cu
//   /tmp/l2_bw > profiles/r02_l2_peak.json
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_k(const float4* __restrict__ p, long long n, int passes, float* out) {
  float acc = 0.0f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < passes; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
      const float4 v = __ldcg(p + i);
      acc += (v.x + v.y) + (v.z + v.w);
    }
  if (acc == 1234.5f) out[0] = acc;   // keeps the loads live
}

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, long long n,
                       int passes) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < passes; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
      __stcg(b + i, __ldcg(a + i));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8, block = 256;
  const size_t big = 1ull << 30;
  float4 *a = nullptr, *b = nullptr;
  float* out = nullptr;
  cudaMalloc(&a, big);
  cudaMalloc(&b, big);
  cudaMalloc(&out, 4);
  cudaMemset(a, 0, big);
  cudaMemset(b, 0, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::printf("{\"sms\": %d, \"grid\": %d, \"block\": %d, \"results\": [\n", sms, grid, block);
  const size_t mbs[] = {8, 16, 32, 48, 64, 1024};
  bool first = true;
  for (size_t mb : mbs) {
    const long long n = (long long)(mb << 20) / 16;
    const int passes = mb >= 1024 ? 4 : (int)(4096 / mb);
    for (int kind = 0; kind < 2; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0)
          read_k<<<grid, block>>>(a, n, passes, out);
        else
          copy_k<<<grid, block>>>(a, b, n / 2, passes);   // footprint mb (half read, half written)
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;   // rep 0 warms L2
      }
      const double bytes = (double)(mb << 20) * passes;   // read: mb; copy: mb/2 in + mb/2 out
      std::printf("%s {\"kind\": \"%s\", \"footprint_mb\": %zu, \"passes\": %d, \"ms\": %.4f, "
                  "\"gbs\": %.1f}",
                  first ? "" : ",\n", kind == 0 ? "read" : "copy", mb, passes, best,
                  bytes / (best * 1e-3) / 1e9);
      first = false;
    }
  }
  std::printf("\n], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
