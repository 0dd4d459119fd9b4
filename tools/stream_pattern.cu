// HBM access-pattern probe for the K3 factor stream: every warp streams its own contiguous region
// of REG KB in 1 KB steps (two 16-byte loads per lane per step, D steps in flight) vs. the same loads interleaved
// across warps.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp tools/stream_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int D, bool INTERLEAVE>
__global__ void k(const double2* __restrict__ p, size_t nsteps_total, int steps_per_region, double* out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (blockDim.x >> 5);
  const size_t nregions = nsteps_total / steps_per_region;
  double s = 0;
  for (size_t r = gw; r < nregions; r += nw) {
    for (int q = 0; q < steps_per_region; q += D) {
      double2 v[D][2];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        size_t step = INTERLEAVE ? ((size_t)(q + d) * nregions + r) : (r * steps_per_region + q + d);
        const double2* a = p + step * 64 + lane;
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v[d][0].x), "=d"(v[d][0].y) : "l"(a));
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v[d][1].x), "=d"(v[d][1].y) : "l"(a + 32));
      }
#pragma unroll
      for (int d = 0; d < D; ++d) s += v[d][0].x + v[d][1].y;
    }
  }
  if (s == 12345.0) out[0] = s;
}
template <int D, bool IL>
void run(const double2* buf, size_t bytes, int spr, int wps, int nsm, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t nsteps = bytes / 1024;
  k<D, IL><<<nsm * wps / 8, 256>>>(buf, nsteps, spr, out);
  cudaEventRecord(e0); k<D, IL><<<nsm * wps / 8, 256>>>(buf, nsteps, spr, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%s D %d region %3d KB warps/SM %2d: %.0f GB/s\n", IL ? "interleaved" : "per-warp   ", D, spr, wps, bytes / (ms * 1e-3) / 1e9);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 64);
  const size_t bytes = 512ull << 20; double2* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 0, bytes);
  for (int spr : {16, 64}) for (int wps : {16, 32}) {
    run<2, false>(buf, bytes, spr, wps, nsm, out); run<2, true>(buf, bytes, spr, wps, nsm, out);
    run<4, false>(buf, bytes, spr, wps, nsm, out); run<4, true>(buf, bytes, spr, wps, nsm, out);
  }
  return 0;
}
