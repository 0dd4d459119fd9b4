// DMMA issue/latency and HBM in-flight probes for the K3 design: TF/s of m8n8k4 f64 chains with K
// independent accumulators per warp at W warps per SM, and HBM GB/s of a plain stream at W warps/SM with D 16-byte
// loads in flight per lane.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int K>
__global__ void k_chain(double* out, int iters) {
  double c[K][2];
  for (int k = 0; k < K; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
  const double a = 1.0000001, b = 0.5;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) dmma(c[k][0], c[k][1], a, b);
  double s = 0;
  for (int k = 0; k < K; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}
template <int D>
__global__ void k_str(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i + (D - 1) * stride < n2; i += D * stride) {
    double2 v[D];
#pragma unroll
    for (int d = 0; d < D; ++d) asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v[d].x), "=d"(v[d].y) : "l"(p + i + d * stride));
#pragma unroll
    for (int d = 0; d < D; ++d) s += v[d].x;
  }
  if (s == 12345.0) out[0] = s;
}
template <int K>
void chain(int nsm, int wps, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048 / K * 8;
  k_chain<K><<<nsm, 32 * wps>>>(out, 16);
  cudaEventRecord(e0); k_chain<K><<<nsm, 32 * wps>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("dmma K %2d warps/SM %2d: %.1f TFLOP/s\n", K, wps, 2.0 * 256 * K * iters * (double)nsm * wps / (ms * 1e-3) / 1e12);
}
template <int D>
void str(int nsm, int wps, const double2* buf, size_t bytes, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_str<D><<<nsm, 32 * wps>>>(buf, bytes / 16, out);
  cudaEventRecord(e0); k_str<D><<<nsm, 32 * wps>>>(buf, bytes / 16, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("stream D %2d warps/SM %2d (in flight %3d KB/SM): %.0f GB/s\n", D, wps, wps * 32 * 16 * D / 1024, bytes / (ms * 1e-3) / 1e9);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 64);
  for (int wps : {4, 8, 12, 16, 32}) { chain<1>(nsm, wps, out); chain<4>(nsm, wps, out); chain<8>(nsm, wps, out); chain<12>(nsm, wps, out); chain<16>(nsm, wps, out); }
  const size_t bytes = 1ull << 30; double2* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 0, bytes);
  for (int wps : {8, 16, 32}) { str<1>(nsm, wps, buf, bytes, out); str<2>(nsm, wps, buf, bytes, out); str<4>(nsm, wps, buf, bytes, out); str<8>(nsm, wps, buf, bytes, out); }
  return 0;
}
