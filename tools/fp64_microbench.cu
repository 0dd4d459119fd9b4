// Throughput probes that decide the K3 design on sm_100a:
//   dfma      fp64 FMA pipe (8 independent chains per thread)
//   dmma      fp64 tensor MMA mma.sync.m8n8k4 (8 independent accumulators per warp)
//   mixed     half of the warps on each pipe at the same time
//   stream    HBM read bandwidth (ld.global.nc 16 B per lane, 1 GiB buffer)
//   stream+dfma  read 8-byte "factor" elements and do 24 FMAs each against register operands (R = 24 columns)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64mb tools/fp64_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a) {
  double c[8];
  for (int k = 0; k < 8; ++k) c[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma(c[k], a, 1e-9);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k];
  if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters, double a) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
  const double b = a * 0.5;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_mixed(double* out, int iters_mma, int iters_fma, double a) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double c[8][2];
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters_mma; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, a);
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  } else {
    double c[8];
    for (int k = 0; k < 8; ++k) c[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters_fma; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = fma(c[k], a, 1e-9);
    for (int k = 0; k < 8; ++k) s += c[k];
  }
  if (s == 12345.0) out[0] = s;
}

__global__ void k_stream(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p + i));
    s += v.x + v.y;
  }
  if (s == 12345.0) out[0] = s;
}

__global__ void k_stream_fma(const double2* __restrict__ p, size_t n2, double* out) {
  double acc[24];
  for (int k = 0; k < 24; ++k) acc[k] = 0;
  double r[12];
  for (int k = 0; k < 12; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p + i));
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      acc[k] = fma(v.x, r[k], acc[k]);
      acc[12 + k] = fma(v.x, r[(k + 1) % 12], acc[12 + k]);
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      acc[k] = fma(v.y, r[(k + 5) % 12], acc[k]);
      acc[12 + k] = fma(v.y, r[(k + 7) % 12], acc[12 + k]);
    }
  }
  double s = 0;
  for (int k = 0; k < 24; ++k) s += acc[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto tf = [&](double flops) { return flops / (ms * 1e-3) / 1e12; };
  for (int tpb : {128, 256, 512}) {
    const int blocks = nsm * (1024 / tpb) * 2, iters = 4096;
    k_dfma<<<blocks, tpb>>>(out, 64, 1.0000001);
    cudaEventRecord(e0);
    k_dfma<<<blocks, tpb>>>(out, iters, 1.0000001);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dfma   tpb %4d: %.1f TFLOP/s\n", tpb, tf(2.0 * 8 * iters * (double)blocks * tpb));
    k_dmma<<<blocks, tpb>>>(out, 64, 1.0000001);
    cudaEventRecord(e0);
    k_dmma<<<blocks, tpb>>>(out, iters / 4, 1.0000001);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dmma   tpb %4d: %.1f TFLOP/s\n", tpb, tf(2.0 * 256 * 8 * (iters / 4) * (double)blocks * tpb / 32));
  }
  for (int ratio : {1, 2, 4, 8}) {  // fma iterations per mma iteration
    const int tpb = 256, blocks = nsm * 8, im = 1024, ifm = im * ratio;
    k_mixed<<<blocks, tpb>>>(out, 16, 16 * ratio, 1.0000001);
    cudaEventRecord(e0);
    k_mixed<<<blocks, tpb>>>(out, im, ifm, 1.0000001);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (2.0 * 256 * 8 * im * (tpb / 64) + 2.0 * 8 * ifm * (tpb / 2)) * blocks;
    printf("mixed  fma:mma iters %d:1: %.1f TFLOP/s total\n", ratio, tf(fl));
  }
  const size_t bytes = 1ull << 30;
  double2* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  for (int tpb : {256, 512}) {
    const int blocks = nsm * (2048 / tpb);
    k_stream<<<blocks, tpb>>>(buf, bytes / 16, out);
    cudaEventRecord(e0);
    k_stream<<<blocks, tpb>>>(buf, bytes / 16, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream tpb %d: %.0f GB/s\n", tpb, bytes / (ms * 1e-3) / 1e9);
    k_stream_fma<<<blocks, tpb>>>(buf, bytes / 16, out);
    cudaEventRecord(e0);
    k_stream_fma<<<blocks, tpb>>>(buf, bytes / 16, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream+24fma/elem tpb %d: %.0f GB/s, %.1f TFLOP/s\n", tpb, bytes / (ms * 1e-3) / 1e9,
           tf(48.0 * bytes / 8));
  }
  return 0;
}
