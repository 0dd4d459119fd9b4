// Prototype of the register-streaming K3 work unit (round 2): one warp = one task = a 32-lane
// output tile x 24 columns over a run of k-groups; the factor block (fragment order, 1 KB per k-group) and the
// right-hand-side rows are loaded straight into registers P k-groups ahead (no shared memory, no barriers),
// 12 DMMA m8n8k4 per k-group.  Synthetic: NTASK tasks of KG k-groups over a 300 MB factor stream, RHS rows from
// an L2-resident [nrows][24] matrix (contiguous rows per task), persistent warps taking tasks from a counter.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k3p tools/k3_proto.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 ldg2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg1(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int P, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_proto(const double2* __restrict__ A, const double* __restrict__ Z,
                                                    int R, int ntask, int KG, int nrows, int* counter,
                                                    double* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(counter, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= ntask) break;
    const double2* a = A + (size_t)task * KG * 64 + lane;    // k-group q: a[q*64], a[q*64 + 32]
    const int row0 = (int)(((long long)task * 977) % (nrows - 4 * KG));
    const double* z = Z + (size_t)row0 * R + t * R + g;       // k = 4q + t, col = 8n + g
    double acc[4][3][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    double2 ra[P][2];
    double rb[P][3];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (p < KG) {
        ra[p][0] = ldg2(a + p * 64);
        ra[p][1] = ldg2(a + p * 64 + 32);
#pragma unroll
        for (int n = 0; n < 3; ++n) rb[p][n] = ldg1(z + (size_t)(4 * p) * R + 8 * n);
      }
    }
    for (int q0 = 0; q0 < KG; q0 += P) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int q = q0 + p;
        if (q < KG) {
          const double2 a01 = ra[p][0], a23 = ra[p][1];
          double b[3] = {rb[p][0], rb[p][1], rb[p][2]};
          const int qn = q + P;
          if (qn < KG) {
            ra[p][0] = ldg2(a + qn * 64);
            ra[p][1] = ldg2(a + qn * 64 + 32);
#pragma unroll
            for (int n = 0; n < 3; ++n) rb[p][n] = ldg1(z + (size_t)(4 * qn) * R + 8 * n);
          }
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            dmma(acc[0][n][0], acc[0][n][1], a01.x, b[n]);
            dmma(acc[1][n][0], acc[1][n][1], a01.y, b[n]);
            dmma(acc[2][n][0], acc[2][n][1], a23.x, b[n]);
            dmma(acc[3][n][0], acc[3][n][1], a23.y, b[n]);
          }
        }
      }
    }
    double* o = out + (size_t)task * 32 * 24;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n)
        *reinterpret_cast<double2*>(o + (4 * g + m) * 24 + 8 * n + 2 * t) = make_double2(acc[m][n][0], acc[m][n][1]);
  }
}

template <int P, int WPB>
int run(const double2* A, const double* Z, double* out, int* ctr, int ntask, int KG, int nrows, int nsm, int ctas_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * ctas_per_sm;
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(e0);
    k_proto<P, WPB><<<grid, 32 * WPB>>>(A, Z, 24, ntask, KG, nrows, ctr, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_proto<P, WPB>);
  const double bytes = (double)ntask * KG * 1024;
  printf("P %d WPB %2d ctas/SM %d KG %3d regs %3d: %.1f us  factor %.0f GB/s  %.1f TFLOP/s\n", P, WPB, ctas_per_sm, KG,
         fa.numRegs, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 8 * 48 / (best * 1e-3) / 1e12);
  return 0;
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t abytes = 300ull << 20;
  double2* A;
  double *Z, *out;
  int* ctr;
  const int nrows = 72000;
  CK(cudaMalloc(&A, abytes));
  CK(cudaMemset(A, 0, abytes));
  CK(cudaMalloc(&Z, (size_t)nrows * 24 * 8));
  CK(cudaMemset(Z, 0, (size_t)nrows * 24 * 8));
  CK(cudaMalloc(&ctr, 4));
  for (int KG : {8, 16, 32, 64}) {
    const int ntask = (int)(abytes / 1024 / KG);
    CK(cudaMalloc(&out, (size_t)ntask * 32 * 24 * 8));
    run<4, 4>(A, Z, out, ctr, ntask, KG, nrows, nsm, 4);
    run<4, 8>(A, Z, out, ctr, ntask, KG, nrows, nsm, 2);
    run<6, 4>(A, Z, out, ctr, ntask, KG, nrows, nsm, 3);
    run<8, 4>(A, Z, out, ctr, ntask, KG, nrows, nsm, 3);
    run<2, 8>(A, Z, out, ctr, ntask, KG, nrows, nsm, 3);
    cudaFree(out);
  }
  // a 30 MB "level": per-launch fixed cost
  for (int KG : {8, 16}) {
    const int ntask = (int)((30ull << 20) / 1024 / KG);
    CK(cudaMalloc(&out, (size_t)ntask * 32 * 24 * 8));
    printf("30 MB level:\n");
    run<4, 4>(A, Z, out, ctr, ntask, KG, nrows, nsm, 4);
    run<6, 4>(A, Z, out, ctr, ntask, KG, nrows, nsm, 3);
    cudaFree(out);
  }
  return 0;
}
