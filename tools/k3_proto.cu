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

template <int P, int WPB, bool STATIC, bool RHS>
__global__ void __launch_bounds__(32 * WPB) k_proto(const double2* __restrict__ A, const double* __restrict__ Z,
                                                    int R, int ntask, int KG, int nrows, int* counter,
                                                    double* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int gw = blockIdx.x * WPB + (threadIdx.x >> 5), nw = gridDim.x * WPB;
  for (int it = 0;; ++it) {
    int task = 0;
    if (STATIC) {
      task = gw + it * nw;
    } else {
      if (lane == 0) task = atomicAdd(counter, 1);
      task = __shfl_sync(0xffffffffu, task, 0);
    }
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
        for (int n = 0; n < 3; ++n) rb[p][n] = RHS ? ldg1(z + (size_t)(4 * p) * R + 8 * n) : 1.0 + n;
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
            for (int n = 0; n < 3; ++n) rb[p][n] = RHS ? ldg1(z + (size_t)(4 * qn) * R + 8 * n) : b[n] * 0.5;
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

template <int P, int WPB, bool STATIC = true, bool RHS = true>
int run(const double2* A, const double* Z, double* out, int* ctr, int ntask, int KG, int nrows, int nsm, int ctas_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * ctas_per_sm;
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(e0);
    k_proto<P, WPB, STATIC, RHS><<<grid, 32 * WPB>>>(A, Z, 24, ntask, KG, nrows, ctr, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_proto<P, WPB, STATIC, RHS>);
  const double bytes = (double)ntask * KG * 1024;
  printf("%s%s P %d WPB %2d ctas/SM %d KG %3d regs %3d: %.1f us  factor %.0f GB/s  %.1f TFLOP/s\n",
         STATIC ? "static" : "atomic", RHS ? "" : " noRHS", P, WPB, ctas_per_sm, KG, fa.numRegs, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 8 * 48 / (best * 1e-3) / 1e12);
  return 0;
}


// Variant: lane-private cp.async ring of S k-groups per warp (no register cost for the prefetch, no barrier:
// each lane reads back only what it copied).  Per k-group and lane: 2 x 16 B of factor (A fragments) and 3 x 8 B
// of right-hand side (B fragments).
__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
template <int S, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_ring(const double2* __restrict__ A, const double* __restrict__ Z, int R,
                                                   int ntask, int KG, int nrows, double* __restrict__ out) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  // per warp: S slots x (2 double2 + 3 double (+1 pad)) per lane, lane-major inside a slot: slot stride 32 * 8 doubles
  double* ring = smem + (size_t)w * S * 32 * 8 + lane * 8;
  const int gw = blockIdx.x * WPB + w, nw = gridDim.x * WPB;
  for (int task = gw; task < ntask; task += nw) {
    const double2* a = A + (size_t)task * KG * 64 + lane;
    const int row0 = (int)(((long long)task * 977) % (nrows - 4 * KG));
    const double* z = Z + (size_t)row0 * R + t * R + g;
    double acc[4][3][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    auto issue = [&](int q) {
      double* sl = ring + (q % S) * 32 * 8;
      if (q < KG) {
        cpa16(sl, a + q * 64);
        cpa16(sl + 2, a + q * 64 + 32);
#pragma unroll
        for (int n = 0; n < 3; ++n) cpa8(sl + 4 + n, z + (size_t)(4 * q) * R + 8 * n);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int q = 0; q < S - 1; ++q) issue(q);
    for (int q = 0; q < KG; ++q) {
      issue(q + S - 1);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 1) : "memory");
      const double* sl = ring + (q % S) * 32 * 8;
      const double2 a01 = *reinterpret_cast<const double2*>(sl);
      const double2 a23 = *reinterpret_cast<const double2*>(sl + 2);
      const double b0 = sl[4], b1 = sl[5], b2 = sl[6];
      const double b[3] = {b0, b1, b2};
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        dmma(acc[0][n][0], acc[0][n][1], a01.x, b[n]);
        dmma(acc[1][n][0], acc[1][n][1], a01.y, b[n]);
        dmma(acc[2][n][0], acc[2][n][1], a23.x, b[n]);
        dmma(acc[3][n][0], acc[3][n][1], a23.y, b[n]);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    double* o = out + (size_t)task * 32 * 24;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n)
        *reinterpret_cast<double2*>(o + (4 * g + m) * 24 + 8 * n + 2 * t) = make_double2(acc[m][n][0], acc[m][n][1]);
  }
}

template <int S, int WPB>
int run_ring(const double2* A, const double* Z, double* out, int ntask, int KG, int nrows, int nsm, int ctas_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sm = (size_t)WPB * S * 32 * 8 * 8;
  CK(cudaFuncSetAttribute(k_ring<S, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ring<S, WPB>, 32 * WPB, sm);
  const int cps = ctas_per_sm < occ ? ctas_per_sm : occ;
  const int grid = nsm * cps;
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_ring<S, WPB><<<grid, 32 * WPB, sm>>>(A, Z, 24, ntask, KG, nrows, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_ring<S, WPB>);
  const double bytes = (double)ntask * KG * 1024;
  printf("ring S %2d WPB %2d ctas/SM %d (smem %zu KB) KG %3d regs %3d: %.1f us  factor %.0f GB/s  %.1f TFLOP/s\n", S, WPB,
         cps, sm / 1024, KG, fa.numRegs, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 8 * 48 / (best * 1e-3) / 1e12);
  return 0;
}

// Variant: per-warp TMA ring.  Each warp owns S stages of (16 k-steps x 32 rows of factor = 4 KB, 16 RHS rows x 24
// columns = 3 KB), filled by cp.async.bulk issued from lane 0 and completing on the stage's mbarrier; the ring runs
// across the warp's consecutive tasks (static round robin).  No CTA barrier anywhere.
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned ph) {
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}
template <int S, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_tma(const double2* __restrict__ A, const double* __restrict__ Z, int R,
                                                  int ntask, int KG, int nrows, double* __restrict__ out) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[WPB][S];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  constexpr int STAGE = 16 * 32 + 16 * 24;   // doubles: factor 16 k x 32 rows, RHS 16 rows x 24
  double* ring = smem + (size_t)w * S * STAGE;
  if (lane == 0)
    for (int i = 0; i < S; ++i) mb_init(&bars[w][i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * WPB + w, nw = gridDim.x * WPB;
  const int nst = KG / 4;                     // stages per task
  // global stage sequence of this warp: (task index j -> task gw + j*nw, stage st)
  const int my_tasks = gw < ntask ? (ntask - 1 - gw) / nw + 1 : 0;
  const int total = my_tasks * nst;
  auto issue = [&](int idx) {
    if (idx >= total) return;
    const int j = idx / nst, st = idx - j * nst;
    const int task = gw + j * nw;
    const int slot = idx % S;
    double* sb = ring + slot * STAGE;
    const double2* a = A + (size_t)task * KG * 64 + (size_t)st * 4 * 64;
    const int row0 = (int)(((long long)task * 977) % (nrows - 4 * KG));
    const double* z = Z + (size_t)(row0 + st * 16) * R;
    if (lane == 0) {
      mb_expect(&bars[w][slot], 16 * 32 * 8 + 16 * 24 * 8);
      bulk(sb, a, 16 * 32 * 8, &bars[w][slot]);
      bulk(sb + 16 * 32, z, 16 * 24 * 8, &bars[w][slot]);
    }
  };
  for (int i = 0; i < S - 1; ++i) issue(i);
  int idx = 0;
  for (int j = 0; j < my_tasks; ++j) {
    const int task = gw + j * nw;
    double acc[4][3][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int st = 0; st < nst; ++st, ++idx) {
      __syncwarp();
      issue(idx + S - 1);   // refills the slot consumed at idx - 1 (all lanes are past it: syncwarp above)
      const int slot = idx % S;
      mb_wait(&bars[w][slot], (idx / S) & 1);
      const double2* As = reinterpret_cast<const double2*>(ring + slot * STAGE);
      const double* Zs = ring + slot * STAGE + 16 * 32;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 a01 = As[(q * 2) * 32 + lane], a23 = As[(q * 2 + 1) * 32 + lane];
        double b[3];
#pragma unroll
        for (int n = 0; n < 3; ++n) b[n] = Zs[(4 * q + t) * 24 + 8 * n + g];
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          dmma(acc[0][n][0], acc[0][n][1], a01.x, b[n]);
          dmma(acc[1][n][0], acc[1][n][1], a01.y, b[n]);
          dmma(acc[2][n][0], acc[2][n][1], a23.x, b[n]);
          dmma(acc[3][n][0], acc[3][n][1], a23.y, b[n]);
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

template <int S, int WPB>
int run_tma(const double2* A, const double* Z, double* out, int ntask, int KG, int nrows, int nsm, int ctas_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sm = (size_t)WPB * S * (16 * 32 + 16 * 24) * 8;
  CK(cudaFuncSetAttribute(k_tma<S, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma<S, WPB>, 32 * WPB, sm);
  const int cps = ctas_per_sm < occ ? ctas_per_sm : occ;
  const int grid = nsm * cps;
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_tma<S, WPB><<<grid, 32 * WPB, sm>>>(A, Z, 24, ntask, KG, nrows, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_tma<S, WPB>);
  const double bytes = (double)ntask * KG * 1024;
  printf("tma  S %2d WPB %2d ctas/SM %d (smem %zu KB) KG %3d regs %3d: %.1f us  factor %.0f GB/s  %.1f TFLOP/s\n", S, WPB,
         cps, sm / 1024, KG, fa.numRegs, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 8 * 48 / (best * 1e-3) / 1e12);
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
  for (int KG : {16, 64}) {
    const int ntask = (int)(abytes / 1024 / KG);
    CK(cudaMalloc(&out, (size_t)ntask * 32 * 24 * 8));
    run<2, 8>(A, Z, out, ctr, ntask, KG, nrows, nsm, 4);
    run_tma<4, 4>(A, Z, out, ntask, KG, nrows, nsm, 2);
    run_tma<4, 6>(A, Z, out, ntask, KG, nrows, nsm, 1);
    run_tma<6, 4>(A, Z, out, ntask, KG, nrows, nsm, 1);
    run_tma<3, 8>(A, Z, out, ntask, KG, nrows, nsm, 1);
    run_tma<4, 8>(A, Z, out, ntask, KG, nrows, nsm, 1);
    run_tma<3, 4>(A, Z, out, ntask, KG, nrows, nsm, 2);
    run_tma<8, 4>(A, Z, out, ntask, KG, nrows, nsm, 1);
    cudaFree(out);
  }
  for (int KG : {8, 16, 32}) {
    const int ntask = (int)((30ull << 20) / 1024 / KG);
    CK(cudaMalloc(&out, (size_t)ntask * 32 * 24 * 8));
    printf("30 MB level:\n");
    run<2, 8>(A, Z, out, ctr, ntask, KG, nrows, nsm, 3);
    run_tma<4, 4>(A, Z, out, ntask, KG, nrows, nsm, 2);
    run_tma<4, 6>(A, Z, out, ntask, KG, nrows, nsm, 1);
    run_tma<3, 8>(A, Z, out, ntask, KG, nrows, nsm, 1);
    run_tma<4, 8>(A, Z, out, ntask, KG, nrows, nsm, 1);
    cudaFree(out);
  }
  return 0;
}
