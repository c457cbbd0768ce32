// Microbenchmark + layout probe for tcgen05.mma (kind::f16, bf16 in, fp32 accum) on sm_100a.
// Purpose: (1) verify the no-swizzle K-major SMEM descriptor layout used by the conv kernels,
// including the "shifted start address" trick (implicit-GEMM taps as descriptor offsets) and
// the LBO=0 trick (duplicate K-chunk); (2) measure MMA issue rate vs N at M=128 SS mode, to
// decide how the 3x3 conv maps onto the tensor core (SURVEY.md §7 hard part 1).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------- correctness probe ----------------
// A_big: rows 0..(128+8) x K=16, layout addr(m,kc) = m*16 + kc*LBO_A, LBO_A = 144*16
// B: N x 16, addr(n,kc) = n*16 + kc*LBO_B, LBO_B = N*16
// mode 0: D = A[0:128] B^T ; mode 1: start shifted by 3 rows ; mode 2: LBO_A = 0
template <int N>
__global__ void probe_kernel(const float* a_host_vals, const float* b_vals, int mode, float* out /*128 x N*/) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int ROWS = 144;
  __nv_bfloat16* A = (__nv_bfloat16*)smem;                // ROWS*16*2 = 4608 B
  __nv_bfloat16* B = (__nv_bfloat16*)(smem + 8192);
  const uint32_t LBO_A = ROWS * 16, LBO_B = N * 16;
  for (int i = threadIdx.x; i < ROWS * 16; i += blockDim.x) {
    int m = i / 16, k = i % 16;
    A[(m * 16 + (k / 8) * LBO_A + (k % 8) * 2) / 2] = __float2bfloat16(a_host_vals[i]);
  }
  for (int i = threadIdx.x; i < N * 16; i += blockDim.x) {
    int n = i / 16, k = i % 16;
    B[(n * 16 + (k / 8) * LBO_B + (k % 8) * 2) / 2] = __float2bfloat16(b_vals[i]);
  }
  fence_async_smem();
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    uint32_t a_addr = smem_u32(A) + (mode == 1 ? 3 * 16 : 0);
    uint64_t ad = make_desc(a_addr, mode == 2 ? 0 : LBO_A, 128);
    uint64_t bd = make_desc(smem_u32(B), LBO_B, 128);
    mma_ss(tbase, ad, bd, make_idesc(128, N), 0);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  int m = threadIdx.x;  // 128 threads, lane = m
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int i = 0; i < 8; ++i) out[m * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tbase));
}

// ---------------- throughput ----------------
// One CTA per SM. Thread 0 issues ITERS MMAs (M=128, N, K=16) into one accumulator, cycling the A
// start address over NSHIFT offsets (to mimic 3x3 taps). Reports cycles per MMA.
template <int N>
__global__ void tput_kernel(int iters, int nshift, long long* cyc, unsigned long long* ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    uint32_t abase = smem_u32(smem);
    uint32_t bbase = abase + 48 * 1024;
    constexpr uint32_t LBO_A = 400 * 16;  // A rows: 400 positions, 4 chunks of 8 channels
    constexpr uint32_t LBO_B = N * 16;
    const uint32_t idesc = make_idesc(128, N);
    const uint64_t a0 = make_desc(abase, LBO_A, 128), b0 = make_desc(bbase, LBO_B, 128);
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    long long c0 = clock64();
    for (int it = 0; it < iters; it += 18) {
      const uint32_t tacc = tbase + (uint32_t)((it / 18) & 1) * 256;
#pragma unroll
      for (int t = 0; t < 9; ++t)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t aoff = nshift > 1 ? (uint32_t)(((t / 3) * 130 + (t % 3)) + j * 2 * (LBO_A / 16)) : (uint32_t)(j * 2 * (LBO_A / 16));
          mma_ss(tacc, a0 + aoff, b0 + (uint32_t)((t * 2 + j) & 1) * (8192 / 16), idesc, (t | j) != 0);
        }
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    long long c1 = clock64();
    unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    cyc[blockIdx.x] = c1 - c0;
    ns[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}


// pattern kernel: N=96 M=128 SS; mode selects the D-column pattern
//  0: D at col 0 always; 1: D at col 32 always; 2: D alternates 0/32 per MMA;
//  3: SLIDE pattern: 6 MMAs per "row" into window at col base(r) = ((16 - r) & 15) * 32 (wrapped to 3 slots)
//     (only the non-wrapping windows are used: r cycles over windows at cols 0,32,...,416)
//  4: like 0 but A LBO = 2048
template <int N>
__global__ void pattern_kernel(int iters, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    uint32_t abase = smem_u32(smem);
    uint32_t bbase = abase + 48 * 1024;
    const uint32_t LBO_A = mode == 4 ? 2048 : 400 * 16;
    const uint32_t idesc = make_idesc(128, N);
    const uint64_t a0 = make_desc(abase, LBO_A, 128), b0 = make_desc(bbase, N * 16, 128);
    __shared__ uint64_t bar2, bar3;
    mbar_init(smem_u32(&bar2), 1);
    mbar_init(smem_u32(&bar3), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // complete bar3's phase 0 once so waits on parity 0 succeed immediately
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" :: "r"(smem_u32(&bar3)) : "memory");
    long long c0 = clock64();
    for (int it = 0; it < iters; it += 6) {
      uint32_t d;
      const int row = it / 6;
      if (mode == 5 || mode == 8) mma_commit(smem_u32(&bar2));
      if (mode == 6 || mode == 8) tc_fence_after();
      if (mode == 7 || mode == 8) mbar_wait(smem_u32(&bar3), 0);
      if (mode == 9) { mma_commit(smem_u32(&bar2)); mma_commit(smem_u32(&bar2)); mma_commit(smem_u32(&bar2)); }
      if (mode == 10) {
        uint32_t ok;
        do {
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(ok) : "r"(smem_u32(&bar3)), "r"(0) : "memory");
        } while (!ok);
      }
      if (mode == 11) { while (*(volatile uint32_t*)&tmem_base == 0xFFFFFFFFu) {} }
      if (mode == 12 && (row & 3) == 0) { mbar_wait(smem_u32(&bar3), 0); }
      if (mode == 13) {
        uint32_t ok;
        do {
          asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(ok) : "r"(smem_u32(&bar3)), "r"(0) : "memory");
        } while (!ok);
      }
      if (mode == 3) d = tbase + (uint32_t)((13 - (row % 14)) * 32);
      else d = tbase + (mode == 1 ? 32u : 0u);
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        uint32_t dd = (mode == 2 && (j & 1)) ? tbase + 32 : d;
        mma_ss(dd, a0 + (uint32_t)(j * 8), b0 + (uint32_t)((j & 1) * 512), idesc, 1u);
      }
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    cyc[blockIdx.x] = clock64() - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1 || warp == 0) {}
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

void run_pattern(int mode) {
  long long* dcyc; CK(cudaMalloc(&dcyc, 148 * 8));
  int smem = 120 * 1024;
  CK(cudaFuncSetAttribute(pattern_kernel<96>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 6 * 2000;
  for (int rep = 0; rep < 2; ++rep) pattern_kernel<96><<<148, 128, smem>>>(iters, mode, dcyc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<long long> cyc(148);
  CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
  long long mx = 0; for (auto c : cyc) mx = c > mx ? c : mx;
  printf("pattern N=96 mode=%d : %.1f cyc/mma\n", mode, (double)mx / iters);
  cudaFree(dcyc);
}


// group kernel: per group: 2 waits on completed barriers, G*6 MMAs (N=96), 2 commits.
// variant v: 0 = as described; 1 = no waits/commits; 2 = only commits; 3 = only waits; 4 = 8 ALU ops per row
template <int G>
__global__ void group_kernel(int ngroups, int v, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1); mbar_init(smem_u32(&bar2), 1); mbar_init(smem_u32(&bar3), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" :: "r"(smem_u32(&bar3)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    uint32_t abase = smem_u32(smem);
    uint32_t bbase = abase + 48 * 1024;
    const uint32_t idesc = make_idesc(128, 96);
    const uint64_t a0 = make_desc(abase, 6400, 128), b0 = make_desc(bbase, 96 * 16, 128);
    uint32_t x = threadIdx.x + 7;
    long long c0 = clock64();
    for (int g = 0; g < ngroups; ++g) {
      if (v == 0 || v == 3) { mbar_wait(smem_u32(&bar3), 0); mbar_wait(smem_u32(&bar3), 0); }
#pragma unroll
      for (int r = 0; r < G; ++r) {
        const uint32_t d = tbase + (uint32_t)(((13 - r) & 15) * 32);
#pragma unroll
        for (int j = 0; j < 6; ++j) mma_ss(d, a0 + (uint32_t)(j * 8 + r), b0 + (uint32_t)((j & 1) * 512), idesc, 1u);
        if (v == 4) {
#pragma unroll
          for (int k = 0; k < 8; ++k) x = x * 1664525u + 1013904223u;
        }
      }
      if (v == 0 || v == 2) { mma_commit(smem_u32(&bar2)); mma_commit(smem_u32(&bar2)); }
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    cyc[blockIdx.x] = clock64() - c0 + (x == 12345 ? 1 : 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

template <int G>
void run_group(int v) {
  long long* dcyc; CK(cudaMalloc(&dcyc, 148 * 8));
  int smem = 120 * 1024;
  CK(cudaFuncSetAttribute(group_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int ng = 12000 / (6 * G);
  for (int rep = 0; rep < 2; ++rep) group_kernel<G><<<148, 128, smem>>>(ng, v, dcyc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<long long> cyc(148);
  CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
  long long mx = 0; for (auto c : cyc) mx = c > mx ? c : mx;
  printf("group G=%d v=%d : %.1f cyc/mma  (%.0f cyc/group)\n", G, v, (double)mx / (ng * 6 * G), (double)mx / ng);
  cudaFree(dcyc);
}

template <int N>
bool run_probe(int mode) {
  const int ROWS = 144;
  std::vector<float> a(ROWS * 16), b(N * 16), out(128 * N);
  for (int m = 0; m < ROWS; ++m) for (int k = 0; k < 16; ++k) a[m * 16 + k] = (float)(((m * 3 + k * 5) % 7) - 3);
  for (int n = 0; n < N; ++n) for (int k = 0; k < 16; ++k) b[n * 16 + k] = (float)(((n * 5 + k * 3 + 1) % 5) - 2);
  float *da, *db, *dout;
  CK(cudaMalloc(&da, a.size() * 4)); CK(cudaMalloc(&db, b.size() * 4)); CK(cudaMalloc(&dout, out.size() * 4));
  CK(cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  probe_kernel<N><<<1, 128, 32768>>>(da, db, mode, dout);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    double ref = 0;
    int ms = m + (mode == 1 ? 3 : 0);
    for (int k = 0; k < 16; ++k) {
      double av = (mode == 2) ? a[ms * 16 + (k % 8)] : a[ms * 16 + k];
      ref += av * b[n * 16 + k];
    }
    if (out[m * N + n] != (float)ref) { if (bad < 5) printf("  mismatch m=%d n=%d got %f ref %f\n", m, n, out[m * N + n], ref); ++bad; }
  }
  printf("probe N=%d mode=%d : %s (%d bad)\n", N, mode, bad ? "FAIL" : "ok", bad);
  cudaFree(da); cudaFree(db); cudaFree(dout);
  return bad == 0;
}

template <int N>
void run_tput(int nshift) {
  int nsm = 148; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  long long* dcyc; unsigned long long* dns;
  CK(cudaMalloc(&dcyc, nsm * 8)); CK(cudaMalloc(&dns, nsm * 8));
  int smem = 120 * 1024;
  CK(cudaFuncSetAttribute(tput_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 18 * 1200;
  for (int rep = 0; rep < 2; ++rep) tput_kernel<N><<<nsm, 128, smem>>>(iters, nshift, dcyc, dns);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<long long> cyc(nsm); std::vector<unsigned long long> ns(nsm);
  CK(cudaMemcpy(cyc.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ns.data(), dns, nsm * 8, cudaMemcpyDeviceToHost));
  double cmax = 0, nmax = 0; for (int i = 0; i < nsm; ++i) { cmax = cyc[i] > cmax ? cyc[i] : cmax; nmax = ns[i] > nmax ? ns[i] : nmax; }
  double flops = 2.0 * 128 * N * 16 * (double)iters * nsm;
  printf("tput M=128 N=%3d nshift=%d : %.2f cyc/mma (ideal %.1f)  chip %.1f TFLOP/s  clk %.0f MHz\n", N, nshift,
         cmax / iters, 128.0 * N / 256.0, flops / (nmax * 1e-9) / 1e12, cmax / nmax * 1e3);
  cudaFree(dcyc); cudaFree(dns);
}

int main() {
  bool ok = true;
  for (int v = 0; v < 5; ++v) { run_group<1>(v); run_group<2>(v); run_group<4>(v); run_group<8>(v); }
  printf("ALL_PROBES %s\n", ok ? "OK" : "FAIL");
  return 0;
}
