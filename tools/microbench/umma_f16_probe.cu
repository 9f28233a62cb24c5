// Probe of tcgen05.mma kind::f16 with fp32 accumulation, A in tensor memory (packed f16x2 per
// 32-bit column, row = lane) and B in shared memory (K-major, SWIZZLE_NONE, 16-bit elements):
// D[128x32] = A[128x32] . B[32x32]^T, "3xFP16" split (A_hi B_hi + A_hi B_lo + A_lo B_hi) with
// hi = x with the 13 low mantissa bits cleared (exact in fp16 for |x| >= 2^-14), lo = x - hi.
// Checks which half of a TMEM column holds the even K element (variant 0: low half) and prints the
// max error against an fp64 host reference.  Also times a long chain of MMAs of the production
// shape (M = 128, N = 64, K = 16) against the same chain in kind::tf32 (K = 8).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_f16_probe umma_f16_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, N = 32, K = 32;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// byte offset of element (r, k) of a K-major 16-bit operand with K columns: 8-element (16-byte)
// chunks along K, 8 rows x 16 B core matrices, chunk stride 128 B, 8-row group stride K/8 * 128 B
__host__ __device__ __forceinline__ unsigned kmaj16(int r, int k) {
  return (unsigned)((k >> 3) * 128 + (r >> 3) * (K / 8) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc(unsigned saddr, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ float hi13(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ unsigned pack2(float lo_elem, float hi_elem) {   // lo_elem -> bits 0..15
  unsigned r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}

template <int VARIANT>
__global__ void __launch_bounds__(128) probe(const float *A, const float *B, float *D) {
  __shared__ __align__(128) unsigned char sm[2 * N * K * 2];    // B_hi, B_lo (fp16)
  __shared__ __align__(8) unsigned long long bar;
  __shared__ unsigned tmem_base;
  unsigned char *Bhi = sm, *Blo = sm + N * K * 2;
  const int t = threadIdx.x;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (t < N)
    for (int k = 0; k < K; ++k) {
      const float x = B[t * K + k], h = hi13(x);
      *reinterpret_cast<__half *>(Bhi + kmaj16(t, k)) = __float2half_rn(h);
      *reinterpret_cast<__half *>(Blo + kmaj16(t, k)) = __float2half_rn(x - h);
    }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;          // cols [0,16) A_hi, [16,32) A_lo, [64,96) D
  unsigned hv[16], lv[16];
  for (int c = 0; c < K / 2; ++c) {
    const float x0 = A[t * K + 2 * c], x1 = A[t * K + 2 * c + 1];
    const float h0 = hi13(x0), h1 = hi13(x1);
    if (VARIANT == 0) { hv[c] = pack2(h0, h1); lv[c] = pack2(x0 - h0, x1 - h1); }
    else { hv[c] = pack2(h1, h0); lv[c] = pack2(x1 - h1, x0 - h0); }
  }
  const unsigned lane_base = (unsigned)((t >> 5) * 32) << 16;
#define ST16(addr, v) asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
    ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory")
  ST16(tmem + lane_base + 0, hv);
  ST16(tmem + lane_base + 16, lv);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    // kind::f16: c_format F32 (bits 4-5 = 1), a/b_format F16 (0), K-major, N >> 3, M >> 4
    const unsigned idesc = (1u << 4) | ((unsigned)(N >> 3) << 17) | ((unsigned)(M >> 4) << 24);
    const unsigned acol[3] = {0u, 0u, 16u};
    const unsigned char *Bs[3] = {Bhi, Blo, Bhi};
    int first = 1;
    for (int p = 0; p < 3; ++p)
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint64_t db = sdesc(su32(Bs[p]) + ks * 256, 128, (K / 8) * 128);
        const unsigned acc = first ? 0u : 1u;
        asm volatile("{\n .reg .pred pa;\n setp.ne.b32 pa, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, pa;\n}"
                     ::"r"(tmem + 64), "r"(tmem + acol[p] + ks * 8), "l"(db), "r"(idesc), "r"(acc));
        first = 0;
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)su32(&bar)));
  }
  {
    unsigned ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                   " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    } while (!ok);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  unsigned v[32];
  const unsigned taddr = tmem + 64 + lane_base;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                 "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                 "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < N; ++n) D[t * N + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// Throughput: one CTA per SM (x4 CTAs), thread 0 issues R rounds of the production MMA group
// (3 products x 2 K-steps of kind::f16 K=16, or 3 x 4 K-steps of kind::tf32 K=8), N = 64, M = 128,
// each round committed and awaited (as the kernel does per antenna).  Operand contents irrelevant.
template <bool F16>
__global__ void __launch_bounds__(128) mma_rate(int rounds, long long *cyc) {
  __shared__ __align__(128) unsigned char sm[2 * 64 * 32 * 4];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ unsigned tmem_base;
  const int t = threadIdx.x;
  for (int i = t; i < (int)sizeof(sm) / 4; i += 128) reinterpret_cast<float *>(sm)[i] = 0.f;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;
  if (t == 0) {
    const int NN = 64;
    const unsigned idesc = F16 ? ((1u << 4) | ((unsigned)(NN >> 3) << 17) | ((unsigned)(128 >> 4) << 24))
                               : ((1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(NN >> 3) << 17) |
                                  ((unsigned)(128 >> 4) << 24));
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      for (int p = 0; p < 3; ++p)
        for (int ks = 0; ks < (F16 ? 2 : 4); ++ks) {
          const uint64_t db = sdesc(su32(sm) + ks * 256, 128, F16 ? 512 : 1024);
          if (F16)
            asm volatile("{\n .reg .pred pa;\n setp.ne.b32 pa, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, pa;\n}"
                         ::"r"(tmem + 64), "r"(tmem + ks * 8), "l"(db), "r"(idesc), "r"(p | ks));
          else
            asm volatile("{\n .reg .pred pa;\n setp.ne.b32 pa, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, pa;\n}"
                         ::"r"(tmem + 64), "r"(tmem + ks * 8), "l"(db), "r"(idesc), "r"(p | ks));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)su32(&bar)));
      unsigned ok = 0;
      do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(&bar)), "r"((unsigned)(r & 1)) : "memory");
      } while (!ok);
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) * (1.0f / 16777216.0f) * 2.f - 1.f; };
  for (auto &x : A) x = rnd();
  for (auto &x : B) x = rnd() * (rnd() > 0.8f ? 1e-3f : 1.f);   // some small elements too
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dD, 0, D.size() * 4);
    if (variant == 0) probe<0><<<1, 128>>>(dA, dB, dD); else probe<1><<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0, se = 0, sr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[n * K + k];
        const double d = r - D[m * N + n];
        maxerr = fmax(maxerr, fabs(d)); maxref = fmax(maxref, fabs(r)); se += d * d; sr += r * r;
      }
    printf("{\"variant\":%d,\"even_k_in\":\"%s\",\"max_abs_err\":%.3e,\"max_ref\":%.3e,\"rel_l2\":%.3e,\"cuda\":\"%s\"}\n",
           variant, variant == 0 ? "low half" : "high half", maxerr, maxref, sqrt(se / sr), cudaGetErrorString(e));
  }
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *dc; cudaMalloc(&dc, sizeof(long long) * nsm * 4);
  std::vector<long long> cyc(nsm * 4);
  const int rounds = 20000;
  for (int f16 = 1; f16 >= 0; --f16) {
    for (int ctas = 1; ctas <= 4; ctas *= 2) {
      if (f16) mma_rate<true><<<nsm * ctas, 128>>>(rounds, dc); else mma_rate<false><<<nsm * ctas, 128>>>(rounds, dc);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(cyc.data(), dc, sizeof(long long) * nsm * ctas, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < nsm * ctas; ++i) mx = fmax(mx, (double)cyc[i]);
      // per SM: ctas CTAs each doing `rounds` rounds of 128 x 64 x 32 complex-real MACs x 3
      const double macs = 3.0 * 128 * 64 * 32 * rounds * ctas;
      printf("{\"kind\":\"%s\",\"ctas_per_sm\":%d,\"cycles_per_round_per_cta\":%.1f,\"mac_per_sm_cycle\":%.1f,\"cuda\":\"%s\"}\n",
             f16 ? "f16" : "tf32", ctas, mx / rounds, macs / mx, cudaGetErrorString(e));
    }
  }
  return 0;
}
