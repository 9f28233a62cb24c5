// Probe of the tcgen05 (UMMA) tf32 path used by the tensor-core adjoint: D[128x32] = A[128x32] .
// B[32x32]^T with both operands K-major in the SWIZZLE_NONE ("interleave") canonical layout,
// 3xTF32 split (A_hi B_hi + A_hi B_lo + A_lo B_hi), accumulator in TMEM read back with
// tcgen05.ld.32x32b.x32.  Prints the max relative error against an fp64 host reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_tf32_probe umma_tf32_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 32;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// byte offset of element (r, k) of a K-major interleaved operand with K columns
__host__ __device__ __forceinline__ unsigned kmaj_off(int r, int k) {
  return (unsigned)((k >> 2) * 128 + (r >> 3) * (K / 4) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t sdesc(unsigned saddr, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                     // version = 1 (Blackwell)
  return d;                                   // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}
__device__ __forceinline__ float tf32_hi(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(128) probe(const float *A, const float *B, float *D, int mode) {
  __shared__ __align__(128) unsigned char sm[2 * M * K * 4 + 2 * N * K * 4];   // A_hi, A_lo, B_hi, B_lo
  __shared__ __align__(8) unsigned long long bar;
  __shared__ unsigned tmem_base;
  unsigned char *Ahi = sm, *Alo = sm + M * K * 4, *Bhi = sm + 2 * M * K * 4, *Blo = Bhi + N * K * 4;
  const int t = threadIdx.x;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // operands: row t of A; rows of B by threads < N
  for (int k = 0; k < K; ++k) {
    const float x = A[t * K + k];
    const float h = mode ? tf32_hi(x) : x;
    *reinterpret_cast<float *>(Ahi + kmaj_off(t, k)) = h;
    *reinterpret_cast<float *>(Alo + kmaj_off(t, k)) = x - h;
  }
  if (t < N)
    for (int k = 0; k < K; ++k) {
      const float x = B[t * K + k];
      const float h = mode ? tf32_hi(x) : x;
      *reinterpret_cast<float *>(Bhi + kmaj_off(t, k)) = h;
      *reinterpret_cast<float *>(Blo + kmaj_off(t, k)) = x - h;
    }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;
  if (t == 0) {
    const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(N >> 3) << 17) |
                           ((unsigned)(M >> 4) << 24);
    const unsigned char *As[3] = {Ahi, Ahi, Alo}, *Bs[3] = {Bhi, Blo, Bhi};
    const int nprod = mode == 2 ? 3 : 1;
    int first = 1;
    for (int p = 0; p < nprod; ++p)
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t da = sdesc(su32(As[p]) + ks * 256, 128, (K / 4) * 128);
        const uint64_t db = sdesc(su32(Bs[p]) + ks * 256, 128, (K / 4) * 128);
        const unsigned acc = first ? 0u : 1u;
        asm volatile("{\n .reg .pred pa;\n setp.ne.b32 pa, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, pa;\n}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        first = 0;
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)su32(&bar)));
  }
  // wait for the MMAs
  {
    unsigned ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, 1000000;\n"
                   " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    } while (!ok);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  unsigned v[32];
  const unsigned taddr = tmem + ((unsigned)((t >> 5) * 32) << 16);
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
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

// TS variant: A (hi, lo) written to TMEM with tcgen05.st.32x32b.x32 (row = lane), B from smem.
__global__ void __launch_bounds__(128) probe_ts(const float *A, const float *B, float *D) {
  __shared__ __align__(128) unsigned char sm[2 * N * K * 4];    // B_hi, B_lo
  __shared__ __align__(8) unsigned long long bar;
  __shared__ unsigned tmem_base;
  unsigned char *Bhi = sm, *Blo = sm + N * K * 4;
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
      const float x = B[t * K + k];
      const float h = tf32_hi(x);
      *reinterpret_cast<float *>(Bhi + kmaj_off(t, k)) = h;
      *reinterpret_cast<float *>(Blo + kmaj_off(t, k)) = x - h;
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;          // cols [0,32) A_hi, [32,64) A_lo, [64,96) D
  unsigned hv[32], lv[32];
  for (int k = 0; k < K; ++k) {
    const float x = A[t * K + k];
    const float h = tf32_hi(x);
    hv[k] = __float_as_uint(h);
    lv[k] = __float_as_uint(x - h);
  }
  const unsigned lane_base = (unsigned)((t >> 5) * 32) << 16;
#define ST32(addr, v) asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
    ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), \
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory")
  ST32(tmem + lane_base + 0, hv);
  ST32(tmem + lane_base + 32, lv);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(N >> 3) << 17) |
                           ((unsigned)(M >> 4) << 24);
    const unsigned acol[3] = {0u, 0u, 32u};
    const unsigned char *Bs[3] = {Bhi, Blo, Bhi};
    int first = 1;
    for (int p = 0; p < 3; ++p)
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t db = sdesc(su32(Bs[p]) + ks * 256, 128, (K / 4) * 128);
        const unsigned acc = first ? 0u : 1u;
        asm volatile("{\n .reg .pred pa;\n setp.ne.b32 pa, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, pa;\n}"
                     ::"r"(tmem + 64), "r"(tmem + acol[p] + ks * 8), "l"(db), "r"(idesc), "r"(acc));
        first = 0;
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)su32(&bar)));
  }
  {
    unsigned ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, 1000000;\n"
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

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) * (1.0f / 16777216.0f) * 2.f - 1.f; };
  for (auto &x : A) x = rnd();
  for (auto &x : B) x = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    if (mode < 3) probe<<<1, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(r - D[m * N + n]));
        maxref = fmax(maxref, fabs(r));
      }
    if (mode == 3) { cudaMemset(dD, 0, D.size() * 4); probe_ts<<<1, 128>>>(dA, dB, dD); e = cudaDeviceSynchronize(); cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost); }
    if (mode == 3) {
      printf("rows with err>1e-3:");
      for (int m = 0; m < M; ++m) { double e = 0; for (int n = 0; n < N; ++n) { double r = 0; for (int k = 0; k < K; ++k) r += (double)A[m*K+k]*B[n*K+k]; e = fmax(e, fabs(r - D[m*N+n])); } if (e > 1e-3) printf(" %d", m); }
      printf("\nrow 40 got/ref:"); for (int n = 0; n < 4; ++n) { double r = 0; for (int k = 0; k < K; ++k) r += (double)A[40*K+k]*B[n*K+k]; printf(" %.4f/%.4f", D[40*N+n], r); }
      printf("\nrow 20 got/ref:"); for (int n = 0; n < 4; ++n) { double r = 0; for (int k = 0; k < K; ++k) r += (double)A[20*K+k]*B[n*K+k]; printf(" %.4f/%.4f", D[20*N+n], r); }
      printf("\n");
    }
    printf("{\"mode\":%d,\"what\":\"%s\",\"max_abs_err\":%.3e,\"max_ref\":%.3e,\"rel\":%.3e,\"cuda\":\"%s\","
           "\"D00\":%.6f}\n", mode, mode == 0 ? "tf32 raw" : mode == 1 ? "tf32 hi only" : mode == 2 ? "3xTF32 SS" : "3xTF32 TS (A in TMEM)",
           maxerr, maxref, maxerr / maxref, cudaGetErrorString(e), D[0]);
  }
  return 0;
}
