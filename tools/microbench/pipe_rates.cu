// Pipe-rate microbenchmark for the B200 (sm_100a): FP32 FFMA (3-register, packed f32x2),
// FADD, FP64 DFMA, MUFU sin/cos, F2F conversions, and the forward kernel's inner step
// (Chebyshev recurrence + accumulate).  Used to fix the ALU roofline denominators in DESIGN.md.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu
// Each test: grid = n_sm * BPS blocks of TPB threads, ITERS iterations of U independent chains.
// Reported: lane-ops per SM per cycle (from clock64 in each block, median over blocks)
// and lane-ops/s from CUDA events.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int TPB = 512;
constexpr int ITERS = 4096;

__device__ long long g_cyc[4096];

template <int U>
__global__ void k_ffma(float *out, float b, float c) {
  float a[U];
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = threadIdx.x * 1e-3f + u;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = fmaf(a[u], b, c);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) s += a[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// 3 distinct register sources per FFMA (b[u], c[u] differ per chain)
template <int U>
__global__ void k_ffma3(float *out, float b0, float c0) {
  float a[U], b[U], c[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { a[u] = threadIdx.x * 1e-3f + u; b[u] = b0 + u * 1e-7f; c[u] = c0 - u * 1e-7f; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = fmaf(a[u], b[u], c[u]);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) s += a[u] + b[u] + c[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void upk(unsigned long long r, float &x, float &y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int U>
__global__ void k_ffma2(float *out, float b0, float c0) {
  unsigned long long a[U];
  unsigned long long b = pk(b0, b0 * 0.5f), c = pk(c0, c0 * 0.25f);
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = pk(threadIdx.x * 1e-3f + u, u * 0.5f);
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = ffma2(a[u], b, c);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) { float x, y; upk(a[u], x, y); s += x + y; }
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// Forward inner step, scalar: y_{m+1} = k*y_m - y_{m-1} (re, im), acc_m += y_m.
// 4 lane-ops per complex contribution.  U bins unrolled, accumulators in registers.
template <int U>
__global__ void k_cheb(float *out, float k0) {
  float ar[U], ai[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { ar[u] = 0.f; ai[u] = 0.f; }
  float k = k0 + threadIdx.x * 1e-9f;
  float y0r = 0.3f, y0i = 0.2f, y1r = 0.25f, y1i = 0.1f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS / U * 4; ++it) {
    float pr = y0r, pi = y0i, cr = y1r, ci = y1i;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ar[u] += pr; ai[u] += pi;
      float nr = fmaf(k, cr, -pr), ni = fmaf(k, ci, -pi);
      pr = cr; pi = ci; cr = nr; ci = ni;
    }
    y0r = pr * 0.999f; y0i = pi; y1r = cr; y1i = ci * 1.0001f;
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) s += ar[u] + ai[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// Same step with packed f32x2 and the period-4 sign trick q_m = sigma_m y_m, sigma = (+,+,-,-):
// q_{m+1} = (+-k) q_m + q_{m-1}, acc_m += q_m (sign fixed at write-out): 1 FFMA2 + 1 FADD2.
template <int U>
__global__ void k_cheb2(float *out, float k0) {
  unsigned long long acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0ull;
  float kk = k0 + threadIdx.x * 1e-9f;
  unsigned long long kp = pk(kk, kk), kn = pk(-kk, -kk);
  unsigned long long y0 = pk(0.3f, 0.2f), y1 = pk(0.25f, 0.1f);
  long long t0 = clock64();
  for (int it = 0; it < ITERS / U * 4; ++it) {
    unsigned long long p = y0, c = y1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = fadd2(acc[u], c);
      unsigned long long n = ffma2((u & 1) ? kn : kp, c, p);
      p = c; c = n;
    }
    y0 = c; y1 = p;
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) { float x, y; upk(acc[u], x, y); s += x + y; }
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// Horner with packed f32x2: h' = hr*(wr,wi) + hi*(-wi,wr) + G : 2 FFMA2 per complex contribution.
template <int S>
__global__ void k_horner2(float *out, float wr0, float wi0) {
  unsigned long long h[S], wa[S], wb[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    h[s] = 0ull; float a = wr0 + s * 1e-6f, b = wi0 - s * 1e-6f;
    wa[s] = pk(a, b); wb[s] = pk(-b, a);
  }
  unsigned long long G = pk(threadIdx.x * 1e-4f, 0.5f), dG = pk(1e-7f, 0.f);
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float hr, hi; upk(h[s], hr, hi);
      unsigned long long t = ffma2(pk(hr, hr), wa[s], G);
      h[s] = ffma2(pk(hi, hi), wb[s], t);
    }
    G = fadd2(G, dG);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < S; ++q) { float x, y; upk(h[q], x, y); s += x + y; }
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// Horner step (backward/filter): h = h*w + G_m : 4 FFMA per complex contribution; S independent pairs.
template <int S>
__global__ void k_horner(float *out, float wr0, float wi0) {
  float hr[S], hi[S], wr[S], wi[S];
#pragma unroll
  for (int s = 0; s < S; ++s) { hr[s] = 0.f; hi[s] = 0.f; wr[s] = wr0 + s * 1e-6f; wi[s] = wi0 - s * 1e-6f; }
  float gr = threadIdx.x * 1e-4f, gi = 0.5f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float nr = fmaf(hr[s], wr[s], fmaf(-hi[s], wi[s], gr));
      float ni = fmaf(hr[s], wi[s], fmaf(hi[s], wr[s], gi));
      hr[s] = nr; hi[s] = ni;
    }
    gr += 1e-7f;
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < S; ++q) s += hr[q] + hi[q];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int U>
__global__ void k_dfma(float *out, double b, double c) {
  double a[U];
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = threadIdx.x * 1e-3 + u;
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = fma(a[u], b, c);
  }
  long long t1 = clock64();
  double s = 0.;
#pragma unroll
  for (int u = 0; u < U; ++u) s += a[u];
  if (s == 12345.) out[0] = (float)s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int U>
__global__ void k_mufu(float *out, float b) {
  float a[U];
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = threadIdx.x * 1e-3f + u;
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __sinf(a[u]) + b;   // MUFU.SIN + FADD (+ FMUL range scale)
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) s += a[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int U>
__global__ void k_f2f(float *out, float b) {
  float a[U];
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = threadIdx.x * 1e-3f + u;
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) { double d = (double)a[u]; d = d * 1.0000001; a[u] = (float)d; }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) s += a[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <typename K, typename... Args>
void run(const char *name, double ops_per_thread, int bps, K kern, Args... args) {
  int dev; CK(cudaGetDevice(&dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int nsm = p.multiProcessorCount;
  int grid = nsm * bps;
  float *out; CK(cudaMalloc(&out, 4));
  kern<<<grid, TPB>>>(out, args...);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, TPB>>>(out, args...);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> cyc(grid);
  CK(cudaMemcpyFromSymbol(cyc.data(), g_cyc, sizeof(long long) * grid));
  std::sort(cyc.begin(), cyc.end());
  double med = (double)cyc[grid / 2];
  double tot_ops = ops_per_thread * TPB * grid;
  double per_sm_cyc = ops_per_thread * TPB * bps / med;
  double rate = tot_ops / (ms * 1e-3);
  // implied clock: cycles per block (median) / kernel time (rough, includes launch)
  printf("{\"test\":\"%s\",\"lane_ops_per_sm_per_cycle\":%.2f,\"lane_ops_per_s\":%.4e,\"ms\":%.3f,"
         "\"implied_mhz\":%.0f,\"n_sm\":%d}\n",
         name, per_sm_cyc, rate, ms, med / (ms * 1e-3) / 1e6, nsm);
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\":\"%s\",\"sm\":%d,\"cc\":\"%d.%d\",\"clock_khz\":%d}\n", p.name,
         p.multiProcessorCount, p.major, p.minor, p.clockRate);
  run("ffma_imm_like_U8", (double)ITERS * 8, 4, k_ffma<8>, 0.999f, 0.001f);
  run("ffma_3reg_U8", (double)ITERS * 8, 4, k_ffma3<8>, 0.999f, 0.001f);
  run("ffma2_U8(x2 lanes)", (double)ITERS * 8 * 2, 4, k_ffma2<8>, 0.999f, 0.001f);
  run("cheb_scalar_U16(4 ops/contrib)", (double)(ITERS / 16 * 4) * 16 * 4, 4, k_cheb<16>, 1.9f);
  run("cheb_f32x2_U16(4 ops/contrib)", (double)(ITERS / 16 * 4) * 16 * 4, 4, k_cheb2<16>, 1.9f);
  run("horner_S4(4 ffma/contrib)", (double)ITERS * 4 * 4, 4, k_horner<4>, 0.9f, 0.1f);
  run("horner_S8(4 ffma/contrib)", (double)ITERS * 8 * 4, 2, k_horner<8>, 0.9f, 0.1f);
  run("horner2_S4(4 lane-ffma/contrib)", (double)ITERS * 4 * 4, 4, k_horner2<4>, 0.9f, 0.1f);
  run("horner2_S8(4 lane-ffma/contrib)", (double)ITERS * 8 * 4, 2, k_horner2<8>, 0.9f, 0.1f);
  run("dfma_U8", (double)(ITERS / 8) * 8, 4, k_dfma<8>, 0.999, 0.001);
  run("mufu_sin+fadd_U8(per sin)", (double)(ITERS / 8) * 8, 4, k_mufu<8>, 0.1f);
  run("f2f_roundtrip+dmul_U8(per elem)", (double)(ITERS / 8) * 8, 4, k_f2f<8>, 0.1f);
  return 0;
}
