// Horner inner-loop shapes for K3/K4 on sm_100a: measure packed-FP32 (FFMA2) throughput of the
// straight-line complex Horner h = h w + X_m over NF bins with X broadcast from shared memory, for
// C independent chains per sample (bin blocks sharing w) and S samples per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o horner_shapes horner_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk(float x, float y) { f2x r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 upk(f2x r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ f2x ffma2(f2x a, f2x b, f2x c) { f2x d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

constexpr int NF = 256, NANT = 16, REP = 4, TPB = 128;

template <int C, int S>
__global__ void __launch_bounds__(TPB) horner(const float2 *Xg, float2 *out) {
  __shared__ float4 xs4[NANT * NF / 2];
  float2 *xs = reinterpret_cast<float2 *>(xs4);
  constexpr int Q = NF / C;
  for (int i = threadIdx.x; i < NANT * NF; i += TPB) {
    const int row = i / NF, col = i % NF, c = col / Q, m = col % Q;
    xs[row * NF + m * C + c] = Xg[i];
  }
  __syncthreads();
  float2 acc = make_float2(0.f, 0.f);
  const float th0 = (blockIdx.x * TPB + threadIdx.x) * 1e-5f;
  for (int a = 0; a < NANT * REP; ++a) {
    f2x w[S], h[S][C];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      float sn, cs;
      __sincosf(th0 + s * 1e-3f + a * 1e-4f, &sn, &cs);
      w[s] = pk(cs, sn);
#pragma unroll
      for (int c = 0; c < C; ++c) h[s][c] = 0ull;
    }
    const float4 *X4 = xs4 + (a % NANT) * NF / 2;
#pragma unroll
    for (int m = Q - 1; m >= 0; --m) {
      float2 xv[C];
#pragma unroll
      for (int c = 0; c < C; c += 2) {
        const float4 v = X4[(m * C + c) / 2];
        xv[c] = make_float2(v.x, v.y);
        xv[c + 1] = make_float2(v.z, v.w);
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const float2 wv = upk(w[s]);
        const f2x w2 = pk(-wv.y, wv.x);
        f2x t[C];
#pragma unroll
        for (int c = 0; c < C; ++c) { const float2 v = upk(h[s][c]); t[c] = ffma2(w[s], pk(v.x, v.x), pk(xv[c].x, xv[c].y)); }
#pragma unroll
        for (int c = 0; c < C; ++c) { const float2 v = upk(h[s][c]); h[s][c] = ffma2(w2, pk(v.y, v.y), t[c]); }
      }
    }
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int c = 0; c < C; ++c) { const float2 v = upk(h[s][c]); acc.x += v.x; acc.y += v.y; }
  }
  out[blockIdx.x * TPB + threadIdx.x] = acc;
}

template <int C, int S>
void run(const char *name, const float2 *X, float2 *out, int nsm) {
  const int grid = nsm * 8 * 16 / S;   // same total samples x antennas work per shape
  horner<C, S><<<grid, TPB>>>(X, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) horner<C, S><<<grid, TPB>>>(X, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double lane_ops = 5.0 * grid * TPB * (double)S * NANT * REP * NF * 4;   // 4 lane-FMA per bin
  const double peak = nsm * 128.0 * 1.965e9;
  printf("{\"shape\":\"%s\",\"ms\":%.3f,\"lane_ops_per_s\":%.4e,\"frac_of_1965MHz_peak\":%.3f,\"err\":\"%s\"}\n",
         name, ms / 5, lane_ops / (ms * 1e-3), lane_ops / (ms * 1e-3) / peak,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float2 *X, *out;
  cudaMalloc(&X, NANT * NF * sizeof(float2));
  cudaMalloc(&out, nsm * 8 * 16 * TPB * sizeof(float2));
  cudaMemset(X, 0, NANT * NF * sizeof(float2));
  run<2, 1>("C2_S1", X, out, nsm);
  run<4, 1>("C4_S1", X, out, nsm);
  run<8, 1>("C8_S1", X, out, nsm);
  run<2, 2>("C2_S2", X, out, nsm);
  run<4, 2>("C4_S2", X, out, nsm);
  run<2, 4>("C2_S4", X, out, nsm);
  run<4, 4>("C4_S4", X, out, nsm);
  return 0;
}
