// rfr_tc_gemm.cu -- the r2 engine's two dense complex contractions on the 5th-generation tensor
// cores (tcgen05.mma.kind::f16, accumulators in TMEM), SURVEY 8(f) NEXT-2's tensor-core half.
//
// Both contract one antenna's row against the SAME table a[m][q] = eps_q (-j)^q J_q(2 pi m' delta_g)
// (the global Jacobi-Anger / Chebyshev expansion of DESIGN 5b / 5e, Eq. 3, Eq. 4
// P:L231-234), so over a block of 128 antennas they are plain GEMMs with a shared operand:
//
//   expansion of the adjoint rows (K3 App. A.5, K4 Eq. 3):
//       G_i[q] = sum_m Y_i[m] conj(a[m][q]),   Y_i[m] = X_i[m] e^{+j 2 pi m' u_g,i}
//       real form D[i][2q + c] = sum_k A[i][k] B[2q + c][k] with k = 2m + c' (Re, Im interleaved):
//       B[2q][2m] = Re a, B[2q][2m+1] = Im a, B[2q+1][2m] = -Im a, B[2q+1][2m+1] = Re a;
//   bins of the forward (the last step of k2_fout):
//       s_i[m] = e^{-j 2 pi m' u_g,i} sum_q a[m][q] M_g,i[q]
//       B[2m][2q] = Re a, B[2m][2q+1] = -Im a, B[2m+1][2q] = Im a, B[2m+1][2q+1] = Re a.
//
// fp32-level accuracy from the "3xFP16" split (A_hi B_hi + A_hi B_lo + A_lo B_hi, hi = x with the
// 13 low mantissa bits cleared, lo = x - hi; 22 significant bits, the scheme of rfr_tc.cu), A rows
// scaled by a power of two to max |Y| (or |M_g|) in [0.5, 1) for fp16's range and unscaled in the
// epilogue; |a| <= 2 needs no scaling.  A (per-antenna, built by the threads: thread = antenna =
// TMEM lane) is written to tensor memory with tcgen05.st; B (the shared table) is split once per
// plan into fp16 images (k2_tc_bimg) that one thread brings into shared memory with bulk copies on
// the TMA engine (cp.async.bulk, mbarrier completion), double-buffered over K for the expansion.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "rfr_device.cuh"
#include "rfr_tcgen05.cuh"
#include "rfr_tiled.h"

namespace rfr {

namespace {


// byte offset of fp16 element (row n, column k) of a K-major SWIZZLE_NONE operand whose rows are
// KW elements wide: core matrices of 8 rows x 16 B; K-adjacent core matrices 128 B apart (LBO),
// row groups KW * 16 B apart (SBO)
__host__ __device__ __forceinline__ unsigned kmaj16(int n, int k, int KW) {
  return (unsigned)((k >> 3) * 128 + (n >> 3) * (KW * 16) + (n & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ int gexp_N(int Pg) { return (2 * Pg + 15) & ~15; }    // <= 96
__device__ __forceinline__ int bins_KP(int Pg) { return (2 * Pg + 31) & ~31; }   // <= 96
__device__ __forceinline__ unsigned short f2h(float x) {
  unsigned short r;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void put_split(unsigned char *hi, unsigned char *lo, unsigned off,
                                          float v) {
  const float h = tf32_hi(v);
  *reinterpret_cast<unsigned short *>(hi + off) = f2h(h);
  *reinterpret_cast<unsigned short *>(lo + off) = f2h(v - h);
}
// power-of-two scale bringing a row's max modulus into [0.5, 1) (1 for a zero row)
__device__ __forceinline__ void row_scale(float mx2, float &sc, float &inv) {
  sc = inv = 1.f;
  if (mx2 > 0.f) {
    int ex;
    frexpf(sqrtf(mx2), &ex);
    sc = ldexpf(1.f, -ex);
    inv = ldexpf(1.f, ex);
  }
}

// fp16 hi / lo images of the a table for both GEMMs (one launch per plan, after k2_tables)
__global__ void __launch_bounds__(256) k2_tc_bimg(T2Args a) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0 || pl.Pg == 0) return;
  const int Pg = pl.Pg, nf = a.n_f, N = gexp_N(Pg), KP = bins_KP(Pg);
  const int NCg = (nf + 31) / 32, NCb = (nf + 127) / 128;
  const float2 *am = a.acoef + (int64_t)kT2PgMax * nf;            // [m][q]
  const int64_t ng = (int64_t)NCg * N * 64, nb = (int64_t)NCb * 256 * KP;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < ng + nb;
       w += (int64_t)gridDim.x * blockDim.x) {
    if (w < ng) {
      const int c = (int)(w / (N * 64)), r = (int)(w % (N * 64)), n = r / 64, k = r % 64;
      const int m = 32 * c + (k >> 1), q = n >> 1;
      float v = 0.f;
      if (m < nf && q < Pg) {
        const float2 e = am[(int64_t)m * kT2PgMax + q];
        v = (n & 1) ? ((k & 1) ? e.x : -e.y) : ((k & 1) ? e.y : e.x);
      }
      unsigned char *hi = a.tcimg + (size_t)c * kT2GexpImg;
      put_split(hi, hi + (size_t)N * 64 * 2, kmaj16(n, k, 64), v);
    } else {
      const int64_t u = w - ng;
      const int b = (int)(u / (256 * KP)), r = (int)(u % (256 * KP)), n = r / KP, k = r % KP;
      const int m = 128 * b + (n >> 1), q = k >> 1;
      float v = 0.f;
      if (m < nf && q < Pg) {
        const float2 e = am[(int64_t)m * kT2PgMax + q];
        v = (n & 1) ? ((k & 1) ? e.x : e.y) : ((k & 1) ? -e.y : e.x);
      }
      unsigned char *hi = a.tcimg + (size_t)NCg * kT2GexpImg + (size_t)b * kT2BinsImg;
      put_split(hi, hi + (size_t)256 * KP * 2, kmaj16(n, k, KP), v);
    }
  }
}

__device__ __forceinline__ void tmem_alloc(unsigned *dst, unsigned cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free(unsigned base, unsigned cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
}
__device__ __forceinline__ void tc_commit(unsigned long long *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];"
               ::"l"((uint64_t)smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// G[row][i][q] for a block of 128 antennas (thread = antenna = TMEM lane); K = 2 n_f in chunks of
// 32 bins (64 fp16 columns: A_hi at TMEM columns [0, 32), A_lo at [32, 64), D at [64, 64 + N))
__global__ void __launch_bounds__(128, 2) k2_gexp_tc(T2Args a, const float2 *X0, const float2 *X1) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0 || pl.Pg == 0) return;
  extern __shared__ __align__(128) unsigned char bsm[];              // [2][kT2GexpImg]
  __shared__ __align__(8) unsigned long long full[2], mbar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int Pg = pl.Pg, N = gexp_N(Pg), nf = a.n_f, NC = (nf + 31) / 32;
  const int row = blockIdx.y;
  const float2 *X = row == 0 ? X0 : X1;
  const int64_t i = (int64_t)blockIdx.x * 128 + tid;
  const bool valid = i < a.n_a;
  const unsigned cbytes = (unsigned)(N * 64 * 2 * 2);
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < 2 && b < NC; ++b) {
      mbar_arrive_expect_tx(&full[b], cbytes);
      bulk_g2s(bsm + (size_t)b * kT2GexpImg, a.tcimg + (size_t)b * kT2GexpImg, cbytes, &full[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = tbase, lane = (unsigned)(warp * 32) << 16;
  const unsigned a_hi = tmem, a_lo = tmem + 32, d = tmem + 64;
  const unsigned idesc = (1u << 4) | ((unsigned)(N >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
  const float2 *Xi = X + (valid ? i : 0) * (int64_t)nf;
  float mx2 = 0.f;
  if (valid)
    for (int m = 0; m < nf; ++m) {
      const float2 v = Xi[m];
      mx2 = fmaxf(mx2, fmaf(v.x, v.x, v.y * v.y));
    }
  float sc, inv;
  row_scale(mx2, sc, inv);
  const double ug = valid ? a.lg[i * 3] * a.kd : 0.0;
  for (int c = 0; c < NC; ++c) {
    unsigned hv[32], lv[32];
#pragma unroll
    for (int mm = 0; mm < 32; ++mm) {
      const int m = 32 * c + mm;
      float yr = 0.f, yi = 0.f;
      if (valid && m < nf) {
        const double cc = (double)(m - nf / 2) * ug;
        float ps, pc;                                  // e^{+j 2 pi m' u_g}
        sincospif(2.f * (float)(cc - rint(cc)), &ps, &pc);
        const float2 v = Xi[m];
        yr = fmaf(pc, v.x, -ps * v.y) * sc;
        yi = fmaf(pc, v.y, ps * v.x) * sc;
      }
      const float hr = tf32_hi(yr), hi_ = tf32_hi(yi);
      hv[mm] = pack_h2(hr, hi_);
      lv[mm] = pack_h2(yr - hr, yi - hi_);
    }
    if (c > 0) mbar_wait(&mbar, (unsigned)((c - 1) & 1));   // MMAs of chunk c-1 done with A, B
    tc_fence_after();
    if (tid == 0 && c > 0 && c + 1 < NC) {
      const int b = (c + 1) & 1;
      mbar_arrive_expect_tx(&full[b], cbytes);
      bulk_g2s(bsm + (size_t)b * kT2GexpImg, a.tcimg + (size_t)(c + 1) * kT2GexpImg, cbytes,
               &full[b]);
    }
    tmem_st16(a_hi + lane, *reinterpret_cast<const unsigned(*)[16]>(hv));
    tmem_st16(a_hi + 16 + lane, *reinterpret_cast<const unsigned(*)[16]>(hv + 16));
    tmem_st16(a_lo + lane, *reinterpret_cast<const unsigned(*)[16]>(lv));
    tmem_st16(a_lo + 16 + lane, *reinterpret_cast<const unsigned(*)[16]>(lv + 16));
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      mbar_wait(&full[c & 1], (unsigned)((c >> 1) & 1));
      const unsigned char *Bh = bsm + (size_t)(c & 1) * kT2GexpImg, *Bl = Bh + N * 64 * 2;
      const unsigned acol[3] = {a_hi, a_hi, a_lo};
      const unsigned char *bs[3] = {Bh, Bl, Bh};
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_f16_ts(d, acol[p] + 8 * ks, umma_sdesc(smem_u32(bs[p]) + ks * 256, 128, 64 * 16),
                      idesc, (c | p | ks) ? 1u : 0u);
      tc_commit(&mbar);
    }
  }
  mbar_wait(&mbar, (unsigned)((NC - 1) & 1));
  tc_fence_after();
  float2 *G = a.gexp + ((int64_t)row * a.n_a + (valid ? i : 0)) * kT2PgMax;
  for (int c0 = 0; c0 < N; c0 += 16) {
    unsigned v[16];
    tmem_ld16(d + c0 + lane, v);
    tmem_wait_ld();
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int q = c0 / 2 + h;
      if (valid && q < Pg)
        G[q] = make_float2(__uint_as_float(v[2 * h]) * inv, __uint_as_float(v[2 * h + 1]) * inv);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 256);
}

// bins of the forward for a block of 128 antennas: D at TMEM columns [0, 256) (one N chunk of 128
// bins), A_hi at [256, 256 + KP/2), A_lo after it; the B chunk images stream through one shared
// buffer (the next chunk's bulk copy overlaps this chunk's epilogue)
__global__ void __launch_bounds__(128, 1) k2_bins_tc(T2Args a, float2 *__restrict__ out) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0 || pl.Pg == 0) return;
  extern __shared__ __align__(128) unsigned char bsm[];              // [kT2BinsImg]
  __shared__ __align__(8) unsigned long long full, mbar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int Pg = pl.Pg, KP = bins_KP(Pg), nf = a.n_f, NCb = (nf + 127) / 128;
  const int64_t i = (int64_t)blockIdx.x * 128 + tid;
  const bool valid = i < a.n_a;
  const unsigned cbytes = (unsigned)(256 * KP * 2 * 2);
  const unsigned char *img = a.tcimg + (size_t)((nf + 31) / 32) * kT2GexpImg;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    mbar_init(&full, 1);
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(&full, cbytes);
    bulk_g2s(bsm, img, cbytes, &full);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = tbase, lane = (unsigned)(warp * 32) << 16;
  const unsigned d = tmem, a_hi = tmem + 256, a_lo = tmem + 256 + KP / 2;
  {
    float2 M[kT2PgMax];
    float mx2 = 0.f;
#pragma unroll
    for (int q = 0; q < kT2PgMax; ++q) {
      M[q] = (valid && q < Pg) ? a.mg[i * kT2PgMax + q] : make_float2(0.f, 0.f);
      mx2 = fmaxf(mx2, fmaf(M[q].x, M[q].x, M[q].y * M[q].y));
    }
    float sc, inv;
    row_scale(mx2, sc, inv);
    unsigned hv[kT2PgMax], lv[kT2PgMax];           // column q = (Re M_q, Im M_q)
#pragma unroll
    for (int q = 0; q < kT2PgMax; ++q) {
      const float mr = M[q].x * sc, mi = M[q].y * sc;
      const float hr = tf32_hi(mr), hi_ = tf32_hi(mi);
      hv[q] = pack_h2(hr, hi_);
      lv[q] = pack_h2(mr - hr, mi - hi_);
    }
#pragma unroll
    for (int s = 0; s < kT2PgMax / 16; ++s)
      if (s < KP / 32) {
        tmem_st16(a_hi + 16 * s + lane, *reinterpret_cast<const unsigned(*)[16]>(hv + 16 * s));
        tmem_st16(a_lo + 16 * s + lane, *reinterpret_cast<const unsigned(*)[16]>(lv + 16 * s));
      }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const double ug = valid ? a.lg[i * 3] * a.kd : 0.0;
    const int KS = KP / 16;
    for (int b = 0; b < NCb; ++b) {
      const int NB = min(128, ((nf - 128 * b) + 7) & ~7), N = 2 * NB;
      if (tid == 0) {
        mbar_wait(&full, (unsigned)(b & 1));
        const unsigned idesc = (1u << 4) | ((unsigned)(N >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
        const unsigned char *Bh = bsm, *Bl = bsm + (size_t)256 * KP * 2;
        const unsigned acol[3] = {a_hi, a_hi, a_lo};
        const unsigned char *bs[3] = {Bh, Bl, Bh};
        for (int p = 0; p < 3; ++p)
          for (int ks = 0; ks < KS; ++ks)
            umma_f16_ts(d, acol[p] + 8 * ks, umma_sdesc(smem_u32(bs[p]) + ks * 256, 128, KP * 16),
                        idesc, (p | ks) ? 1u : 0u);
        tc_commit(&mbar);
      }
      mbar_wait(&mbar, (unsigned)(b & 1));
      tc_fence_after();
      if (tid == 0 && b + 1 < NCb) {                   // the B buffer is free: next chunk
        mbar_arrive_expect_tx(&full, cbytes);
        bulk_g2s(bsm, img + (size_t)(b + 1) * kT2BinsImg, cbytes, &full);
      }
      for (int g = 0; g < NB / 8; ++g) {
        unsigned v[16];
        tmem_ld16(d + 16 * g + lane, v);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const int m = 128 * b + 8 * g + h;
            if (m < nf) {
              const float re = __uint_as_float(v[2 * h]) * inv, im = __uint_as_float(v[2 * h + 1]) * inv;
              const double cc = (double)(m - nf / 2) * ug;
              float ps, pc;                            // e^{-j 2 pi m' u_g}
              sincospif(2.f * (float)(cc - rint(cc)), &ps, &pc);
              out[i * nf + m] = make_float2(fmaf(pc, re, ps * im), fmaf(pc, im, -ps * re));
            }
          }
        }
      }
      tc_fence_before();
      __syncthreads();                                 // D read before the next chunk's MMAs
      tc_fence_after();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

}  // namespace

bool t2_tc_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RFR_T2TC");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

cudaError_t t2_tc_images(const T2Args &a, cudaStream_t st) {
  if (!t2_tc_enabled() || a.n_f <= 0) return cudaSuccess;
  const int64_t n = (int64_t)((a.n_f + 31) / 32) * 96 * 64 + (int64_t)((a.n_f + 127) / 128) * 256 * 96;
  k2_tc_bimg<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

cudaError_t t2_gexp_tc(const T2Args &a, const float2 *X0, const float2 *X1, cudaStream_t st) {
  if (a.n_a <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k2_gexp_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(2 * kT2GexpImg));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 g((unsigned)((a.n_a + 127) / 128), X1 ? 2u : 1u);
  k2_gexp_tc<<<g, 128, 2 * kT2GexpImg, st>>>(a, X0, X1);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

cudaError_t t2_bins_tc(const T2Args &a, float2 *out, cudaStream_t st) {
  if (a.n_a <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k2_bins_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kT2BinsImg);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k2_bins_tc<<<(unsigned)((a.n_a + 127) / 128), 128, kT2BinsImg, st>>>(a, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

}  // namespace rfr
