// rfr_tc.cu -- tensor-core (tcgen05 / TMEM) form of the adjoint sums K3 (backward) and K4 (filter).
//
// Both compute, per (sample or query j, antenna i), the bin sum
//     h_ij = sum_{m < NF} X_i[m] w_ij^m,   w_ij = e^{+j 2 pi df tau_ij}
// (X = G for K3, X = s for K4; App. A.5, Eq. 3).  With m = 16 m1 + m0 it
// factorises EXACTLY (no approximation) into a dense complex contraction over m0 followed by a
// short Horner sum over m1:
//     U_ij[m1] = sum_{m0 < 16} X_i[16 m1 + m0] w_ij^{m0},      h_ij = sum_{m1} (w_ij^16)^{m1} U_ij[m1].
// For a fixed antenna i the first step is a real GEMM D = A B^T over a tile of 128 samples, with
// complex values interleaved (re, im) along both K and N so that packed f32x2 registers map 1:1
// onto tensor-memory columns:
//     A[j][2 m0 + c]        : c = 0 -> Re w^m0, c = 1 -> Im w^m0                    (M = 128, K = 32)
//     B^T[2 m1][2 m0 + c]   : (Re X, -Im X)[c] of bin 16 m1 + m0   -> D[j][2 m1]     = Re U[m1]
//     B^T[2 m1 + 1][2m0 + c]: (Im X,  Re X)[c]                     -> D[j][2 m1 + 1] = Im U[m1]
//                                                                   (N = 2P, P = NF / 16)
// run on the 5th-generation tensor cores as tcgen05.mma.kind::f16 (fp16 operands, fp32
// accumulation) with A in tensor memory (each thread writes its own row with tcgen05.st, two fp16
// per 32-bit column, even K element in the low half), B in shared memory (K-major, no swizzle) and
// D in tensor memory.  fp32 accuracy comes from the "3xFP16" split (A_hi B_hi + A_hi B_lo +
// A_lo B_hi, hi = x with the 13 low mantissa bits cleared, exact in fp16, lo = x - hi): 22
// significant bits, like 3xTF32 (fp16 and tf32 share the 10-bit mantissa), at twice the tf32 MMA
// rate (tools/microbench/umma_f16_probe.cu: rel-L2 4.7e-7; 232 vs 432 tensor cycles per 128 x 64
// x 32 x 3 round).  fp16's range is handled by scaling every B row (antenna, X) by a power of two
// to max |component| in [0.5, 1) in k_prep_bt; the epilogue undoes it.  The per-pair SIMT work
// (fp64 geometry, the 16 powers of w, the Horner over m1, the Eq. 5 epilogue) overlaps the MMAs
// of the previous antenna.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "rfr_device.cuh"
#include "rfr_launch.h"
#include "rfr_tcgen05.cuh"

namespace rfr {

namespace {

// byte offset of element (row n, column k) of a K-major 16-bit operand with 32 columns: 16-byte
// chunks of 8 columns; 8 rows x 16 B core matrices; chunk stride 128 B, row-group stride 512 B
__device__ __forceinline__ unsigned bT_off(int n, int k) {
  return (unsigned)((k >> 3) * 128 + (n >> 3) * 512 + (n & 7) * 16 + (k & 7) * 2);
}
// per-pair state carried from the SIMT part of antenna a to its epilogue
struct PairTC {
  PairBwd g;
  float ec, es;     // E = e^{+j 2 pi f0 tau}
  float Wc, Ws;     // W = w^16
  float inv[2];     // 1 / (B row scale) of the antenna's X rows
};

}  // namespace

template <int NF, int NX>
struct TCShape {
  static constexpr int P = NF / 16;                  // m1 values
  static constexpr int N1 = 2 * P;                   // D columns per X row
  static constexpr int N = NX * N1;                  // D columns (NX = 2: [G | s] side by side)
  // D double-buffered (epilogue of antenna a-1 overlaps the MMA of antenna a) unless that would
  // halve the CTAs per SM; single-buffered D reads antenna a-1 before the MMA of a is issued.
  static constexpr int DBUF = (32 + 2 * N <= 128) ? 2 : 1;
  static constexpr int COLS = 32 + DBUF * N;         // A_hi, A_lo (16 f16x2 each) + D buffers
  static constexpr int ALLOC = COLS <= 128 ? 128 : (COLS <= 256 ? 256 : 512);
  static constexpr int MINB = 512 / ALLOC;           // CTAs per SM (512 TMEM columns)
};

// MODE == kModeBoth: K3 and K4 in one sweep (the filter's queries are the samples): the pair
// geometry, the powers of w and the A operand are shared; B^T stacks the G rows over the signal
// rows, so one MMA with N = 2 N1 yields both U_G and U_s.
template <int MODE, bool MONO, bool CORR, int NF>
__global__ void __launch_bounds__(kAdjThreads, TCShape<NF, MODE == kModeBoth ? 2 : 1>::MINB)
    k_adjoint_tc(AdjArgs a) {
  constexpr int NX = MODE == kModeBoth ? 2 : 1;
  using S = TCShape<NF, NX>;
  constexpr int P = S::P, N1 = S::N1, N = S::N, DBUF = S::DBUF;
  constexpr int GEO = MODE == kModeFlt ? kModeFlt : kModeBwd;     // geometry / record kind
  constexpr unsigned BBYTES = 2u * N * 64u;                        // B_hi | B_lo fp16 image
  static_assert(kAdjThreads == 128, "one TMEM lane per thread");
  // B^T images of antennas a (buffer a & 1), prepared by k_prep_bt and brought in by the bulk-copy
  // engine two antennas ahead: no thread of the CTA touches B
  extern __shared__ __align__(128) unsigned char bsm_raw[];
  unsigned char(*bsm)[BBYTES] = reinterpret_cast<unsigned char(*)[BBYTES]>(bsm_raw);
  __shared__ __align__(8) unsigned long long mma_bar, full_bar[2];
  __shared__ unsigned tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (a.skip && a.skip->sel) return;              // the Chebyshev adjoint was chosen
  const int64_t j = (int64_t)blockIdx.x * kAdjThreads + tid;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  const int na = (int)max(i_hi - i_lo, (int64_t)0);
  const bool valid = j < a.n_s;
  const bool no_gain = a.no_gain;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&tmem_base_sh)), "n"(S::ALLOC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const unsigned char *bsrc = a.bprep + (size_t)i_lo * BBYTES;
  const float2 *bscale = reinterpret_cast<const float2 *>(a.bprep + (size_t)a.n_a * BBYTES);
  if (tid == 0) {
    mbar_init(&mma_bar, 1);
    mbar_init(&full_bar[0], 1);
    mbar_init(&full_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < 2 && b < na; ++b) {
      mbar_arrive_expect_tx(&full_bar[b], BBYTES);
      bulk_g2s(bsm[b], bsrc + (size_t)b * BBYTES, BBYTES, &full_bar[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = tmem_base_sh;
  const unsigned lane_off = (unsigned)(warp * 32) << 16;
  const unsigned a_hi = tmem, a_lo = tmem + 16, d0 = tmem + 32;
  // kind::f16: fp16 A and B, fp32 accumulate, both operands K-major, M = 128, N
  const unsigned idesc = (1u << 4) | ((unsigned)(N >> 3) << 17) | ((unsigned)(128 >> 4) << 24);

  const Rec rec = load_point<GEO>(a, j, valid);
  float S1 = 0.f, S2 = 0.f, S3x = 0.f, S3y = 0.f, S3z = 0.f;
  float M1 = 0.f, M2 = 0.f;                       // kModeBoth: the filter's complex M
  bool domain = false;
  PairTC prev;
  const double kd16 = a.kd * 16.0;
  // antenna records prefetched one antenna ahead (the global-load latency was exposed at the
  // first fp64 difference of the pair geometry)
  AntF nxt;
  float2 nxt_inv = make_float2(1.f, 1.f);
  if (na > 0) { nxt = load_antf<MONO>(a, i_lo); nxt_inv = bscale[i_lo]; }

  // epilogue of antenna ai-1: U from TMEM, Horner over m1, Eq. 5 / M sums
  auto epilogue = [&](int ai) {
    const unsigned d = d0 + (unsigned)((DBUF == 2 ? ((ai - 1) & 1) : 0) * N) + lane_off;
#pragma unroll
    for (int x = 0; x < NX; ++x) {
      float Ur[P], Ui[P];
#pragma unroll
      for (int c = 0; c < N1; c += 16) {
        unsigned v[16];
        tmem_ld16(d + x * N1 + c, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
          Ur[(c + q) / 2] = __uint_as_float(v[q]);
          Ui[(c + q) / 2] = __uint_as_float(v[q + 1]);
        }
      }
      const f2x W = pk(prev.Wc, prev.Ws), W2 = pk(-prev.Ws, prev.Wc);
      f2x h = pk(Ur[P - 1], Ui[P - 1]);
#pragma unroll
      for (int m1 = P - 2; m1 >= 0; --m1) {
        const float2 hv = upk(h);
        const f2x t = ffma2(W, pk(hv.x, hv.x), pk(Ur[m1], Ui[m1]));
        h = ffma2(W2, pk(hv.y, hv.y), t);
      }
      const float2 hh = upk(fmul2(h, pk(prev.inv[x], prev.inv[x])));
      if (MODE != kModeBoth)
        adj_accumulate<MODE>(prev.g, prev.ec, prev.es, hh.x, hh.y, S1, S2, S3x, S3y, S3z);
      else if (x == 0)
        adj_accumulate<kModeBwd>(prev.g, prev.ec, prev.es, hh.x, hh.y, S1, S2, S3x, S3y, S3z);
      else
        adj_accumulate<kModeFlt>(prev.g, prev.ec, prev.es, hh.x, hh.y, M1, M2, S3x, S3y, S3z);
    }
  };

  for (int ai = 0; ai <= na; ++ai) {
    PairTC cur;
    if (ai < na) {
      // ---------------- SIMT: pair data and the powers of w for antenna ai (overlaps MMA ai-1)
      const int64_t ia = i_lo + ai;
      const AntD an = widen_ant<MONO>(nxt);
      cur.inv[0] = nxt_inv.x;
      cur.inv[1] = nxt_inv.y;
      if (ai + 1 < na) { nxt = load_antf<MONO>(a, ia + 1); nxt_inv = bscale[ia + 1]; }
      double L;
      if (GEO == kModeBwd) {
        pair_geometry<MONO, CORR>(rec, an, no_gain, cur.g);
        domain |= valid && !cur.g.ok;
        L = cur.g.L;
      } else {
        L = pair_length<MONO>(rec, an);
      }
      const float fr0 = frac_cycles(L * a.k0);
      const float frd = frac_cycles(L * a.kd);
      const float f16 = frac_cycles(L * kd16);
      __sincosf(kTwoPi * fr0, &cur.es, &cur.ec);
      float zs, zc;
      sincospif(2.f * frd, &zs, &zc);            // w (accurate)
      // W = w^16 from the fp64 cycle count; MUFU (abs. error ~4e-7): the Horner over m1 amplifies
      // it at most P - 1 times, well inside the 1e-4 / 1e-3 tolerances
      __sincosf(kTwoPi * f16, &cur.Ws, &cur.Wc);
      unsigned hv[16], lv[16];
      {
        // powers p_k = w^k (packed complex mults) by binary expansion -- dependency depth 4
        // instead of a 15-long chain -- and their hi / lo split
        f2x pw[16];
        pw[0] = pk(1.f, 0.f);
        pw[1] = pk(zc, zs);
        pw[2] = cmul2(pw[1], pw[1]);
        pw[4] = cmul2(pw[2], pw[2]);
        pw[8] = cmul2(pw[4], pw[4]);
        pw[3] = cmul2(pw[2], pw[1]);
        pw[5] = cmul2(pw[4], pw[1]);
        pw[6] = cmul2(pw[4], pw[2]);
        pw[7] = cmul2(pw[4], pw[3]);
#pragma unroll
        for (int k = 9; k < 16; ++k) pw[k] = cmul2(pw[8], pw[k - 8]);
#pragma unroll
        for (int k = 0; k < 16; ++k) {          // column k = (Re, Im) of w^k: K elements 2k, 2k+1
          const float2 pv = upk(pw[k]);
          const float hr = tf32_hi(pv.x), hi_ = tf32_hi(pv.y);
          const float2 lo = upk(fadd2(pw[k], pk(-hr, -hi_)));
          hv[k] = pack_h2(hr, hi_);
          lv[k] = pack_h2(lo.x, lo.y);
        }
      }
      // ---------------- MMA ai-1 must be done before A / B (and a single D) are reused
      if (ai > 0) mbar_wait(&mma_bar, (unsigned)((ai - 1) & 1));
      tc_fence_after();
      // the MMA of ai-1 released B buffer (ai + 1) & 1: bring in antenna ai + 1
      if (tid == 0 && ai > 0 && ai + 1 < na) {
        const int b = (ai + 1) & 1;
        mbar_arrive_expect_tx(&full_bar[b], BBYTES);
        bulk_g2s(bsm[b], bsrc + (size_t)(ai + 1) * BBYTES, BBYTES, &full_bar[b]);
      }
      tmem_st16(a_hi + lane_off, hv);
      tmem_st16(a_lo + lane_off, lv);
      if (DBUF == 1 && ai > 0) epilogue(ai);      // read D of ai-1 before the MMA of ai
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      // all A rows and B chunks written before the MMA is issued.  (An mbarrier that only the
      // issuing thread waits on measured slower: the other warps then reach the single-buffered A
      // of the next antenna before the late-issued MMA has finished with it.)
      __syncthreads();
      tc_fence_after();
      if (tid == 0) {
        mbar_wait(&full_bar[ai & 1], (unsigned)((ai >> 1) & 1));   // B^T of antenna ai landed
        const unsigned d = d0 + (unsigned)((DBUF == 2 ? (ai & 1) : 0) * N);
        const unsigned acol[3] = {a_hi, a_hi, a_lo};
        const unsigned char *Bhi = bsm[ai & 1], *Blo = Bhi + N * 64;
        const unsigned char *bs[3] = {Bhi, Blo, Bhi};
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            umma_f16_ts(d, acol[p] + 8 * ks,
                        umma_sdesc(smem_u32(bs[p]) + ks * 256, 128, 512), idesc,
                        (p | ks) ? 1u : 0u);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];"
                     ::"l"((uint64_t)smem_u32(&mma_bar)) : "memory");
      }
      if (DBUF == 2 && ai > 0) epilogue(ai);
    } else if (ai > 0) {
      mbar_wait(&mma_bar, (unsigned)((ai - 1) & 1));
      tc_fence_after();
      epilogue(ai);
    }
    prev = cur;
  }
  if (domain) atomicOr(a.flags, 1u);
  if (valid) {
    if (MODE != kModeBoth) {
      adj_store<MODE>(a, j, S1, S2, S3x, S3y, S3z);
    } else {
      adj_store<kModeBwd>(a, j, S1, S2, S3x, S3y, S3z);
      reinterpret_cast<float2 *>(a.out2)[(int64_t)blockIdx.y * a.n_s + j] = make_float2(M1, M2);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(S::ALLOC));
}

// B^T images for the tensor-core adjoint, one per antenna: [B_hi | B_lo], each N rows of 32 fp16
// columns in the canonical K-major no-swizzle layout (bT_off).  Row n = x N1 + 2 m1 + c of X row
// x (G then s for kModeBoth), column 2 m0 + c' holds bin 16 m1 + m0 as (Re, -Im) for c = 0 and
// (Im, Re) for c = 1 (the complex product's sign pattern), scaled by 2^-e so that the row's max
// |component| lies in [0.5, 1) (fp16 range), split hi = x with 13 low mantissa bits cleared,
// lo = x - hi.  The inverse scales 2^e go to a float2 per antenna after the images.  One warp
// per antenna; HBM-bound, ~0.05 ms at c3.
__global__ void k_prep_bt(const float2 *__restrict__ X, const float2 *__restrict__ X2, int64_t n_a,
                          int nf, int nx, unsigned char *__restrict__ out, const ChebHdr *skip) {
  if (skip && skip->sel) return;
  const int lane = threadIdx.x & 31;
  const int N1 = nf / 8, N = nx * N1;
  const size_t bbytes = (size_t)N * 128;                 // hi + lo, N rows x 64 B each
  float2 *scales = reinterpret_cast<float2 *>(out + (size_t)n_a * bbytes);
  for (int64_t ia = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ia < n_a;
       ia += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float sc[2] = {1.f, 1.f}, inv[2] = {1.f, 1.f};
    for (int x = 0; x < nx; ++x) {
      const float4 *row = reinterpret_cast<const float4 *>((x == 0 ? X : X2) + ia * nf);
      float m = 0.f;
      for (int q = lane; q < nf / 2; q += 32) {
        const float4 v = row[q];
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (m > 0.f && isfinite(m)) {
        int e;
        frexpf(m, &e);                                   // m = f 2^e, f in [0.5, 1)
        sc[x] = ldexpf(1.f, -e);
        inv[x] = ldexpf(1.f, e);
      }
    }
    if (lane == 0) scales[ia] = make_float2(inv[0], inv[1]);
    unsigned char *img = out + (size_t)ia * bbytes;
    // 16-byte chunk (row n, columns 8c .. 8c+7) = bins 16 (n' / 2) + 4c .. +3 of row x
    for (int q = lane; q < N * 4; q += 32) {
      const int n = q % N, c = q / N;
      const int x = n / N1, nn = n % N1;
      const float4 *row = reinterpret_cast<const float4 *>((x == 0 ? X : X2) + ia * nf);
      const int b = 16 * (nn >> 1) + 4 * c;
      const float4 u = row[b >> 1], w = row[(b >> 1) + 1];
      float v[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
      unsigned hv[4], lv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float re = v[2 * t] * sc[x], im = v[2 * t + 1] * sc[x];
        const float e0 = (n & 1) ? im : re, e1 = (n & 1) ? re : -im;
        const float h0 = tf32_hi(e0), h1 = tf32_hi(e1);
        hv[t] = pack_h2(h0, h1);
        lv[t] = pack_h2(e0 - h0, e1 - h1);
      }
      *reinterpret_cast<uint4 *>(img + bT_off(n, 8 * c)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<uint4 *>(img + N * 64 + bT_off(n, 8 * c)) =
          make_uint4(lv[0], lv[1], lv[2], lv[3]);
    }
  }
}

template <int MODE, bool MONO, bool CORR, int NF>
static cudaError_t tc_launch(const AdjArgs &a, dim3 grid, cudaStream_t st) {
  using S = TCShape<NF, MODE == kModeBoth ? 2 : 1>;
  const size_t smem = (size_t)2 * 2 * S::N * 64;         // two B^T image buffers (fp16 hi | lo)
  auto k = k_adjoint_tc<MODE, MONO, CORR, NF>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kAdjThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int MODE, bool MONO, bool CORR>
static cudaError_t tc_nf(const AdjArgs &a, dim3 grid, cudaStream_t st) {
  switch (a.n_f) {
    case 128: return tc_launch<MODE, MONO, CORR, 128>(a, grid, st);
    case 256: return tc_launch<MODE, MONO, CORR, 256>(a, grid, st);
    case 512: return tc_launch<MODE, MONO, CORR, 512>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

bool adjoint_tc_supported(int n_f) { return n_f == 128 || n_f == 256 || n_f == 512; }

cudaError_t launch_adjoint_tc(const AdjArgs &a, int mode, bool mono, bool corr, int n_splits,
                              cudaStream_t st) {
  if (!a.bprep) return cudaErrorInvalidValue;
  if (a.n_a > 0) {
    const int nx = mode == kModeBoth ? 2 : 1;
    const unsigned g = (unsigned)std::min<int64_t>((a.n_a + 7) / 8, 148 * 32);   // 8 warps / CTA
    k_prep_bt<<<g, 256, 0, st>>>(a.X, a.X2, a.n_a, a.n_f, nx, a.bprep, a.skip);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)((a.n_s + kAdjThreads - 1) / kAdjThreads), (unsigned)n_splits);
  if (mode == kModeBwd) {
    if (mono) return corr ? tc_nf<kModeBwd, true, true>(a, grid, st)
                          : tc_nf<kModeBwd, true, false>(a, grid, st);
    return corr ? tc_nf<kModeBwd, false, true>(a, grid, st)
                : tc_nf<kModeBwd, false, false>(a, grid, st);
  }
  if (mode == kModeBoth) {
    if (mono) return corr ? tc_nf<kModeBoth, true, true>(a, grid, st)
                          : tc_nf<kModeBoth, true, false>(a, grid, st);
    return corr ? tc_nf<kModeBoth, false, true>(a, grid, st)
                : tc_nf<kModeBoth, false, false>(a, grid, st);
  }
  return mono ? tc_nf<kModeFlt, true, false>(a, grid, st)
              : tc_nf<kModeFlt, false, false>(a, grid, st);
}

}  // namespace rfr
