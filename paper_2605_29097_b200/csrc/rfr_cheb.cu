// rfr_cheb.cu -- forward signal tracing (Eq. 4) by a Jacobi-Anger / Chebyshev
// factorisation of the bin dependence ("range-profile factorisation").
//
// For antenna i write the per-pair delay in cycles per bin step as u_ij = L_ij df / c and centre it
// on the antenna: u_ij = u_c,i + delta x_ij with |x_ij| <= 1, where [u_c,i -+ delta_i] bounds the
// delays of every sample of the call (from the samples' bounding box) and delta = max_i delta_i.
// With centred bins m' = m - N/2 and c_ij = A_ij exp(-j 2 pi f_c tau_ij), f_c = f0 + (N/2) df:
//     s_i[m] = exp(-j 2 pi m' u_c,i) sum_j c_ij exp(-j z_m' x_ij),      z_m' = 2 pi m' delta,
//     exp(-j z x) = sum_p eps_p (-j)^p J_p(z) T_p(x)                     (Jacobi-Anger)
// so the N_f-bin sum of every pair collapses to P Chebyshev moments M_i[p] = sum_j c_ij T_p(x_ij),
// and the bins come from one small dense complex product per antenna,
//     s_i[m] = exp(-j 2 pi m' u_c,i) sum_p a[m][p] M_i[p],    a[m][p] = eps_p (-j)^p J_p(z_m').
// The truncation after P terms is below 1e-7 of sum |c| for |z| <= z_P (P = 16 / 24 / 28 / 32 / 48
// for z <= 4.7 / 9.9 / 12.9 / 15.8 / 28.6); wider delay spreads fall back to the direct kernels.
// Per pair: the fp64 geometry, one MUFU sincos and P steps of Reinsch's stabilised Chebyshev
// recurrence (d_{p+1} = 2 (x - 1) T_p + d_p, T_{p+1} = T_p + d_{p+1}: absolute error O(p u) up to
// |x| = 1, where the plain three-term recurrence grows like p^2 u) with one complex-real FFMA2 each:
// ~4 FP32 lane-ops per moment instead of 4 per bin.  No atomics: split-K partial moments summed in
// fixed order, results bitwise reproducible.
//
// The choice between this path and K2 is taken on the device (the delay spread is only known
// there): k_cheb_setup writes the selected P (0 = direct) into the workspace header, and the kernels
// of the path not taken return at once.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "rfr_device.cuh"
#include "rfr_launch.h"

namespace rfr {

namespace {
constexpr int kBoxBlocks = 256;
constexpr int kChebThreads = 128;
constexpr int kChebTJ = 32;                       // records per shared-memory tile
}  // namespace

// ---------------------------------------------------------- empty-space skipping (forward)
// A sample contributes A_ij = w_j g gamma T_t T_r to the forward: nothing when w_j = p a alpha is
// exactly 0 (alpha underflows to 0 in fp32 a few millimetres from any surface at s = 2e4 / m) or,
// without the Eq. 7 correction, when T_j is exactly 0 (behind a surface).  The forward's Chebyshev
// path runs over the compacted list of the other records (order preserved: an ordered stream
// compaction, deterministic); the count stays on the device.
constexpr int kCompactBlock = 1024;

// forward: w = p a alpha != 0; backward (aflag given): alpha != 0 -- every gradient of a sample
// with alpha = 0 in fp32 is 0 or carries a factor sigma(-s f) below the fp32 range (DESIGN 5c)
__device__ __forceinline__ bool rec_active(const Rec &r, bool corr, const unsigned char *aflag,
                                           int64_t j) {
  return (aflag ? aflag[j] != 0 : r.w != 0.f) && (corr || r.T != 0.f);
}

__global__ void __launch_bounds__(kCompactBlock) k_compact_count(const Rec *__restrict__ rec,
                                                                 int64_t n, bool corr,
                                                                 const unsigned char *aflag,
                                                                 int *__restrict__ cnt) {
  const int64_t j = (int64_t)blockIdx.x * kCompactBlock + threadIdx.x;
  const bool act = j < n && rec_active(rec[j], corr, aflag, j);
  const int c = __syncthreads_count(act);
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

// exclusive scan of the block counts (one CTA, sequential over chunks of 1024) and the total
__global__ void __launch_bounds__(1024) k_compact_scan(int *__restrict__ cnt, int nb,
                                                       int64_t *__restrict__ total) {
  __shared__ int sh[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int v = b < nb ? cnt[b] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {            // Hillis-Steele inclusive scan
      const int u = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += u;
      __syncthreads();
    }
    if (b < nb) cnt[b] = (int)(carry + sh[threadIdx.x] - v);
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kCompactBlock) k_compact_write(const Rec *__restrict__ rec,
                                                                 int64_t n, bool corr,
                                                                 const unsigned char *aflag,
                                                                 const int *__restrict__ off,
                                                                 Rec *__restrict__ out,
                                                                 int *__restrict__ idx) {
  __shared__ int wsum[kCompactBlock / 32];
  const int64_t j = (int64_t)blockIdx.x * kCompactBlock + threadIdx.x;
  Rec r;
  bool act = false;
  if (j < n) { r = rec[j]; act = rec_active(r, corr, aflag, j); }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, act);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int base = off[blockIdx.x];
  for (int w = 0; w < warp; ++w) base += wsum[w];
  if (act) {
    const int pos = base + __popc(bal & ((1u << lane) - 1u));
    out[pos] = r;
    if (idx) idx[pos] = (int)j;
  }
}

cudaError_t launch_compact(const Rec *rec, int64_t n, bool corr, int *cnt, int64_t *total, Rec *out,
                           cudaStream_t st, const unsigned char *aflag, int *idx) {
  const int nb = (int)((n + kCompactBlock - 1) / kCompactBlock);
  if (nb == 0) return cudaMemsetAsync(total, 0, sizeof(int64_t), st);
  k_compact_count<<<nb, kCompactBlock, 0, st>>>(rec, n, corr, aflag, cnt);
  k_compact_scan<<<1, 1024, 0, st>>>(cnt, nb, total);
  k_compact_write<<<nb, kCompactBlock, 0, st>>>(rec, n, corr, aflag, cnt, out, idx);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(3);
  return e;
}
int compact_blocks(int64_t n) { return (int)((n + kCompactBlock - 1) / kCompactBlock); }

// query points as records (fp64 position; only the box kernel reads them)
__global__ void k_pack_points(const float *__restrict__ x, const float *__restrict__ y,
                              const float *__restrict__ z, int64_t n, Rec *__restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    Rec r;
    r.x = x[q]; r.y = y[q]; r.z = z[q];
    r.w = 0.f; r.T = 1.f; r.nx = r.ny = 0.f; r.nz = 1.f; r.papr = 1.f;
    out[q] = r;
  }
}

cudaError_t launch_pack_points(const float *x, const float *y, const float *z, int64_t n, Rec *out,
                               int n_sm, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)n_sm * 8);
  k_pack_points<<<g, 256, 0, st>>>(x, y, z, n, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

// ------------------------------------------------------------------ bounding box of the samples
__global__ void k_cheb_box(const Rec *__restrict__ rec, int64_t n, const int64_t *n_dev,
                           double *__restrict__ part) {
  if (n_dev) n = *n_dev;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const Rec r = rec[j];
    lo[0] = fmin(lo[0], r.x); hi[0] = fmax(hi[0], r.x);
    lo[1] = fmin(lo[1], r.y); hi[1] = fmax(hi[1], r.y);
    lo[2] = fmin(lo[2], r.z); hi[2] = fmax(hi[2], r.z);
  }
  __shared__ double sh[6][256];
  for (int c = 0; c < 3; ++c) { sh[c][threadIdx.x] = lo[c]; sh[3 + c][threadIdx.x] = hi[c]; }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int c = 0; c < 3; ++c) {
        sh[c][threadIdx.x] = fmin(sh[c][threadIdx.x], sh[c][threadIdx.x + s]);
        sh[3 + c][threadIdx.x] = fmax(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

// distance range [dmin, dmax] from a point to an axis-aligned box
__device__ __forceinline__ void box_dist(const double *b, double px, double py, double pz,
                                         double &dmin, double &dmax) {
  const double p[3] = {px, py, pz};
  double s0 = 0.0, s1 = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double l = b[c], h = b[3 + c];
    const double out = fmax(fmax(l - p[c], p[c] - h), 0.0);
    s0 += out * out;
    const double far = fmax(fabs(p[c] - l), fabs(p[c] - h));
    s1 += far * far;
  }
  dmin = sqrt(s0);
  dmax = sqrt(s1);
}

// truncation tail sum_{p>=P} eps_p |J_p(z)| < 1e-7 of sum |c|, 10^3 below the 1e-4 signal
// tolerance (tests/test_cheb_math.py); 0: spread too wide for the moment path
__device__ __forceinline__ int cheb_select_P(double zmax) {
  if (zmax <= 4.7) return 16;
  if (zmax <= 9.9) return 24;
  if (zmax <= 12.9) return 28;
  if (zmax <= 15.8) return 32;
  if (zmax <= 28.6) return 48;
  return 0;
}

// ----------------------------------------------- per-antenna delay centre, global spread, P choice
// One CTA of 1024 threads.  lc[i] = centre path length (m) of antenna i; hdr gets the selected P
// (0: delay spread too wide -> direct kernel), delta and kd / delta.
__global__ void __launch_bounds__(1024) k_cheb_setup(double *__restrict__ part, int nblk,
                                                     ChebArgs a, double *__restrict__ lc,
                                                     ChebHdr *__restrict__ hdr) {
  __shared__ double box[6];
  __shared__ double red[1024];
  if (threadIdx.x < 6) {
    double v = threadIdx.x < 3 ? 1e300 : -1e300;
    for (int b = 0; b < nblk; ++b) {
      const double u = part[b * 6 + threadIdx.x];
      v = threadIdx.x < 3 ? fmin(v, u) : fmax(v, u);
    }
    box[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0 && !(box[0] <= box[3])) {   // no points (empty compacted list): any box
    for (int c = 0; c < 6; ++c) box[c] = 0.0;       // gives zero moments; keep the centres finite
  }
  __syncthreads();
  if (threadIdx.x < 6) part[nblk * 6 + threadIdx.x] = box[threadIdx.x];   // the box, for later kernels
  double dmax_half = 0.0;
  for (int64_t i = threadIdx.x; i < a.n_a; i += blockDim.x) {
    double tmin, tmax, rmin, rmax;
    box_dist(box, a.tx_x[i], a.tx_y[i], a.tx_z[i], tmin, tmax);
    if (a.rx_x) box_dist(box, a.rx_x[i], a.rx_y[i], a.rx_z[i], rmin, rmax);
    else { rmin = tmin; rmax = tmax; }
    const double Lmin = tmin + rmin, Lmax = tmax + rmax;
    lc[i] = 0.5 * (Lmin + Lmax);
    dmax_half = fmax(dmax_half, 0.5 * (Lmax - Lmin));
  }
  red[threadIdx.x] = dmax_half;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // spread in cycles per bin, with a small margin for the fp32 rounding of the positions
    const double delta = fmax(red[0] * a.kd * (1.0 + 1e-6), 1e-30);
    const double zmax = 2.0 * 3.14159265358979323846 * (double)(a.n_f / 2 + 1) * delta;
    const int P = a.enable ? cheb_select_P(zmax) : 0;
    hdr->sel = P > 0 ? 1u : 0u;
    hdr->P = P;
    hdr->delta = delta;
    hdr->inv = a.kd / delta;
  }
}

// ------------------------------------------------ a[m][p] = eps_p (-j)^p J_p(2 pi (m - N/2) delta)
// One thread per bin: Bessel J_0..J_{P-1} by Miller's backward recurrence in fp64 (rescaled
// against overflow), normalised by J_0 + 2 sum_k J_2k = 1.
__global__ void k_cheb_coef(const ChebHdr *__restrict__ hdr, int n_f, int pmax,
                            float2 *__restrict__ coef) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_f || hdr->sel == 0) return;
  const int P = hdr->P;
  const double z0 = 2.0 * 3.14159265358979323846 * (double)(m - n_f / 2) * hdr->delta;
  const double z = fabs(z0);
  double J[128];
  if (z < 1e-12) {
    for (int p = 0; p < P; ++p) J[p] = p == 0 ? 1.0 : 0.0;
  } else {
    const int top = min(127, P + 24 + (int)z);
    double jp1 = 0.0, jp = 1e-30, norm = 0.0;   // jp = J_k, jp1 = J_{k+1} (common scale)
    for (int k = top; k >= 1; --k) {
      if (k < P) J[k] = jp;
      if ((k & 1) == 0) norm += 2.0 * jp;
      const double jm1 = (2.0 * k / z) * jp - jp1;
      jp1 = jp;
      jp = jm1;
      if (fabs(jp) > 1e200) {                    // rescale everything accumulated so far
        jp *= 1e-200; jp1 *= 1e-200; norm *= 1e-200;
        for (int q = k; q < P; ++q) J[q] *= 1e-200;
      }
    }
    J[0] = jp;
    norm += jp;
    for (int p = 0; p < P; ++p) J[p] /= norm;
  }
  for (int p = 0; p < P; ++p) {
    double v = (p == 0 ? 1.0 : 2.0) * J[p];
    if (z0 < 0.0 && (p & 1)) v = -v;             // J_p(-z) = (-1)^p J_p(z)
    // (-j)^p = 1, -j, -1, j
    const int q = p & 3;
    const float2 c = q == 0 ? make_float2((float)v, 0.f)
                   : q == 1 ? make_float2(0.f, (float)-v)
                   : q == 2 ? make_float2((float)-v, 0.f)
                            : make_float2(0.f, (float)v);
    coef[(int64_t)m * pmax + p] = c;
  }
}

// ------------------------------------------------------------------------- moments M_i[p]
// Thread = antenna; the CTA walks its split's samples in tiles of kChebTJ records staged in shared
// memory (every thread reads the same record: broadcast).  KIND == kFwdMFAdj: the records are the
// K5 query records {x, y, z, w = Re c_q, T = Im c_q} and the pair amplitude is c_q.
template <int P, bool MONO, int KIND>
constexpr int kFwdUnroll = (MONO && P == 28 && KIND == kFwdTrace) ? 2 : 1;
template <int P, bool MONO, bool CORR, int KIND>
__global__ void __launch_bounds__(kChebThreads, (MONO && P == 28 && KIND == kFwdTrace) ? 3 : ((MONO && P <= 28) || P <= 16 ? 5 : (P <= 32 ? 4 : 3))) k_cheb_fwd(ChebArgs a) {
  if (a.hdr->P != P) return;                     // another P (or the direct kernel) was chosen
  __shared__ __align__(16) Rec rb[2][kChebTJ];
  const int tid = threadIdx.x;
  const int64_t ia = (int64_t)blockIdx.x * kChebThreads + tid;
  const bool ant_ok = ia < a.n_a;
  // point range of this split: from the device count when the records are a compacted list
  const int64_t n_pts = a.n_dev ? *a.n_dev : a.n_s;
  const int64_t per = a.n_dev ? (n_pts + gridDim.y - 1) / gridDim.y : a.samples_per_split;
  const int64_t j_lo = (int64_t)blockIdx.y * per;
  const int64_t j_hi = min(n_pts, j_lo + per);
  AntF af;
  if (ant_ok) af = load_antf<MONO>(a, ia);
  else { af.x = af.y = 0.f; af.z = 1.f; af.rx = af.ry = 0.f; af.rz = 1.f; af.ptx = af.prx = 1.f; }
  const AntD an = widen_ant<MONO>(af);
  const double Lc = ant_ok ? a.lc[ia] : 0.0;
  const double inv = a.hdr->inv;
  const bool no_gain = a.no_gain;
  f2x M[P];
#pragma unroll
  for (int p = 0; p < P; ++p) M[p] = 0ull;
  bool domain = false;

  auto prefetch = [&](int64_t jt, int b) {
    const int nv = (int)min((int64_t)kChebTJ, j_hi - jt);
    const float4 *src = reinterpret_cast<const float4 *>(a.rec + jt);
    float4 *dst = reinterpret_cast<float4 *>(rb[b]);
    if (tid < kChebTJ * 3) {
      if (tid < 3 * nv) cp_async16(dst + tid, src + tid);
      else dst[tid] = make_float4(0.f, 0.f, 0.f, 0.f);      // tail: w = 0 records
    }
    cp_async_commit();
  };
  if (j_lo < j_hi) prefetch(j_lo, 0);
  int b = 0;
  for (int64_t jt = j_lo; jt < j_hi; jt += kChebTJ, b ^= 1) {
    cp_async_wait_all();
    __syncthreads();
    if (jt + kChebTJ < j_hi) prefetch(jt + kChebTJ, b ^ 1);
    const int nv = (int)min((int64_t)kChebTJ, j_hi - jt);
    // two samples per step: their Reinsch recurrences run packed in one FFMA2 / FADD2 (lanes =
    // samples), each moment update is one FFMA2 per sample.  An odd tail pairs the last record
    // with a zero record of the tile (w = 0).
#pragma unroll 1
    for (int jj = 0; jj < nv; jj += 2) {
      f2x cc0 = 0ull, co0 = 0ull, cc1 = 0ull, co1 = 0ull;
      float xv0 = 0.f, xv1 = 0.f;
#pragma unroll (kFwdUnroll<P, MONO, KIND>)
      for (int u = 0; u < 2; ++u) {
        const Rec rec = rb[b][jj + u];
        double L;
        float Ar, Ai;
        if (KIND == kFwdTrace) {
          PairBwd g;
          pair_geometry<MONO, CORR>(rec, an, no_gain, g);
          domain |= ant_ok && (jj + u < nv) && !g.ok;
          Ar = rec.w * g.gg * g.Tt * g.Tr;
          Ai = 0.f;
          L = g.L;
        } else {
          L = pair_length<MONO>(rec, an);
          Ar = rec.w;
          Ai = rec.T;
        }
        // c = A exp(-j 2 pi f_c tau) from the fp64 cycle count at the centre frequency
        float es, ec;
        __sincosf(kTwoPi * frac_cycles(L * a.kc), &es, &ec);
        const f2x c = (KIND == kFwdTrace) ? pk(Ar * ec, -Ar * es)
                                          : pk(fmaf(Ar, ec, Ai * es), fmaf(Ai, ec, -Ar * es));
        float x = (float)((L - Lc) * inv);
        x = fminf(fmaxf(x, -1.f), 1.f);
        const f2x cneg = x < 0.f ? pk(-upk(c).x, -upk(c).y) : c;   // odd moments: T_p(x) = -T_p(|x|)
        if (u == 0) { cc0 = c; co0 = cneg; xv0 = fabsf(x) - 1.f; }
        else { cc1 = c; co1 = cneg; xv1 = fabsf(x) - 1.f; }
      }
      const f2x cc[2] = {cc0, cc1}, co[2] = {co0, co1};
      const f2x xm1 = pk(xv0, xv1), two_xm1 = pk(2.f * xv0, 2.f * xv1);
      f2x d = xm1, t = pk(1.f, 1.f);
      acc2(M[0], cc[0]);
      acc2(M[0], cc[1]);
      t = fadd2(t, d);                                     // (T_1, T_1')
      {
        const float2 tv = upk(t);
        M[1] = ffma2(pk(tv.x, tv.x), co[0], M[1]);
        M[1] = ffma2(pk(tv.y, tv.y), co[1], M[1]);
      }
#pragma unroll
      for (int p = 2; p < P; ++p) {
        d = ffma2(two_xm1, t, d);
        t = fadd2(t, d);
        const float2 tv = upk(t);
        M[p] = ffma2(pk(tv.x, tv.x), (p & 1) ? co[0] : cc[0], M[p]);
        M[p] = ffma2(pk(tv.y, tv.y), (p & 1) ? co[1] : cc[1], M[p]);
      }
    }
  }
  cp_async_wait_all();
  if (domain) atomicOr(a.flags, 1u);
  if (ant_ok) {
    float2 *dst = a.part + ((int64_t)blockIdx.y * a.n_a + ia) * a.pmax;
#pragma unroll
    for (int p = 0; p < P; ++p) dst[p] = upk(M[p]);
  }
}

// ------------------------------------------------ bins: s_i[m] = e^{-j 2pi m' u_c} sum_p a M_i[p]
__global__ void k_cheb_out(ChebArgs a, int splits, float2 *__restrict__ out) {
  if (a.hdr->sel == 0) return;
  const int P = a.hdr->P;
  __shared__ float2 Ms[64];
  const int64_t i = blockIdx.x;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    float2 v = make_float2(0.f, 0.f);
    for (int s = 0; s < splits; ++s) {          // fixed order over the splits
      const float2 u = a.part[((int64_t)s * a.n_a + i) * a.pmax + p];
      v.x += u.x;
      v.y += u.y;
    }
    Ms[p] = v;
  }
  __syncthreads();
  const double uc = a.lc[i] * a.kd;
  for (int m = threadIdx.x; m < a.n_f; m += blockDim.x) {
    const float2 *cf = a.coef + (int64_t)m * a.pmax;
    float re = 0.f, im = 0.f;
    for (int p = 0; p < P; ++p) {
      const float2 c = cf[p], v = Ms[p];
      re = fmaf(c.x, v.x, fmaf(-c.y, v.y, re));
      im = fmaf(c.x, v.y, fmaf(c.y, v.x, im));
    }
    float ps, pc;
    sincospif(2.f * frac_cycles((double)(m - a.n_f / 2) * uc), &ps, &pc);   // e^{-j 2 pi m' u_c}
    out[i * a.n_f + m] = make_float2(fmaf(pc, re, ps * im), fmaf(pc, im, -ps * re));
  }
}

// =============================================================================== adjoint
// E_ij h_ij = sum_m X_i[m] e^{+j 2 pi f_m tau_ij} = e^{+j 2 pi f_c tau_ij} sum_p T_p(x_ij) B_i[p],
//     B_i[p] = sum_m X_i[m] e^{+j 2 pi m' u_c,i} conj(a[m][p])
// (the conjugate expansion e^{+j z x} = sum_p eps_p j^p J_p(z) T_p(x)).  k_cheb_adj_prep forms the
// antenna moments B (fixed-order sums), k_cheb_adj runs one thread per sample over the antennas of
// its split with the Reinsch recurrence and the Eq. 5 / matched-filter epilogue of the direct
// kernels.  bmom layout: [n_a][kChebPMax][2] float2 (X row 0 = G or the signal, row 1 = the signal
// in the fused sweep), so one 16-byte load feeds both MACs of a moment.
constexpr int kAdjPrepThreads = 256;

__global__ void __launch_bounds__(kAdjPrepThreads) k_cheb_adj_prep(ChebArgs c, const float2 *X0,
                                                                   const float2 *X1, int nx,
                                                                   float2 *__restrict__ bmom) {
  if (c.hdr->sel == 0) return;
  extern __shared__ float2 ysh[];                 // [n_f] rotated row, then [8][64] partials
  const int P = c.hdr->P;
  const int64_t i = blockIdx.x;
  const double uc = c.lc[i] * c.kd;
  const int N = c.n_f;
  float2 *part = ysh + N;
  for (int x = 0; x < nx; ++x) {
    const float2 *row = (x == 0 ? X0 : X1) + i * N;
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
      float ps, pc;                                // e^{+j 2 pi m' u_c}
      sincospif(2.f * frac_cycles((double)(m - N / 2) * uc), &ps, &pc);
      const float2 v = row[m];
      ysh[m] = make_float2(fmaf(pc, v.x, -ps * v.y), fmaf(pc, v.y, ps * v.x));
    }
    __syncthreads();
    // thread (p, q): partial over bins m = q, q + 8, ... ; then a fixed-order sum over q
    const int p = threadIdx.x & 63, q = threadIdx.x >> 6;     // 64 x 4
    float re = 0.f, im = 0.f;
    if (p < P)
      for (int m = q; m < N; m += 4) {
        const float2 a = c.coef[(int64_t)m * c.pmax + p], y = ysh[m];   // y conj(a)
        re = fmaf(y.x, a.x, fmaf(y.y, a.y, re));
        im = fmaf(y.y, a.x, fmaf(-y.x, a.y, im));
      }
    part[q * 64 + p] = make_float2(re, im);
    __syncthreads();
    if (threadIdx.x < P) {
      float2 v = part[threadIdx.x];
      for (int qq = 1; qq < 4; ++qq) {
        v.x += part[qq * 64 + threadIdx.x].x;
        v.y += part[qq * 64 + threadIdx.x].y;
      }
      bmom[(i * kChebPMax + threadIdx.x) * 2 + x] = v;
    }
    __syncthreads();
  }
}

constexpr int kChebGA = 16;                        // antennas per shared-memory stage

// Two samples per thread (j and j + 128 of a 256-sample CTA tile): their Reinsch recurrences run
// packed (one FFMA2 + one FADD2 per moment for both) and every B[p] load from shared memory feeds
// the moment updates of both samples.
template <int P, int MODE, bool MONO, bool CORR>
__global__ void __launch_bounds__(kChebThreads, 4) k_cheb_adj(ChebArgs c, AdjArgs a,
                                                              const float2 *__restrict__ bmom) {
  if (c.hdr->P != P) return;
  constexpr int NX = MODE == kModeBoth ? 2 : 1;
  constexpr int GEO = MODE == kModeFlt ? kModeFlt : kModeBwd;
  __shared__ __align__(16) float4 bs[kChebGA][P];   // (B_0[p], B_1[p]) per antenna of the stage
  __shared__ AntF as[kChebGA];
  __shared__ double ls[kChebGA];
  __shared__ float4 gs[kChebGA][2];                 // F32G: tile-relative antenna geometry
  const int tid = threadIdx.x;
  // points: all n_s, or the compacted list of c.n_dev points (records at a.rec, original index
  // c.idx[j] for the outputs)
  const int64_t n_pts = c.n_dev ? *c.n_dev : a.n_s;
  const int64_t jb = (int64_t)blockIdx.x * (2 * kChebThreads) + tid;
  if ((int64_t)blockIdx.x * (2 * kChebThreads) >= n_pts) return;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  bool valid[2];
  Rec rec[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    valid[u] = jb + u * kChebThreads < n_pts;
    rec[u] = load_point<GEO>(a, jb + u * kChebThreads, valid[u]);
  }
  const bool row1 = NX == 1 && c.row == 1;
  const bool no_gain = a.no_gain;
  const double inv = c.hdr->inv;
  float S1[2] = {0.f, 0.f}, S2[2] = {0.f, 0.f}, S3x[2] = {0.f, 0.f}, S3y[2] = {0.f, 0.f},
        S3z[2] = {0.f, 0.f}, M1[2] = {0.f, 0.f}, M2[2] = {0.f, 0.f};
  bool domain = false;
  for (int64_t i0 = i_lo; i0 < i_hi; i0 += kChebGA) {
    const int ga = (int)min((int64_t)kChebGA, i_hi - i0);
    __syncthreads();
    for (int t = tid; t < ga * P; t += kChebThreads) {
      const int aa = t / P, p = t % P;
      bs[aa][p] = reinterpret_cast<const float4 *>(bmom)[(i0 + aa) * kChebPMax + p];
    }
    if (tid < ga) {
      as[tid] = load_antf<MONO>(a, i0 + tid);
      ls[tid] = c.lc[i0 + tid];
    }
    __syncthreads();
#pragma unroll 1
    for (int aa = 0; aa < ga; ++aa) {
      const AntD an = widen_ant<MONO>(as[aa]);
      PairBwd g[2];
      float ec[2], es[2], xv[2], sg[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double L;
        if (GEO == kModeBwd) {
          pair_geometry<MONO, CORR>(rec[u], an, no_gain, g[u]);
          domain |= valid[u] && !g[u].ok;
          L = g[u].L;
        } else {
          L = pair_length<MONO>(rec[u], an);
        }
        __sincosf(kTwoPi * frac_cycles(L * c.kc), &es[u], &ec[u]);   // E_c = e^{+j 2 pi f_c tau}
        float x = (float)((L - ls[aa]) * inv);
        x = fminf(fmaxf(x, -1.f), 1.f);
        xv[u] = fabsf(x) - 1.f;
        sg[u] = x < 0.f ? -1.f : 1.f;
      }
      const float4 *B = bs[aa];
      // single-row modes read only their row of (B_0[p], B_1[p]): one 8-byte load per moment
      const float2 *B1 = reinterpret_cast<const float2 *>(B) + (row1 ? 1 : 0);
      auto ldb = [&](int p) -> float4 {
        if (NX == 2) return B[p];
        const float2 v = B1[2 * p];
        return make_float4(v.x, v.y, 0.f, 0.f);
      };
      // even / odd partial sums in T_p(|x|) per sample and X row; T_p(x) = (-1)^p T_p(|x|)
      f2x he[2][2], ho[2][2];
      float4 b = ldb(0);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        he[u][0] = pk(b.x, b.y); he[u][1] = pk(b.z, b.w);
        ho[u][0] = 0ull; ho[u][1] = 0ull;
      }
      const f2x two_xm1 = pk(2.f * xv[0], 2.f * xv[1]);
      f2x d = pk(xv[0], xv[1]);
      f2x t = fadd2(pk(1.f, 1.f), d);                // (T_1, T_1')
      b = ldb(1);
      {
        const float2 tv = upk(t);
        ho[0][0] = ffma2(pk(tv.x, tv.x), pk(b.x, b.y), ho[0][0]);
        ho[1][0] = ffma2(pk(tv.y, tv.y), pk(b.x, b.y), ho[1][0]);
        if (NX == 2) {
          ho[0][1] = ffma2(pk(tv.x, tv.x), pk(b.z, b.w), ho[0][1]);
          ho[1][1] = ffma2(pk(tv.y, tv.y), pk(b.z, b.w), ho[1][1]);
        }
      }
#pragma unroll
      for (int p = 2; p < P; ++p) {
        d = ffma2(two_xm1, t, d);
        t = fadd2(t, d);
        b = ldb(p);
        const float2 tv = upk(t);
        f2x(&h)[2][2] = (p & 1) ? ho : he;
        h[0][0] = ffma2(pk(tv.x, tv.x), pk(b.x, b.y), h[0][0]);
        h[1][0] = ffma2(pk(tv.y, tv.y), pk(b.x, b.y), h[1][0]);
        if (NX == 2) {
          h[0][1] = ffma2(pk(tv.x, tv.x), pk(b.z, b.w), h[0][1]);
          h[1][1] = ffma2(pk(tv.y, tv.y), pk(b.z, b.w), h[1][1]);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float2 h0 = upk(ffma2(pk(sg[u], sg[u]), ho[u][0], he[u][0]));
        if (MODE == kModeBwd) {
          adj_accumulate<kModeBwd>(g[u], ec[u], es[u], h0.x, h0.y, S1[u], S2[u], S3x[u], S3y[u],
                                   S3z[u]);
        } else if (MODE == kModeFlt) {
          adj_accumulate<kModeFlt>(g[u], ec[u], es[u], h0.x, h0.y, M1[u], M2[u], S3x[u], S3y[u],
                                   S3z[u]);
        } else {
          const float2 h1 = upk(ffma2(pk(sg[u], sg[u]), ho[u][1], he[u][1]));
          adj_accumulate<kModeBwd>(g[u], ec[u], es[u], h0.x, h0.y, S1[u], S2[u], S3x[u], S3y[u],
                                   S3z[u]);
          adj_accumulate<kModeFlt>(g[u], ec[u], es[u], h1.x, h1.y, M1[u], M2[u], S3x[u], S3y[u],
                                   S3z[u]);
        }
      }
    }
  }
  if (domain) atomicOr(a.flags, 1u);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!valid[u]) continue;
    const int64_t j = c.idx ? (int64_t)c.idx[jb + u * kChebThreads] : jb + u * kChebThreads;
    if (MODE == kModeBwd) {
      adj_store<kModeBwd>(a, j, S1[u], S2[u], S3x[u], S3y[u], S3z[u]);
    } else if (MODE == kModeFlt) {
      adj_store<kModeFlt>(a, j, M1[u], M2[u], 0.f, 0.f, 0.f);
    } else {
      adj_store<kModeBwd>(a, j, S1[u], S2[u], S3x[u], S3y[u], S3z[u]);
      reinterpret_cast<float2 *>(a.out2)[(int64_t)blockIdx.y * a.n_s + j] =
          make_float2(M1[u], M2[u]);
    }
  }
}

// Matched filter only (the fused sweep's pass over every sample, and rfr_filter): four query
// points per thread -- two packed recurrence chains, and every B[p] load (8 bytes, this row
// only) feeds four moment updates.  No amplitude factors (Eq. 3): the pair needs only its path
// length.  Output: M partials [split][n_s] complex at a.out.
template <int P, bool MONO>
__global__ void __launch_bounds__(kChebThreads, 4) k_cheb_flt4(ChebArgs c, AdjArgs a,
                                                               const float2 *__restrict__ bmom) {
  if (c.hdr->P != P) return;
  constexpr int SPT = 4;
  __shared__ __align__(16) float2 bs[kChebGA][P];
  __shared__ AntF as[kChebGA];
  __shared__ double ls[kChebGA];
  __shared__ float4 gs[kChebGA][2];                 // F32G: tile-relative antenna geometry
  const int tid = threadIdx.x;
  const int64_t jb = (int64_t)blockIdx.x * (SPT * kChebThreads) + tid;
  if ((int64_t)blockIdx.x * (SPT * kChebThreads) >= a.n_s) return;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  Rec q[SPT];
  bool valid[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    valid[u] = jb + u * kChebThreads < a.n_s;
    q[u] = load_point<kModeFlt>(a, jb + u * kChebThreads, valid[u]);
  }
  const double inv = c.hdr->inv;
  const int row = c.row;
  float M1[SPT], M2[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) { M1[u] = 0.f; M2[u] = 0.f; }
  float d0 = 0.f, d1 = 0.f, d2 = 0.f;               // unused S3 slots of adj_accumulate
  for (int64_t i0 = i_lo; i0 < i_hi; i0 += kChebGA) {
    const int ga = (int)min((int64_t)kChebGA, i_hi - i0);
    __syncthreads();
    for (int t = tid; t < ga * P; t += kChebThreads) {
      const int aa = t / P, p = t % P;
      bs[aa][p] = bmom[((i0 + aa) * kChebPMax + p) * 2 + row];
    }
    if (tid < ga) {
      as[tid] = load_antf<MONO>(a, i0 + tid);
      ls[tid] = c.lc[i0 + tid];
    }
    __syncthreads();
#pragma unroll 1
    for (int aa = 0; aa < ga; ++aa) {
      const AntD an = widen_ant<MONO>(as[aa]);
      float ec[SPT], es[SPT], xv[SPT], sg[SPT];
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        const double L = pair_length<MONO>(q[u], an);
        __sincosf(kTwoPi * frac_cycles(L * c.kc), &es[u], &ec[u]);   // E_c = e^{+j 2 pi f_c tau}
        float x = (float)((L - ls[aa]) * inv);
        x = fminf(fmaxf(x, -1.f), 1.f);
        xv[u] = fabsf(x) - 1.f;
        sg[u] = x < 0.f ? -1.f : 1.f;
      }
      const float2 *B = bs[aa];
      f2x he[SPT], ho[SPT];
      const float2 b0 = B[0];
#pragma unroll
      for (int u = 0; u < SPT; ++u) { he[u] = pk(b0.x, b0.y); ho[u] = 0ull; }
      const f2x two01 = pk(2.f * xv[0], 2.f * xv[1]), two23 = pk(2.f * xv[2], 2.f * xv[3]);
      f2x d01 = pk(xv[0], xv[1]), d23 = pk(xv[2], xv[3]);
      f2x t01 = fadd2(pk(1.f, 1.f), d01), t23 = fadd2(pk(1.f, 1.f), d23);   // T_1
      {
        const float2 b = B[1];
        const f2x pb = pk(b.x, b.y);
        const float2 v01 = upk(t01), v23 = upk(t23);
        ho[0] = ffma2(pk(v01.x, v01.x), pb, ho[0]);
        ho[1] = ffma2(pk(v01.y, v01.y), pb, ho[1]);
        ho[2] = ffma2(pk(v23.x, v23.x), pb, ho[2]);
        ho[3] = ffma2(pk(v23.y, v23.y), pb, ho[3]);
      }
#pragma unroll
      for (int p = 2; p < P; ++p) {
        d01 = ffma2(two01, t01, d01);
        d23 = ffma2(two23, t23, d23);
        t01 = fadd2(t01, d01);
        t23 = fadd2(t23, d23);
        const float2 b = B[p];
        const f2x pb = pk(b.x, b.y);
        const float2 v01 = upk(t01), v23 = upk(t23);
        f2x *h = (p & 1) ? ho : he;
        h[0] = ffma2(pk(v01.x, v01.x), pb, h[0]);
        h[1] = ffma2(pk(v01.y, v01.y), pb, h[1]);
        h[2] = ffma2(pk(v23.x, v23.x), pb, h[2]);
        h[3] = ffma2(pk(v23.y, v23.y), pb, h[3]);
      }
      PairBwd g;                                      // unused by the filter epilogue
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        const float2 hh = upk(ffma2(pk(sg[u], sg[u]), ho[u], he[u]));
        adj_accumulate<kModeFlt>(g, ec[u], es[u], hh.x, hh.y, M1[u], M2[u], d0, d1, d2);
      }
    }
  }
  float2 *out = reinterpret_cast<float2 *>(a.out) + (int64_t)blockIdx.y * a.n_s;
#pragma unroll
  for (int u = 0; u < SPT; ++u)
    if (valid[u]) out[jb + u * kChebThreads] = make_float2(M1[u], M2[u]);
}

// =============================================================== tiled matched filter (5d)
constexpr int kTileBlock = 1024;
constexpr int kTileChunk = 4 * kChebThreads;       // points per filter CTA (TileArgs.chunk)
#ifndef RFR_TILE_FLT_MINB
#define RFR_TILE_FLT_MINB 5
#endif
constexpr int kTileFltMinBlocks = RFR_TILE_FLT_MINB;  // CTAs per SM of the tiled filter

int tile_count_blocks(int64_t n) { return (int)((n + kTileBlock - 1) / kTileBlock); }

__device__ __forceinline__ int tile_of(const double *b, float x, float y, float z) {
  const float p[3] = {x, y, z};
  int id = 0;
  for (int c = 2; c >= 0; --c) {
    const double w = b[3 + c] - b[c];
    int k = w > 0.0 ? (int)((p[c] - b[c]) / w * kTileDim) : 0;
    k = min(max(k, 0), kTileDim - 1);
    id = id * kTileDim + k;
  }
  return id;
}

// per-warp counts of each tile by ballots -> smem [warps][kTiles]
__device__ __forceinline__ void warp_tile_counts(int t, bool ok, int (*wc)[kTiles]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = 0; q < kTiles; ++q) {
    const unsigned b = __ballot_sync(0xffffffffu, ok && t == q);
    if (lane == 0) wc[warp][q] = __popc(b);
  }
}

__global__ void __launch_bounds__(kTileBlock) k_tile_count(TileArgs a) {
  if (a.ghdr->sel == 0) return;
  __shared__ int wc[kTileBlock / 32][kTiles];
  const int64_t n = a.n_dev ? *a.n_dev : a.n;
  const int64_t j = (int64_t)blockIdx.x * kTileBlock + threadIdx.x;
  const bool ok = j < n;
  int t = 0;
  if (ok) {
    t = a.rec ? tile_of(a.gbox, (float)a.rec[j].x, (float)a.rec[j].y, (float)a.rec[j].z)
              : tile_of(a.gbox, a.qx[j], a.qy[j], a.qz[j]);
    a.tile[j] = (unsigned char)t;
  }
  warp_tile_counts(t, ok, wc);
  __syncthreads();
  if (threadIdx.x < kTiles) {
    int c = 0;
    for (int w = 0; w < kTileBlock / 32; ++w) c += wc[w][threadIdx.x];
    a.bcnt[(int64_t)blockIdx.x * kTiles + threadIdx.x] = c;
  }
}

// thread q: exclusive offsets of tile q over the blocks; then the tile and CTA starts
__global__ void k_tile_scan(TileArgs a, int nb) {
  if (a.ghdr->sel == 0) return;
  __shared__ int tot[kTiles];
  const int q = threadIdx.x;
  int run = 0;
  for (int b = 0; b < nb; ++b) {
    const int c = a.bcnt[(int64_t)b * kTiles + q];
    a.bcnt[(int64_t)b * kTiles + q] = run;
    run += c;
  }
  tot[q] = run;
  __syncthreads();
  if (q == 0) {
    int s = 0, cs = 0;
    for (int k = 0; k < kTiles; ++k) {
      a.tstart[k] = s;
      a.cstart[k] = cs;
      s += tot[k];
      cs += (tot[k] + a.chunk - 1) / a.chunk;
    }
    a.tstart[kTiles] = s;
    a.cstart[kTiles] = cs;
  }
}

__global__ void __launch_bounds__(kTileBlock) k_tile_write(TileArgs a) {
  if (a.ghdr->sel == 0) return;
  __shared__ int wc[kTileBlock / 32][kTiles];
  const int64_t n = a.n_dev ? *a.n_dev : a.n;
  const int64_t j = (int64_t)blockIdx.x * kTileBlock + threadIdx.x;
  const bool ok = j < n;
  const int t = ok ? (int)a.tile[j] : 0;
  warp_tile_counts(t, ok, wc);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned m = __match_any_sync(0xffffffffu, ok ? t : -1);
  if (ok) {
    int pos = a.tstart[t] + a.bcnt[(int64_t)blockIdx.x * kTiles + t];
    for (int w = 0; w < warp; ++w) pos += wc[w][t];
    pos += __popc(m & ((1u << lane) - 1u));
    a.perm[pos] = (int)j;
    if (a.rec) {
      const Rec r = a.rec[j];
      a.rs[pos] = r;
      a.qs[pos] = make_float4((float)r.x, (float)r.y, (float)r.z, 0.f);
    } else {
      a.qs[pos] = make_float4(a.qx[j], a.qy[j], a.qz[j], 0.f);
    }
  }
}

__global__ void k_tile_box(TileArgs a) {
  if (a.ghdr->sel == 0) return;
  const int t = blockIdx.x;
  const int lo = a.tstart[t], hi = a.tstart[t + 1];
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const float4 v = a.qs[k];
    mn[0] = fmin(mn[0], (double)v.x); mx[0] = fmax(mx[0], (double)v.x);
    mn[1] = fmin(mn[1], (double)v.y); mx[1] = fmax(mx[1], (double)v.y);
    mn[2] = fmin(mn[2], (double)v.z); mx[2] = fmax(mx[2], (double)v.z);
  }
  __shared__ double sh[6][256];
  for (int c = 0; c < 3; ++c) { sh[c][threadIdx.x] = mn[c]; sh[3 + c][threadIdx.x] = mx[c]; }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int c = 0; c < 3; ++c) {
        sh[c][threadIdx.x] = fmin(sh[c][threadIdx.x], sh[c][threadIdx.x + s]);
        sh[3 + c][threadIdx.x] = fmax(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) a.tbox[t * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

// fp32 centre of a tile's box (the same rounding wherever it is evaluated)
__device__ __forceinline__ float tile_centre(const double *b, int c) {
  return (float)(0.5 * (b[c] + b[3 + c]));
}

// per (antenna, tile): centre path length; max half-spread over everything (fp64 bits, atomicMax:
// order-independent)
__global__ void k_tile_setup(TileArgs a) {
  if (a.ghdr->sel == 0) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double dm = 0.0;
  if (i < a.n_a) {
    for (int t = 0; t < kTiles; ++t) {
      const double *b = a.tbox + t * 6;
      if (!(b[0] <= b[3])) { a.lc[(int64_t)t * a.n_a + i] = 0.0; continue; }   // empty tile
      double tmin, tmax, rmin, rmax;
      box_dist(b, a.tx_x[i], a.tx_y[i], a.tx_z[i], tmin, tmax);
      if (a.rx_x) box_dist(b, a.rx_x[i], a.rx_y[i], a.rx_z[i], rmin, rmax);
      else { rmin = tmin; rmax = tmax; }
      const double Lc = 0.5 * (tmin + rmin + tmax + rmax);
      a.lc[(int64_t)t * a.n_a + i] = Lc;
      dm = fmax(dm, 0.5 * (tmax + rmax - tmin - rmin));
      if (!a.rx_x) {
        // monostatic tile-relative geometry around the fp32 tile centre c_t: a' = a - c_t,
        // D = |a'|^2, d_a = sqrt(D); per pair d - d_a = delta / (d + d_a) with
        // delta = |q'|^2 - 2 a'.q' in fp32 (k_tile_flt4 F32G)
        double ap[3];
        const double av[3] = {a.tx_x[i], a.tx_y[i], a.tx_z[i]};
        for (int c = 0; c < 3; ++c) ap[c] = av[c] - (double)tile_centre(b, c);
        const double D = ap[0] * ap[0] + ap[1] * ap[1] + ap[2] * ap[2];
        const double da = sqrt(D);
        float4 *g = a.tgeo + ((int64_t)t * a.n_a + i) * 2;
        g[0] = make_float4((float)(-2.0 * ap[0]), (float)(-2.0 * ap[1]), (float)(-2.0 * ap[2]),
                           (float)D);
        g[1] = make_float4((float)da, frac_cycles(2.0 * da * a.kc), (float)(2.0 * da - Lc), 0.f);
      }
    }
  }
  __shared__ double red[256];
  red[threadIdx.x] = dm;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(a.dmax, (unsigned long long)__double_as_longlong(red[0]));
}

__global__ void k_tile_select(TileArgs a) {
  const double delta = fmax(__longlong_as_double((long long)*a.dmax) * a.kd * (1.0 + 1e-6), 1e-30);
  const double zmax = 2.0 * 3.14159265358979323846 * (double)(a.n_f / 2 + 1) * delta;
  const int P = a.ghdr->sel ? cheb_select_P(zmax) : 0;
  a.hdr->sel = P > 0 ? 1u : 0u;
  a.hdr->P = P;
  a.hdr->delta = delta;
  a.hdr->inv = a.kd / delta;
  if (a.pub) *a.pub = P;
}

// B[i][t][p] = sum_m X_i[m] e^{+j 2 pi m' u_c,i,t} conj(a[m][p]); one CTA per antenna: per tile
// the rotated row (one sincospi per bin) into shared memory, then fixed-order partial sums
__global__ void __launch_bounds__(kAdjPrepThreads) k_tile_bprep(TileArgs a) {
  if (a.hdr->sel == 0) return;
  extern __shared__ float2 xs[];                    // [n_f] row, [n_f] rotated row, [4][64]
  const int P = a.hdr->P;
  const int64_t i = blockIdx.x;
  const int N = a.n_f;
  float2 *ys = xs + N, *part = xs + 2 * N;
  for (int m = threadIdx.x; m < N; m += blockDim.x) xs[m] = a.X[i * N + m];
  // thread (p, q): moment p over the bins m = q, q + Q, ...; PP = P rounded up to a power of two
  const int PP = P <= 16 ? 16 : (P <= 32 ? 32 : 64), Q = kAdjPrepThreads / PP;
  const int p = threadIdx.x % PP, q = threadIdx.x / PP;
  for (int t = 0; t < kTiles; ++t) {
    if (a.tstart[t + 1] == a.tstart[t]) continue;   // empty tile: never read
    const double uc = a.lc[(int64_t)t * a.n_a + i] * a.kd;
    __syncthreads();
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
      float ps, pc;                                 // e^{+j 2 pi m' u_c}
      sincospif(2.f * frac_cycles((double)(m - N / 2) * uc), &ps, &pc);
      const float2 v = xs[m];
      ys[m] = make_float2(fmaf(pc, v.x, -ps * v.y), fmaf(pc, v.y, ps * v.x));
    }
    __syncthreads();
    float re = 0.f, im = 0.f;
    if (p < P)
      for (int m = q; m < N; m += Q) {
        const float2 y = ys[m], c = a.coef[(int64_t)m * kChebPMax + p];   // y conj(c)
        re = fmaf(y.x, c.x, fmaf(y.y, c.y, re));
        im = fmaf(y.y, c.x, fmaf(-y.x, c.y, im));
      }
    part[q * PP + p] = make_float2(re, im);
    __syncthreads();
    if (threadIdx.x < P) {                          // fixed-order sum over the Q partials
      float2 v = part[threadIdx.x];
      for (int qq = 1; qq < Q; ++qq) {
        v.x += part[qq * PP + threadIdx.x].x;
        v.y += part[qq * PP + threadIdx.x].y;
      }
      a.bmom[(i * kTiles + t) * kChebPMax + threadIdx.x] = v;
    }
  }
}

// the filter over the sorted points: CTA -> (tile, chunk of kTileChunk points), 4 per thread
template <int P, bool MONO, bool F32G = false, bool STD = false>
__global__ void __launch_bounds__(kChebThreads, kTileFltMinBlocks) k_tile_flt4(TileArgs a) {
  if (a.hdr->P != P) return;
  constexpr int SPT = 4;
  const int blk = blockIdx.x;
  if (blk >= a.cstart[kTiles]) return;
  int t = 0;
  while (a.cstart[t + 1] <= blk) ++t;               // the tile of this CTA (kTiles entries)
  const int64_t base = a.tstart[t] + (int64_t)(blk - a.cstart[t]) * a.chunk;
  const int64_t end = a.tstart[t + 1];
  __shared__ __align__(16) float2 bs[kChebGA][P];
  __shared__ AntD as[kChebGA];                      // widened once per stage
  __shared__ double ls[kChebGA];
  __shared__ float4 gs[kChebGA][2];                 // F32G: tile-relative antenna geometry
  const int tid = threadIdx.x;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  Rec q[SPT];
  bool valid[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    const int64_t k = base + tid + u * kChebThreads;
    valid[u] = k < end;
    const float4 v = valid[u] ? a.qs[k] : make_float4(0.f, 0.f, 1.f, 0.f);
    q[u].x = v.x; q[u].y = v.y; q[u].z = v.z;
    q[u].w = 0.f; q[u].T = 1.f; q[u].nx = q[u].ny = 0.f; q[u].nz = 1.f; q[u].papr = 1.f;
  }
  // F32G: the points relative to the tile centre (fp32) and |q'|^2
  float qp[SPT][4];
  if (F32G) {
    const double *tb = a.tbox + t * 6;
    const float cx = tile_centre(tb, 0), cy = tile_centre(tb, 1), cz = tile_centre(tb, 2);
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      qp[u][0] = (float)(q[u].x - (double)cx);
      qp[u][1] = (float)(q[u].y - (double)cy);
      qp[u][2] = (float)(q[u].z - (double)cz);
      qp[u][3] = fmaf(qp[u][0], qp[u][0], fmaf(qp[u][1], qp[u][1], qp[u][2] * qp[u][2]));
    }
  }
  const double inv = a.hdr->inv;
  const float kc2f = (float)(2.0 * a.kc), inv2f = (float)(2.0 * inv);
  // monostatic: L = 2 d, so the cycle count is d (2 kc) and x = d (2 inv) - L_c inv (one DFMA)
  const double kc2 = 2.0 * a.kc, inv2 = 2.0 * inv;
  float M1[SPT], M2[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) { M1[u] = 0.f; M2[u] = 0.f; }
  float d0 = 0.f, d1 = 0.f, d2 = 0.f;
  for (int64_t i0 = i_lo; i0 < i_hi; i0 += kChebGA) {
    const int ga = (int)min((int64_t)kChebGA, i_hi - i0);
    __syncthreads();
    for (int w = tid; w < ga * P; w += kChebThreads) {
      const int aa = w / P, p = w % P;
      float2 v = a.bmom[((i0 + aa) * kTiles + t) * kChebPMax + p];
      if (STD && ((p >> 1) & 1)) { v.x = -v.x; v.y = -v.y; }   // B'_p = s_p B_p, s = (+ + - -)
      bs[aa][p] = v;
    }
    if (tid < ga) {
      AntF f;
      const int64_t ia = i0 + tid;
      f.x = a.tx_x[ia]; f.y = a.tx_y[ia]; f.z = a.tx_z[ia];
      if (MONO) { f.rx = f.ry = f.rz = 0.f; }
      else { f.rx = a.rx_x[ia]; f.ry = a.rx_y[ia]; f.rz = a.rx_z[ia]; }
      f.ptx = f.prx = 1.f;
      as[tid] = widen_ant<MONO>(f);
      ls[tid] = a.lc[(int64_t)t * a.n_a + ia] * (MONO ? inv : 1.0);   // L_c inv (mono) or L_c
      if (F32G) {
        const float4 *g = a.tgeo + ((int64_t)t * a.n_a + ia) * 2;
        float4 g1 = g[1];
        g1.z = (float)((double)g1.z * inv);          // x at the antenna's tile distance d_a
        gs[tid][0] = g[0];
        gs[tid][1] = g1;
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int aa = 0; aa < ga; ++aa) {
      const AntD an = as[aa];
      float ec[SPT], es[SPT], xv[SPT], sg[SPT];
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        if (F32G) {
          // d - d_a = delta / (d + d_a), delta = |q'|^2 - 2 a'.q' (fp32, all terms small);
          // cycles = frac(2 d_a kc) + 2 kc (d - d_a), x = (2 d_a - L_c) inv + 2 inv (d - d_a)
          const float4 g0 = gs[aa][0], g1 = gs[aa][1];
          const float del = fmaf(g0.x, qp[u][0], fmaf(g0.y, qp[u][1], fmaf(g0.z, qp[u][2], qp[u][3])));
          const float s2 = g0.w + del;
          const float dd = s2 * rsqrtf(s2);
          const float dl = __fdividef(del, dd + g1.x);
          float cy = fmaf(dl, kc2f, g1.y);
          cy -= rintf(cy);
          __sincosf(kTwoPi * cy, &es[u], &ec[u]);
          float x = fmaf(dl, inv2f, g1.z);
          x = fminf(fmaxf(x, -1.f), 1.f);
          xv[u] = STD ? x : fabsf(x) - 1.f;
          sg[u] = x < 0.f ? -1.f : 1.f;
          continue;
        }
        double cyc, xd;
        if (MONO) {
          const double dx = q[u].x - an.x, dy = q[u].y - an.y, dz = q[u].z - an.z;
          const double d = dist64(fma(dx, dx, fma(dy, dy, dz * dz)));
          cyc = d * kc2;
          xd = fma(d, inv2, -ls[aa]);
        } else {
          const double L = pair_length64<MONO>(q[u], an);
          cyc = L * a.kc;
          xd = (L - ls[aa]) * inv;
        }
        __sincosf(kTwoPi * frac_cycles(cyc), &es[u], &ec[u]);
        float x = (float)xd;
        x = fminf(fmaxf(x, -1.f), 1.f);
        xv[u] = fabsf(x) - 1.f;
        sg[u] = x < 0.f ? -1.f : 1.f;
      }
      const float2 *B = bs[aa];
      if (STD) {
        // plain three-term recurrence on v_p = s_p T_p(x), s = (+ + - -) repeating, so that
        // v_p = (-1)^(p+1) 2x v_{p-1} + v_{p-2} is one FFMA2 per two points (P <= 16: the
        // recurrence's ~p^2 u error stays < 2e-5); h = sum_p v_p B'_p, B'_p = s_p B_p
        const f2x x01 = pk(xv[0], xv[1]), x23 = pk(xv[2], xv[3]);
        const f2x tp01 = pk(2.f * xv[0], 2.f * xv[1]), tp23 = pk(2.f * xv[2], 2.f * xv[3]);
        const f2x tn01 = pk(-2.f * xv[0], -2.f * xv[1]), tn23 = pk(-2.f * xv[2], -2.f * xv[3]);
        f2x h[SPT];
        const float2 b0 = B[0], b1 = B[1];
        const f2x pb0 = pk(b0.x, b0.y), pb1 = pk(b1.x, b1.y);
        h[0] = ffma2(pk(xv[0], xv[0]), pb1, pb0);
        h[1] = ffma2(pk(xv[1], xv[1]), pb1, pb0);
        h[2] = ffma2(pk(xv[2], xv[2]), pb1, pb0);
        h[3] = ffma2(pk(xv[3], xv[3]), pb1, pb0);
        f2x v2_01 = pk(1.f, 1.f), v2_23 = pk(1.f, 1.f), v1_01 = x01, v1_23 = x23;
#pragma unroll
        for (int p = 2; p < P; ++p) {
          const f2x v01 = ffma2((p & 1) ? tp01 : tn01, v1_01, v2_01);
          const f2x v23 = ffma2((p & 1) ? tp23 : tn23, v1_23, v2_23);
          v2_01 = v1_01; v1_01 = v01;
          v2_23 = v1_23; v1_23 = v23;
          const float2 b = B[p];
          const f2x pb = pk(b.x, b.y);
          const float2 w01 = upk(v01), w23 = upk(v23);
          h[0] = ffma2(pk(w01.x, w01.x), pb, h[0]);
          h[1] = ffma2(pk(w01.y, w01.y), pb, h[1]);
          h[2] = ffma2(pk(w23.x, w23.x), pb, h[2]);
          h[3] = ffma2(pk(w23.y, w23.y), pb, h[3]);
        }
        PairBwd g;
#pragma unroll
        for (int u = 0; u < SPT; ++u) {
          const float2 hh = upk(h[u]);
          adj_accumulate<kModeFlt>(g, ec[u], es[u], hh.x, hh.y, M1[u], M2[u], d0, d1, d2);
        }
        continue;
      }
      f2x he[SPT], ho[SPT];
      const float2 b0 = B[0];
#pragma unroll
      for (int u = 0; u < SPT; ++u) { he[u] = pk(b0.x, b0.y); ho[u] = 0ull; }
      const f2x two01 = pk(2.f * xv[0], 2.f * xv[1]), two23 = pk(2.f * xv[2], 2.f * xv[3]);
      f2x d01 = pk(xv[0], xv[1]), d23 = pk(xv[2], xv[3]);
      f2x t01 = fadd2(pk(1.f, 1.f), d01), t23 = fadd2(pk(1.f, 1.f), d23);
      {
        const float2 b = B[1];
        const f2x pb = pk(b.x, b.y);
        const float2 v01 = upk(t01), v23 = upk(t23);
        ho[0] = ffma2(pk(v01.x, v01.x), pb, ho[0]);
        ho[1] = ffma2(pk(v01.y, v01.y), pb, ho[1]);
        ho[2] = ffma2(pk(v23.x, v23.x), pb, ho[2]);
        ho[3] = ffma2(pk(v23.y, v23.y), pb, ho[3]);
      }
#pragma unroll
      for (int p = 2; p < P; ++p) {
        d01 = ffma2(two01, t01, d01);
        d23 = ffma2(two23, t23, d23);
        t01 = fadd2(t01, d01);
        t23 = fadd2(t23, d23);
        const float2 b = B[p];
        const f2x pb = pk(b.x, b.y);
        const float2 v01 = upk(t01), v23 = upk(t23);
        f2x *h = (p & 1) ? ho : he;
        h[0] = ffma2(pk(v01.x, v01.x), pb, h[0]);
        h[1] = ffma2(pk(v01.y, v01.y), pb, h[1]);
        h[2] = ffma2(pk(v23.x, v23.x), pb, h[2]);
        h[3] = ffma2(pk(v23.y, v23.y), pb, h[3]);
      }
      PairBwd g;
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        const float2 hh = upk(ffma2(pk(sg[u], sg[u]), ho[u], he[u]));
        adj_accumulate<kModeFlt>(g, ec[u], es[u], hh.x, hh.y, M1[u], M2[u], d0, d1, d2);
      }
    }
  }
  float2 *out = a.out + (int64_t)blockIdx.y * a.n;
#pragma unroll
  for (int u = 0; u < SPT; ++u)
    if (valid[u]) out[a.perm[base + tid + u * kChebThreads]] = make_float2(M1[u], M2[u]);
}

// ------------------------------------------------ packed tiled filter (monostatic, fp32 geometry)
// k_tile_flt4<P, mono, F32G, STD> with every per-pair step after the moment staging in f32x2
// instructions over point pairs (0,1) and (2,3): on sm_100a a scalar 3-register FFMA / FMUL / FADD
// occupies the FMA pipe as long as one FFMA2 does (B300_MICROARCH "rt_SMSP = 2"), so the scalar
// geometry and epilogue were half of the kernel's FMA-pipe time (r02w SASS: 88 FFMA2 + 84 scalar
// FP32 per antenna and 4 points).  MUFU operands use the .ftz forms (no denormal rescaling
// sequences), and the epilogue keeps M = A1 + j A2 with A1 = sum ec h, A2 = sum es h (two FFMA2
// per pair instead of four FFMA).  Same arithmetic as k_tile_flt4 otherwise (DESIGN 5d).
__device__ __forceinline__ f2x bc(float v) { return pk(v, v); }
__device__ __forceinline__ float rsqrt_ftz(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float rcp_ftz(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ void sincos_ftz(float v, float &s, float &c) {
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(v));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(v));
}
__device__ __forceinline__ float rint_f(float v) {
  float r;
  asm("cvt.rni.f32.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
// per point pair: the tile-relative geometry of k_tile_flt4 (F32G), returning E = (cos, sin) of
// the centre phase per point and x per point, packed
struct PairGeo2 {
  f2x c, s, x;
};
__device__ __forceinline__ PairGeo2 tile_geo2(const float4 &g0, const float4 &g1, f2x qx, f2x qy,
                                              f2x qz, f2x qw, float kc2f, float inv2f) {
  // delta = |q'|^2 - 2 a'.q';  d - d_a = delta / (sqrt(D + delta) + d_a)
  const f2x del = ffma2(bc(g0.x), qx, ffma2(bc(g0.y), qy, ffma2(bc(g0.z), qz, qw)));
  const f2x s2 = fadd2(bc(g0.w), del);
  const float2 s2v = upk(s2);
  const f2x dd = fmul2(s2, pk(rsqrt_ftz(s2v.x), rsqrt_ftz(s2v.y)));
  const float2 den = upk(fadd2(dd, bc(g1.x)));
  const f2x dl = fmul2(del, pk(rcp_ftz(den.x), rcp_ftz(den.y)));
  // cycles = frac(2 d_a kc) + 2 kc (d - d_a), reduced to [-1/2, 1/2] (exact subtraction)
  const f2x cy = ffma2(dl, bc(kc2f), bc(g1.y));
  const float2 cv = upk(cy);
  const f2x ang = fmul2(fadd2(cy, pk(-rint_f(cv.x), -rint_f(cv.y))), bc(kTwoPi));
  const float2 av = upk(ang);
  PairGeo2 o;
  float s0, c0, s1, c1;
  sincos_ftz(av.x, s0, c0);
  sincos_ftz(av.y, s1, c1);
  o.c = pk(c0, c1);
  o.s = pk(s0, s1);
  const float2 xv = upk(ffma2(dl, bc(inv2f), bc(g1.z)));
  o.x = pk(fminf(fmaxf(xv.x, -1.f), 1.f), fminf(fmaxf(xv.y, -1.f), 1.f));
  return o;
}

// PIPE: the next antenna's geometry (MUFU chains) is issued ahead of the current antenna's moment
// loop, so its latency hides under the FFMA2 stream of the same warp
template <int P, bool PIPE, int MINB>
__global__ void __launch_bounds__(kChebThreads, MINB) k_tile_flt_pk(TileArgs a) {
  if (a.hdr->P != P) return;
  constexpr int SPT = 4;
  const int blk = blockIdx.x;
  if (blk >= a.cstart[kTiles]) return;
  int t = 0;
  while (a.cstart[t + 1] <= blk) ++t;
  const int64_t base = a.tstart[t] + (int64_t)(blk - a.cstart[t]) * a.chunk;
  const int64_t end = a.tstart[t + 1];
  __shared__ __align__(16) float2 bs[kChebGA][P];
  __shared__ float4 gs[kChebGA][2];
  const int tid = threadIdx.x;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  bool valid[SPT];
  float qp[SPT][4];
  {
    const double *tb = a.tbox + t * 6;
    const float cx = tile_centre(tb, 0), cy = tile_centre(tb, 1), cz = tile_centre(tb, 2);
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const int64_t k = base + tid + u * kChebThreads;
      valid[u] = k < end;
      const float4 v = valid[u] ? a.qs[k] : make_float4(cx, cy, cz, 0.f);
      qp[u][0] = (float)((double)v.x - (double)cx);
      qp[u][1] = (float)((double)v.y - (double)cy);
      qp[u][2] = (float)((double)v.z - (double)cz);
      qp[u][3] = fmaf(qp[u][0], qp[u][0], fmaf(qp[u][1], qp[u][1], qp[u][2] * qp[u][2]));
    }
  }
  const f2x qx01 = pk(qp[0][0], qp[1][0]), qy01 = pk(qp[0][1], qp[1][1]),
            qz01 = pk(qp[0][2], qp[1][2]), qw01 = pk(qp[0][3], qp[1][3]);
  const f2x qx23 = pk(qp[2][0], qp[3][0]), qy23 = pk(qp[2][1], qp[3][1]),
            qz23 = pk(qp[2][2], qp[3][2]), qw23 = pk(qp[2][3], qp[3][3]);
  const double inv = a.hdr->inv;
  const float kc2f = (float)(2.0 * a.kc), inv2f = (float)(2.0 * inv);
  f2x A1[SPT], A2[SPT];                             // sum ec h, sum es h (complex, packed)
#pragma unroll
  for (int u = 0; u < SPT; ++u) { A1[u] = 0ull; A2[u] = 0ull; }
  for (int64_t i0 = i_lo; i0 < i_hi; i0 += kChebGA) {
    const int ga = (int)min((int64_t)kChebGA, i_hi - i0);
    __syncthreads();
    for (int w = tid; w < ga * P; w += kChebThreads) {
      const int aa = w / P, p = w % P;
      float2 v = a.bmom[((i0 + aa) * kTiles + t) * kChebPMax + p];
      if ((p >> 1) & 1) { v.x = -v.x; v.y = -v.y; }   // B'_p = s_p B_p, s = (+ + - -)
      bs[aa][p] = v;
    }
    if (tid < ga) {
      const int64_t ia = i0 + tid;
      const float4 *g = a.tgeo + ((int64_t)t * a.n_a + ia) * 2;
      float4 g1 = g[1];
      g1.z = (float)((double)g1.z * inv);            // x at the antenna's tile distance d_a
      gs[tid][0] = g[0];
      gs[tid][1] = g1;
    }
    __syncthreads();
    PairGeo2 n01, n23;
    if (PIPE) {
      const float4 g0 = gs[0][0], g1 = gs[0][1];
      n01 = tile_geo2(g0, g1, qx01, qy01, qz01, qw01, kc2f, inv2f);
      n23 = tile_geo2(g0, g1, qx23, qy23, qz23, qw23, kc2f, inv2f);
    }
#pragma unroll 1
    for (int aa = 0; aa < ga; ++aa) {
      PairGeo2 e01, e23;
      if (PIPE) {
        e01 = n01;
        e23 = n23;
        const int an = aa + 1 < ga ? aa + 1 : aa;       // (the last one recomputes: no branch)
        const float4 g0 = gs[an][0], g1 = gs[an][1];
        n01 = tile_geo2(g0, g1, qx01, qy01, qz01, qw01, kc2f, inv2f);
        n23 = tile_geo2(g0, g1, qx23, qy23, qz23, qw23, kc2f, inv2f);
      } else {
        const float4 g0 = gs[aa][0], g1 = gs[aa][1];
        e01 = tile_geo2(g0, g1, qx01, qy01, qz01, qw01, kc2f, inv2f);
        e23 = tile_geo2(g0, g1, qx23, qy23, qz23, qw23, kc2f, inv2f);
      }
      const float2 *B = bs[aa];
      // v_p = s_p T_p(x): v_p = (-1)^(p+1) 2x v_{p-1} + v_{p-2}; h = sum_p v_p B'_p
      const f2x tp01 = fadd2(e01.x, e01.x), tp23 = fadd2(e23.x, e23.x);
      const f2x tn01 = fmul2(e01.x, bc(-2.f)), tn23 = fmul2(e23.x, bc(-2.f));
      const float2 x01 = upk(e01.x), x23 = upk(e23.x);
      const float2 b0 = B[0], b1 = B[1];
      const f2x pb0 = pk(b0.x, b0.y), pb1 = pk(b1.x, b1.y);
      f2x h[SPT];
      h[0] = ffma2(bc(x01.x), pb1, pb0);
      h[1] = ffma2(bc(x01.y), pb1, pb0);
      h[2] = ffma2(bc(x23.x), pb1, pb0);
      h[3] = ffma2(bc(x23.y), pb1, pb0);
      f2x v2_01 = bc(1.f), v2_23 = bc(1.f), v1_01 = e01.x, v1_23 = e23.x;
#pragma unroll
      for (int p = 2; p < P; ++p) {
        const f2x v01 = ffma2((p & 1) ? tp01 : tn01, v1_01, v2_01);
        const f2x v23 = ffma2((p & 1) ? tp23 : tn23, v1_23, v2_23);
        v2_01 = v1_01; v1_01 = v01;
        v2_23 = v1_23; v1_23 = v23;
        const float2 b = B[p];
        const f2x pb = pk(b.x, b.y);
        const float2 w01 = upk(v01), w23 = upk(v23);
        h[0] = ffma2(bc(w01.x), pb, h[0]);
        h[1] = ffma2(bc(w01.y), pb, h[1]);
        h[2] = ffma2(bc(w23.x), pb, h[2]);
        h[3] = ffma2(bc(w23.y), pb, h[3]);
      }
      const float2 c01 = upk(e01.c), s01 = upk(e01.s), c23 = upk(e23.c), s23 = upk(e23.s);
      A1[0] = ffma2(bc(c01.x), h[0], A1[0]); A2[0] = ffma2(bc(s01.x), h[0], A2[0]);
      A1[1] = ffma2(bc(c01.y), h[1], A1[1]); A2[1] = ffma2(bc(s01.y), h[1], A2[1]);
      A1[2] = ffma2(bc(c23.x), h[2], A1[2]); A2[2] = ffma2(bc(s23.x), h[2], A2[2]);
      A1[3] = ffma2(bc(c23.y), h[3], A1[3]); A2[3] = ffma2(bc(s23.y), h[3], A2[3]);
    }
  }
  float2 *out = a.out + (int64_t)blockIdx.y * a.n;
#pragma unroll
  for (int u = 0; u < SPT; ++u)
    if (valid[u]) {
      const float2 p1 = upk(A1[u]), p2 = upk(A2[u]);   // M = A1 + j A2
      out[a.perm[base + tid + u * kChebThreads]] = make_float2(p1.x - p2.y, p1.y + p2.x);
    }
}

static bool tile_fltpk() {          // RFR_FLTPK=0: the scalar-geometry k_tile_flt4 (A/B)
  static int v = -1;
  if (v < 0) { const char *e = getenv("RFR_FLTPK"); v = (e && e[0] == '0') ? 0 : 1; }
  return v == 1;
}

static bool tile_stdrec() {         // RFR_STDREC=0: the Reinsch recurrence at P = 16 too (A/B)
  static int v = -1;
  if (v < 0) { const char *e = getenv("RFR_STDREC"); v = (e && e[0] == '0') ? 0 : 1; }
  return v == 1;
}
static bool tile_f32g() {           // RFR_F32G=0: the fp64 per-pair geometry (A/B)
  static int v = -1;
  if (v < 0) { const char *e = getenv("RFR_F32G"); v = (e && e[0] == '0') ? 0 : 1; }
  return v == 1;
}
template <bool MONO>
static void tile_flt_all(const TileArgs &a, dim3 g, cudaStream_t st) {
  if (MONO && tile_f32g() && tile_stdrec() && tile_fltpk()) {
    static int pipe = -1;
    if (pipe < 0) { const char *e = getenv("RFR_FLTPIPE"); pipe = e ? atoi(e) : 1; }
    if (pipe == 1) k_tile_flt_pk<16, true, 4><<<g, kChebThreads, 0, st>>>(a);
    else if (pipe == 2) k_tile_flt_pk<16, true, 5><<<g, kChebThreads, 0, st>>>(a);
    else k_tile_flt_pk<16, false, kTileFltMinBlocks><<<g, kChebThreads, 0, st>>>(a);
  }
  else if (MONO && tile_f32g() && tile_stdrec())
    k_tile_flt4<16, MONO, true, true><<<g, kChebThreads, 0, st>>>(a);
  else if (MONO && tile_f32g()) k_tile_flt4<16, MONO, true><<<g, kChebThreads, 0, st>>>(a);
  else k_tile_flt4<16, MONO><<<g, kChebThreads, 0, st>>>(a);
  // P = 24 is the widest tiled variant: a tile spreads ~1/4 of the global delay range, so under
  // the global gate z <= 28.6 (P <= 48 untiled) no tile needs more (z_tile <= ~7 -> P <= 24)
  k_tile_flt4<24, MONO><<<g, kChebThreads, 0, st>>>(a);
}

static cudaError_t tile_prepare(const TileArgs &a, cudaStream_t st, bool bprep = true) {
  const int nb = tile_count_blocks(a.n);
  k_tile_count<<<nb, kTileBlock, 0, st>>>(a);
  k_tile_scan<<<1, kTiles, 0, st>>>(a, nb);
  k_tile_write<<<nb, kTileBlock, 0, st>>>(a);
  k_tile_box<<<kTiles, 256, 0, st>>>(a);
  cudaError_t e = cudaMemsetAsync(a.dmax, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  k_tile_setup<<<(unsigned)((a.n_a + 255) / 256), 256, 0, st>>>(a);
  k_tile_select<<<1, 1, 0, st>>>(a);
  k_cheb_coef<<<(a.n_f + 127) / 128, 128, 0, st>>>(a.hdr, a.n_f, kChebPMax, a.coef);
  if (!bprep) {
    if ((e = cudaGetLastError()) == cudaSuccess) add_launches(8);
    return e;
  }
  const size_t sm = (2 * (size_t)a.n_f + 4 * 64) * sizeof(float2);
  if (sm > 48 * 1024) {
    e = cudaFuncSetAttribute(k_tile_bprep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  k_tile_bprep<<<(unsigned)a.n_a, kAdjPrepThreads, sm, st>>>(a);
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(9);
  return e;
}

cudaError_t launch_tiled_filter(const TileArgs &a0, bool mono, int n_splits, cudaStream_t st) {
  if (a0.n_a <= 0 || a0.n <= 0) return cudaSuccess;
  TileArgs a = a0;
  a.chunk = kTileChunk;
  cudaError_t e = tile_prepare(a, st);
  if (e != cudaSuccess) return e;
  dim3 g((unsigned)((a.n + kTileChunk - 1) / kTileChunk + kTiles), (unsigned)n_splits);
  if (mono) tile_flt_all<true>(a, g, st);
  else tile_flt_all<false>(a, g, st);
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(2);
  return e;
}

// --------------------------------------------------- tiled K5 (matched-filter adjoint, DESIGN 6b)
// dL/ds_i[m] = sum_q c_q e^{-j 2 pi f_m tau_iq} is forward-shaped: per (antenna, tile) the moments
// M_it[p] = sum_{q in t} c_q e^{-j 2 pi f_c tau_iq} T_p(x_iqt) around the tile's own centre
// (x_iqt = (L_iq - L_c,it) inv), then s_i[m] = sum_t e^{-j 2 pi m' u_c,it} sum_p a[m][p] M_it[p].
// CTA = (128 antennas, one chunk of one tile's sorted query records), as k_cheb_fwd.
int64_t tile_fwd_chunk(int64_t n) { return std::max<int64_t>(256, (n + 63) / 64); }
int64_t tile_fwd_blocks(int64_t n) {
  return n > 0 ? (n + tile_fwd_chunk(n) - 1) / tile_fwd_chunk(n) + kTiles : 0;
}

template <int P, bool MONO, int MINB, bool QUAD = false, bool F32G = false, bool STD = false>
__global__ void __launch_bounds__(kChebThreads, MINB) k_tile_fwd(TileArgs a) {
  if (a.hdr->P != P) return;
  const int blk = blockIdx.y;
  if (blk >= a.cstart[kTiles]) return;
  int t = 0;
  while (a.cstart[t + 1] <= blk) ++t;               // the tile of this CTA (kTiles entries)
  const int64_t j_lo = a.tstart[t] + (int64_t)(blk - a.cstart[t]) * a.chunk;
  const int64_t j_hi = min((int64_t)a.tstart[t + 1], j_lo + a.chunk);
  __shared__ __align__(16) Rec rb[2][kChebTJ];
  const int tid = threadIdx.x;
  const int64_t ia = (int64_t)blockIdx.x * kChebThreads + tid;
  const bool ant_ok = ia < a.n_a;
  AntF af;
  if (ant_ok) af = load_antf<MONO>(a, ia);
  else { af.x = af.y = 0.f; af.z = 1.f; af.rx = af.ry = 0.f; af.rz = 1.f; af.ptx = af.prx = 1.f; }
  const AntD an = widen_ant<MONO>(af);
  const double Lc = ant_ok ? a.lc[(int64_t)t * a.n_a + ia] : 0.0;
  const double inv = a.hdr->inv;
  const double kc2 = 2.0 * a.kc, inv2 = 2.0 * inv, lsi = Lc * inv;
  // F32G (monostatic): tile-relative fp32 geometry as k_tile_flt4 (DESIGN 5d); the records'
  // q' = q - c_t and |q'|^2 once per staged record
  __shared__ float4 qf[kChebTJ];
  float4 g0 = make_float4(0.f, 0.f, 0.f, 1.f), g1 = make_float4(1.f, 0.f, 0.f, 0.f);
  float ctx = 0.f, cty = 0.f, ctz = 0.f;
  const float kc2f = (float)kc2, inv2f = (float)inv2;
  if (F32G) {
    const double *tb = a.tbox + t * 6;
    ctx = tile_centre(tb, 0); cty = tile_centre(tb, 1); ctz = tile_centre(tb, 2);
    if (ant_ok) {
      const float4 *g = a.tgeo + ((int64_t)t * a.n_a + ia) * 2;
      g0 = g[0];
      g1 = g[1];
      g1.z = (float)((double)g1.z * inv);
    }
  }
  f2x M[P];
#pragma unroll
  for (int p = 0; p < P; ++p) M[p] = 0ull;
  auto prefetch = [&](int64_t jt, int b) {
    const int nv = (int)min((int64_t)kChebTJ, j_hi - jt);
    const float4 *src = reinterpret_cast<const float4 *>(a.rs + jt);
    float4 *dst = reinterpret_cast<float4 *>(rb[b]);
    if (tid < kChebTJ * 3) {
      if (tid < 3 * nv) cp_async16(dst + tid, src + tid);
      else dst[tid] = make_float4(0.f, 0.f, 0.f, 0.f);      // tail: c = 0 records
    }
    cp_async_commit();
  };
  if (j_lo < j_hi) prefetch(j_lo, 0);
  int b = 0;
  for (int64_t jt = j_lo; jt < j_hi; jt += kChebTJ, b ^= 1) {
    cp_async_wait_all();
    __syncthreads();
    if (F32G) {
      if (tid < kChebTJ) {
        const Rec &r = rb[b][tid];
        const float x = (float)r.x - ctx, y = (float)r.y - cty, z = (float)r.z - ctz;
        qf[tid] = make_float4(x, y, z, fmaf(x, x, fmaf(y, y, z * z)));
      }
      __syncthreads();
    }
    if (jt + kChebTJ < j_hi) prefetch(jt + kChebTJ, b ^ 1);
    const int nv = (int)min((int64_t)kChebTJ, j_hi - jt);
#pragma unroll 1
    for (int jj = 0; jj < nv; jj += (MONO && P <= 16 && QUAD) ? 4 : 2) {
      f2x cc0 = 0ull, co0 = 0ull, cc1 = 0ull, co1 = 0ull;
      float xv0 = 0.f, xv1 = 0.f;
      auto geom = [&](int k, f2x &c, f2x &cn, float &xv) {
        const Rec &rec = rb[b][k];
        if (F32G) {        // d - d_a = delta / (d + d_a), delta = |q'|^2 - 2 a'.q'
          const float4 qv = qf[k];
          const float del = fmaf(g0.x, qv.x, fmaf(g0.y, qv.y, fmaf(g0.z, qv.z, qv.w)));
          const float s2 = g0.w + del;
          const float dl = __fdividef(del, s2 * rsqrtf(s2) + g1.x);
          float cy = fmaf(dl, kc2f, g1.y);
          cy -= rintf(cy);
          float es, ec;
          __sincosf(kTwoPi * cy, &es, &ec);
          const float Ar = rec.w, Ai = rec.T;
          c = pk(fmaf(Ar, ec, Ai * es), fmaf(Ai, ec, -Ar * es));
          float x = fmaf(dl, inv2f, g1.z);
          x = fminf(fmaxf(x, -1.f), 1.f);
          cn = x < 0.f ? pk(-upk(c).x, -upk(c).y) : c;
          xv = STD ? x : fabsf(x) - 1.f;
          return;
        }
        double cyc, xd;
        if (MONO) {      // L = 2 d: cycles d (2 kc), x = d (2 inv) - L_c inv (as k_tile_flt4)
          const double dx = rec.x - an.x, dy = rec.y - an.y, dz = rec.z - an.z;
          const double dd = dist64(fma(dx, dx, fma(dy, dy, dz * dz)));
          cyc = dd * kc2;
          xd = fma(dd, inv2, -lsi);
        } else {
          const double L = pair_length64<MONO>(rec, an);
          cyc = L * a.kc;
          xd = (L - Lc) * inv;
        }
        const float Ar = rec.w, Ai = rec.T;               // c_q (k_mf_adj_pack)
        float es, ec;
        __sincosf(kTwoPi * frac_cycles(cyc), &es, &ec);
        c = pk(fmaf(Ar, ec, Ai * es), fmaf(Ai, ec, -Ar * es));
        float x = (float)xd;
        x = fminf(fmaxf(x, -1.f), 1.f);
        cn = x < 0.f ? pk(-upk(c).x, -upk(c).y) : c;     // odd moments: T_p(x) = -T_p(|x|)
        xv = fabsf(x) - 1.f;
      };
      if (MONO && P <= 16 && QUAD) {   // four records per step: two packed recurrences
        f2x cc2, co2, cc3, co3;
        float xv2, xv3;
        geom(jj, cc0, co0, xv0);
        geom(jj + 1, cc1, co1, xv1);
        geom(jj + 2, cc2, co2, xv2);
        geom(jj + 3, cc3, co3, xv3);
        if (STD) {       // plain recurrence on v_p = s_p T_p(x) (k_tile_flt4); M'[p] = s_p M[p]
          const f2x tp01 = pk(2.f * xv0, 2.f * xv1), tp23 = pk(2.f * xv2, 2.f * xv3);
          const f2x tn01 = pk(-2.f * xv0, -2.f * xv1), tn23 = pk(-2.f * xv2, -2.f * xv3);
          acc2(M[0], cc0);
          acc2(M[0], cc1);
          acc2(M[0], cc2);
          acc2(M[0], cc3);
          M[1] = ffma2(pk(xv0, xv0), cc0, M[1]);
          M[1] = ffma2(pk(xv1, xv1), cc1, M[1]);
          M[1] = ffma2(pk(xv2, xv2), cc2, M[1]);
          M[1] = ffma2(pk(xv3, xv3), cc3, M[1]);
          f2x v2_01 = pk(1.f, 1.f), v2_23 = pk(1.f, 1.f), v1_01 = pk(xv0, xv1), v1_23 = pk(xv2, xv3);
#pragma unroll
          for (int p = 2; p < P; ++p) {
            const f2x v01 = ffma2((p & 1) ? tp01 : tn01, v1_01, v2_01);
            const f2x v23 = ffma2((p & 1) ? tp23 : tn23, v1_23, v2_23);
            v2_01 = v1_01; v1_01 = v01;
            v2_23 = v1_23; v1_23 = v23;
            const float2 w01 = upk(v01), w23 = upk(v23);
            M[p] = ffma2(pk(w01.x, w01.x), cc0, M[p]);
            M[p] = ffma2(pk(w01.y, w01.y), cc1, M[p]);
            M[p] = ffma2(pk(w23.x, w23.x), cc2, M[p]);
            M[p] = ffma2(pk(w23.y, w23.y), cc3, M[p]);
          }
          continue;
        }
        const f2x two01 = pk(2.f * xv0, 2.f * xv1), two23 = pk(2.f * xv2, 2.f * xv3);
        f2x d01 = pk(xv0, xv1), d23 = pk(xv2, xv3);
        acc2(M[0], cc0);
        acc2(M[0], cc1);
        acc2(M[0], cc2);
        acc2(M[0], cc3);
        f2x t01 = fadd2(pk(1.f, 1.f), d01), t23 = fadd2(pk(1.f, 1.f), d23);
        {
          const float2 v01 = upk(t01), v23 = upk(t23);
          M[1] = ffma2(pk(v01.x, v01.x), co0, M[1]);
          M[1] = ffma2(pk(v01.y, v01.y), co1, M[1]);
          M[1] = ffma2(pk(v23.x, v23.x), co2, M[1]);
          M[1] = ffma2(pk(v23.y, v23.y), co3, M[1]);
        }
#pragma unroll
        for (int p = 2; p < P; ++p) {
          d01 = ffma2(two01, t01, d01);
          d23 = ffma2(two23, t23, d23);
          t01 = fadd2(t01, d01);
          t23 = fadd2(t23, d23);
          const float2 v01 = upk(t01), v23 = upk(t23);
          M[p] = ffma2(pk(v01.x, v01.x), (p & 1) ? co0 : cc0, M[p]);
          M[p] = ffma2(pk(v01.y, v01.y), (p & 1) ? co1 : cc1, M[p]);
          M[p] = ffma2(pk(v23.x, v23.x), (p & 1) ? co2 : cc2, M[p]);
          M[p] = ffma2(pk(v23.y, v23.y), (p & 1) ? co3 : cc3, M[p]);
        }
        continue;
      }
      if (MONO && P <= 16) {     // both geometries in flight (ILP; no spills at this size)
        geom(jj, cc0, co0, xv0);
        geom(jj + 1, cc1, co1, xv1);
      } else {
#pragma unroll 1
        for (int u = 0; u < 2; ++u) {
          f2x c, cn;
          float xv;
          geom(jj + u, c, cn, xv);
          if (u == 0) { cc0 = c; co0 = cn; xv0 = xv; }
          else { cc1 = c; co1 = cn; xv1 = xv; }
        }
      }
      const f2x cc[2] = {cc0, cc1}, co[2] = {co0, co1};
      const f2x xm1 = pk(xv0, xv1), two_xm1 = pk(2.f * xv0, 2.f * xv1);
      f2x d = xm1, tt = pk(1.f, 1.f);
      acc2(M[0], cc[0]);
      acc2(M[0], cc[1]);
      tt = fadd2(tt, d);
      {
        const float2 tv = upk(tt);
        M[1] = ffma2(pk(tv.x, tv.x), co[0], M[1]);
        M[1] = ffma2(pk(tv.y, tv.y), co[1], M[1]);
      }
#pragma unroll
      for (int p = 2; p < P; ++p) {
        d = ffma2(two_xm1, tt, d);
        tt = fadd2(tt, d);
        const float2 tv = upk(tt);
        M[p] = ffma2(pk(tv.x, tv.x), (p & 1) ? co[0] : cc[0], M[p]);
        M[p] = ffma2(pk(tv.y, tv.y), (p & 1) ? co[1] : cc[1], M[p]);
      }
    }
  }
  cp_async_wait_all();
  if (ant_ok) {
    float2 *dst = a.fpart + ((int64_t)blk * a.n_a + ia) * kChebPMax;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      float2 v = upk(M[p]);
      if (STD && ((p >> 1) & 1)) { v.x = -v.x; v.y = -v.y; }   // M[p] = s_p M'[p]
      dst[p] = v;
    }
  }
}

// bins: one CTA per antenna; the tiles' moments (fixed-order sums over their chunks) in shared
// memory, one thread per bin with its coefficient row in registers, tiles in order
template <int P>
__global__ void __launch_bounds__(256) k_tile_out(TileArgs a, float2 *__restrict__ out) {
  if (a.hdr->P != P) return;
  __shared__ float2 Ms[kTiles][P];
  __shared__ double uc[kTiles];
  __shared__ int live[kTiles];
  const int64_t i = blockIdx.x;
  for (int w = threadIdx.x; w < kTiles * P; w += blockDim.x) {
    const int t = w / P, p = w % P;
    float2 v = make_float2(0.f, 0.f);
    for (int c = a.cstart[t]; c < a.cstart[t + 1]; ++c) {
      const float2 u = a.fpart[((int64_t)c * a.n_a + i) * kChebPMax + p];
      v.x += u.x;
      v.y += u.y;
    }
    Ms[t][p] = v;
  }
  if (threadIdx.x < kTiles) {
    const int t = threadIdx.x;
    live[t] = a.cstart[t + 1] > a.cstart[t];
    uc[t] = a.lc[(int64_t)t * a.n_a + i] * a.kd;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < a.n_f; m += blockDim.x) {
    float2 cf[P];
#pragma unroll
    for (int p = 0; p < P; ++p) cf[p] = a.coef[(int64_t)m * kChebPMax + p];
    const double mc = (double)(m - a.n_f / 2);
    float re = 0.f, im = 0.f;
#pragma unroll 1
    for (int t = 0; t < kTiles; ++t) {
      if (!live[t]) continue;
      float vr = 0.f, vi = 0.f;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float2 c = cf[p], v = Ms[t][p];
        vr = fmaf(c.x, v.x, fmaf(-c.y, v.y, vr));
        vi = fmaf(c.x, v.y, fmaf(c.y, v.x, vi));
      }
      float ps, pc;                                   // e^{-j 2 pi m' u_c,it}
      sincospif(2.f * frac_cycles(mc * uc[t]), &ps, &pc);
      re += fmaf(pc, vr, ps * vi);
      im += fmaf(pc, vi, -ps * vr);
    }
    out[i * a.n_f + m] = make_float2(re, im);
  }
}

template <int P, bool MONO>
constexpr int tile_fwd_minb() { return (MONO && P <= 28) || P <= 16 ? 5 : (P <= 32 ? 4 : 3); }
template <bool MONO>
static void tile_fwd_all(const TileArgs &a, dim3 g, cudaStream_t st) {
  // P = 16: four records per step at 4 CTAs / SM (r02m: 64.7 ms at c3 against 68.3 ms for two
  // records at 5 CTAs / SM); RFR_TFWD_MINB=5 selects the latter (A/B)
  static int two = -1;
  if (two < 0) { const char *e = getenv("RFR_TFWD_MINB"); two = (e && e[0] == '5') ? 1 : 0; }
  if (two) k_tile_fwd<16, MONO, tile_fwd_minb<16, MONO>()><<<g, kChebThreads, 0, st>>>(a);
  else if (MONO && tile_f32g() && tile_stdrec())
    k_tile_fwd<16, MONO, 4, true, true, true><<<g, kChebThreads, 0, st>>>(a);
  else if (MONO && tile_f32g()) k_tile_fwd<16, MONO, 4, true, true><<<g, kChebThreads, 0, st>>>(a);
  else k_tile_fwd<16, MONO, 4, true><<<g, kChebThreads, 0, st>>>(a);
  k_tile_fwd<24, MONO, tile_fwd_minb<24, MONO>()><<<g, kChebThreads, 0, st>>>(a);
}

cudaError_t launch_tiled_mfadj(const TileArgs &a0, bool mono, float2 *out, cudaStream_t st) {
  if (a0.n_a <= 0 || a0.n <= 0) return cudaSuccess;
  TileArgs a = a0;
  a.chunk = (int)tile_fwd_chunk(a.n);
  cudaError_t e = tile_prepare(a, st, false);
  if (e != cudaSuccess) return e;
  dim3 g((unsigned)((a.n_a + kChebThreads - 1) / kChebThreads), (unsigned)tile_fwd_blocks(a.n));
  if (mono) tile_fwd_all<true>(a, g, st);
  else tile_fwd_all<false>(a, g, st);
  const unsigned na = (unsigned)a.n_a;
  k_tile_out<16><<<na, 256, 0, st>>>(a, out);
  k_tile_out<24><<<na, 256, 0, st>>>(a, out);
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(4);
  return e;
}

// ------------------------------------------------- tiled backward (compacted active samples)
// As k_cheb_adj (kModeBwd, two samples per thread) over the tile-sorted compacted records, with
// the per-(antenna, tile) centres and moments of G; partials at the original sample index.
template <int P, bool MONO, bool CORR, bool STD = false>
__global__ void __launch_bounds__(kChebThreads, 4) k_tile_bwd(TileArgs ta, AdjArgs a) {
  if (ta.hdr->P != P) return;
  const int blk = blockIdx.x;
  if (blk >= ta.cstart[kTiles]) return;
  int t = 0;
  while (ta.cstart[t + 1] <= blk) ++t;
  const int64_t base = ta.tstart[t] + (int64_t)(blk - ta.cstart[t]) * ta.chunk;
  const int64_t end = ta.tstart[t + 1];
  __shared__ __align__(16) float2 bs[kChebGA][P];
  __shared__ AntF as[kChebGA];
  __shared__ double ls[kChebGA];
  __shared__ float4 gs[kChebGA][2];                 // F32G: tile-relative antenna geometry
  const int tid = threadIdx.x;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  bool valid[2];
  Rec rec[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int64_t k = base + tid + u * kChebThreads;
    valid[u] = k < end;
    if (valid[u]) rec[u] = ta.rs[k];
    else { rec[u].x = rec[u].y = 0.0; rec[u].z = 1.0; rec[u].w = 0.f; rec[u].T = 0.f;
           rec[u].nx = rec[u].ny = 0.f; rec[u].nz = 1.f; rec[u].papr = 1.f; }
  }
  const bool no_gain = a.no_gain;
  const double inv = ta.hdr->inv;
  float S1[2] = {0.f, 0.f}, S2[2] = {0.f, 0.f}, S3x[2] = {0.f, 0.f}, S3y[2] = {0.f, 0.f},
        S3z[2] = {0.f, 0.f};
  bool domain = false;
  for (int64_t i0 = i_lo; i0 < i_hi; i0 += kChebGA) {
    const int ga = (int)min((int64_t)kChebGA, i_hi - i0);
    __syncthreads();
    for (int w = tid; w < ga * P; w += kChebThreads) {
      const int aa = w / P, p = w % P;
      float2 v = ta.bmom[((i0 + aa) * kTiles + t) * kChebPMax + p];
      if (STD && ((p >> 1) & 1)) { v.x = -v.x; v.y = -v.y; }   // B'_p = s_p B_p (k_tile_flt4)
      bs[aa][p] = v;
    }
    if (tid < ga) {
      as[tid] = load_antf<MONO>(a, i0 + tid);
      ls[tid] = ta.lc[(int64_t)t * ta.n_a + i0 + tid];
    }
    __syncthreads();
#pragma unroll 1
    for (int aa = 0; aa < ga; ++aa) {
      const AntD an = widen_ant<MONO>(as[aa]);
      PairBwd g[2];
      float ec[2], es[2], xv[2], sg[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        pair_geometry<MONO, CORR>(rec[u], an, no_gain, g[u]);
        domain |= valid[u] && !g[u].ok;
        const double L = g[u].L;
        __sincosf(kTwoPi * frac_cycles(L * ta.kc), &es[u], &ec[u]);
        float x = (float)((L - ls[aa]) * inv);
        x = fminf(fmaxf(x, -1.f), 1.f);
        xv[u] = STD ? x : fabsf(x) - 1.f;
        sg[u] = x < 0.f ? -1.f : 1.f;
      }
      const float2 *B = bs[aa];
      if (STD) {           // plain three-term recurrence on v_p = s_p T_p(x), as k_tile_flt4
        const f2x tp = pk(2.f * xv[0], 2.f * xv[1]), tn = pk(-2.f * xv[0], -2.f * xv[1]);
        const float2 b0 = B[0], b1 = B[1];
        const f2x pb0 = pk(b0.x, b0.y), pb1 = pk(b1.x, b1.y);
        f2x h0v = ffma2(pk(xv[0], xv[0]), pb1, pb0), h1v = ffma2(pk(xv[1], xv[1]), pb1, pb0);
        f2x v2 = pk(1.f, 1.f), v1 = pk(xv[0], xv[1]);
#pragma unroll
        for (int p = 2; p < P; ++p) {
          const f2x v = ffma2((p & 1) ? tp : tn, v1, v2);
          v2 = v1;
          v1 = v;
          const float2 b = B[p];
          const f2x pb = pk(b.x, b.y);
          const float2 w = upk(v);
          h0v = ffma2(pk(w.x, w.x), pb, h0v);
          h1v = ffma2(pk(w.y, w.y), pb, h1v);
        }
        const float2 h0 = upk(h0v), h1 = upk(h1v);
        adj_accumulate<kModeBwd>(g[0], ec[0], es[0], h0.x, h0.y, S1[0], S2[0], S3x[0], S3y[0],
                                 S3z[0]);
        adj_accumulate<kModeBwd>(g[1], ec[1], es[1], h1.x, h1.y, S1[1], S2[1], S3x[1], S3y[1],
                                 S3z[1]);
        continue;
      }
      const float2 b0 = B[0];
      f2x he0 = pk(b0.x, b0.y), he1 = he0, ho0 = 0ull, ho1 = 0ull;
      const f2x two_xm1 = pk(2.f * xv[0], 2.f * xv[1]);
      f2x d = pk(xv[0], xv[1]);
      f2x tt = fadd2(pk(1.f, 1.f), d);
      {
        const float2 b = B[1];
        const float2 tv = upk(tt);
        ho0 = ffma2(pk(tv.x, tv.x), pk(b.x, b.y), ho0);
        ho1 = ffma2(pk(tv.y, tv.y), pk(b.x, b.y), ho1);
      }
#pragma unroll
      for (int p = 2; p < P; ++p) {
        d = ffma2(two_xm1, tt, d);
        tt = fadd2(tt, d);
        const float2 b = B[p];
        const f2x pb = pk(b.x, b.y);
        const float2 tv = upk(tt);
        if (p & 1) {
          ho0 = ffma2(pk(tv.x, tv.x), pb, ho0);
          ho1 = ffma2(pk(tv.y, tv.y), pb, ho1);
        } else {
          he0 = ffma2(pk(tv.x, tv.x), pb, he0);
          he1 = ffma2(pk(tv.y, tv.y), pb, he1);
        }
      }
      const float2 h0 = upk(ffma2(pk(sg[0], sg[0]), ho0, he0));
      const float2 h1 = upk(ffma2(pk(sg[1], sg[1]), ho1, he1));
      adj_accumulate<kModeBwd>(g[0], ec[0], es[0], h0.x, h0.y, S1[0], S2[0], S3x[0], S3y[0],
                               S3z[0]);
      adj_accumulate<kModeBwd>(g[1], ec[1], es[1], h1.x, h1.y, S1[1], S2[1], S3x[1], S3y[1],
                               S3z[1]);
    }
  }
  if (domain) atomicOr(a.flags, 1u);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!valid[u]) continue;
    const int64_t j = ta.idx[ta.perm[base + tid + u * kChebThreads]];
    adj_store<kModeBwd>(a, j, S1[u], S2[u], S3x[u], S3y[u], S3z[u]);
  }
}

template <bool MONO, bool CORR>
static void tile_bwd_all(const TileArgs &ta, const AdjArgs &a, dim3 g, cudaStream_t st) {
  if (tile_stdrec()) k_tile_bwd<16, MONO, CORR, true><<<g, kChebThreads, 0, st>>>(ta, a);
  else k_tile_bwd<16, MONO, CORR><<<g, kChebThreads, 0, st>>>(ta, a);
  k_tile_bwd<24, MONO, CORR><<<g, kChebThreads, 0, st>>>(ta, a);
}

cudaError_t launch_tiled_backward(const TileArgs &t0, const AdjArgs &a, bool mono, bool corr,
                                  int n_splits, cudaStream_t st) {
  if (t0.n_a <= 0 || t0.n <= 0) return cudaSuccess;
  TileArgs t = t0;
  t.chunk = 2 * kChebThreads;
  cudaError_t e = tile_prepare(t, st);
  if (e != cudaSuccess) return e;
  dim3 g((unsigned)((t.n + t.chunk - 1) / t.chunk + kTiles), (unsigned)n_splits);
  if (mono) {
    if (corr) tile_bwd_all<true, true>(t, a, g, st);
    else tile_bwd_all<true, false>(t, a, g, st);
  } else {
    if (corr) tile_bwd_all<false, true>(t, a, g, st);
    else tile_bwd_all<false, false>(t, a, g, st);
  }
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(2);
  return e;
}

// B moments of row a.X only (row 0), for a later launch_cheb_adj(..., prep_nx = -1)
cudaError_t launch_cheb_adj_prep_only(const ChebArgs &c, const AdjArgs &a, float2 *bmom,
                                      cudaStream_t st) {
  if (a.n_a <= 0) return cudaSuccess;
  const size_t sm = ((size_t)c.n_f + 4 * 64) * sizeof(float2);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_cheb_adj_prep,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  k_cheb_adj_prep<<<(unsigned)a.n_a, kAdjPrepThreads, sm, st>>>(c, a.X, a.X, 1, bmom);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

cudaError_t launch_cheb_flt(const ChebArgs &c, const AdjArgs &a, float2 *bmom, bool mono,
                            int n_splits, cudaStream_t st, int prep_nx) {
  if (a.n_a <= 0 || a.n_s <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (prep_nx >= 0) {
    const int nx = prep_nx > 0 ? prep_nx : 1;
    const size_t sm = ((size_t)c.n_f + 4 * 64) * sizeof(float2);
    if (sm > 48 * 1024) {
      e = cudaFuncSetAttribute(k_cheb_adj_prep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sm);
      if (e != cudaSuccess) return e;
    }
    k_cheb_adj_prep<<<(unsigned)a.n_a, kAdjPrepThreads, sm, st>>>(c, a.X, nx == 2 ? a.X2 : a.X,
                                                                  nx, bmom);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  dim3 g((unsigned)((a.n_s + 4 * kChebThreads - 1) / (4 * kChebThreads)), (unsigned)n_splits);
  if (mono) {
    k_cheb_flt4<16, true><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<24, true><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<28, true><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<32, true><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<48, true><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  } else {
    k_cheb_flt4<16, false><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<24, false><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<28, false><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<32, false><<<g, kChebThreads, 0, st>>>(c, a, bmom);
    k_cheb_flt4<48, false><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  }
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(prep_nx >= 0 ? 6 : 5);
  return e;
}

template <int MODE, bool MONO, bool CORR>
static cudaError_t cheb_adj_all(const ChebArgs &c, const AdjArgs &a, const float2 *bmom, dim3 g,
                                cudaStream_t st) {
  k_cheb_adj<16, MODE, MONO, CORR><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  k_cheb_adj<24, MODE, MONO, CORR><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  k_cheb_adj<28, MODE, MONO, CORR><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  k_cheb_adj<32, MODE, MONO, CORR><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  k_cheb_adj<48, MODE, MONO, CORR><<<g, kChebThreads, 0, st>>>(c, a, bmom);
  return cudaGetLastError();
}

cudaError_t launch_cheb_adj(const ChebArgs &c, const AdjArgs &a, float2 *bmom, int mode,
                            bool mono, bool corr, int n_splits, cudaStream_t st, int prep_nx) {
  if (a.n_a <= 0 || a.n_s <= 0) return cudaSuccess;
  const int nx = prep_nx > 0 ? prep_nx : (mode == kModeBoth ? 2 : 1);
  const size_t sm = ((size_t)c.n_f + 4 * 64) * sizeof(float2);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_cheb_adj_prep,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaSuccess;
  if (prep_nx >= 0) {                              // prep_nx < 0: B already prepared
    k_cheb_adj_prep<<<(unsigned)a.n_a, kAdjPrepThreads, sm, st>>>(
        c, a.X, (mode == kModeBoth || nx == 2) ? a.X2 : a.X, nx, bmom);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  dim3 g((unsigned)((a.n_s + 2 * kChebThreads - 1) / (2 * kChebThreads)), (unsigned)n_splits);
  if (mode == kModeBwd)
    e = mono ? (corr ? cheb_adj_all<kModeBwd, true, true>(c, a, bmom, g, st)
                     : cheb_adj_all<kModeBwd, true, false>(c, a, bmom, g, st))
             : (corr ? cheb_adj_all<kModeBwd, false, true>(c, a, bmom, g, st)
                     : cheb_adj_all<kModeBwd, false, false>(c, a, bmom, g, st));
  else if (mode == kModeBoth)
    e = mono ? (corr ? cheb_adj_all<kModeBoth, true, true>(c, a, bmom, g, st)
                     : cheb_adj_all<kModeBoth, true, false>(c, a, bmom, g, st))
             : (corr ? cheb_adj_all<kModeBoth, false, true>(c, a, bmom, g, st)
                     : cheb_adj_all<kModeBoth, false, false>(c, a, bmom, g, st));
  else
    e = mono ? cheb_adj_all<kModeFlt, true, false>(c, a, bmom, g, st)
             : cheb_adj_all<kModeFlt, false, false>(c, a, bmom, g, st);
  if (e == cudaSuccess) add_launches(prep_nx >= 0 ? 6 : 5);
  return e;
}

// ------------------------------------------------------------------------------- launchers
template <int P, bool MONO, bool CORR, int KIND>
static cudaError_t cheb_fwd_t(const ChebArgs &a, dim3 g, cudaStream_t st) {
  k_cheb_fwd<P, MONO, CORR, KIND><<<g, kChebThreads, 0, st>>>(a);
  return cudaGetLastError();
}
template <bool MONO, bool CORR, int KIND>
static cudaError_t cheb_fwd_all(const ChebArgs &a, dim3 g, cudaStream_t st) {
  cudaError_t e;
  if ((e = cheb_fwd_t<16, MONO, CORR, KIND>(a, g, st)) != cudaSuccess) return e;
  if ((e = cheb_fwd_t<24, MONO, CORR, KIND>(a, g, st)) != cudaSuccess) return e;
  if ((e = cheb_fwd_t<28, MONO, CORR, KIND>(a, g, st)) != cudaSuccess) return e;
  if ((e = cheb_fwd_t<32, MONO, CORR, KIND>(a, g, st)) != cudaSuccess) return e;
  return cheb_fwd_t<48, MONO, CORR, KIND>(a, g, st);
}

int cheb_box_blocks() { return kBoxBlocks; }
int cheb_threads() { return kChebThreads; }

cudaError_t launch_cheb_prepare(const ChebArgs &a, double *box_part, cudaStream_t st) {
  k_cheb_box<<<kBoxBlocks, 256, 0, st>>>(a.rec, a.n_s, a.n_dev, box_part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_cheb_setup<<<1, 1024, 0, st>>>(box_part, kBoxBlocks, a, a.lc, a.hdr);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_cheb_coef<<<(a.n_f + 127) / 128, 128, 0, st>>>(a.hdr, a.n_f, a.pmax, a.coef);
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(3);
  return e;
}

cudaError_t launch_cheb_fwd(const ChebArgs &a, bool mono, bool corr, int kind, int splits,
                            float2 *out, cudaStream_t st) {
  if (a.n_a <= 0) return cudaSuccess;
  dim3 g((unsigned)((a.n_a + kChebThreads - 1) / kChebThreads), (unsigned)splits);
  cudaError_t e;
  if (kind == kFwdMFAdj)
    e = mono ? cheb_fwd_all<true, false, kFwdMFAdj>(a, g, st)
             : cheb_fwd_all<false, false, kFwdMFAdj>(a, g, st);
  else if (mono)
    e = corr ? cheb_fwd_all<true, true, kFwdTrace>(a, g, st)
             : cheb_fwd_all<true, false, kFwdTrace>(a, g, st);
  else
    e = corr ? cheb_fwd_all<false, true, kFwdTrace>(a, g, st)
             : cheb_fwd_all<false, false, kFwdTrace>(a, g, st);
  if (e != cudaSuccess) return e;
  k_cheb_out<<<(unsigned)a.n_a, 256, 0, st>>>(a, splits, out);
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(6);
  return e;
}

}  // namespace rfr
