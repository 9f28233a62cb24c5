// rfr_kernels.cu -- sm_100a kernels of the lensless RF volumetric renderer.
//
//   k_blend        K1  per primary ray: NeuS alpha / transmittance -> 48 B
//                      records {fp64 position, w = p a alpha, T, n, Phi_apr} + (1 - alpha)
//   k_trace_fwd    K2  Eq. 4 tracing: per (antenna, 32-bin block) register
//                      accumulators, per-pair anchors staged in shared memory, Chebyshev phasor
//                      recurrence in packed f32x2 (FFMA2 + FADD2 per complex contribution)
//   k_adjoint      K3  App. A.5 adjoint: per sample, Horner over bins
//                  K4  Eq. 3 matched filter: same Horner core, complex epilogue
//   k_blend_bwd    K1' reverse scan through Eq. 5 and the blend (division-free)
//   k_loss_*       K6  residual and L2 loss
//   reductions     fixed-order split sums (deterministic, no float atomics)
#include "rfr_device.cuh"
#include "rfr_launch.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace rfr {

// ================================================================================== K1 blend
__global__ void k_blend(BlendArgs a) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const int nz = a.n_per_ray;
  const int64_t j0 = r * nz;
  float T = 1.f;
  float fk = a.sdf[j0];
  bool bad = false;
  for (int k = 0; k < nz; ++k) {
    const int64_t j = j0 + k;
    const bool has_next = (k + 1 < nz);
    const float fk1 = has_next ? a.sdf[j + 1] : 0.f;
    float alpha, oma;
    blend_step(a.s, fk, fk1, has_next, alpha, oma);
    const float p = a.power[j], refl = a.refl[j];
    const float x = a.x[j], y = a.y[j], z = a.z[j];
    const float nx = a.nx[j], ny = a.ny[j], nz_ = a.nz[j];
    const float papr = a.phi_origin ? a.phi_origin[j] : 1.f;
    if (a.check_finite) {
      bad |= !isfinite(p) || !isfinite(refl) || !isfinite(x) || !isfinite(y) || !isfinite(z) ||
             !isfinite(nx) || !isfinite(ny) || !isfinite(nz_) || !isfinite(fk) || !isfinite(papr);
    }
    Rec rec;
    rec.x = (double)x; rec.y = (double)y; rec.z = (double)z;
    rec.w = p * refl * alpha;
    if (a.aflag) a.aflag[j] = alpha != 0.f ? 1 : 0;
    rec.T = T;
    rec.nx = nx; rec.ny = ny; rec.nz = nz_;
    rec.papr = papr;
    a.rec[j] = rec;
    T *= oma;
    fk = fk1;
  }
  if (bad) atomicOr(a.flags, 2u);
}

// Warp per ray, lane = sample (chunks of 32 samples): every load and store is coalesced along the
// ray-major sample index, and the transmittance T_k = prod_{l<k} (1 - alpha_l) is an
// exclusive product scan over the lanes with the running product carried across chunks.  Same
// per-sample arithmetic as k_blend; only the association of the products differs (a tree instead
// of a left fold), and exact factors stay exact: a (1 - alpha) of 0 or 1 gives the same T.
// (c3: 84 -> ~20 us per call; the thread-per-ray form kept its rays' 32 samples in one thread,
// with only 256 warps in flight on 148 SMs.)
__global__ void __launch_bounds__(256) k_blend_warp(BlendArgs a) {
  const int lane = (int)(threadIdx.x & 31);
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= a.n_rays) return;                        // warp-uniform
  const int nz = a.n_per_ray;
  const int64_t j0 = r * nz;
  float Tc = 1.f;                                   // product of (1 - alpha) over the chunks so far
  bool bad = false;
  for (int k0 = 0; k0 < nz; k0 += 32) {
    const int k = k0 + lane;
    const bool in = k < nz;
    const int64_t j = j0 + k;
    float alpha = 0.f, oma = 1.f, fk = 0.f;
    if (in) {
      const bool has_next = (k + 1 < nz);
      fk = a.sdf[j];
      const float fk1 = has_next ? a.sdf[j + 1] : 0.f;
      blend_step(a.s, fk, fk1, has_next, alpha, oma);
    }
    float incl = oma;                               // inclusive product scan over the lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const float v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl *= v;
    }
    float excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 1.f;
    const float T = Tc * excl;
    Tc *= __shfl_sync(0xffffffffu, incl, 31);
    if (in) {
      const float p = a.power[j], refl = a.refl[j];
      const float x = a.x[j], y = a.y[j], z = a.z[j];
      const float nx = a.nx[j], ny = a.ny[j], nz_ = a.nz[j];
      const float papr = a.phi_origin ? a.phi_origin[j] : 1.f;
      if (a.check_finite) {
        bad |= !isfinite(p) || !isfinite(refl) || !isfinite(x) || !isfinite(y) || !isfinite(z) ||
               !isfinite(nx) || !isfinite(ny) || !isfinite(nz_) || !isfinite(fk) || !isfinite(papr);
      }
      Rec rec;
      rec.x = (double)x; rec.y = (double)y; rec.z = (double)z;
      rec.w = p * refl * alpha;
      if (a.aflag) a.aflag[j] = alpha != 0.f ? 1 : 0;
      rec.T = T;
      rec.nx = nx; rec.ny = ny; rec.nz = nz_;
      rec.papr = papr;
      a.rec[j] = rec;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags, 2u);
}

// ================================================================================== K2 forward
// Warp-independent design (no CTA barriers on the hot loop).  Warp w of a CTA owns taw = 32 / nbc
// antennas (a0 + w taw ...) and all nbc bin blocks of B bins of this CTA's bin chunk; lane
// (my_b, my_a) = (lane / taw, lane % taw) keeps B complex accumulators in registers (packed f32x2).
// The warp walks its CTA's sample split in tiles of TJ samples:
//   prefetch: the next tile's 48 B records are copied global -> shared with cp.async while the
//             current tile runs (no register cost, latency hidden behind phase 2)
//   phase 1:  the taw x TJ (antenna, sample) pairs of the tile, one per lane: fp64 geometry, the
//             Eq. 5 amplitude, anchors y0_b = A e^{-j2pi(f0 + bB df)tau}, y1_b = y0_b z,
//             z = e^{-j2pi df tau}, for every bin block b, into the warp's shared-memory slice
//   phase 2:  each lane runs the Chebyshev recurrence y_{m+1} = 2cos(theta) y_m - y_{m-1} over its
//             B bins in the sign-alternating form q_m = sigma_m y_m (sigma = +,+,-,-): ONE FFMA2
//             per step and ONE FADD2 per accumulate.
// Warps synchronise only with __syncwarp, so the FMA-light phase 1 of one warp overlaps the
// FMA-bound phase 2 of the others.  Bin chunks (blockIdx.z) of 32 blocks cover n_f > 32 B.
//
// KIND == kFwdMFAdj (K5, matched-filter adjoint): the "samples" are filter queries packed by
// k_mf_adj_pack as {x, y, z, w = Re c_q, T = Im c_q} with c_q = (dL/dP_q) M_q / max(P_q, eps); the
// per-pair amplitude is the complex c_q itself (no gain, decay or transmittance), so the kernel
// computes dL/ds(i,m) = sum_q c_q e^{-j 2 pi f_m tau_iq} with the same anchors and recurrence.
// NB > 0: compile-time bin blocks per warp (n_f = 32 NB x chunks, no partial chunk), so the
// per-pair loops and the slot arithmetic of phase 1 fold to constants; NB == 0: runtime.
template <int B, bool MONO, bool CORR, int KIND, int NB>
__global__ void __launch_bounds__(kFwdThreads, fwd_min_blocks(B)) k_trace_fwd(FwdArgs a) {
  constexpr int TJ = fwd_tj(B);
  if (a.skip && a.skip->sel) return;              // the Chebyshev-moment path was chosen
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbc = NB > 0 ? NB : a.nb, taw = NB > 0 ? 32 / NB : a.taw;
  unsigned char *wb = smem_raw + (size_t)warp * a.warp_smem;
  // fixed strides (32 slots per sample) so that phase-2 addresses are compile-time offsets
  float4 *anc = reinterpret_cast<float4 *>(wb);                          // [TJ][32]: slot b*taw+aa
  float *kv = reinterpret_cast<float *>(wb + TJ * 32 * 16);          // [TJ][32]: slot aa
  AntD *ant = reinterpret_cast<AntD *>(wb + TJ * 32 * 20);           // [taw]
  Rec *rbuf = reinterpret_cast<Rec *>(wb + TJ * 32 * 20 + 32 * sizeof(AntD));  // [2][TJ]
  const int64_t a0 = ((int64_t)blockIdx.x * kFwdWarps + warp) * taw;
  const int64_t j_lo = (int64_t)blockIdx.y * a.samples_per_split;
  const int64_t j_hi = min(a.n_s, j_lo + a.samples_per_split);
  const int chunk = blockIdx.z;
  const double k0 = a.k0 + (double)chunk * a.kchunk;                    // f0 of this bin chunk / c
  const int nb_here = NB > 0 ? NB : min(nbc, a.nb_total - chunk * nbc);   // blocks in this chunk
  const bool no_gain = a.no_gain;

  for (int aa = lane; aa < taw; aa += 32) {
    const int64_t ia = a0 + aa;
    AntD d;
    if (ia < a.n_a) {
      d.x = a.tx_x[ia]; d.y = a.tx_y[ia]; d.z = a.tx_z[ia];
      if (MONO) { d.rx = d.x; d.ry = d.y; d.rz = d.z; }
      else { d.rx = a.rx_x[ia]; d.ry = a.rx_y[ia]; d.rz = a.rx_z[ia]; }
      d.ptx = a.phi_tx ? a.phi_tx[ia] : 1.f;
      d.prx = a.phi_rx ? a.phi_rx[ia] : (MONO ? d.ptx : 1.f);
    } else {
      d.x = d.y = 0.0; d.z = 1.0; d.rx = d.ry = 0.0; d.rz = 1.0; d.ptx = d.prx = 1.f;
    }
    ant[aa] = d;
  }
  const int my_a = lane % taw, my_b = lane / taw;
  const bool active = my_b < nb_here;
  f2x acc[B];
#pragma unroll
  for (int m = 0; m < B; ++m) acc[m] = 0ull;
  bool domain = false;

  // records of one tile: TJ x 48 B = 3 TJ chunks of 16 B spread over the lanes
  // the tile's records are one contiguous run of TJ x 48 B: copy it as 16-byte chunks
  auto prefetch = [&](int64_t jt, int buf) {
    const int n_chunks = 3 * (int)min((int64_t)TJ, j_hi - jt);
    const float4 *src = reinterpret_cast<const float4 *>(a.rec + jt);
    float4 *dst = reinterpret_cast<float4 *>(rbuf + buf * TJ);
#pragma unroll
    for (int c0 = 0; c0 < TJ * 3; c0 += 32) {
      const int c = c0 + lane;
      if (c < n_chunks) cp_async16(dst + c, src + c);
      else if (c < TJ * 3) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);   // tail: w = 0 records
    }
    cp_async_commit();
  };
  if (j_lo < j_hi) prefetch(j_lo, 0);
  int buf = 0;
  for (int64_t jt = j_lo; jt < j_hi; jt += TJ, buf ^= 1) {
    cp_async_wait_all();
    __syncwarp();
    if (jt + TJ < j_hi) prefetch(jt + TJ, buf ^ 1);
    // ---------------- phase 1: per-pair geometry and anchors (one pair per lane).  Branch-free:
    // tail samples carry zero records (w = 0) and padded antennas a zero amplitude, so a lane's
    // pairs are independent straight-line code the scheduler can interleave.
#pragma unroll
    for (int pr = lane; pr < taw * TJ; pr += 32) {
      const int aa = pr % taw, jj = pr / taw;
      const bool valid = (jt + jj < j_hi) && (a0 + aa < a.n_a);
      float4 *dst = anc + jj * 32 + aa;
      const Rec rec = rbuf[buf * TJ + jj];
      double L;
      float Ar, Ai;
      if (KIND == kFwdTrace) {
        PairBwd g;
        pair_geometry<MONO, CORR>(rec, ant[aa], no_gain, g);
        domain |= valid && !g.ok;
        Ar = valid ? rec.w * g.gg * g.Tt * g.Tr : 0.f;
        Ai = 0.f;
        L = g.L;
      } else {
        L = pair_length<MONO>(rec, ant[aa]);
        Ar = valid ? rec.w : 0.f;
        Ai = valid ? rec.T : 0.f;
      }
      // phase anchors from fp64 cycle counts (cycles = L f / c), reduced to [-0.5, 0.5]
      const float fr0 = frac_cycles(L * k0);
      const float frd = frac_cycles(L * a.kd);
      const float frw = frac_cycles(L * a.kw);
      float es, ec, zs, zc, ws, wc;
      __sincosf(kTwoPi * fr0, &es, &ec);            // anchor phase: MUFU, error not amplified
      sincospif(2.f * frd, &zs, &zc);               // recurrence step: accurate (sets 2cos theta)
      __sincosf(kTwoPi * frw, &ws, &wc);            // block step
      // A e^{-j theta0} (real A: trace; complex A: matched-filter adjoint)
      f2x c = (KIND == kFwdTrace) ? pk(Ar * ec, -Ar * es)
                                  : pk(fmaf(Ar, ec, Ai * es), fmaf(Ai, ec, -Ar * es));
      const f2x zz = pk(zc, -zs), ww = pk(wc, -ws);
      for (int b = 0; b < nb_here; ++b) {
        const float2 y0 = upk(c), y1 = upk(cmul2(c, zz));
        dst[b * taw] = make_float4(y0.x, y0.y, y1.x, y1.y);
        c = cmul2(c, ww);
      }
      kv[jj * 32 + aa] = 2.f * zc;
    }
    __syncwarp();
    // ---------------- phase 2: bin recurrences, two samples interleaved (independent chains)
    if (active) {
      const float4 *ap = anc + my_b * taw + my_a;
      const float *kp_ = kv + my_a;
#pragma unroll 1
      for (int jj = 0; jj < TJ; jj += 2) {
        const float4 Ya = ap[jj * 32], Yb = ap[(jj + 1) * 32];
        const float ka = kp_[jj * 32], kb = kp_[(jj + 1) * 32];
        const f2x kpa = pk(ka, ka), kna = pk(-ka, -ka), kpb = pk(kb, kb), knb = pk(-kb, -kb);
        f2x a0 = pk(Ya.x, Ya.y), a1 = pk(Ya.z, Ya.w);
        f2x b0 = pk(Yb.x, Yb.y), b1 = pk(Yb.z, Yb.w);
        acc2(acc[0], a0); acc2(acc[0], b0);
        acc2(acc[1], a1); acc2(acc[1], b1);
#pragma unroll
        for (int m = 1; m < B - 1; ++m) {
          const f2x a2 = ffma2((m & 1) ? kna : kpa, a1, a0);
          const f2x b2 = ffma2((m & 1) ? knb : kpb, b1, b0);
          acc2(acc[m + 1], a2); acc2(acc[m + 1], b2);
          a0 = a1; a1 = a2;
          b0 = b1; b1 = b2;
        }
      }
    }
  }
  cp_async_wait_all();
  if (domain) atomicOr(a.flags, 1u);
  const int64_t ia = a0 + my_a;
  if (active && ia < a.n_a) {
    const int bin0 = (chunk * nbc + my_b) * B;
    float2 *dst = a.out + ((int64_t)blockIdx.y * a.n_a + ia) * a.n_f + bin0;
    const int lim = min(B, a.n_f - bin0);
#pragma unroll
    for (int m = 0; m < B; ++m) {
      if (m < lim) {
        const float2 v = upk(acc[m]);
        const float sg = (m & 2) ? -1.f : 1.f;       // undo sigma_m
        dst[m] = make_float2(sg * v.x, sg * v.y);
      }
    }
  }
}

// ================================================================================== K3 / K4
// One thread owns one sample (or query) and loops over the antennas of its split.  Per pair:
// fp64 path length, E = e^{+j2pi f0 tau}, w = e^{+j2pi df tau}; Horner h = sum_m X(i,m) w^m over the
// bins with X(i, .) broadcast from shared memory (2 FFMA2 per complex step).
//   MODE_BWD: R = Re(E h) -> per-sample sums S1, S2, S3 (Eq. 5 chain), written as partials.
//   MODE_FLT: M += E h (complex) -> partial matched-filter output.
// NF > 0 (the configs' bin counts): straight-line code over two independent Horner chains that
// share w -- bins [NF/2, NF) and [0, NF/2), merged as h = h_lo + w^{NF/2} h_hi.  Both FFMA2 of a
// step read w from the same register (ptxas folds the (-Im, Re) swizzle into the operand), so w
// stays in the operand reuse cache across the chains and each FFMA2 reads at most two registers
// per bank: the issue interval drops from 3 to 2 cycles (tools/sass_banks.py).  X is staged
// interleaved, X'[m] = (X[m], X[m + NF/2]), one LDS.128 per step.  NF == 0: rolled single chain.
// Specialised bin count NF (64/128/256/512).  Warps 0..3 are consumers (one sample or query per
// thread); warp 4 is the producer: its lane 0 streams the X rows of the split, kAdjRowsStage
// antennas per stage, through a kAdjStages-deep shared-memory ring with the bulk-copy (TMA)
// engine, signalled by "full" mbarriers (transaction bytes) and released by "empty" mbarriers
// (one arrive per consumer warp).  No CTA-wide barrier on the hot path: a consumer warp waits
// only for the bytes it needs, so warps that drift apart are absorbed by the ring.
// Horner: two chains per sample stepping by v = w^2 over the even and odd bins, h = h_e + w h_o;
// one LDS.128 = (X[2k], X[2k+1]) feeds both, and both FFMA2 of a step read v from one register
// (operand reuse cache), so each FFMA2 reads at most two registers per bank.
template <int MODE, bool MONO, bool CORR, int NF>
__global__ void __launch_bounds__(kAdjThreads + 32, 4) k_adjoint_tma(AdjArgs a) {
  if (a.skip && a.skip->sel) return;
  constexpr int GA = adj_stage_ants(NF);
  constexpr int NS = kAdjStages;
  constexpr int H = NF / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2 *Xs = reinterpret_cast<float2 *>(smem_raw);                          // [NS][GA][NF]
  unsigned long long *full = reinterpret_cast<unsigned long long *>(
      smem_raw + (size_t)NS * GA * NF * sizeof(float2));
  unsigned long long *empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  const int n_stages = (int)((max(i_hi - i_lo, (int64_t)0) + GA - 1) / GA);
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kAdjThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kAdjThreads / 32) {                 // ------------------------------ producer
    if (lane == 0) {
      for (int st = 0; st < n_stages; ++st) {
        const int b = st % NS;
        if (st >= NS) mbar_wait_sleep(&empty[b], ((st / NS) - 1) & 1);
        const int64_t ic = i_lo + (int64_t)st * GA;
        const int ga = (int)min((int64_t)GA, i_hi - ic);
        const unsigned bytes = (unsigned)(ga * NF * sizeof(float2));
        mbar_arrive_expect_tx(&full[b], bytes);
        bulk_g2s(Xs + (size_t)b * GA * NF, a.X + ic * NF, bytes, &full[b]);
      }
    }
    return;
  }

  // ------------------------------------------------------------------------------ consumers
  const int64_t j = (int64_t)blockIdx.x * kAdjThreads + tid;
  const bool valid = j < a.n_s;
  const Rec rec = load_point<MODE>(a, j, valid);
  const bool no_gain = a.no_gain;
  float S1 = 0.f, S2 = 0.f, S3x = 0.f, S3y = 0.f, S3z = 0.f;
  bool domain = false;
  // antenna coordinates prefetched one pair ahead (floats; widened to fp64 at use)
  float nx_ = 0.f, ny_ = 0.f, nz_ = 0.f;
  if (n_stages > 0) { nx_ = a.tx_x[i_lo]; ny_ = a.tx_y[i_lo]; nz_ = a.tx_z[i_lo]; }
  for (int st = 0; st < n_stages; ++st) {
    const int b = st % NS;
    const int64_t ic = i_lo + (int64_t)st * GA;
    const int ga = (int)min((int64_t)GA, i_hi - ic);
    mbar_wait(&full[b], (st / NS) & 1);
    const float2 *X = Xs + (size_t)b * GA * NF;
    for (int aa = 0; aa < ga; ++aa) {
      AntD an;
      if (MONO && !a.phi_tx) {
        an.x = nx_; an.y = ny_; an.z = nz_;
        an.rx = an.x; an.ry = an.y; an.rz = an.z;
        an.ptx = an.prx = 1.f;
      } else {
        an = load_ant<MONO>(a, ic + aa);
      }
      if (ic + aa + 1 < i_hi) {                   // prefetch the next antenna
        nx_ = a.tx_x[ic + aa + 1]; ny_ = a.tx_y[ic + aa + 1]; nz_ = a.tx_z[ic + aa + 1];
      }
      PairBwd g;
      pair_geometry<MONO, CORR>(rec, an, no_gain, g);
      domain |= (MODE == kModeBwd) && valid && !g.ok;
      const float fr0 = frac_cycles(g.L * a.k0);
      const float frd = frac_cycles(g.L * a.kd);
      float es, ec, zs, zc, vs_, vc_;
      __sincosf(kTwoPi * fr0, &es, &ec);
      sincospif(2.f * frd, &zs, &zc);             // w = e^{+j theta_d}
      sincospif(4.f * frd, &vs_, &vc_);           // v = w^2, accurate
      const f2x v = pk(vc_, vs_);
      const float4 *X4 = reinterpret_cast<const float4 *>(X + aa * NF);
      f2x he = 0ull, ho = 0ull;
#pragma unroll
      for (int k = H - 1; k >= 0; --k) {
        const float4 xv = X4[k];                  // (X[2k], X[2k+1])
        const float2 ve = upk(he), vo = upk(ho);
        const f2x te = ffma2(v, pk(ve.x, ve.x), pk(xv.x, xv.y));
        const f2x to = ffma2(v, pk(vo.x, vo.x), pk(xv.z, xv.w));
        const f2x v2 = pk(-vs_, vc_);
        he = ffma2(v2, pk(ve.y, ve.y), te);
        ho = ffma2(v2, pk(vo.y, vo.y), to);
      }
      const float2 ve = upk(he), vo = upk(ho);
      const float hr = ve.x + (zc * vo.x - zs * vo.y);
      const float hi = ve.y + (zc * vo.y + zs * vo.x);
      adj_accumulate<MODE>(g, ec, es, hr, hi, S1, S2, S3x, S3y, S3z);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);       // this warp is done with buffer b
  }
  if (domain) atomicOr(a.flags, 1u);
  if (valid) adj_store<MODE>(a, j, S1, S2, S3x, S3y, S3z);
}

// Backward (K3) at specialised bin counts: two samples per thread share every X load (LDS.64
// broadcast, half the shared-memory wavefronts of the one-sample kernels), single Horner chain per
// sample in straight-line code, one CTA barrier per stage of kAdjGA antennas.  Measured faster
// than the TMA-ring kernel for the backward, whose heavier per-pair epilogue (Eq. 5 gradient
// sums) favours sharing the stage across two samples.
template <int MODE, bool MONO, bool CORR, int NF>
__global__ void __launch_bounds__(kAdjThreads) k_adjoint_s2(AdjArgs a) {
  if (a.skip && a.skip->sel) return;
  constexpr int SPT = 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2 *X = reinterpret_cast<float2 *>(smem_raw);                      // [GA][n_f]
  AntD *ant = reinterpret_cast<AntD *>(smem_raw + a.smem_ant_off);       // [GA]
  const int tid = threadIdx.x;
  constexpr int nf = NF;
  const int64_t base = (int64_t)blockIdx.x * (kAdjThreads * SPT);
  const int64_t i_lo = (int64_t)blockIdx.y * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  const bool no_gain = a.no_gain;

  Rec rec[SPT];
  bool valid[SPT];
  float S1[SPT], S2[SPT], S3x[SPT], S3y[SPT], S3z[SPT];
#pragma unroll
  for (int s = 0; s < SPT; ++s) {
    const int64_t j = base + s * kAdjThreads + tid;
    valid[s] = j < a.n_s;
    if (MODE == kModeBwd) {
      if (valid[s]) rec[s] = a.rec[j];
      else { rec[s].x = rec[s].y = 0.0; rec[s].z = 1.0; rec[s].w = 0.f; rec[s].T = 0.f;
             rec[s].nx = rec[s].ny = 0.f; rec[s].nz = 1.f; rec[s].papr = 1.f; }
    } else {
      rec[s].x = valid[s] ? (double)a.qx[j] : 0.0;
      rec[s].y = valid[s] ? (double)a.qy[j] : 0.0;
      rec[s].z = valid[s] ? (double)a.qz[j] : 1.0;
      rec[s].w = 0.f; rec[s].T = 1.f; rec[s].nx = rec[s].ny = 0.f; rec[s].nz = 1.f;
      rec[s].papr = 1.f;
    }
    S1[s] = S2[s] = S3x[s] = S3y[s] = S3z[s] = 0.f;
  }
  bool domain = false;

  for (int64_t ic = i_lo; ic < i_hi; ic += kAdjGA) {
    const int ga = (int)min((int64_t)kAdjGA, i_hi - ic);
    __syncthreads();
    {   // stage X rows [ga][nf] (contiguous in global memory) and the antennas
      const float2 *src = a.X + ic * nf;
      const int n2 = ga * nf;
      for (int t = tid; t < n2; t += kAdjThreads) X[t] = src[t];
      for (int aa = tid; aa < ga; aa += kAdjThreads) {
        const int64_t ia = ic + aa;
        AntD d;
        d.x = a.tx_x[ia]; d.y = a.tx_y[ia]; d.z = a.tx_z[ia];
        if (MONO) { d.rx = d.x; d.ry = d.y; d.rz = d.z; }
        else { d.rx = a.rx_x[ia]; d.ry = a.rx_y[ia]; d.rz = a.rx_z[ia]; }
        d.ptx = a.phi_tx ? a.phi_tx[ia] : 1.f;
        d.prx = a.phi_rx ? a.phi_rx[ia] : (MONO ? d.ptx : 1.f);
        ant[aa] = d;
      }
    }
    __syncthreads();
    for (int aa = 0; aa < ga; ++aa) {
      const AntD an = ant[aa];   // (staged per stage, broadcast)
      PairBwd g[SPT];
      f2x w1[SPT], w2[SPT], h[SPT];
      float Er[SPT], Ei[SPT];
#pragma unroll
      for (int s = 0; s < SPT; ++s) {
        pair_geometry<MONO, CORR>(rec[s], an, no_gain, g[s]);
        domain |= (MODE == kModeBwd) && valid[s] && !g[s].ok;
        const float fr0 = frac_cycles(g[s].L * a.k0);
        const float frd = frac_cycles(g[s].L * a.kd);
        float es, ec, zs, zc;
        __sincosf(kTwoPi * fr0, &es, &ec);
        sincospif(2.f * frd, &zs, &zc);
        Er[s] = ec; Ei[s] = es;                    // E = e^{+j theta0}
        w1[s] = pkv(zc, zs);                       // w = e^{+j theta_d}
        w2[s] = pkv(-zs, zc);                      // (opaque: keeps ptxas from re-deriving it in the loop)
        h[s] = 0ull;
      }
      const float2 *Xa = X + aa * nf;
      // Horner from the top bin down: h = h w + X_m  (2 FFMA2 per complex step).  With NF > 0
      // the bin loop is straight-line code (no loop-carried register renames: in a rolled loop
      // ptxas spent ~25% extra FMA-pipe slots on IMAD.MOV / re-derived w2 at every back edge).
      {
#pragma unroll
        for (int m = NF - 1; m >= 0; --m) {
          const float2 xv = Xa[m];
          const f2x xm = pk(xv.x, xv.y);
#pragma unroll
          for (int s = 0; s < SPT; ++s) {
            const float2 hv = upk(h[s]);
            const f2x t = ffma2(pk(hv.x, hv.x), w1[s], xm);
            h[s] = ffma2(pk(hv.y, hv.y), w2[s], t);
          }
        }
      }
#pragma unroll
      for (int s = 0; s < SPT; ++s) {
        const float2 hv = upk(h[s]);
        if (MODE == kModeBwd) {
          const float R = Er[s] * hv.x - Ei[s] * hv.y;      // Re(E h)
          const float TT = g[s].Tt * g[s].Tr;
          const float Rg = R * g[s].gg;
          S1[s] = fmaf(Rg, TT, S1[s]);
          S2[s] = fmaf(Rg, g[s].Tr * g[s].chit + g[s].Tt * g[s].chir, S2[s]);
          const float Rc = R * g[s].gamma * TT;
          S3x[s] = fmaf(Rc, g[s].dgx, S3x[s]);
          S3y[s] = fmaf(Rc, g[s].dgy, S3y[s]);
          S3z[s] = fmaf(Rc, g[s].dgz, S3z[s]);
        } else {
          // M += E h
          S1[s] = fmaf(Er[s], hv.x, fmaf(-Ei[s], hv.y, S1[s]));
          S2[s] = fmaf(Er[s], hv.y, fmaf(Ei[s], hv.x, S2[s]));
        }
      }
    }
  }
  if (domain) atomicOr(a.flags, 1u);
#pragma unroll
  for (int s = 0; s < SPT; ++s) {
    const int64_t j = base + s * kAdjThreads + tid;
    if (!valid[s]) continue;
    if (MODE == kModeBwd) {
      float *P = a.out + (int64_t)blockIdx.y * 5 * a.n_s;     // [split][5][n_s]
      P[j] = S1[s];
      P[a.n_s + j] = S2[s];
      P[2 * a.n_s + j] = S3x[s];
      P[3 * a.n_s + j] = S3y[s];
      P[4 * a.n_s + j] = S3z[s];
    } else {
      float2 *M = reinterpret_cast<float2 *>(a.out) + (int64_t)blockIdx.y * a.n_s;
      M[j] = make_float2(S1[s], S2[s]);
    }
  }
}

// Generic bin count (or unaligned rows): one buffer of kAdjGA antennas, CTA barriers, rolled Horner.
// One (sample tile bx, antenna split by) per call.
template <int MODE, bool MONO, bool CORR>
__device__ __forceinline__ void adjoint_generic(const AdjArgs &a, unsigned char *smem_raw,
                                                int64_t bx, int64_t by) {
  float2 *X = reinterpret_cast<float2 *>(smem_raw);                      // [GA][n_f]
  AntD *ant = reinterpret_cast<AntD *>(smem_raw + a.smem_ant_off);       // [GA]
  const int tid = threadIdx.x;
  const int nf = a.n_f;
  const int64_t j = bx * kAdjThreads + tid;
  const int64_t i_lo = by * a.ants_per_split;
  const int64_t i_hi = min(a.n_a, i_lo + a.ants_per_split);
  const bool no_gain = a.no_gain;
  const bool valid = j < a.n_s;
  const Rec rec = load_point<MODE>(a, j, valid);
  float S1 = 0.f, S2 = 0.f, S3x = 0.f, S3y = 0.f, S3z = 0.f;
  bool domain = false;
  for (int64_t ic = i_lo; ic < i_hi; ic += kAdjGA) {
    const int ga = (int)min((int64_t)kAdjGA, i_hi - ic);
    __syncthreads();
    const float2 *src = a.X + ic * nf;
    for (int t = tid; t < ga * nf; t += kAdjThreads) X[t] = src[t];
    for (int aa = tid; aa < ga; aa += kAdjThreads) ant[aa] = load_ant<MONO>(a, ic + aa);
    __syncthreads();
    for (int aa = 0; aa < ga; ++aa) {
      const AntD an = ant[aa];
      PairBwd g;
      pair_geometry<MONO, CORR>(rec, an, no_gain, g);
      domain |= (MODE == kModeBwd) && valid && !g.ok;
      const float fr0 = frac_cycles(g.L * a.k0);
      const float frd = frac_cycles(g.L * a.kd);
      float es, ec, zs, zc;
      __sincosf(kTwoPi * fr0, &es, &ec);
      sincospif(2.f * frd, &zs, &zc);
      const f2x w = pk(zc, zs);                   // w = e^{+j theta_d}
      const f2x w2 = pkv(-zs, zc);
      const float2 *Xa = X + aa * nf;
      f2x h = 0ull;
#pragma unroll 4
      for (int m = nf - 1; m >= 0; --m) {
        const float2 xv = Xa[m];
        const float2 hv = upk(h);
        const f2x t = ffma2(w, pk(hv.x, hv.x), pk(xv.x, xv.y));
        h = ffma2(w2, pk(hv.y, hv.y), t);
      }
      const float2 hv = upk(h);
      adj_accumulate<MODE>(g, ec, es, hv.x, hv.y, S1, S2, S3x, S3y, S3z);
    }
  }
  if (domain) atomicOr(a.flags, 1u);
  if (valid) adj_store<MODE>(a, j, S1, S2, S3x, S3y, S3z, by);
}
// a.vgx > 0 (the r2 engine's direct fallback): a persistent grid walks the virtual grid
// vgx x vgy, so the launch that returns at once when the plan applied is one short wave
template <int MODE, bool MONO, bool CORR>
__global__ void __launch_bounds__(kAdjThreads) k_adjoint(AdjArgs a) {
  if (a.skip && a.skip->sel) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (a.vgx == 0) {
    adjoint_generic<MODE, MONO, CORR>(a, smem_raw, blockIdx.x, blockIdx.y);
    return;
  }
  const int64_t nv = (int64_t)a.vgx * a.vgy;
  for (int64_t v = blockIdx.x; v < nv; v += gridDim.x) {
    __syncthreads();                               // the previous virtual block's staging
    adjoint_generic<MODE, MONO, CORR>(a, smem_raw, v % a.vgx, v / a.vgx);
  }
}

// ================================================================================== K1' backward
// Per ray, reverse order.  With gT_k = w_k S2_k, Q_l = gT_{l+1} + (1-alpha_{l+1}) Q_{l+1} gives
// dL/d(1-alpha_l) = T_l Q_l without dividing by (1 - alpha) (exactly 0 at surface entries).
__global__ void k_blend_bwd(BlendBwdArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n_rays) return;
  const int nz = a.n_per_ray;
  const int64_t j0 = r * nz, ns = a.n_s;
  float Q = 0.f, carry = 0.f, gs = 0.f;
  float gT_next = 0.f, oma_next = 1.f;
  float f_next = 0.f, sm_next = 0.f;
  for (int l = nz - 1; l >= 0; --l) {
    const int64_t j = j0 + l;
    const float f = a.sdf[j];
    const float p = a.power[j], refl = a.refl[j];
    const Rec rec = a.rec[j];
    const float S1 = a.partials[j], S2 = a.partials[ns + j];
    const float S3x = a.partials[2 * ns + j], S3y = a.partials[3 * ns + j],
                S3z = a.partials[4 * ns + j];
    const bool has_next = l + 1 < nz;
    float alpha, oma;
    blend_step(a.s, f, f_next, has_next, alpha, oma);
    const float w = rec.w;
    a.g_power[j] = refl * alpha * S1;
    a.g_refl[j] = p * alpha * S1;
    a.g_nx[j] = w * S3x;
    a.g_ny[j] = w * S3y;
    a.g_nz[j] = w * S3z;
    if (has_next) Q = gT_next + oma_next * Q;
    const float dalpha = p * refl * S1 - rec.T * Q;
    const float sm = sig_minus(a.s, f);
    float gf_here = 0.f;
    if (has_next && alpha > 0.f) {
      const float c = dalpha * oma;
      gf_here = c * a.s * sm;
      carry -= c * a.s * sm_next;
      gs += c * (f * sm - f_next * sm_next);
    }
    if (has_next) a.g_sdf[j + 1] = carry;
    carry = gf_here;
    gT_next = w * S2;
    oma_next = oma;
    f_next = f;
    sm_next = sm;
  }
  a.g_sdf[j0] = carry;
  a.ds_part[r] = gs;
}

// Warp per ray, lane = sample, chunks of 32 samples from the ray's end: the recurrence
// Q_l = gT_{l+1} + (1 - alpha_{l+1}) Q_{l+1} is a suffix scan of affine maps over the lanes
// (Q_l = B_l + A_l Q_in, Q_in = the Q of the first sample of the later chunk), everything else is
// per sample or between neighbouring samples (shuffles; the later chunk's first sample carried).
// Same per-sample expressions as k_blend_bwd; the scan and the ray sum of d/ds associate
// differently (trees instead of folds).
__global__ void __launch_bounds__(256) k_blend_bwd_warp(BlendBwdArgs a) {
  const unsigned full = 0xffffffffu;
  const int lane = (int)(threadIdx.x & 31);
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= a.n_rays) return;                        // warp-uniform
  const int nz = a.n_per_ray;
  const int64_t j0 = r * nz, ns = a.n_s;
  float gs = 0.f;
  // carried from the later chunk (its first sample): Q, gT, 1 - alpha, gf_here
  float Qin = 0.f, gT_c = 0.f, oma_c = 1.f, gfh_c = 0.f;
  for (int k0 = ((nz - 1) / 32) * 32; k0 >= 0; k0 -= 32) {
    const int l = k0 + lane;
    const bool in = l < nz;
    const int64_t j = j0 + l;
    const bool has_next = in && l + 1 < nz;
    float f = 0.f, f_next = 0.f, p = 0.f, refl = 0.f, w = 0.f, Tl = 0.f;
    float S1 = 0.f, S2 = 0.f, S3x = 0.f, S3y = 0.f, S3z = 0.f;
    if (in) {
      f = a.sdf[j];
      f_next = has_next ? a.sdf[j + 1] : 0.f;
      p = a.power[j]; refl = a.refl[j];
      const Rec rec = a.rec[j];
      w = rec.w; Tl = rec.T;
      S1 = a.partials[j]; S2 = a.partials[ns + j];
      S3x = a.partials[2 * ns + j]; S3y = a.partials[3 * ns + j]; S3z = a.partials[4 * ns + j];
    }
    float alpha, oma;
    blend_step(a.s, f, f_next, has_next, alpha, oma);
    if (!in) { alpha = 0.f; oma = 1.f; }
    const float sm = in ? sig_minus(a.s, f) : 0.f;
    const float gT = w * S2;
    // neighbours: the next sample's gT, 1 - alpha, sigma(-s f) (lane 31: the later chunk's first)
    float gT_n = __shfl_down_sync(full, gT, 1), oma_n = __shfl_down_sync(full, oma, 1);
    float sm_n = __shfl_down_sync(full, sm, 1);
    if (lane == 31) { gT_n = gT_c; oma_n = oma_c; sm_n = has_next ? sig_minus(a.s, f_next) : 0.f; }
    // affine map of this sample: Q_l = b + aQ_{l+1}; the last sample of the ray (and lanes past
    // it) map everything to 0
    float A = has_next ? oma_n : 0.f, B = has_next ? gT_n : 0.f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const float A2 = __shfl_down_sync(full, A, d), B2 = __shfl_down_sync(full, B, d);
      if (lane + d < 32) { B = fmaf(A, B2, B); A *= A2; }
    }
    const float Q = fmaf(A, Qin, B);
    float c = 0.f, gf_here = 0.f;
    if (in) {
      a.g_power[j] = refl * alpha * S1;
      a.g_refl[j] = p * alpha * S1;
      a.g_nx[j] = w * S3x;
      a.g_ny[j] = w * S3y;
      a.g_nz[j] = w * S3z;
      const float dalpha = p * refl * S1 - Tl * Q;
      if (has_next && alpha > 0.f) {
        c = dalpha * oma;
        gf_here = c * a.s * sm;
        gs += c * (f * sm - f_next * sm_n);
      }
    }
    float gfh_n = __shfl_down_sync(full, gf_here, 1);
    if (lane == 31) gfh_n = gfh_c;
    if (has_next) a.g_sdf[j + 1] = gfh_n - c * a.s * sm_n;
    if (k0 == 0 && lane == 0) a.g_sdf[j0] = gf_here;
    Qin = __shfl_sync(full, Q, 0);
    gT_c = __shfl_sync(full, gT, 0);
    oma_c = __shfl_sync(full, oma, 0);
    gfh_c = __shfl_sync(full, gf_here, 0);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) gs += __shfl_xor_sync(full, gs, d);
  if (lane == 0) a.ds_part[r] = gs;
}

// ================================================================================== reductions
// out[k] = sum_{s < S} part[s * n + k], fixed order (float2 / float granularity via float4 loads)
__global__ void k_sum_splits(const float4 *__restrict__ part, int S, int64_t n4,
                             float4 *__restrict__ out, const ChebHdr *skip) {
  if (skip && skip->sel) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4;
       k += (int64_t)gridDim.x * blockDim.x) {
    float4 v = part[k];
    for (int s = 1; s < S; ++s) {
      const float4 u = part[(int64_t)s * n4 + k];
      v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
    }
    out[k] = v;
  }
}
__global__ void k_sum_splits_tail(const float *__restrict__ part, int S, int64_t n, int64_t lo,
                                  float *__restrict__ out, const ChebHdr *skip) {
  if (skip && skip->sel) return;
  const int64_t k = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  float v = part[k];
  for (int s = 1; s < S; ++s) v += part[(int64_t)s * n + k];
  out[k] = v;
}

// |M| for the filter (M already summed)
__global__ void k_abs(const float2 *__restrict__ m, int64_t n, float *__restrict__ p) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = m[k];
    p[k] = sqrtf(fmaf(v.x, v.x, v.y * v.y));
  }
}

// Block-level fixed-order sum of n floats into out[blockIdx.x] (grid-stride over the input)
__device__ __forceinline__ float block_sum(float v, float *sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.f;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_reduce_sum(const float *__restrict__ x, int64_t n, float *__restrict__ out) {
  __shared__ float sh[32];
  float v = 0.f;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    v += x[k];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

// ================================================================================== K6 loss
__global__ void k_loss_partial(const float2 *__restrict__ s, const float2 *__restrict__ y,
                               int64_t n, float2 *__restrict__ g, float *__restrict__ part) {
  __shared__ float sh[32];
  float v = 0.f;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const float2 a = s[k], b = y[k];
    const float2 d = make_float2(a.x - b.x, a.y - b.y);
    g[k] = d;
    v = fmaf(d.x, d.x, fmaf(d.y, d.y, v));
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = 0.5f * v;
}

// ================================================================================== launchers
static inline unsigned grid1(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// count of kernels this library launched (diagnostic for the bench's gpu_launches claim)
static unsigned long long g_launches = 0;
static inline cudaError_t counted(cudaError_t e, int n = 1) {
  if (e == cudaSuccess) __atomic_add_fetch(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED);
  return e;
}
unsigned long long launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }
void add_launches(int n) { __atomic_add_fetch(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

cudaError_t launch_blend(const BlendArgs &a, cudaStream_t st) {
  if (a.n_rays <= 0) return cudaSuccess;
  // warp per ray (default); RFR_K1=thread: the thread-per-ray form
  static int warp = -1;
  if (warp < 0) { const char *e = getenv("RFR_K1"); warp = (e && !strcmp(e, "thread")) ? 0 : 1; }
  if (warp) k_blend_warp<<<grid1(a.n_rays * 32, 256), 256, 0, st>>>(a);
  else k_blend<<<grid1(a.n_rays, 128), 128, 0, st>>>(a);
  return counted(cudaGetLastError());
}

template <int B, bool MONO, bool CORR, int KIND>
static cudaError_t fwd_t(const FwdArgs &a, dim3 grid, size_t smem, cudaStream_t st) {
  const bool full = a.nb_total % a.nb == 0;
  auto k = (B == 32 && full && a.nb == 8) ? k_trace_fwd<B, MONO, CORR, KIND, 8>
         : (B == 32 && full && a.nb == 16) ? k_trace_fwd<B, MONO, CORR, KIND, 16>
         : (B == 32 && full && a.nb == 4) ? k_trace_fwd<B, MONO, CORR, KIND, 4>
         : (B == 32 && full && a.nb == 2) ? k_trace_fwd<B, MONO, CORR, KIND, 2>
                                          : k_trace_fwd<B, MONO, CORR, KIND, 0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kFwdThreads, smem, st>>>(a);
  return counted(cudaGetLastError());
}

template <int B>
static cudaError_t fwd_b(const FwdArgs &a, bool mono, bool corr, int kind, dim3 g, size_t sm,
                         cudaStream_t st) {
  if (kind == kFwdMFAdj)
    return mono ? fwd_t<B, true, false, kFwdMFAdj>(a, g, sm, st)
                : fwd_t<B, false, false, kFwdMFAdj>(a, g, sm, st);
  if (mono)
    return corr ? fwd_t<B, true, true, kFwdTrace>(a, g, sm, st)
                : fwd_t<B, true, false, kFwdTrace>(a, g, sm, st);
  return corr ? fwd_t<B, false, true, kFwdTrace>(a, g, sm, st)
              : fwd_t<B, false, false, kFwdTrace>(a, g, sm, st);
}

cudaError_t launch_trace_fwd(const FwdArgs &a, int B, bool mono, bool corr, int kind, int n_splits,
                             cudaStream_t st) {
  const int64_t ta = (int64_t)kFwdWarps * a.taw;
  const int64_t n_tiles = (a.n_a + ta - 1) / ta;
  const int chunks = (a.nb_total + a.nb - 1) / a.nb;
  dim3 grid((unsigned)n_tiles, (unsigned)n_splits, (unsigned)chunks);
  const size_t smem = (size_t)kFwdWarps * a.warp_smem;
  switch (B) {
    case 8: return fwd_b<8>(a, mono, corr, kind, grid, smem, st);
    case 16: return fwd_b<16>(a, mono, corr, kind, grid, smem, st);
    case 32: return fwd_b<32>(a, mono, corr, kind, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

// K5 prep: c_q = (dL/dP_q) M_q / max(P_q, eps) packed with the fp64 query position.
__global__ void k_mf_adj_pack(const float *__restrict__ gP, const float2 *__restrict__ M,
                              const float *__restrict__ P, float eps, const float *__restrict__ qx,
                              const float *__restrict__ qy, const float *__restrict__ qz,
                              int64_t n, Rec *__restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float2 m = M[q];
    const float p = P ? P[q] : sqrtf(fmaf(m.x, m.x, m.y * m.y));
    // subgradient of |M| at M = 0 is 0: a query with P = 0 (zero signal) adds nothing, also for
    // eps = 0 (a 0/0 here would make every antenna's dL/ds NaN through the sum over queries)
    const float sc = p > 0.f ? gP[q] / fmaxf(p, eps) : 0.f;
    Rec r;
    r.x = (double)qx[q]; r.y = (double)qy[q]; r.z = (double)qz[q];
    r.w = sc * m.x;
    r.T = sc * m.y;
    r.nx = r.ny = 0.f; r.nz = 1.f; r.papr = 1.f;
    out[q] = r;
  }
}

cudaError_t launch_mf_adj_pack(const float *gP, const float *M, const float *P, float eps,
                               const float *qx, const float *qy, const float *qz, int64_t n,
                               Rec *out, int n_sm, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>(grid1(n, 256), (int64_t)n_sm * 8);
  k_mf_adj_pack<<<g, 256, 0, st>>>(gP, reinterpret_cast<const float2 *>(M), P, eps, qx, qy, qz, n,
                                   out);
  return counted(cudaGetLastError());
}

// ================================================================================== K7 heatmap loss
// Masked heatmap-domain L2 with the dynamic loss mask of P:L392-402:
// keep_q = !(H[cell_q] > thr_hi && P_q < ratio H[cell_q]) against the history BEFORE this call.
__global__ void k_heat_loss(const float *__restrict__ P, const float *__restrict__ Pgt, int64_t n,
                            const int *__restrict__ cell, const float *__restrict__ H,
                            float thr_hi, float ratio, float *__restrict__ gP,
                            unsigned char *__restrict__ mask, float *__restrict__ part) {
  __shared__ float sh[32];
  float v = 0.f;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float p = P[q];
    bool keep = true;
    if (H) {
      const float h = H[cell[q]];
      keep = !(h > thr_hi && p < ratio * h);
    }
    const float d = p - Pgt[q];
    gP[q] = keep ? d : 0.f;
    if (mask) mask[q] = keep ? 1 : 0;
    if (keep) v = fmaf(d, d, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = 0.5f * v;
}

// H[c] = max(H[c], P_q): order-independent (integer max on the bits of non-negative floats)
__global__ void k_heat_hist(const float *__restrict__ P, int64_t n, const int *__restrict__ cell,
                            float *H) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float p = P[q];
    if (p > 0.f) atomicMax(reinterpret_cast<int *>(H) + cell[q], __float_as_int(p));
  }
}

cudaError_t launch_heat_loss(const float *P, const float *Pgt, int64_t n, const int *cell, float *H,
                             float thr_hi, float ratio, float *gP, unsigned char *mask, float *tmp,
                             int tmp_n, float *loss, cudaStream_t st) {
  k_heat_loss<<<tmp_n, 256, 0, st>>>(P, Pgt, n, cell, H, thr_hi, ratio, gP, mask, tmp);
  k_reduce_sum<<<1, 256, 0, st>>>(tmp, tmp_n, loss);
  int launched = 2;
  if (H && n > 0) {
    k_heat_hist<<<tmp_n, 256, 0, st>>>(P, n, cell, H);
    ++launched;
  }
  return counted(cudaGetLastError(), launched);
}

template <int MODE, bool MONO, bool CORR>
static cudaError_t adj_t(const AdjArgs &a, dim3 grid, cudaStream_t st) {
  // bin counts with the TMA-ring / straight-line Horner specialisation (the configs' 64 / 128 /
  // 256 / 512); the bulk copies need 16-byte aligned rows
  const bool al = (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  const int nf = al ? a.n_f : 0;
  const bool spec = a.n_f == 256 || a.n_f == 512 || a.n_f == 128 || a.n_f == 64;
  if (a.gated) {
    // the r2 engine's direct fallback: the generic kernel on a persistent grid (one short wave
    // when the plan applied and it returns at once; the whole virtual grid when it did not)
    auto k = k_adjoint<MODE, MONO, CORR>;
    AdjArgs b = a;
    b.smem_ant_off = adj_smem_ant_off(a.n_f);
    b.vgx = grid.x;
    b.vgy = grid.y;
    const size_t smem = adj_smem_bytes(a.n_f);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kAdjThreads, smem) != cudaSuccess ||
        occ < 1)
      occ = 1;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
    const unsigned g = (unsigned)std::min<int64_t>((int64_t)grid.x * grid.y, (int64_t)sms * occ);
    k<<<g, kAdjThreads, smem, st>>>(b);
    return counted(cudaGetLastError());
  }
  if (MODE == kModeBwd && spec) {
    auto k = a.n_f == 256 ? k_adjoint_s2<MODE, MONO, CORR, 256>
           : a.n_f == 512 ? k_adjoint_s2<MODE, MONO, CORR, 512>
           : a.n_f == 128 ? k_adjoint_s2<MODE, MONO, CORR, 128>
                          : k_adjoint_s2<MODE, MONO, CORR, 64>;
    AdjArgs b = a;
    b.smem_ant_off = adj_smem_ant_off(a.n_f);
    const size_t smem = adj_smem_bytes(a.n_f);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 g2((unsigned)((a.n_s + 2 * kAdjThreads - 1) / (2 * kAdjThreads)), grid.y);
    k<<<g2, kAdjThreads, smem, st>>>(b);
    return counted(cudaGetLastError());
  }
  if (nf == 256 || nf == 512 || nf == 128 || nf == 64) {
    auto k = nf == 256 ? k_adjoint_tma<MODE, MONO, CORR, 256>
           : nf == 512 ? k_adjoint_tma<MODE, MONO, CORR, 512>
           : nf == 128 ? k_adjoint_tma<MODE, MONO, CORR, 128>
                       : k_adjoint_tma<MODE, MONO, CORR, 64>;
    const size_t smem = adj_tma_smem_bytes(nf);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kAdjThreads + 32, smem, st>>>(a);
    return counted(cudaGetLastError());
  }
  auto k = k_adjoint<MODE, MONO, CORR>;
  AdjArgs b = a;
  b.smem_ant_off = adj_smem_ant_off(a.n_f);
  const size_t smem = adj_smem_bytes(a.n_f);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kAdjThreads, smem, st>>>(b);
  return counted(cudaGetLastError());
}

// K3/K4 implementation: tensor-core factorisation (rfr_tc.cu) where the bin count allows, else
// SIMT.  RFR_ADJOINT=simt forces the SIMT kernels (A/B measurements).
static bool use_tensor_cores() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RFR_ADJOINT");
    v = (e && strcmp(e, "simt") == 0) ? 0 : 1;
  }
  return v == 1;
}

cudaError_t launch_adjoint(const AdjArgs &a, int mode, bool mono, bool corr, int n_splits,
                           cudaStream_t st) {
  const size_t bneed = (size_t)a.n_a * tc_bprep_bytes_per_ant(a.n_f, mode == kModeBoth ? 2 : 1);
  if (!a.gated && use_tensor_cores() && adjoint_tc_supported(a.n_f) && a.bprep && bneed <= a.bprep_cap &&
      (reinterpret_cast<uintptr_t>(a.X) & 15) == 0 &&
      (mode != kModeBoth || (reinterpret_cast<uintptr_t>(a.X2) & 15) == 0))
    return counted(launch_adjoint_tc(a, mode, mono, corr, n_splits, st));
  if (mode == kModeBoth) {          // SIMT: the two sweeps one after the other
    cudaError_t e = launch_adjoint(a, kModeBwd, mono, corr, n_splits, st);
    if (e != cudaSuccess) return e;
    AdjArgs f = a;
    f.X = a.X2;
    f.out = a.out2;
    return launch_adjoint(f, kModeFlt, mono, false, n_splits, st);
  }
  const int64_t per_cta = (int64_t)kAdjThreads;
  dim3 grid((unsigned)((a.n_s + per_cta - 1) / per_cta), (unsigned)n_splits);
  if (mode == kModeBwd) {
    if (mono) return corr ? adj_t<kModeBwd, true, true>(a, grid, st)
                          : adj_t<kModeBwd, true, false>(a, grid, st);
    return corr ? adj_t<kModeBwd, false, true>(a, grid, st)
                : adj_t<kModeBwd, false, false>(a, grid, st);
  }
  return mono ? adj_t<kModeFlt, true, false>(a, grid, st)
              : adj_t<kModeFlt, false, false>(a, grid, st);
}

cudaError_t launch_blend_bwd(const BlendBwdArgs &a, cudaStream_t st) {
  if (a.n_rays <= 0) return cudaSuccess;
  static int warp = -1;
  if (warp < 0) { const char *e = getenv("RFR_K1"); warp = (e && !strcmp(e, "thread")) ? 0 : 1; }
  if (warp) k_blend_bwd_warp<<<grid1(a.n_rays * 32, 256), 256, 0, st>>>(a);
  else k_blend_bwd<<<grid1(a.n_rays, 128), 128, 0, st>>>(a);
  return counted(cudaGetLastError());
}

cudaError_t launch_sum_splits(const float *part, int S, int64_t n, float *out, int n_sm,
                              cudaStream_t st, const ChebHdr *skip) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = n / 4;
  if (n4 > 0) {
    const unsigned g = (unsigned)std::min<int64_t>(grid1(n4, 256), (int64_t)n_sm * 8);
    // the float4 view of split s starts at s * n floats: needs n % 4 == 0 for alignment
    if (n % 4 == 0) {
      k_sum_splits<<<g, 256, 0, st>>>(reinterpret_cast<const float4 *>(part), S, n4,
                                      reinterpret_cast<float4 *>(out), skip);
      return counted(cudaGetLastError());
    }
  }
  k_sum_splits_tail<<<grid1(n, 256), 256, 0, st>>>(part, S, n, 0, out, skip);
  return counted(cudaGetLastError());
}

cudaError_t launch_abs(const float *m, int64_t n, float *p, int n_sm, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>(grid1(n, 256), (int64_t)n_sm * 8);
  k_abs<<<g, 256, 0, st>>>(reinterpret_cast<const float2 *>(m), n, p);
  return counted(cudaGetLastError());
}

cudaError_t launch_reduce_sum(const float *x, int64_t n, float *tmp, int tmp_n, float *out,
                              cudaStream_t st) {
  // two fixed-shape passes: tmp_n blocks -> 1 block
  k_reduce_sum<<<tmp_n, 256, 0, st>>>(x, n, tmp);
  k_reduce_sum<<<1, 256, 0, st>>>(tmp, tmp_n, out);
  return counted(cudaGetLastError(), 2);
}

cudaError_t launch_loss(const float *s, const float *y, int64_t n, float *g, float *tmp,
                        int tmp_n, float *loss, cudaStream_t st) {
  k_loss_partial<<<tmp_n, 256, 0, st>>>(reinterpret_cast<const float2 *>(s),
                                        reinterpret_cast<const float2 *>(y), n,
                                        reinterpret_cast<float2 *>(g), tmp);
  k_reduce_sum<<<1, 256, 0, st>>>(tmp, tmp_n, loss);
  return counted(cudaGetLastError(), 2);
}

}  // namespace rfr
