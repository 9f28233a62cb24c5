// rfr_device.cuh -- device-side building blocks of the sm_100a renderer kernels.
//
// Packed-FP32 (f32x2) arithmetic, the per-(sample, antenna) geometry of Eq. 2 / Eq. 5, the NeuS
// blend step and the phase anchors.  The CPU oracle (oracle/) shares nothing with this file.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rfr_launch.h"

namespace rfr {

// ------------------------------------------------------------------------------ packed f32x2
// One 64-bit register pair holds a complex value (re, im).  FFMA2 / FADD2 issue one instruction
// for two FP32 lanes, which halves the issue pressure of the bin loops (the FP32 pipe, not the
// issue slot, becomes the bound).
typedef unsigned long long f2x;

__device__ __forceinline__ f2x pk(float x, float y) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
// same, but opaque to the optimiser (a loop-invariant pair stays one register pair)
__device__ __forceinline__ f2x pkv(float x, float y) {
  f2x r;
  asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 upk(f2x r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ f2x ffma2(f2x a, f2x b, f2x c) {
  f2x d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2x fadd2(f2x a, f2x b) {
  f2x d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// acc += x in place (register-stable accumulators: no MOV rotation at the loop end)
__device__ __forceinline__ void acc2(f2x &acc, f2x x) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(x));
}
__device__ __forceinline__ f2x fmul2(f2x a, f2x b) {
  f2x d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// complex product a*b = a.re*(b.re, b.im) + a.im*(-b.im, b.re)
__device__ __forceinline__ f2x cmul2(f2x a, f2x b) {
  float2 av = upk(a), bv = upk(b);
  return ffma2(pk(av.y, av.y), pk(-bv.y, bv.x), fmul2(pk(av.x, av.x), b));
}

// ------------------------------------------------------------------------------ data records
// K1 output per sample (48 B): fp64 position (phase geometry runs in fp64) + fp32 blend state.
struct __align__(16) Rec {
  double x, y, z;
  float w;      // p * a * alpha  (Eq. 5 weight without the per-pair factors)
  float T;      // primary-ray transmittance T_j
  float nx, ny, nz;
  float papr;   // Phi_s at the primary-ray origin (Eq. 7); 1 if not supplied
};
static_assert(sizeof(Rec) == 48, "Rec layout");

// antenna staged in shared memory
struct AntD {
  double x, y, z;      // transmitter
  double rx, ry, rz;   // receiver (== transmitter when monostatic)
  float ptx, prx;      // Phi_s at the real-ray origins (Eq. 7)
};

constexpr float kInv16Pi2 = 0.00633257759406206f;   // 1 / (4 pi)^2  (Q3)
constexpr double kUmin = 1e-3;                       // u_min guard (Q24)
constexpr float kTwoPi = 6.283185307179586f;

// fractional part of a cycle count, in [-0.5, 0.5], computed in fp64 then rounded to fp32
__device__ __forceinline__ float frac_cycles(double cyc) { return (float)(cyc - rint(cyc)); }

// ------------------------------------------------------------------------------ NeuS blend step
// log Phi_s(f1) - log Phi_s(f0) with log Phi_s(f) = -softplus(-s f), evaluated so that the large
// linear parts cancel exactly when both samples are deep inside (s*|f| ~ 1e3).
__device__ __forceinline__ float log_phi_ratio(float s, float f0, float f1) {
  float x0 = -s * f0, x1 = -s * f1;
  float hinge = (x0 >= 0.f && x1 >= 0.f) ? -s * (f0 - f1) : fmaxf(x0, 0.f) - fmaxf(x1, 0.f);
  float t0 = log1pf(__expf(-fabsf(x0))), t1 = log1pf(__expf(-fabsf(x1)));
  return hinge + (t0 - t1);
}
// sigma(-s f) = 1 - Phi_s(f)
__device__ __forceinline__ float sig_minus(float s, float f) {
  float x = -s * f;
  return x >= 0.f ? 1.f / (1.f + __expf(-x)) : __expf(x) / (1.f + __expf(x));
}
// alpha_k and (1 - alpha_k) for the interval (f_k, f_{k+1}); inactive (0, 1) unless f decreases.
__device__ __forceinline__ void blend_step(float s, float fk, float fk1, bool has_next, float &alpha,
                                           float &oma) {
  alpha = 0.f;
  oma = 1.f;
  if (has_next && fk1 < fk) {
    float d = fminf(log_phi_ratio(s, fk, fk1), 0.f);
    alpha = -expm1f(d);
    oma = __expf(d);
  }
}

// ------------------------------------------------------------------------------ pair geometry
struct PairFwd {
  float A;        // Eq. 5 amplitude A_ij
  double L;       // path length d_t + d_r (m): tau = L / c
};

struct PairBwd {
  float gg;           // g * gamma
  float gamma;
  float Tt, Tr;       // clamped transmittances
  float chit, chir;   // 1 where the clamp is inactive
  float dgx, dgy, dgz;// d g / d n (0 where clamped or RFR_NO_GAIN)
  double L;
  bool ok;            // false: closer than u_min (contributes 0)
};

// Distance in fp64 from its square: r0 = rsqrt in fp32 (MUFU, rel. error ~1e-7), then one Newton
// step in fp64, y + (d2 - y^2) r0 / 2 with y = d2 r0, which leaves a relative error ~1e-14 (enough
// for the phase: 1e-10 of a 0.5 m path is 5e-11 m) without the IEEE fp64 sqrt sequence and its slow
// path.  *inv = r0 ~ 1/d in fp32 for the directions and the path loss.
__device__ __forceinline__ double dist_from_sq(double d2, float *inv) {
  d2 = fmax(d2, 1e-24);            // coincident points stay finite (and fail the u_min guard)
  float r0;                        // MUFU.RSQ without the denormal rescaling (d2 >= 1e-24)
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"((float)d2));
  const double y = d2 * (double)r0;
  const double e = fma(-y, y, d2);
  *inv = r0;
  return fma(e, (double)(0.5f * r0), y);
}

// Same without the fp32 inverse: one fp32->fp64 conversion (the 1/2 r0 of the Newton step is an
// fp64 multiply instead of a second conversion)
__device__ __forceinline__ double dist_only(double d2) {
  d2 = fmax(d2, 1e-24);
  float r0;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"((float)d2));
  const double h = (double)r0;
  const double y = d2 * h;
  const double e = fma(-y, y, d2);
  return fma(e, 0.5 * h, y);
}

// Distance without leaving fp64: r0 = rsqrt.approx.f64 (MUFU.RSQ64H, ~2^-22) and one Newton
// step, ~1e-13 relative -- one XU instruction instead of two conversions and the fp32 rsqrt.
__device__ __forceinline__ double dist64(double d2) {
  d2 = fmax(d2, 1e-24);
  double r0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(d2));
  const double y = d2 * r0;
  const double e = fma(-y, y, d2);
  return fma(e, 0.5 * r0, y);
}
template <bool MONO>
__device__ __forceinline__ double pair_length64(const Rec &r, const AntD &a) {
  double dx = r.x - a.x, dy = r.y - a.y, dz = r.z - a.z;
  double dt = dist64(fma(dx, dx, fma(dy, dy, dz * dz)));
  if (MONO) return 2.0 * dt;
  double ex = a.rx - r.x, ey = a.ry - r.y, ez = a.rz - r.z;
  return dt + dist64(fma(ex, ex, fma(ey, ey, ez * ez)));
}

// Path length d_t + d_r in fp64 only (matched-filter adjoint: no amplitude factors, Eq. 3)
template <bool MONO>
__device__ __forceinline__ double pair_length(const Rec &r, const AntD &a) {
  double dx = r.x - a.x, dy = r.y - a.y, dz = r.z - a.z;
  double dt = dist_only(fma(dx, dx, fma(dy, dy, dz * dz)));
  if (MONO) return 2.0 * dt;
  double ex = a.rx - r.x, ey = a.ry - r.y, ez = a.rz - r.z;
  return dt + dist_only(fma(ex, ex, fma(ey, ey, ez * ez)));
}

// Shared geometry: distances in fp64 (phase precision), directions / gain / decay in fp32.
template <bool MONO, bool CORR>
__device__ __forceinline__ void pair_geometry(const Rec &r, const AntD &a, bool no_gain,
                                              PairBwd &o) {
  double dx = r.x - a.x, dy = r.y - a.y, dz = r.z - a.z;
  float it;
  double dt = dist_from_sq(fma(dx, dx, fma(dy, dy, dz * dz)), &it);
  double dr = dt;
  float wix, wiy, wiz, wrx, wry, wrz;
  wix = (float)dx * it; wiy = (float)dy * it; wiz = (float)dz * it;
  float ir = it;
  if (!MONO) {
    double ex = a.rx - r.x, ey = a.ry - r.y, ez = a.rz - r.z;
    dr = dist_from_sq(fma(ex, ex, fma(ey, ey, ez * ez)), &ir);
    wrx = (float)ex * ir; wry = (float)ey * ir; wrz = (float)ez * ir;
  } else {
    wrx = -wix; wry = -wiy; wrz = -wiz;
  }
  o.L = dt + dr;
  o.ok = (dt >= kUmin) && (dr >= kUmin);
  // gain: w_o . w_r with w_o = w_i - 2 (n.w_i) n, clamped (Q4)
  float nwi = r.nx * wix + r.ny * wiy + r.nz * wiz;
  float nwr = r.nx * wrx + r.ny * wry + r.nz * wrz;
  float graw = (wix * wrx + wiy * wry + wiz * wrz) - 2.f * nwi * nwr;
  float g;
  if (no_gain) {
    g = 1.f; o.dgx = o.dgy = o.dgz = 0.f;
  } else if (graw > 0.f) {
    g = graw;
    o.dgx = -2.f * (nwr * wix + nwi * wrx);
    o.dgy = -2.f * (nwr * wiy + nwi * wry);
    o.dgz = -2.f * (nwr * wiz + nwi * wrz);
  } else {
    g = 0.f; o.dgx = o.dgy = o.dgz = 0.f;
  }
  o.gamma = kInv16Pi2 * it * ir;                     // 1/((4 pi)^2 d_t d_r)
  o.gg = g * o.gamma;
  if (CORR) {                                        // Eq. 7 as printed, clamped (Q11, Q12)
    float tt = r.T + (a.ptx - r.papr), tr = r.T + (a.prx - r.papr);   // T - Phi_apr + Phi_ant
    // clamp derivative (Q25b): the upper clamp acts only for a positive correction
    o.chit = (tt > 0.f && (tt < 1.f || a.ptx - r.papr <= 0.f)) ? 1.f : 0.f;
    o.chir = (tr > 0.f && (tr < 1.f || a.prx - r.papr <= 0.f)) ? 1.f : 0.f;
    o.Tt = fminf(fmaxf(tt, 0.f), 1.f);
    o.Tr = fminf(fmaxf(tr, 0.f), 1.f);
  } else {
    o.Tt = o.Tr = r.T;
    // no correction: T_ij = T_j <= 1 and the clamp is the identity on [0, 1] (Q25b); T_j rounds
    // to 1 in fp32 behind faint (alpha ~ 1e-14) intervals, so T < 1 must not gate the derivative
    float chi = r.T > 0.f ? 1.f : 0.f;
    o.chit = o.chir = chi;
  }
  if (!o.ok) { o.gg = 0.f; o.gamma = 0.f; }
}

// ------------------------------------------------------------------------------ async copies
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }


// ---- mbarrier / bulk-copy (TMA engine) helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
// Wait for the phase with the given parity to complete.  Plain try_wait (the hardware may
// suspend the thread for a short, system-defined time per probe).  A suspend-time hint was tried
// and made things worse: ptxas turns it into NANOSLEEP up to the hint after a failed probe.
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  } while (!ok);
}
// Same with a suspend-time hint (ns): for a producer that is expected to wait long (TMA ring).
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long *bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a), "r"(parity), "r"(20000u) : "memory");
  } while (!ok);
}
// contiguous global -> shared copy by the bulk-copy (TMA) engine, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}


// ------------------------------------------------------------------------------ K3/K4 shared pieces
template <bool MONO>
__device__ __forceinline__ AntD load_ant(const AdjArgs &a, int64_t ia) {
  AntD d;
  d.x = a.tx_x[ia]; d.y = a.tx_y[ia]; d.z = a.tx_z[ia];
  if (MONO) { d.rx = d.x; d.ry = d.y; d.rz = d.z; }
  else { d.rx = a.rx_x[ia]; d.ry = a.rx_y[ia]; d.rz = a.rx_z[ia]; }
  d.ptx = a.phi_tx ? a.phi_tx[ia] : 1.f;
  d.prx = a.phi_rx ? a.phi_rx[ia] : (MONO ? d.ptx : 1.f);
  return d;
}

// fp32 antenna record as stored (prefetched in registers), widened to AntD at use
struct AntF {
  float x, y, z, rx, ry, rz, ptx, prx;
};
template <bool MONO, typename Args>
__device__ __forceinline__ AntF load_antf(const Args &a, int64_t ia) {
  AntF d;
  d.x = a.tx_x[ia]; d.y = a.tx_y[ia]; d.z = a.tx_z[ia];
  if (MONO) { d.rx = d.ry = d.rz = 0.f; }
  else { d.rx = a.rx_x[ia]; d.ry = a.rx_y[ia]; d.rz = a.rx_z[ia]; }
  d.ptx = a.phi_tx ? a.phi_tx[ia] : 1.f;
  d.prx = a.phi_rx ? a.phi_rx[ia] : (MONO ? d.ptx : 1.f);
  return d;
}
template <bool MONO>
__device__ __forceinline__ AntD widen_ant(const AntF &f) {
  AntD d;
  d.x = f.x; d.y = f.y; d.z = f.z;
  if (MONO) { d.rx = d.x; d.ry = d.y; d.rz = d.z; }
  else { d.rx = f.rx; d.ry = f.ry; d.rz = f.rz; }
  d.ptx = f.ptx; d.prx = f.prx;
  return d;
}

template <int MODE>
__device__ __forceinline__ Rec load_point(const AdjArgs &a, int64_t j, bool valid) {
  Rec rec;
  if (MODE == kModeBwd) {
    if (valid) rec = a.rec[j];
    else { rec.x = rec.y = 0.0; rec.z = 1.0; rec.w = 0.f; rec.T = 0.f;
           rec.nx = rec.ny = 0.f; rec.nz = 1.f; rec.papr = 1.f; }
  } else {
    rec.x = valid ? (double)a.qx[j] : 0.0;
    rec.y = valid ? (double)a.qy[j] : 0.0;
    rec.z = valid ? (double)a.qz[j] : 1.0;
    rec.w = 0.f; rec.T = 1.f; rec.nx = rec.ny = 0.f; rec.nz = 1.f; rec.papr = 1.f;
  }
  return rec;
}

// Per-pair epilogue shared by both K3/K4 kernels: R = Re(E h) into the Eq. 5 sums, or M += E h.
template <int MODE>
__device__ __forceinline__ void adj_accumulate(const PairBwd &g, float ec, float es, float hr,
                                               float hi, float &S1, float &S2, float &S3x,
                                               float &S3y, float &S3z) {
  if (MODE == kModeBwd) {
    const float R = ec * hr - es * hi;            // Re(E h), E = e^{+j theta0}
    const float TT = g.Tt * g.Tr;
    const float Rg = R * g.gg;
    S1 = fmaf(Rg, TT, S1);
    S2 = fmaf(Rg, g.Tr * g.chit + g.Tt * g.chir, S2);
    const float Rc = R * g.gamma * TT;
    S3x = fmaf(Rc, g.dgx, S3x);
    S3y = fmaf(Rc, g.dgy, S3y);
    S3z = fmaf(Rc, g.dgz, S3z);
  } else {                                        // M += E h
    S1 = fmaf(ec, hr, fmaf(-es, hi, S1));
    S2 = fmaf(ec, hi, fmaf(es, hr, S2));
  }
}

template <int MODE>
__device__ __forceinline__ void adj_store(const AdjArgs &a, int64_t j, float S1, float S2,
                                          float S3x, float S3y, float S3z, int64_t split = -1) {
  if (split < 0) split = blockIdx.y;                         // the launch's antenna split
  if (MODE == kModeBwd) {
    float *P = a.out + split * 5 * a.n_s;                    // [split][5][n_s]
    P[j] = S1;
    P[a.n_s + j] = S2;
    P[2 * a.n_s + j] = S3x;
    P[3 * a.n_s + j] = S3y;
    P[4 * a.n_s + j] = S3z;
  } else {
    float2 *M = reinterpret_cast<float2 *>(a.out) + split * a.n_s;
    M[j] = make_float2(S1, S2);
  }
}

}  // namespace rfr
