/*
 * rfr_oracle.c -- plain fp64 CPU oracle of the lensless RF volumetric renderer (arxiv 2605.29097).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no source, header, table or helper with
 * the CUDA path (paper_2605_29097_b200/csrc); the two meet only through seeded input arrays.
 *
 * Every function evaluates the paper's definition directly, term by term, in double precision:
 * no recurrences, no tiling, no fusion.  Inputs arrive as float64 arrays (the Python wrapper widens
 * the float32 inputs exactly).  Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn.
 *
 *   O1 blend      NeuS discrete alpha + transmittance along each primary ray
 *                 ("same discretization as NeuS"; App. B.1)
 *   O2 pair       Eq. 2 / Eq. 5 amplitude and round-trip delay of one (sample, antenna) pair
 *                 (Eq. 7 correction P:L335-341)
 *   O3 forward    Eq. 4 signal tracing s(i,m) = sum_j A_ij exp(-j 2 pi f_m tau_ij)
 *                 (Alg. 2 [1] P:L769-782)
 *   O4 filter     Eq. 3 matched filter P(x) = | sum_i sum_m s(i,m) exp(+j 2 pi f_m tau_i(x)) |
 *                 (Alg. 1 [1] P:L734-748)
 *   O5 loss       L = 1/2 sum |s - y|^2, G = s - y (signal-domain L2, north_star)
 *   O6 backward   dL/dA = Re sum_i sum_m G e^{+j phi} (App. A.5, Alg. 2 [2] P:L783-793),
 *                 chained through Eq. 5 and the blend (origin Phi terms detached)
 *
 * Readings of silent / ambiguous passages follow DESIGN.md section "Readings".
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "rfr_oracle.h"

#define ORC_C 299792458.0            /* speed of light, m/s ("c is the speed of light") */
#define ORC_UMIN 1e-3                /* u_min domain guard, SPEC S:L109 (reading Q24) */

/* ---------------------------------------------------------------- O1: blend (per primary ray) */

/* log Phi_s(f), Phi_s(f) = 1/(1+exp(-s f)) the logistic CDF (reading Q7). */
static double log_Phi(double s, double f) {
  double x = -s * f;                                   /* log Phi = -softplus(-s f) */
  return x > 0 ? -(x + log1p(exp(-x))) : -log1p(exp(x));
}

/* sigma(-s f) = 1 - Phi_s(f) = d log Phi_s / d(s f) */
static double sig_minus(double s, double f) {
  double x = -s * f;
  return x >= 0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
}

/* alpha_k = max(1 - Phi_s(f_{k+1}) / Phi_s(f_k), 0)  (P:L811-818 discretised as in NeuS);
 * the ratio is evaluated as exp(log Phi_{k+1} - log Phi_k) so that it is finite when both Phi underflow.
 * Last sample of a ray: alpha = 0 (reading Q8).  T_0 = 1, T_{k+1} = T_k (1 - alpha_k)  (Q9). */
void orc_blend(const double *sdf, int64_t n_rays, int32_t n_per_ray, double s,
               double *alpha, double *oma, double *T) {
  for (int64_t r = 0; r < n_rays; ++r) {
    double t = 1.0;
    for (int32_t k = 0; k < n_per_ray; ++k) {
      int64_t j = r * n_per_ray + k;
      double a = 0.0, o = 1.0;
      if (k + 1 < n_per_ray) {
        double ratio_log = log_Phi(s, sdf[j + 1]) - log_Phi(s, sdf[j]);
        if (ratio_log < 0.0) {            /* 1 - ratio > 0 : the max(., 0) is inactive */
          a = -expm1(ratio_log);
          o = exp(ratio_log);
        }
      }
      if (alpha) alpha[j] = a;
      if (oma) oma[j] = o;
      if (T) T[j] = t;
      t *= o;
    }
  }
}

/* ---------------------------------------------------------------- O2: one (sample, antenna) pair */

typedef struct {
  double A;          /* Eq. 5 amplitude A_ij                                        */
  double tau;        /* round-trip delay (d_t + d_r)/c                              */
  double g, graw;    /* directive gain max(w_o . w_r, 0) and its unclamped value    */
  double gamma;      /* free-space amplitude decay 1/((4 pi)^2 d_t d_r)             */
  double Tt, Tr;     /* clamped lensless transmittances toward TX and RX            */
  int chi_t, chi_r;  /* 1 where the [0,1] clamp is inactive                         */
  double dg_dn[3];   /* d g_raw / d n                                               */
  int domain;        /* 1 if the pair is closer than u_min                          */
} orc_pair_t;

static void pair_eval(const orc_samples *S, int64_t j, double w_j, double T_j,
                      const orc_antennas *Ant, int64_t i, uint32_t flags, orc_pair_t *o) {
  double xj = S->x[j], yj = S->y[j], zj = S->z[j];
  double tx = Ant->tx_x[i], ty = Ant->tx_y[i], tz = Ant->tx_z[i];
  int bistatic = Ant->rx_x != NULL;
  double rx = bistatic ? Ant->rx_x[i] : tx, ry = bistatic ? Ant->rx_y[i] : ty,
         rz = bistatic ? Ant->rx_z[i] : tz;
  /* incoming direction w_i: transmitter -> point; w_r: point -> receiver */
  double dti[3] = {xj - tx, yj - ty, zj - tz};
  double dri[3] = {rx - xj, ry - yj, rz - zj};
  double d_t = sqrt(dti[0] * dti[0] + dti[1] * dti[1] + dti[2] * dti[2]);
  double d_r = sqrt(dri[0] * dri[0] + dri[1] * dri[1] + dri[2] * dri[2]);
  memset(o, 0, sizeof(*o));
  o->tau = (d_t + d_r) / ORC_C;                       /* Eq. 1 with d = d_t + d_r (A2) */
  if (d_t < ORC_UMIN || d_r < ORC_UMIN) { o->domain = 1; return; }
  double wi[3] = {dti[0] / d_t, dti[1] / d_t, dti[2] / d_t};
  double wr[3] = {dri[0] / d_r, dri[1] / d_r, dri[2] / d_r};
  double n[3] = {S->nx[j], S->ny[j], S->nz[j]};
  double n_wi = n[0] * wi[0] + n[1] * wi[1] + n[2] * wi[2];
  double n_wr = n[0] * wr[0] + n[1] * wr[1] + n[2] * wr[2];
  /* w_o = w_i - 2 (n . w_i) n;  gain = w_o . w_r, clamped >= 0 (Q4) */
  double wo[3] = {wi[0] - 2.0 * n_wi * n[0], wi[1] - 2.0 * n_wi * n[1], wi[2] - 2.0 * n_wi * n[2]};
  double graw = wo[0] * wr[0] + wo[1] * wr[1] + wo[2] * wr[2];
  if (flags & ORC_FLAG_NO_GAIN) {                     /* E11 ablation: drop (w_o . w_r) */
    o->graw = 1.0; o->g = 1.0;
  } else {
    o->graw = graw;
    o->g = graw > 0.0 ? graw : 0.0;
    if (graw > 0.0)                                   /* d/dn [w_i.w_r - 2 (n.w_i)(n.w_r)] */
      for (int c = 0; c < 3; ++c) o->dg_dn[c] = -2.0 * (n_wr * wi[c] + n_wi * wr[c]);
  }
  /* amplitude decay (4 pi u)^-2 per leg-pair ("divided from the received amplitude", Q3) */
  o->gamma = 1.0 / ((4.0 * M_PI) * (4.0 * M_PI) * d_t * d_r);
  /* Eq. 7 lensless transmittance correction as printed, clamped to [0,1] (Q11, Q12) */
  double papr = S->phi_origin ? S->phi_origin[j] : 1.0;
  double ptx = Ant->phi_tx ? Ant->phi_tx[i] : 1.0;
  double prx = Ant->phi_rx ? Ant->phi_rx[i] : (Ant->phi_tx && !bistatic ? ptx : 1.0);
  double tt = T_j + (ptx - papr), tr = T_j + (prx - papr);   /* = T - Phi_apr + Phi_ant */
  /* clamp derivative (Q25b): the upper clamp can only act when the correction is positive; with
     Phi_ant - Phi_apr <= 0, T_raw <= T_j <= 1 and the clamp is the identity on the feasible side */
  o->chi_t = (tt > 0.0 && (tt < 1.0 || ptx - papr <= 0.0));
  o->chi_r = (tr > 0.0 && (tr < 1.0 || prx - papr <= 0.0));
  o->Tt = tt < 0.0 ? 0.0 : (tt > 1.0 ? 1.0 : tt);
  o->Tr = tr < 0.0 ? 0.0 : (tr > 1.0 ? 1.0 : tr);
  /* Eq. 5 discretised: A = a * (w_o.w_r) * gamma * T^2 * alpha * A'_tx  (T^2 alpha, Q10) */
  o->A = w_j * o->g * o->gamma * o->Tt * o->Tr;
}

/* per-sample blend state for the whole sample set */
typedef struct { double *alpha, *oma, *T, *w; } blend_t;

static int blend_all(const orc_samples *S, double s, blend_t *b) {
  int64_t n = S->n_rays * (int64_t)S->n_per_ray;
  b->alpha = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  b->oma = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  b->T = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  b->w = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!b->alpha || !b->oma || !b->T || !b->w) return -1;
  orc_blend(S->sdf, S->n_rays, S->n_per_ray, s, b->alpha, b->oma, b->T);
  for (int64_t j = 0; j < n; ++j) b->w[j] = S->power[j] * S->refl[j] * b->alpha[j];
  return 0;
}
static void blend_free(blend_t *b) { free(b->alpha); free(b->oma); free(b->T); free(b->w); }

void orc_pair(const orc_samples *S, int64_t j, double s, const orc_antennas *Ant, int64_t i,
              uint32_t flags, double *A, double *tau) {
  blend_t b;
  if (blend_all(S, s, &b)) { *A = NAN; *tau = NAN; return; }
  orc_pair_t p;
  pair_eval(S, j, b.w[j], b.T[j], Ant, i, flags, &p);
  *A = p.A; *tau = p.tau;
  blend_free(&b);
}

/* ---------------------------------------------------------------- O3: forward (Eq. 4) */

/* Neumaier-compensated accumulator so the oracle's own summation error stays << 1e-10 */
typedef struct { double s, c; } ksum_t;
static inline void kadd(ksum_t *k, double v) {
  double t = k->s + v;
  if (fabs(k->s) >= fabs(v)) k->c += (k->s - t) + v; else k->c += (v - t) + k->s;
  k->s = t;
}

int orc_forward(const orc_samples *S, double s, const orc_antennas *Ant, double f0, double df,
                int32_t n_freq, uint32_t flags, const int64_t *rows, int64_t n_rows, double *out) {
  blend_t b;
  if (blend_all(S, s, &b)) return -1;
  int64_t n_s = S->n_rays * (int64_t)S->n_per_ray;
  int domain = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : domain)
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t i = rows ? rows[r] : r;
    ksum_t *acc = calloc((size_t)n_freq * 2, sizeof(ksum_t));
    for (int64_t j = 0; j < n_s; ++j) {
      orc_pair_t p;
      pair_eval(S, j, b.w[j], b.T[j], Ant, i, flags, &p);
      domain |= p.domain;
      for (int32_t m = 0; m < n_freq; ++m) {
        double f_m = f0 + (double)m * df;                 /* f_m = f0 + m df (reading Q1) */
        double phi = 2.0 * M_PI * f_m * p.tau;            /* exp(-j 2 pi f tau) */
        double sn, cs;
        sincos(phi, &sn, &cs);
        kadd(&acc[2 * m], p.A * cs);
        kadd(&acc[2 * m + 1], -p.A * sn);
      }
    }
    for (int32_t m = 0; m < n_freq; ++m) {
      out[(r * n_freq + m) * 2] = acc[2 * m].s + acc[2 * m].c;
      out[(r * n_freq + m) * 2 + 1] = acc[2 * m + 1].s + acc[2 * m + 1].c;
    }
    free(acc);
  }
  blend_free(&b);
  return domain ? ORC_DOMAIN : 0;
}

/* ---------------------------------------------------------------- O4: matched filter (Eq. 3) */

int orc_filter(const double *signal, const orc_antennas *Ant, double f0, double df, int32_t n_freq,
               const double *qx, const double *qy, const double *qz, int64_t n_query,
               double *M, double *P) {
  int bistatic = Ant->rx_x != NULL;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < n_query; ++q) {
    ksum_t re = {0, 0}, im = {0, 0};
    for (int64_t i = 0; i < Ant->n_ant; ++i) {
      double dt[3] = {qx[q] - Ant->tx_x[i], qy[q] - Ant->tx_y[i], qz[q] - Ant->tx_z[i]};
      double d_t = sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]);
      double d_r = d_t;
      if (bistatic) {
        double dr[3] = {qx[q] - Ant->rx_x[i], qy[q] - Ant->rx_y[i], qz[q] - Ant->rx_z[i]};
        d_r = sqrt(dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2]);
      }
      double tau = (d_t + d_r) / ORC_C;                    /* tau_i(x) round trip */
      for (int32_t m = 0; m < n_freq; ++m) {
        double f_m = f0 + (double)m * df;
        double phi = 2.0 * M_PI * f_m * tau;               /* exp(+j 2 pi f tau), P:L184 (Q2) */
        double sn, cs;
        sincos(phi, &sn, &cs);
        double sr = signal[(i * n_freq + m) * 2], si = signal[(i * n_freq + m) * 2 + 1];
        kadd(&re, sr * cs - si * sn);
        kadd(&im, sr * sn + si * cs);
      }
    }
    double mr = re.s + re.c, mi = im.s + im.c;
    if (M) { M[2 * q] = mr; M[2 * q + 1] = mi; }
    if (P) P[q] = sqrt(mr * mr + mi * mi);                 /* P = |M| */
  }
  return 0;
}

/* ---------------------------------------------------------------- O5: loss */

double orc_loss(const double *s, const double *y, int64_t n_complex, double *G) {
  ksum_t L = {0, 0};
  for (int64_t k = 0; k < 2 * n_complex; ++k) {
    double g = s[k] - y[k];
    if (G) G[k] = g;                                       /* G = dL/dRe s + j dL/dIm s (Q14) */
    kadd(&L, 0.5 * g * g);
  }
  return L.s + L.c;
}

/* ---------------------------------------------------------------- O6: backward */

/* Per-sample antenna sums:
 *   R_ij = Re sum_m G(i,m) exp(+j 2 pi f_m tau_ij)              (App. A.5; Q14)
 *   S1_j = sum_i R g gamma Tt Tr                                 = dL/dw_j
 *   S2_j = sum_i R g gamma (Tr chi_t + Tt chi_r)                 -> dL/dT_j = w_j S2_j
 *   S3_j = sum_i R gamma Tt Tr dg/dn                             -> dL/dn_j = w_j S3_j
 * for the listed samples, over the antennas in Ant with G rows [n_ant][n_freq] matching Ant. */
int orc_backward_partials(const double *G, const orc_samples *S, double s, const orc_antennas *Ant,
                          double f0, double df, int32_t n_freq, uint32_t flags,
                          const int64_t *samples, int64_t n_sel, double *partials /* [n_sel][5] */) {
  blend_t b;
  if (blend_all(S, s, &b)) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < n_sel; ++q) {
    int64_t j = samples ? samples[q] : q;
    double S1 = 0, S2 = 0, S3[3] = {0, 0, 0};
    for (int64_t i = 0; i < Ant->n_ant; ++i) {
      orc_pair_t p;
      pair_eval(S, j, b.w[j], b.T[j], Ant, i, flags, &p);
      if (p.domain) continue;
      double R = 0.0;
      for (int32_t m = 0; m < n_freq; ++m) {
        double f_m = f0 + (double)m * df;
        double phi = 2.0 * M_PI * f_m * p.tau;
        double sn, cs;
        sincos(phi, &sn, &cs);
        double gr = G[(i * n_freq + m) * 2], gi = G[(i * n_freq + m) * 2 + 1];
        R += gr * cs - gi * sn;                              /* Re(G e^{+j phi}) */
      }
      S1 += R * p.g * p.gamma * p.Tt * p.Tr;
      S2 += R * p.g * p.gamma * (p.Tr * p.chi_t + p.Tt * p.chi_r);
      for (int c = 0; c < 3; ++c) S3[c] += R * p.gamma * p.Tt * p.Tr * p.dg_dn[c];
    }
    double *o = partials + 5 * q;
    o[0] = S1; o[1] = S2; o[2] = S3[0]; o[3] = S3[1]; o[4] = S3[2];
  }
  blend_free(&b);
  return 0;
}

/* Chain the per-sample sums through Eq. 5 and the NeuS blend of each listed ray.
 * partials: [n_sel_rays * n_per_ray][5] in the listed rays' sample order.
 * Transmittance backward uses Q_l = sum_{k>l} gT_k prod_{l<m<k} (1-alpha_m), so that
 * dL/d(1-alpha_l) = T_l Q_l with no division by (1 - alpha) (exactly 0 at surface entries). */
int orc_backward_finish(const double *partials, const orc_samples *S, double s,
                        const int64_t *rays, int64_t n_sel_rays,
                        double *g_sdf, double *g_refl, double *g_nx, double *g_ny, double *g_nz,
                        double *g_power, double *g_sharp_per_ray) {
  int32_t nz = S->n_per_ray;
  double *gT = malloc(sizeof(double) * (size_t)(nz > 0 ? nz : 1));
  double *ga = malloc(sizeof(double) * (size_t)(nz > 0 ? nz : 1));
  double *al = malloc(sizeof(double) * (size_t)(nz > 0 ? nz : 1));
  double *om = malloc(sizeof(double) * (size_t)(nz > 0 ? nz : 1));
  double *T = malloc(sizeof(double) * (size_t)(nz > 0 ? nz : 1));
  if (!gT || !ga || !al || !om || !T) return -1;
  for (int64_t rr = 0; rr < n_sel_rays; ++rr) {
    int64_t r = rays ? rays[rr] : rr;
    const double *f = S->sdf + r * nz;
    orc_blend(f, 1, nz, s, al, om, T);
    for (int32_t k = 0; k < nz; ++k) {
      int64_t j = r * nz + k, q = rr * nz + k;
      const double *P = partials + 5 * q;
      double p = S->power[j], a = S->refl[j], w = p * a * al[k];
      g_power[q] = a * al[k] * P[0];                       /* dL/dp */
      g_refl[q] = p * al[k] * P[0];                        /* dL/da */
      g_nx[q] = w * P[2]; g_ny[q] = w * P[3]; g_nz[q] = w * P[4];
      ga[k] = p * a * P[0];                                /* direct dL/dalpha_k */
      gT[k] = w * P[1];                                    /* dL/dT_k */
    }
    double Q = 0.0, gs = 0.0;
    for (int32_t k = 0; k < nz; ++k) g_sdf[rr * nz + k] = 0.0;
    for (int32_t l = nz - 1; l >= 0; --l) {
      if (l < nz - 1) Q = gT[l + 1] + om[l + 1] * Q;       /* Q_l from Q_{l+1} */
      double dalpha = ga[l] - T[l] * Q;                    /* total dL/dalpha_l */
      if (l + 1 < nz && al[l] > 0.0) {                     /* active branch f_{l+1} < f_l */
        double sm0 = sig_minus(s, f[l]), sm1 = sig_minus(s, f[l + 1]);
        /* alpha = 1 - exp(logPhi(f_{l+1}) - logPhi(f_l)), d logPhi/df = s sigma(-s f) */
        g_sdf[rr * nz + l] += dalpha * om[l] * s * sm0;
        g_sdf[rr * nz + l + 1] -= dalpha * om[l] * s * sm1;
        gs += dalpha * om[l] * (f[l] * sm0 - f[l + 1] * sm1);
      }
    }
    if (g_sharp_per_ray) g_sharp_per_ray[rr] = gs;
  }
  free(gT); free(ga); free(al); free(om); free(T);
  return 0;
}

/* ---------------------------------------------------------------- O7: matched-filter adjoint */

/* dL/ds(i,m) for L depending on s only through P = |M| (Eq. 3):
 *   M_q = sum_i sum_m s(i,m) e^{+j phi_iqm},  phi_iqm = 2 pi f_m tau_iq
 *   G_M,q = dL/dRe M_q + j dL/dIm M_q = (dL/dP_q) M_q / max(P_q, eps)            (reading Q15)
 *   dL/ds(i,m) = sum_q G_M,q e^{-j phi_iqm}       (conjugate phase: M is C-linear in s)
 * The paper's App. A.5 and Alg. 1 [2] print (1/P) dL/dP e^{-j phi}, without the
 * M_q factor; that form is not the gradient of |M|.  Here M_q and P_q are inputs
 * (from orc_filter on the same signal), eps guards P = 0.
 * Output rows: the listed antenna rows (all if rows == NULL), complex [n_rows][n_freq][2]. */
int orc_filter_backward(const double *grad_P, const double *M, const double *P, double eps,
                        const orc_antennas *Ant, double f0, double df, int32_t n_freq,
                        const double *qx, const double *qy, const double *qz, int64_t n_query,
                        const int64_t *rows, int64_t n_rows, double *out) {
  int bistatic = Ant->rx_x != NULL;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t i = rows ? rows[r] : r;
    ksum_t *acc = calloc((size_t)n_freq * 2, sizeof(ksum_t));
    for (int64_t q = 0; q < n_query; ++q) {
      double den = P[q] > eps ? P[q] : eps;
      /* reading Q15b: at P_q = 0 the subgradient of |M| is taken as 0, so the query adds nothing
         (also for eps = 0, where M / max(P, eps) would be 0 / 0) */
      double sc = P[q] > 0.0 ? grad_P[q] / den : 0.0;
      double cr = sc * M[2 * q], ci = sc * M[2 * q + 1];                            /* G_M,q */
      double dt[3] = {qx[q] - Ant->tx_x[i], qy[q] - Ant->tx_y[i], qz[q] - Ant->tx_z[i]};
      double d_t = sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]);
      double d_r = d_t;
      if (bistatic) {
        double dr[3] = {qx[q] - Ant->rx_x[i], qy[q] - Ant->rx_y[i], qz[q] - Ant->rx_z[i]};
        d_r = sqrt(dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2]);
      }
      double tau = (d_t + d_r) / ORC_C;
      for (int32_t m = 0; m < n_freq; ++m) {
        double phi = 2.0 * M_PI * (f0 + (double)m * df) * tau;
        double sn, cs;
        sincos(phi, &sn, &cs);
        kadd(&acc[2 * m], cr * cs + ci * sn);              /* Re(G_M e^{-j phi}) */
        kadd(&acc[2 * m + 1], ci * cs - cr * sn);          /* Im(G_M e^{-j phi}) */
      }
    }
    for (int32_t m = 0; m < n_freq; ++m) {
      out[(r * n_freq + m) * 2] = acc[2 * m].s + acc[2 * m].c;
      out[(r * n_freq + m) * 2 + 1] = acc[2 * m + 1].s + acc[2 * m + 1].c;
    }
    free(acc);
  }
  return 0;
}

/* ---------------------------------------------------------------- O8: heatmap loss + masking */

/* Dynamic loss masking: a query q whose cell's historical maximum
 * rendered power H[cell_q] exceeds thr_hi while its current power P_q is below ratio * H[cell_q] is
 * excluded.  mask_q = 0 for excluded points, 1 otherwise (H before this iteration's update).
 * Heatmap-domain L2:  L = 1/2 sum_q mask_q (P_q - Pgt_q)^2,
 * dL/dP_q = mask_q (P_q - Pgt_q).  (Unnormalised; reading Q17b in DESIGN.md.)
 * Then H[c] = max(H[c], P_q) over the queries of cell c (H may be NULL: no masking, no history). */
double orc_heatmap_loss(const double *P, const double *Pgt, int64_t n_query, const int32_t *cell,
                        double *H, double thr_hi, double ratio, double *grad_P, uint8_t *mask) {
  ksum_t L = {0, 0};
  for (int64_t q = 0; q < n_query; ++q) {
    int keep = 1;
    if (H && cell) {
      double h = H[cell[q]];
      if (h > thr_hi && P[q] < ratio * h) keep = 0;
    }
    double d = P[q] - Pgt[q];
    if (mask) mask[q] = (uint8_t)keep;
    if (grad_P) grad_P[q] = keep ? d : 0.0;
    if (keep) kadd(&L, 0.5 * d * d);
  }
  if (H && cell)
    for (int64_t q = 0; q < n_query; ++q)
      if (P[q] > H[cell[q]]) H[cell[q]] = P[q];
  return L.s + L.c;
}
