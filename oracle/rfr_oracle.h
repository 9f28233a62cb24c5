/*
 * rfr_oracle.h -- fp64 CPU oracle API.  TEST INFRASTRUCTURE ONLY (see rfr_oracle.c header).
 * Independent of include/librfr.h: the GPU path and the oracle share no declarations.
 */
#ifndef RFR_ORACLE_H
#define RFR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_FLAG_NO_GAIN 1u   /* drop the directive gain (w_o . w_r) -- E11 ablation */
#define ORC_DOMAIN 3          /* a pair closer than u_min = 1 mm was seen (contributes 0) */

typedef struct {
  const double *x, *y, *z, *sdf, *refl, *nx, *ny, *nz, *power;
  const double *phi_origin;     /* Phi_s at the primary-ray origin per sample; NULL => 1 */
  int64_t n_rays;
  int32_t n_per_ray;            /* samples ray-major, depth-sorted along w_p */
} orc_samples;

typedef struct {
  const double *tx_x, *tx_y, *tx_z;
  const double *rx_x, *rx_y, *rx_z;   /* NULL => monostatic */
  const double *phi_tx, *phi_rx;      /* Phi_s at the real-ray origins; NULL => 1 */
  int64_t n_ant;
} orc_antennas;

void orc_blend(const double *sdf, int64_t n_rays, int32_t n_per_ray, double s,
               double *alpha, double *oma, double *T);
void orc_pair(const orc_samples *S, int64_t j, double s, const orc_antennas *A, int64_t i,
              uint32_t flags, double *amp, double *tau);
int orc_forward(const orc_samples *S, double s, const orc_antennas *A, double f0, double df,
                int32_t n_freq, uint32_t flags, const int64_t *rows, int64_t n_rows,
                double *out /* [n_rows][n_freq][2] */);
int orc_filter(const double *signal /* [n_ant][n_freq][2] */, const orc_antennas *A, double f0,
               double df, int32_t n_freq, const double *qx, const double *qy, const double *qz,
               int64_t n_query, double *M /* [n_query][2] or NULL */, double *P /* [n_query] */);
double orc_loss(const double *s, const double *y, int64_t n_complex, double *G);
int orc_backward_partials(const double *G, const orc_samples *S, double s, const orc_antennas *A,
                          double f0, double df, int32_t n_freq, uint32_t flags,
                          const int64_t *samples, int64_t n_sel, double *partials /* [n_sel][5] */);
int orc_backward_finish(const double *partials, const orc_samples *S, double s,
                        const int64_t *rays, int64_t n_sel_rays, double *g_sdf, double *g_refl,
                        double *g_nx, double *g_ny, double *g_nz, double *g_power,
                        double *g_sharp_per_ray);

int orc_filter_backward(const double *grad_P, const double *M /* [n_query][2] */, const double *P,
                        double eps, const orc_antennas *A, double f0, double df, int32_t n_freq,
                        const double *qx, const double *qy, const double *qz, int64_t n_query,
                        const int64_t *rows, int64_t n_rows, double *out /* [n_rows][n_freq][2] */);
double orc_heatmap_loss(const double *P, const double *Pgt, int64_t n_query, const int32_t *cell,
                        double *H, double thr_hi, double ratio, double *grad_P, uint8_t *mask);

#ifdef __cplusplus
}
#endif
#endif
