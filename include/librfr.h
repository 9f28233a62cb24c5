/*
 * librfr.h -- C ABI of the B200-native lensless RF volumetric renderer (arxiv 2605.29097).
 *
 * The renderer's data-parallel hot path:
 *   K1  blend scan      NeuS discrete alpha / transmittance per primary ray
 *                       (App. B.1; lensless sharing L304, L311)
 *   K2  rfr_forward     Eq. 4 signal tracing with the Eq. 5 amplitude (L231-259), Alg. 2 [1] (L769-782)
 *   K4  rfr_filter      Eq. 3 matched filter (L182-187), Alg. 1 [1] (L734-748)
 *   K6  rfr_loss        signal-domain L2 residual (L211; BASELINE north_star "complex residual")
 *   K3  rfr_backward    App. A.5 tracing adjoint (L725-728), Alg. 2 [2] (L783-793), chained
 *   K1' (finish)        through Eq. 5 and the blend; origin Phi terms detached (L352)
 *
 * Conventions (all calls):
 *  - Every array pointer is a DEVICE pointer owned by the caller.  The library never allocates,
 *    frees or retains caller memory and never allocates on the hot path; its scratch space is the
 *    caller-provided rfr_workspace `ws` (size from rfr_workspace_size, alignment >= 256 bytes).
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream), returns
 *    an rfr_status, and never throws across the ABI.  Argument errors are reported before any
 *    launch; RFR_E_CUDA reports a launch failure (cudaGetLastError).
 *  - Complex arrays are interleaved float pairs (re, im), i.e. complex64, row-major.
 *  - Outputs are overwritten, never accumulated.  Results are bitwise reproducible for a fixed
 *    device and workspace size: no floating-point atomics; split reductions run in fixed order.
 *  - Multi-GPU: a rank passes its antenna slice (pointer offset + count) and the matching rows of
 *    signal / grad_signal.  rfr_forward then produces only local rows (no communication).  The
 *    backward and the filter expose a partial/finish split so the caller can all-reduce (sum) the
 *    partials with NCCL between the two calls; rfr_backward / rfr_filter are partial+finish.
 *  - Readings of passages the paper leaves open are listed in DESIGN.md ("Readings", Q1-Q26).
 */
#ifndef LIBRFR_H
#define LIBRFR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RFR_ABI_VERSION 2

typedef struct CUstream_st *rfr_stream_t; /* == cudaStream_t */

typedef enum {
  RFR_OK = 0,
  RFR_E_ARG = 1,      /* null required pointer, negative size, s <= 0, df <= 0, n_freq <= 0     */
  RFR_E_SHAPE = 2,    /* n_per_ray <= 0, workspace too small, sizes beyond the supported range   */
  RFR_E_DOMAIN = 3,   /* (rfr_poll_flags only) a pair closer than u_min = 1 mm contributed 0     */
  RFR_E_NUMERIC = 4,  /* (rfr_poll_flags only) non-finite input seen with RFR_CHECK_FINITE       */
  RFR_E_CUDA = 5,     /* a kernel launch failed                                                  */
  RFR_E_UNSUPPORTED = 6,
  RFR_E_NCCL = 7      /* an NCCL call of the multi-GPU path failed                               */
} rfr_status;

/* Opaque multi-GPU communicator (one NCCL communicator per rank).  NULL everywhere a
 * `const rfr_comm *` is taken means "single GPU, no communication". */
typedef struct rfr_comm rfr_comm;

/* option flags (rfr_opts.flags) */
#define RFR_NO_GAIN 1u       /* drop the directive gain (w_o . w_r): the E11 ablation   */
#define RFR_CHECK_FINITE 2u  /* K1 checks every sample field for NaN/Inf and raises RFR_FLAG_NUMERIC */
#define RFR_DIRECT 8u        /* run the direct kernels (K2 recurrence / tensor-core adjoint) instead
                                of the Chebyshev-moment path (DESIGN 5b); for A/B comparisons      */
#define RFR_REUSE_BLEND 4u   /* workspace already holds K1's records for THIS sample set and s
                                (set by the caller after rfr_forward on the same inputs); skips K1 */
#define RFR_R1 16u           /* monostatic calls: the r1 kernels (rfr_cheb.cu) instead of the r2
                                tiled engine (DESIGN 5e); for A/B comparisons                       */

/* device-side flags read back by rfr_poll_flags */
#define RFR_FLAG_DOMAIN 1u
#define RFR_FLAG_NUMERIC 2u

/* Uniform frequency grid f_m = f0 + m * df, m = 0 .. n_freq-1: the de-chirped IF samples of
 * Eq. 1 (an IF sample at time t sits at frequency f + k t).  Reading Q1. */
typedef struct {
  double f0_hz;
  double df_hz;
  int32_t n_freq;
} rfr_freq_grid;

/* Full-space samples along primary rays: SoA float32, ray-major, n_per_ray samples
 * per ray sorted by depth along w_p.  sdf = f(x) (inside negative, Q7), refl = reflectivity a,
 * (nx,ny,nz) = surface normal as supplied (grad f, the caller normalises; Q6), power = A'_tx.
 * phi_origin = Phi_s(f(x_apr)) at the sample's primary-ray origin (Eq. 7), NULL => 1. */
typedef struct {
  const float *x, *y, *z, *sdf, *refl, *nx, *ny, *nz, *power;
  const float *phi_origin;
  int64_t n_rays;
  int32_t n_per_ray;
} rfr_samples;

/* Antenna positions (TX and RX), SoA float32.  rx_* == NULL => monostatic, RX = TX.
 * phi_tx / phi_rx = Phi_s(f) at the real-ray origins (Eq. 7); NULL => 1.  A shard is a pointer
 * offset plus a count. */
typedef struct {
  const float *tx_x, *tx_y, *tx_z;
  const float *rx_x, *rx_y, *rx_z;
  const float *phi_tx, *phi_rx;
  int64_t n_ant;
} rfr_antennas;

/* Per-sample gradients, float32 [n_samples] each (overwritten).  sharpness -> one float. */
typedef struct {
  float *sdf, *refl, *nx, *ny, *nz, *power;
  float *sharpness;
} rfr_sample_grads;

typedef struct {
  uint32_t flags; /* RFR_NO_GAIN | RFR_CHECK_FINITE | RFR_REUSE_BLEND | RFR_DIRECT */
} rfr_opts;

/* Caller-owned scratch memory of the library.  `ptr` is DEVICE memory of `bytes` >=
 * rfr_workspace_size(n_samples, n_ant, n_freq, n_query), 256-byte aligned.  The four planning
 * dimensions are upper bounds for every call that uses the workspace (a call with more samples or
 * queries than planned returns RFR_E_SHAPE); the internal layout is a function of them only, so
 * the K1 records cached by rfr_forward (RFR_REUSE_BLEND) survive any filter / loss / adjoint call
 * on the same workspace.  One workspace must not be used by two calls running concurrently. */
typedef struct {
  void *ptr;
  size_t bytes;
  int64_t n_samples;
  int64_t n_ant;
  int32_t n_freq;
  int64_t n_query;
} rfr_workspace;

/* Workspace bytes needed for calls on sample sets of up to n_samples, n_ant antennas, n_freq bins
 * and n_query filter queries, on the current device (split counts depend on its SM count).
 * Pass 0 for a size that will not be used.  Host-only; no device work. */
rfr_status rfr_workspace_size(int64_t n_samples, int64_t n_ant, int32_t n_freq, int64_t n_query,
                              size_t *bytes);

/* Eq. 4 forward: signal[i][m] = sum_j A_ij exp(-j 2 pi f_m tau_ij), complex64 [n_ant][n_freq].
 * A_ij = p_j a_j alpha_j g_ij gamma_ij T_t,ij T_r,ij (Eq. 5 discretised with T^2 alpha, Q10);
 * tau_ij = (d_t + d_r)/c.  Runs K1 (unless RFR_REUSE_BLEND), then K2 and its split reduction. */
rfr_status rfr_forward(const rfr_samples *samples, float sharpness, const rfr_antennas *ants,
                       const rfr_freq_grid *grid, const rfr_opts *opts, float *signal,
                       const rfr_workspace *ws, rfr_stream_t stream);

/* Signal-domain L2 loss (K6): grad_signal = signal - target, *loss = 1/2 sum |signal - target|^2
 * (device float).  n_complex = n_ant * n_freq.  grad_signal may alias signal. */
rfr_status rfr_loss(const float *signal, const float *target, int64_t n_complex, float *grad_signal,
                    float *loss, const rfr_workspace *ws, rfr_stream_t stream);

/* Eq. 3 matched filter at n_query points: M_q = sum_i sum_m s(i,m) exp(+j 2 pi f_m tau_iq),
 * power[q] = |M_q| (float32), mf (optional, complex64 [n_query]) = M_q.  Sign as printed (Q2).
 * comm != NULL: `ants`/`signal` are this rank's antenna slice; the partial M is summed over the
 * ranks (ncclAllReduce on `stream`) before |M|, so every rank returns the full P and M. */
rfr_status rfr_filter(const float *signal, const rfr_antennas *ants, const rfr_freq_grid *grid,
                      const float *qx, const float *qy, const float *qz, int64_t n_query,
                      float *power, float *mf, const rfr_comm *comm, const rfr_workspace *ws,
                      rfr_stream_t stream);
/* Antenna-shard partial of the filter: mf (required) = this shard's complex M_q. */
rfr_status rfr_filter_partial(const float *signal, const rfr_antennas *ants,
                              const rfr_freq_grid *grid, const float *qx, const float *qy,
                              const float *qz, int64_t n_query, float *mf,
                              const rfr_workspace *ws, rfr_stream_t stream);
/* Query-sharded filter (the smaller collective when N_a N_f < N_q, e.g. c5): the ranks'
 * antenna slices (contiguous, sizes from the rfr.shard_range convention over n_ant_total) and their
 * signal rows are all-gathered into the workspace (one ncclBroadcast per rank in a group on
 * `stream`, 8 B x n_freq + 12 B per antenna), then this rank filters its query slice
 * [q_lo, q_hi) = shard_range(n_query, rank, nranks) over every antenna.  power / mf (optional) are
 * [q_hi - q_lo]: the heatmap stays query-sharded (no collective on M).  comm == NULL: the plain
 * filter over all n_query queries.  The workspace must be planned with n_ant >= n_ant_total.
 * RFR_E_SHAPE if ants->n_ant differs from this rank's slice size. */
rfr_status rfr_filter_gather(const float *signal, const rfr_antennas *ants, int64_t n_ant_total,
                             const rfr_freq_grid *grid, const float *qx, const float *qy,
                             const float *qz, int64_t n_query, float *power, float *mf,
                             const rfr_comm *comm, const rfr_workspace *ws, rfr_stream_t stream);
/* power[q] = |mf[q]| after the caller's all-reduce of mf. */
rfr_status rfr_filter_power(const float *mf, int64_t n_query, float *power, rfr_stream_t stream);

/* K5, matched-filter adjoint (NEXT-1; Eq. 3 backward, App. A.5, Alg. 1 [2]
 * P:L750-761).  For a loss that depends on the signal through the filter power P_q = |M_q|:
 *   grad_signal[i][m] = sum_q c_q exp(-j 2 pi f_m tau_iq),  c_q = grad_power[q] M_q / max(P_q, eps)
 * i.e. G = dL/dRe s + j dL/dIm s for the antenna rows of `ants` (complex64 [n_ant][n_freq],
 * overwritten).  The paper prints the weight as grad_power/P without M_q; that is not the
 * derivative of |M| (reading Q15).  mf = complex M_q [n_query] from rfr_filter on the same
 * signal and antennas; power = |M_q| [n_query] or NULL (recomputed from mf); eps >= 0 guards P = 0.
 * ants->phi_tx / phi_rx must be NULL (the filter has no transmittance).  Multi-GPU: each rank passes
 * its antenna slice; the output rows are local (no communication). */
rfr_status rfr_filter_backward(const float *grad_power, const float *mf, const float *power,
                               float eps, const rfr_antennas *ants, const rfr_freq_grid *grid,
                               const float *qx, const float *qy, const float *qz, int64_t n_query,
                               float *grad_signal, const rfr_workspace *ws, rfr_stream_t stream);

/* K7, heatmap-domain L2 with dynamic loss masking (masking P:L392-402, SPEC
 * S:L425-430).  keep_q = !(history[cell[q]] > thr_hi && power[q] < ratio * history[cell[q]])
 * evaluated against the history as it was before this call; grad_power[q] = keep_q (P_q - Pgt_q);
 * *loss (device float) = 1/2 sum_q keep_q (P_q - Pgt_q)^2; mask (optional, uint8 [n_query]) =
 * keep_q.  Then history[c] = max(history[c], P_q) over the queries of cell c (order-independent).
 * cell / history: both NULL (no masking, no history) or both given (int32 [n_query] cell index of
 * each query into the caller's history grid, float [n_cells] >= 0). */
rfr_status rfr_heatmap_loss(const float *power, const float *power_gt, int64_t n_query,
                            const int32_t *cell, float *history, float thr_hi, float ratio,
                            float *grad_power, uint8_t *mask, float *loss,
                            const rfr_workspace *ws, rfr_stream_t stream);

/* Backward: grad_signal = G = dL/dRe s + j dL/dIm s, complex64 [n_ant][n_freq] (Q14).
 * Writes dL/d{sdf, refl, n, power} per sample and dL/dsharpness.  = partial + finish.
 * comm != NULL: `ants`/`grad_signal` are this rank's antenna slice; the per-sample partials are
 * summed over the ranks (ncclAllReduce on `stream`) between K3 and K1', so every rank returns the
 * full gradients. */
rfr_status rfr_backward(const float *grad_signal, const rfr_samples *samples, float sharpness,
                        const rfr_antennas *ants, const rfr_freq_grid *grid, const rfr_opts *opts,
                        const rfr_sample_grads *out, const rfr_comm *comm,
                        const rfr_workspace *ws, rfr_stream_t stream);
/* K3: per-sample antenna sums of this antenna shard, partials float32 SoA [5][n_samples]:
 *   row 0  S1 = sum_i R_ij g gamma T_t T_r                 (= dL/dw_j, w = p a alpha)
 *   row 1  S2 = sum_i R_ij g gamma (T_r chi_t + T_t chi_r)  (dL/dT_j = w_j S2)
 *   rows 2-4 S3 = sum_i R_ij gamma T_t T_r dg/dn            (dL/dn_j = w_j S3)
 * with R_ij = Re sum_m G(i,m) exp(+j 2 pi f_m tau_ij).  Additive over antenna shards. */
rfr_status rfr_backward_partial(const float *grad_signal, const rfr_samples *samples,
                                float sharpness, const rfr_antennas *ants,
                                const rfr_freq_grid *grid, const rfr_opts *opts, float *partials,
                                const rfr_workspace *ws, rfr_stream_t stream);
/* K3 + K4 in ONE sweep over the (sample, antenna) pairs: the backward of rfr_backward (from
 * grad_signal) and the matched filter of rfr_filter (from signal) evaluated at the sample points
 * themselves (queries = samples).  Both are adjoint bin sums over the same pairs
 * (App. A.5 P:L725-728 and Eq. 3), so the fp64 pair geometry, the phasors and the
 * tensor-core A operand are computed once; results equal rfr_backward + rfr_filter(q = samples)
 * to rounding.  signal / grad_signal: [n_ant][n_freq] complex64 (this rank's rows); power:
 * [n_samples] |M| (required); mf: optional complex M [n_samples] (NULL = workspace scratch).  The
 * workspace must be planned with n_query >= n_samples.  comm: the partial M and the partial sums
 * are all-reduced before |M| and K1' (NULL = one GPU).  Errors as rfr_backward / rfr_filter. */
rfr_status rfr_backward_filter(const float *grad_signal, const float *signal,
                               const rfr_samples *samples, float sharpness,
                               const rfr_antennas *ants, const rfr_freq_grid *grid,
                               const rfr_opts *opts, const rfr_sample_grads *out, float *power,
                               float *mf, const rfr_comm *comm, const rfr_workspace *ws,
                               rfr_stream_t stream);
/* The sweep of rfr_backward_filter for one antenna shard, without communication or finish:
 * partials [5][n_samples] as rfr_backward_partial and mf [n_samples] complex64 the partial
 * matched filter M at the samples; both are additive over antenna shards.  The caller sums them
 * over shards and calls rfr_backward_finish / rfr_filter_power. */
rfr_status rfr_backward_filter_partial(const float *grad_signal, const float *signal,
                                       const rfr_samples *samples, float sharpness,
                                       const rfr_antennas *ants, const rfr_freq_grid *grid,
                                       const rfr_opts *opts, float *partials, float *mf,
                                       const rfr_workspace *ws, rfr_stream_t stream);
/* K1': chain the (all-reduced) partials through Eq. 5 and the blend of every ray. */
rfr_status rfr_backward_finish(const float *partials, const rfr_samples *samples, float sharpness,
                               const rfr_opts *opts, const rfr_sample_grads *out,
                               const rfr_workspace *ws, rfr_stream_t stream);

/* Multi-GPU communicator.  Rank 0 calls rfr_comm_unique_id (128 opaque bytes) and the caller
 * distributes the bytes to every rank; each rank then calls rfr_comm_init on its own device (it
 * blocks until all nranks ranks joined).  rfr_comm_destroy frees it.  Host calls; RFR_E_NCCL on an
 * NCCL failure. */
rfr_status rfr_comm_unique_id(void *id /* 128 bytes, written */);
rfr_status rfr_comm_init(const void *id, int nranks, int rank, rfr_comm **out);
rfr_status rfr_comm_destroy(rfr_comm *comm);

/* Read (and clear) the device flags RFR_FLAG_DOMAIN / RFR_FLAG_NUMERIC of the calls queued on
 * `stream` before this one: the read and the clear are ordered on that stream, then the call waits
 * for it (host-synchronous).  A flag raised by work on another stream is seen only if that work was
 * ordered before this call (events).  RFR_E_CUDA on a copy failure.  (ABI 2: takes the stream.) */
rfr_status rfr_poll_flags(const rfr_workspace *ws, uint32_t *flags, rfr_stream_t stream);
const char *rfr_status_string(rfr_status s);
int rfr_abi_version(void);
/* Diagnostic: number of kernels this library has launched in the process so far. */
uint64_t rfr_launch_count(void);

/* Diagnostics of the r2 tiled engine.
 * rfr_plan_state: the plan of the last engine call on `ws` (applied = 1: the engine ran; 0: the
 * direct fallback kernels ran) -- tile grid, moments per tile P, moments of the global expansion
 * Pg (0: direct node evaluation), points, and the tile / global delay half-spreads in cycles per
 * bin.  Host-synchronous on `stream` (a 4-byte flag and the plan header are copied back).
 * rfr_profile_enable(1) clears and starts per-sweep device timing: CUDA events are recorded on the
 * launching stream around each sweep of the engine (ids below); rfr_profile_read returns the
 * accumulated milliseconds and the number of timed launches of one sweep (it waits for the
 * recorded events).  rfr_profile_enable(0) stops.  Both: RFR_E_ARG for an unknown id / NULL. */
#define RFR_SWEEP_PLAN 0        /* box, grid choice, tile boxes, per-(tile, antenna) setup, tables */
#define RFR_SWEEP_SORT 1        /* stable counting sort of a point set into the tiles           */
#define RFR_SWEEP_PREP 2        /* global expansion + per-(tile, antenna) Horner coefficients     */
#define RFR_SWEEP_FILTER 3      /* k2_filter (a4)                                               */
#define RFR_SWEEP_BACKWARD 4    /* k2_bwd + split sum (a6)                                       */
#define RFR_SWEEP_FORWARD 5     /* k2_fwd: per-(tile, antenna) moments (a3 / K5)                 */
#define RFR_SWEEP_FORWARD_OUT 6 /* k2_fout: virtual sources -> global moments -> bins            */
typedef struct {
  int32_t applied, tiles, lx, ly, lz, P, Pg, n_points;
  double delta_t, delta_g;
} rfr_plan_info;
rfr_status rfr_plan_state(const rfr_workspace *ws, rfr_plan_info *out, rfr_stream_t stream);
rfr_status rfr_profile_enable(int on);
rfr_status rfr_profile_read(int32_t sweep, double *ms, uint64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* LIBRFR_H */
