// rfr_launch.h -- internal launch interface between the C ABI (librfr.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace rfr {

struct Rec;

// Chebyshev-moment forward (rfr_cheb.cu): device-side choice written by k_cheb_setup
struct ChebHdr {
  unsigned sel;                    // 1: the Chebyshev path runs, 0: the direct kernel K2 runs
  int P;                           // moments (16 / 32 / 48), 0 if not selected
  double delta;                    // half spread of the delays, cycles per bin step
  double inv;                      // (df / c) / delta: metres of path -> x in [-1, 1]
};


constexpr int kFwdThreads = 128;   // K2 CTA size (4 warps)
constexpr int kFwdMinBlocks = 3;   // K2 CTAs per SM (register budget ~170)
constexpr int kFwdWarps = kFwdThreads / 32;
constexpr int kFwdTJ = 16;         // samples per K2 warp tile (B = 32)
// K2 tile shape per bins-per-lane B: samples per warp tile and CTAs per SM (register budget)
__host__ __device__ constexpr int fwd_tj(int B) { return B == 32 ? 16 : 8; }
__host__ __device__ constexpr int fwd_min_blocks(int B) { return B == 32 ? 4 : 5; }
constexpr int kAdjThreads = 128;   // K3/K4 CTA size
constexpr int kAdjGA = 8;          // antennas per K3/K4 shared-memory stage
constexpr int kModeBwd = 0, kModeFlt = 1;
constexpr int kModeBoth = 2;       // K3 + K4 fused (tensor-core kernel only): X = G, X2 = signal
constexpr int kFwdTrace = 0, kFwdMFAdj = 1;  // K2 signal tracing / K5 matched-filter adjoint

struct BlendArgs {
  const float *x, *y, *z, *sdf, *refl, *nx, *ny, *nz, *power, *phi_origin;
  int64_t n_rays;
  int n_per_ray;
  float s;
  Rec *rec;
  unsigned char *aflag;            // [n_s] 1 where alpha != 0 (the backward's active samples), or NULL
  unsigned int *flags;
  bool check_finite;
};

struct ChebArgs {
  const Rec *rec;
  int64_t n_s;                     // points at rec (upper bound when n_dev is set)
  const int64_t *n_dev;            // device count of a compacted list, or NULL
  const int *idx;                  // adjoint over a compacted list: original index of each point
  int row;                         // single-row adjoint: which B row (0 = G / signal, 1 = signal)
  const float *tx_x, *tx_y, *tx_z, *rx_x, *rx_y, *rx_z, *phi_tx, *phi_rx;
  int64_t n_a;
  int n_f;
  double kd, kc;                   // df / c and the centre frequency f0 + (n_f / 2) df over c
  int64_t samples_per_split;
  double *lc;                      // [n_a] centre path length (m)
  ChebHdr *hdr;
  float2 *coef;                    // [n_f][pmax]
  int pmax;
  float2 *part;                    // [split][n_a][pmax] partial moments
  unsigned int *flags;
  bool no_gain;
  bool enable;                     // false: always the direct kernel
};

struct FwdArgs {
  const ChebHdr *skip;             // non-NULL: return at once when the Chebyshev path was chosen
  const Rec *rec;
  int64_t n_s;
  const float *tx_x, *tx_y, *tx_z, *rx_x, *rx_y, *rx_z, *phi_tx, *phi_rx;
  int64_t n_a;
  int n_f;
  int nb;                          // bin blocks of B bins per chunk (<= 32)
  int nb_total;                    // bin blocks over all n_f bins
  int taw;                         // antennas per warp = 32 / nb
  size_t warp_smem;                // shared-memory bytes per warp
  double k0, kd, kw, kchunk;       // cycles per metre of path: f0/c, df/c, B df/c, 32 B df/c
  int64_t samples_per_split;
  float2 *out;                     // [split][n_a][n_f]
  unsigned int *flags;
  bool no_gain;
};

struct AdjArgs {
  const Rec *rec;                  // K3: sample records
  const float *qx, *qy, *qz;       // K4: query points
  int64_t n_s;                     // samples or queries
  const float *tx_x, *tx_y, *tx_z, *rx_x, *rx_y, *rx_z, *phi_tx, *phi_rx;
  int64_t n_a;
  int n_f;
  double k0, kd;
  const float2 *X;                 // G (K3) or signal (K4), [n_a][n_f]
  int64_t ants_per_split;
  float *out;                      // K3: [split][5][n_s]; K4: [split][n_s] complex
  const float2 *X2;                // kModeBoth: the signal s, [n_a][n_f] (filter at the samples)
  float *out2;                     // kModeBoth: [split][n_s] complex partial M
  const ChebHdr *skip;      // non-NULL: return at once when the Chebyshev adjoint was chosen
  unsigned char *bprep;            // tensor-core path: per-antenna B^T images (hi | lo), or NULL
  size_t bprep_cap;                // bytes available at bprep
  size_t smem_ant_off;
  unsigned int *flags;
  bool no_gain;
  bool gated;                      // r2 fallback: generic SIMT kernel on a persistent grid
  unsigned vgx, vgy;               // (set by launch_adjoint) virtual grid of the persistent launch
};

struct BlendBwdArgs {
  const float *sdf, *refl, *power;
  const Rec *rec;
  const float *partials;           // [5][n_s] (summed over antennas and shards)
  int64_t n_rays, n_s;
  int n_per_ray;
  float s;
  float *g_sdf, *g_refl, *g_nx, *g_ny, *g_nz, *g_power;
  float *ds_part;                  // [n_rays]
};

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// K2 per-warp shared memory: anchors [TJ][32] float4, 2cos(theta) [TJ][32] float, antennas [32]
// (56 B each), double-buffered records [2][TJ] (48 B each)
inline size_t fwd_warp_smem(int B) {
  const int tj = fwd_tj(B);
  return align_up((size_t)tj * 32 * 20 + 32 * 56 + 2 * tj * 48, 128);
}
// K3/K4 staging.  TMA-ring kernel (specialised bin counts): kAdjStages buffers of
// adj_stage_ants(nf) antennas (8 KB of X rows each) + 2 mbarriers per stage.  Generic kernel:
// one buffer of kAdjGA antennas + their AntD records.
constexpr int kAdjStages = 4;
__host__ __device__ constexpr int adj_stage_ants(int nf) {
  return 8192 / (nf * 8) > 0 ? 8192 / (nf * 8) : 1;
}
inline size_t adj_tma_smem_bytes(int nf) {
  return (size_t)kAdjStages * adj_stage_ants(nf) * nf * 8 + 2 * kAdjStages * 8;
}
inline size_t adj_smem_ant_off(int n_f) { return align_up((size_t)kAdjGA * n_f * 8, 16); }
inline size_t adj_smem_bytes(int n_f) { return adj_smem_ant_off(n_f) + (size_t)kAdjGA * 56; }

unsigned long long launch_count();
void add_launches(int n);
cudaError_t launch_blend(const BlendArgs &a, cudaStream_t st);
cudaError_t launch_trace_fwd(const FwdArgs &a, int B, bool mono, bool corr, int kind, int n_splits,
                             cudaStream_t st);
cudaError_t launch_mf_adj_pack(const float *gP, const float *M, const float *P, float eps,
                               const float *qx, const float *qy, const float *qz, int64_t n,
                               Rec *out, int n_sm, cudaStream_t st);
cudaError_t launch_heat_loss(const float *P, const float *Pgt, int64_t n, const int *cell, float *H,
                             float thr_hi, float ratio, float *gP, unsigned char *mask, float *tmp,
                             int tmp_n, float *loss, cudaStream_t st);
cudaError_t launch_adjoint(const AdjArgs &a, int mode, bool mono, bool corr, int n_splits,
                           cudaStream_t st);
bool adjoint_tc_supported(int n_f);
// bytes of the prepared B^T data per antenna (nx X rows): fp16 hi and lo images, nx x n_f / 8
// rows of 32 fp16 columns each, plus the float2 of inverse row scales
inline size_t tc_bprep_bytes_per_ant(int n_f, int nx) { return (size_t)nx * 16 * n_f + 8; }
cudaError_t launch_adjoint_tc(const AdjArgs &a, int mode, bool mono, bool corr, int n_splits,
                              cudaStream_t st);
cudaError_t launch_blend_bwd(const BlendBwdArgs &a, cudaStream_t st);
cudaError_t launch_sum_splits(const float *part, int S, int64_t n, float *out, int n_sm,
                              cudaStream_t st, const ChebHdr *skip = nullptr);
constexpr int kChebPMax = 48;
int cheb_box_blocks();
cudaError_t launch_compact(const Rec *rec, int64_t n, bool corr, int *cnt, int64_t *total, Rec *out,
                           cudaStream_t st, const unsigned char *aflag = nullptr,
                           int *idx = nullptr);
int compact_blocks(int64_t n);
cudaError_t launch_pack_points(const float *x, const float *y, const float *z, int64_t n, Rec *out,
                               int n_sm, cudaStream_t st);
int cheb_threads();
cudaError_t launch_cheb_prepare(const ChebArgs &a, double *box_part, cudaStream_t st);
cudaError_t launch_cheb_fwd(const ChebArgs &a, bool mono, bool corr, int kind, int splits,
                            float2 *out, cudaStream_t st);
// adjoint (K3 / fused K3+K4) by Chebyshev moments: B_i[p] per antenna, then per pair P steps
// Tiled matched filter (rfr_cheb.cu, DESIGN 5d): the query points are sorted into kTiles spatial
// tiles of the points' bounding box; each (antenna, tile) gets its own delay centre, so the spread
// -- and the number of Chebyshev moments -- shrinks with the tile.
constexpr int kTileDim = 4;
constexpr int kTiles = kTileDim * kTileDim * kTileDim;
struct TileArgs {
  const float *qx, *qy, *qz;
  int64_t n;                       // points (upper bound when n_dev is set)
  const Rec *rec;                  // backward: the compacted records instead of qx / qy / qz
  const int64_t *n_dev;            // backward: device count of rec
  Rec *rs;                         // backward: sorted records
  const int *idx;                  // backward: original sample index of each compacted record
  int chunk;                       // points per CTA of the sweep (filter 512, backward 256)
  const float *tx_x, *tx_y, *tx_z, *rx_x, *rx_y, *rx_z;
  const float *phi_tx, *phi_rx;
  int64_t n_a;
  int n_f;
  double kd, kc;
  const ChebHdr *ghdr;             // the call's global choice: sel == 0 -> the direct kernels run
  const double *gbox;              // the points' bounding box [6] (k_cheb_setup)
  unsigned char *tile;             // [n] tile of each point
  int *bcnt;                       // [blocks][kTiles] counts -> block offsets
  int *tstart;                     // [kTiles + 1] first sorted position of each tile
  int *cstart;                     // [kTiles + 1] first CTA of each tile
  int *perm;                       // [n] sorted position -> original index
  float4 *qs;                      // [n] sorted positions
  double *tbox;                    // [kTiles][6]
  double *lc;                      // [kTiles][n_a] centre path lengths
  ChebHdr *hdr;                    // the tiled choice (P, delta)
  int *pub;                        // workspace header slot: the tiled P (diagnostics)
  unsigned long long *dmax;        // max half-spread (fp64 bits)
  float2 *coef;                    // [n_f][kChebPMax]
  float2 *bmom;                    // [n_a][kTiles][kChebPMax]
  const float2 *X;                 // the signal rows [n_a][n_f]
  float2 *out;                     // M partials [split][n]
  int64_t ants_per_split;
  float2 *fpart;                   // tiled K5: moments per (chunk CTA, antenna) [blocks][n_a][kChebPMax]
  float4 *tgeo;                    // monostatic tile-relative geometry [kTiles][n_a][2] (k_tile_setup)
};
cudaError_t launch_tiled_filter(const TileArgs &t, bool mono, int n_splits, cudaStream_t st);
// tiled backward over the compacted active samples (t.rec, t.n_dev, t.idx): partials of a
cudaError_t launch_tiled_backward(const TileArgs &t, const AdjArgs &a, bool mono, bool corr,
                                  int n_splits, cudaStream_t st);
cudaError_t launch_cheb_adj_prep_only(const ChebArgs &c, const AdjArgs &a, float2 *bmom,
                                      cudaStream_t st);
int tile_count_blocks(int64_t n);
// tiled K5 (the matched-filter adjoint, a forward-shaped sweep; DESIGN 6b) over the query records
// t.rec [t.n]: tile sort, per-(antenna, tile) centres and P, moments per (tile chunk, antenna) into
// t.fpart, then the bins of every antenna into out [n_a][n_f] (fixed-order sums throughout)
cudaError_t launch_tiled_mfadj(const TileArgs &t, bool mono, float2 *out, cudaStream_t st);
int64_t tile_fwd_chunk(int64_t n);        // points per CTA of the tiled K5 sweep
int64_t tile_fwd_blocks(int64_t n);       // upper bound of its chunk CTAs (fpart rows)
// matched filter only, four points per thread (row c.row of B); prep_nx as launch_cheb_adj
cudaError_t launch_cheb_flt(const ChebArgs &c, const AdjArgs &a, float2 *bmom, bool mono,
                            int n_splits, cudaStream_t st, int prep_nx = 0);
// prep_nx: 0 = prepare B for the mode's rows, 2 = prepare both rows (X, X2), -1 = B is ready
cudaError_t launch_cheb_adj(const ChebArgs &c, const AdjArgs &a, float2 *bmom, int mode,
                            bool mono, bool corr, int n_splits, cudaStream_t st, int prep_nx = 0);
cudaError_t launch_abs(const float *m, int64_t n, float *p, int n_sm, cudaStream_t st);
cudaError_t launch_reduce_sum(const float *x, int64_t n, float *tmp, int tmp_n, float *out,
                              cudaStream_t st);
cudaError_t launch_loss(const float *s, const float *y, int64_t n, float *g, float *tmp,
                        int tmp_n, float *loss, cudaStream_t st);

}  // namespace rfr
