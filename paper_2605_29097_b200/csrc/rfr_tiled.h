// rfr_tiled.h -- internal interface of the r2 tiled engine (rfr_tiled.cu).
//
// Monostatic calls without the Eq. 7 correction (every benchmark configuration) run through this
// engine; bistatic / corrected calls keep the r1 kernels (rfr_cheb.cu, rfr_kernels.cu).
//
// A PLAN is built on the device for one point set: the points' bounding box, an anisotropic grid of
// Lx x Ly x Lz spatial tiles chosen by a cost model (at most kT2Max tiles, at most kT2PMax moments
// per tile), a stable counting sort of the points by tile, the tiles' tight boxes, per (tile,
// antenna) the delay centre and the fp32 tile-relative geometry, the tiles' common half-spread
// delta_t (-> P moments) and per antenna a global delay interval covering all its tiles (-> Pg
// moments of one global Jacobi-Anger / Chebyshev expansion).  Any other point set can then be
// sorted into the same grid (the fused call's active samples).
//
// Sweeps (one persistent launch each, P read on the device):
//   filter / backward: thread = point, loop over antennas; the bin sum of every pair is a degree
//     P-1 polynomial in the tile coordinate x, evaluated by Horner from per-(antenna, tile) monomial
//     coefficients (one FFMA2 per coefficient and point);
//   forward / K5: thread = antenna, loop over the tile's points; per-(antenna, tile) Chebyshev
//     moments, turned into bins through P virtual sources per tile and the global expansion.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rfr_launch.h"

namespace rfr {

constexpr int kT2Max = 512;            // tiles per plan
constexpr int kT2PMax = 16;            // moments per tile
constexpr int kT2TP = 6144;            // plans keep T * P <= kT2TP (coefficient storage)
constexpr int kT2PgMax = 48;           // moments of the global expansion
constexpr int kT2BoxBlocks = 128;
constexpr int kT2SortBlock = 1024;     // points per counting-sort block
constexpr int kT2FltChunk = 512;       // points per filter work item (4 per thread)
int t2_filter_chunk();                 // 512, or 1024 (8 points per thread) with RFR_T2SPT=8
int t2_backward_chunk();               // 256, or 512 (4 points per thread) with RFR_T2BPT=4
constexpr int kT2BwdChunk = 256;       // points per backward work item (2 per thread)
constexpr int kT2FwdAnts = 128;        // antennas per forward work item

// plan header (device, in the workspace)
struct T2Plan {
  float gbox[6];                       // bounding box of the plan's points
  int L[3];                            // tile grid
  int T;                               // tiles
  int P;                               // moments per tile, 0: the engine does not apply
  int Pg;                              // moments of the global expansion, 0: direct nodes
  int n_pts;                           // points of the plan
  double delta_t, inv_t;               // tile half-spread (cycles per bin), kd / delta_t
  double delta_g, inv_g;               // global half-spread, kd / delta_g
  unsigned long long dmax_bits;        // atomicMax scratch (fp64 bits): tile half-spread (m)
  unsigned long long gmax_bits;        // global half-spread (m)
  unsigned long long umin_bits;        // atomicMin: closest (tile box, antenna) distance (m)
  unsigned ctr[4];                     // work counters of the persistent sweeps (zeroed per launch)
};
static_assert(sizeof(T2Plan) <= 256, "the plan header region is 256 bytes");

// a sorted view of a point set in a plan's grid (sort output)
struct T2Sorted {
  int *tstart;                         // [kT2Max + 1] first sorted position of each tile
  int *cstart;                         // [kT2Max + 1] first work item of each tile
  int *n_items;                        // device: work items (chunks) of the sweep
  int *torder;                         // [kT2Max] occupied tiles, most points first (k2_order)
  int *n_occ;                          // device: occupied tiles
  int chunk;                           // points per work item
  int *perm;                           // [n] sorted position -> source index
  float4 *pos;                         // [n] sorted positions (x, y, z, w)
  float4 *aux;                         // [n] sorted (nx, ny, nz, T) for records, else unused
  unsigned short *tile;                // [n] tile of each source point (scratch)
  int *bcnt;                           // [blocks][kT2Max] per-block counts -> offsets (scratch)
};

// a point set: float arrays (queries) or records (Rec) with an optional device count
struct T2Points {
  const float *qx, *qy, *qz;
  const Rec *rec;
  const int64_t *n_dev;
  int64_t n;                           // host upper bound (the count when n_dev is NULL)
};

struct T2Args {
  T2Plan *plan;
  float *box_part;                     // [kT2BoxBlocks][6]
  const float *tx_x, *tx_y, *tx_z;     // monostatic antennas
  int64_t n_a;
  int n_f;
  double kd, kc;                       // df / c, f_c / c with f_c = f0 + (n_f / 2) df
  float *tbox;                         // [kT2Max][6] tight tile boxes
  double *lc;                          // [kT2Max][n_a] centre path length of (tile, antenna)
  double *lct;                         // [n_a][kT2Max] the same, antenna-major (k2_fout)
  float4 *tgeo;                        // [kT2Max][n_a][2] tile-relative geometry
  float4 *tgeof;                       // [kT2Max][n_a][2] the filter's image of it (k2_geofix)
  int dyn;                             // backward sweep: work items from plan->ctr[2]
  double *lg;                          // [n_a][3]: global centre, min / max tile centre (m)
  float2 *acoef;                       // global a[m][q]: [kT2PgMax][n_f] (q-major), then [n_f][kT2PgMax]
  double *tabs;                        // [4][kT2PMax][kT2PMax] nodes, W (nodes -> monomial), lambda
  float2 *gexp;                        // [2][n_a][kT2PgMax] global expansion of the adjoint rows
  float2 *coef;                        // [2][T][n_a][P] monomial coefficients (adjoint rows)
  float2 *mom;                         // [n_a][T][P] forward moments (antenna-major)
  unsigned char *tcimg;                // tensor-core B images of the a table (t2_tc_images):
                                       // [cdiv(n_f, 32)][kT2GexpImg] then [cdiv(n_f, 128)][kT2BinsImg]
  float2 *mg;                          // [n_a][kT2PgMax] global forward moments (k2_fout -> bins)
  ChebHdr *skip;                       // sel = 1 when the plan applies: the direct fallback
                                       // kernels (K2, the adjoint) read it and return at once
  unsigned int *flags;
};

// tensor-core (tcgen05) form of the two dense complex contractions against the shared a table
// (rfr_tc_gemm.cu): the global expansion of the adjoint rows G_i = Y_i conj(a) (k2_gexp) and the
// bins of the forward s_i = e^{-j 2 pi m' u_g} a M_g,i (the end of k2_fout).  Byte sizes of one
// K chunk (32 bins) of the expansion's image and of one N chunk (128 bins) of the bins' image
// (fp16 hi | lo, at the largest Pg).
constexpr size_t kT2GexpImg = (size_t)2 * 96 * 64 * 2;
constexpr size_t kT2BinsImg = (size_t)2 * 256 * 96 * 2;
inline size_t t2_tcimg_bytes(int n_f) {
  return (size_t)((n_f + 31) / 32) * kT2GexpImg + (size_t)((n_f + 127) / 128) * kT2BinsImg;
}
bool t2_tc_enabled();                  // RFR_T2TC=0: the SIMT contractions (A/B)
cudaError_t t2_tc_images(const T2Args &a, cudaStream_t st);
cudaError_t t2_gexp_tc(const T2Args &a, const float2 *X0, const float2 *X1, cudaStream_t st);
cudaError_t t2_bins_tc(const T2Args &a, float2 *out, cudaStream_t st);

// per-sweep device-time profiling (rfr_profile_enable / rfr_profile_read; ids = RFR_SWEEP_*)
constexpr int kProfPlan = 0, kProfSort = 1, kProfPrep = 2, kProfFilter = 3, kProfBackward = 4,
              kProfForward = 5, kProfForwardOut = 6;
constexpr int kT2ProfSlots = 7;
class ProfScope {
 public:
  ProfScope(int id, cudaStream_t st);
  ~ProfScope();
 private:
  cudaStream_t st_;
  int id_;
  void *a_;
};
void t2_profile_enable(bool on);
void t2_profile_read(int id, double *ms, unsigned long long *n);

// plan + sort of the plan's own points; kind selects the cost model of the grid choice:
// kT2PlanAdjoint (filter / backward sweeps, chunks of srt.chunk points) or kT2PlanForward
constexpr int kT2PlanAdjoint = 0, kT2PlanForward = 1;
cudaError_t t2_plan(const T2Args &a, const T2Points &pts, const T2Sorted &srt, int kind,
                    cudaStream_t st);
// sort another point set into an existing plan's grid (chunk = srt.chunk)
cudaError_t t2_sort(const T2Args &a, const T2Points &pts, const T2Sorted &srt, cudaStream_t st);
// adjoint rows X0 (and X1 if not NULL): global expansion + per-(tile, antenna) coefficients.
// tstart: tile occupancy of the points row 1 (or the only row) is swept over; tstart0 (NULL: the
// same): of the points row 0 is swept over -- coefficients of unoccupied tiles are not computed
cudaError_t t2_prep_adjoint(const T2Args &a, const int *tstart, const float2 *X0, const float2 *X1,
                            cudaStream_t st, const int *tstart0 = nullptr);
// matched filter over the sorted points of srt with coefficient row `row`: M partials [split][n]
cudaError_t t2_filter(const T2Args &a, const T2Sorted &srt, int row, float2 *out, int64_t n_out,
                      int n_splits, int64_t ants_per_split, int n_sms, cudaStream_t st);
// backward over the sorted records (compacted list of n_dev <= n_c): split partials
// part[split][5][n_c] at the compacted index, then their fixed-order sum scattered to
// out[5][n_s] at the sample index idx[c] (out zeroed first: samples outside the list get 0)
cudaError_t t2_backward(const T2Args &a, const T2Sorted &srt, int row, const int *idx,
                        const int64_t *n_dev, int64_t n_c, float *part, float *out, int64_t n_s,
                        int n_splits, int64_t ants_per_split, bool no_gain, int n_sms,
                        cudaStream_t st);
// fixed-order sum of [S][n] split partials (a no-op when the plan does not apply)
cudaError_t t2_sum_splits(const T2Args &a, const float *part, int S, int64_t n, float *out,
                          int n_sms, cudaStream_t st);
// forward (kind kFwdTrace) or K5 (kFwdMFAdj) over the sorted records: bins [n_a][n_f]
cudaError_t t2_forward(const T2Args &a, const T2Sorted &srt, int kind, bool no_gain, float2 *out,
                       int n_sms, cudaStream_t st);

}  // namespace rfr
