// librfr.cu -- C ABI (include/librfr.h): argument validation, workspace planning, kernel launches,
// and the library-owned NCCL communicator of the multi-GPU path.
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <new>

#include "../../include/librfr.h"
#include "rfr_device.cuh"
#include "rfr_launch.h"
#include "rfr_tiled.h"

using namespace rfr;

namespace {

constexpr double kC = 299792458.0;
constexpr size_t kHdr = 256;                   // workspace header: flags word at offset 0
constexpr size_t kChebHdrOff = 64;             // ChebHdr of the Chebyshev-moment forward
constexpr size_t kActiveOff = 128;             // int64 count of the compacted active records
constexpr size_t kActiveBwdOff = 136;          // int64 count of the backward's active samples
constexpr size_t kTilePOff = 144;              // int: moments of the last tiled filter
constexpr size_t kT2SkipOff = 192;             // ChebHdr: sel = 1 when the r2 engine's plan applies
constexpr int kTmpN = 512;                     // reduction scratch (floats)
constexpr size_t kSplitCap = size_t(2) << 30;  // cap on each split-partial region (bytes)

int device_sms() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> g(mu);
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------- K2 / K5 tiling
// B bins per lane, nb blocks per warp (one bin chunk), taw = 32 / nb antennas per warp.
struct FwdGeom {
  int B = 32, nb = 1, nb_total = 1, taw = 32, chunks = 1;
};
// bins per lane: 32 (3 CTAs / SM) or, with RFR_FWD_B=16, 16 (5 CTAs / SM, twice the anchors)
int fwd_b_pref() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RFR_FWD_B");
    v = (e && atoi(e) == 16) ? 16 : 32;
  }
  return v;
}
bool fwd_geom(int32_t n_f, FwdGeom &g) {
  const int nf = n_f > 0 ? n_f : 1;
  g.B = nf >= 32 ? fwd_b_pref() : (nf >= 16 ? 16 : 8);
  g.nb_total = (int)cdiv(nf, g.B);
  if (g.nb_total > 256) return false;                      // n_freq > 8192: unsupported
  g.nb = std::min(g.nb_total, 32);
  g.chunks = (int)cdiv(g.nb_total, g.nb);
  g.taw = 32 / g.nb;
  return true;
}

struct Split {
  int splits = 1;
  int64_t per_split = 0;   // points (K2/K5) or antennas (K3/K4) per split
};

// split-K over the summed points of K2 / K5: ~32 waves of kFwdMinBlocks CTAs per SM, bounded by
// the points and by the partial-buffer capacity `cap` (bytes); splits == 1 writes the output
// directly (no partial buffer).
Split fwd_split(int64_t n_pts, int64_t n_a, int32_t n_f, const FwdGeom &g, size_t cap) {
  const int64_t n_tiles =
      (n_a > 0 ? cdiv(n_a, (int64_t)kFwdWarps * g.taw) : 1) * g.chunks;
  const int tj = fwd_tj(g.B);
  int64_t s = cdiv((int64_t)device_sms() * fwd_min_blocks(g.B) * 32, n_tiles);
  s = std::min<int64_t>(s, std::max<int64_t>(1, cdiv(n_pts, tj * 16)));
  const size_t per = (size_t)std::max<int64_t>(n_a, 1) * std::max(n_f, 1) * 8;
  s = std::min<int64_t>(s, std::max<int64_t>(1, (int64_t)(std::min(cap, kSplitCap) / per)));
  s = std::max<int64_t>(s, 1);
  Split r;
  r.per_split = cdiv(cdiv(std::max<int64_t>(n_pts, 1), s), tj) * tj;
  r.splits = (int)std::max<int64_t>(1, cdiv(n_pts, r.per_split));
  if (r.splits == 1) r.per_split = std::max<int64_t>(n_pts, 1);
  return r;
}

// split over antennas of K3 / K4 (one thread per point): ~16 waves of 4 CTAs per SM
Split adj_split(int64_t n_pts, int64_t n_a, int floats_per_pt, size_t cap) {
  const int64_t per_cta = (int64_t)kAdjThreads;
  const int64_t tiles = std::max<int64_t>(1, cdiv(n_pts, per_cta));
  int64_t s = cdiv((int64_t)device_sms() * 4 * 16, tiles);
  s = std::min<int64_t>(s, std::max<int64_t>(1, cdiv(n_a, kAdjGA)));
  const size_t per = (size_t)std::max<int64_t>(n_pts, 1) * floats_per_pt * 4;
  s = std::min<int64_t>(s, std::max<int64_t>(1, (int64_t)(std::min(cap, kSplitCap) / per)));
  s = std::max<int64_t>(s, 1);
  Split r;
  r.per_split = cdiv(cdiv(std::max<int64_t>(n_a, 1), s), kAdjGA) * kAdjGA;
  r.splits = (int)std::max<int64_t>(1, cdiv(n_a, r.per_split));
  return r;
}

// split-K over the points of the Chebyshev-moment forward: ~8 waves of 4 CTAs of 128 antennas per
// SM, at least 512 points per split
Split cheb_split(int64_t n_pts, int64_t n_a) {
  const int64_t tiles = std::max<int64_t>(1, cdiv(n_a, cheb_threads()));
  int64_t s = cdiv((int64_t)device_sms() * 4 * 8, tiles);
  s = std::min<int64_t>(s, std::max<int64_t>(1, cdiv(n_pts, 512)));
  s = std::max<int64_t>(s, 1);
  Split r;
  r.per_split = cdiv(std::max<int64_t>(n_pts, 1), s);
  r.splits = (int)std::max<int64_t>(1, cdiv(n_pts, r.per_split));
  return r;
}
// the Chebyshev path is on unless RFR_FWD=direct (A/B measurements)
bool cheb_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RFR_FWD");
    v = (e && strcmp(e, "direct") == 0) ? 0 : 1;
  }
  return v == 1;
}

// ---------------------------------------------------------------------------- workspace layout
// The layout depends ONLY on the workspace's planning dimensions, so every call that shares a
// workspace sees the same regions: K1's records (the RFR_REUSE_BLEND cache) are never touched by
// the filter, K5 or the loss.
//   header | records [n_s] 48 B | ray ds [n_s] | tmp | backward sums [5][n_s] | filter M [n_q] |
//   K5 query records [n_q] 48 B | K2/K5 split partials | K3 split partials | K4 split partials
struct Layout {
  size_t off_rec = 0, off_ds = 0, off_tmp = 0, off_bwds = 0, off_fltm = 0, off_qrec = 0,
         off_fwdp = 0, off_bwdp = 0, off_fltp = 0, off_bprep = 0, off_cbox = 0, off_clc = 0,
         off_ccoef = 0, off_cpart = 0, off_cbadj = 0, off_recc = 0, off_ccnt = 0, off_aflag = 0,
         off_idxc = 0, off_ttile = 0, off_tbcnt = 0, off_tstart = 0, off_tperm = 0, off_tqs = 0,
         off_tbox = 0, off_tlc = 0, off_thdr = 0, off_tcoef = 0, off_tbmom = 0, off_trs = 0,
         off_tfp = 0, off_tgeo = 0, off_t2geof = 0, total = 0;
  // r2 tiled engine (rfr_tiled.h): plan, tables, per-(tile, antenna) data, two sorted views
  size_t off_t2plan = 0, off_t2boxp = 0, off_t2tabs = 0, off_t2tbox = 0, off_t2lc = 0,
         off_t2geo = 0, off_t2lg = 0, off_t2acoef = 0, off_t2gexp = 0, off_t2coef = 0,
         off_t2mom = 0, off_t2bwdp = 0, off_t2lct = 0, off_t2tcimg = 0, off_t2mg = 0,
         off_t2fltp = 0;
  int t2_flt_cap = 1;               // antenna splits the r2 filter's partial buffer holds
  size_t off_t2v[2][7] = {};        // per view: tstart+cstart+n_items+torder+n_occ, perm, pos, aux, bcnt
  size_t off_gsig = 0, off_gant = 0; // rfr_filter_gather: gathered signal rows and positions
  int t2_bwd_splits = 1;
  size_t cap_trs = 0, cap_tfp = 0;
  size_t cap_cpart = 0;
  size_t cap_fwdp = 0, cap_bwdp = 0, cap_fltp = 0;
};

// antenna splits of the r2 filter sweep: enough work items (chunk of points x antenna split) for
// ~24 per resident CTA slot (5 per SM), so the persistent grid's last round is short (equal-cost
// items: with ~6 per slot the makespan was 7 items for 6.2 on average), at least 64 antennas per
// split, at most `cap`, and the partials [S][n] within 1 GiB
int t2_flt_splits(int64_t n_pts, int chunk, int64_t n_a, int cap) {
  const int64_t items = std::max<int64_t>(1, cdiv(n_pts, chunk));
  static int per_slot = -1;                         // items per resident CTA slot (A/B: RFR_T2SPL)
  if (per_slot < 0) { const char *e = getenv("RFR_T2SPL"); per_slot = e ? std::max(1, atoi(e)) : 24; }
  int64_t s = cdiv((int64_t)device_sms() * 5 * per_slot, items);
  s = std::min<int64_t>(s, std::max<int64_t>(1, cdiv(n_a, 64)));
  s = std::min<int64_t>(s, std::max<int64_t>(1, (int64_t(1) << 30) / (std::max<int64_t>(n_pts, 1) * 8)));
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, cap));
}

bool make_layout(int64_t n_s, int64_t n_a, int32_t n_f, int64_t n_q, Layout &L) {
  if (n_s < 0 || n_a < 0 || n_q < 0 || n_f < 0) return false;
  FwdGeom g;
  if (!fwd_geom(n_f, g)) return false;
  const int32_t nf = std::max(n_f, 1);
  const Split f2 = fwd_split(n_s, n_a, nf, g, kSplitCap);
  const Split f5 = fwd_split(n_q, n_a, nf, g, kSplitCap);
  const Split b3 = adj_split(n_s, n_a, 5, kSplitCap);
  const Split b4 = adj_split(n_q, n_a, 2, kSplitCap);
  const int fsp = std::max(f2.splits, f5.splits);
  L.cap_fwdp = fsp > 1 ? (size_t)fsp * n_a * nf * 8 : 0;
  L.cap_bwdp = b3.splits > 1 ? (size_t)b3.splits * 5 * n_s * 4 : 0;
  L.cap_fltp = b4.splits > 1 ? (size_t)b4.splits * n_q * 8 : 0;
  size_t o = kHdr;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.off_rec = take((size_t)n_s * sizeof(Rec));
  L.off_ds = take((size_t)n_s * 4);
  L.off_tmp = take((size_t)kTmpN * 4);
  L.off_bwds = take((size_t)5 * n_s * 4);
  L.off_fltm = take((size_t)n_q * 8);
  L.off_qrec = take((size_t)n_q * sizeof(Rec));
  L.off_fwdp = take(L.cap_fwdp);
  L.off_bwdp = take(L.cap_bwdp);
  L.off_fltp = take(L.cap_fltp);
  // tensor-core adjoint: per-antenna B^T images (sized for the fused sweep's two X rows)
  L.off_bprep = take(adjoint_tc_supported(nf) ? (size_t)n_a * tc_bprep_bytes_per_ant(nf, 2) : 0);
  // Chebyshev-moment forward: box partials, per-antenna centres, coefficients, partial moments
  const Split cs = cheb_split(std::max(n_s, n_q), n_a);
  L.cap_cpart = (size_t)cs.splits * std::max<int64_t>(n_a, 1) * kChebPMax * 8;
  L.off_cbox = take((size_t)(cheb_box_blocks() + 1) * 6 * 8);   // block partials + the box
  L.off_clc = take((size_t)std::max<int64_t>(n_a, 1) * 8);
  L.off_ccoef = take((size_t)nf * kChebPMax * 8);
  L.off_cpart = take(L.cap_cpart);
  L.off_cbadj = take((size_t)std::max<int64_t>(n_a, 1) * kChebPMax * 2 * 8);
  L.off_recc = take((size_t)n_s * sizeof(Rec));             // compacted active records
  L.off_ccnt = take((size_t)(compact_blocks(n_s) + 1) * 4);
  L.off_aflag = take((size_t)n_s);                           // K1: alpha != 0 per sample
  L.off_idxc = take((size_t)n_s * 4);                        // compacted list: original index
  // tiled matched filter (DESIGN 5d): tile of each point, counts, starts, sorted points, tiles'
  // boxes and per-(antenna, tile) centres, its own choice header, coefficients and moments
  {
    const int64_t np = std::max(n_s, n_q);
    const int64_t na1 = std::max<int64_t>(n_a, 1);
    L.off_ttile = take((size_t)np);
    L.off_tbcnt = take((size_t)(tile_count_blocks(np) + 1) * kTiles * 4);
    L.off_tstart = take((size_t)2 * (kTiles + 1) * 4);
    L.off_tperm = take((size_t)np * 4);
    L.off_tqs = take((size_t)np * 16);
    L.off_tbox = take((size_t)kTiles * 6 * 8);
    L.off_tlc = take((size_t)kTiles * na1 * 8);
    L.off_thdr = take(64);
    L.off_tcoef = take((size_t)nf * kChebPMax * 8);
    L.off_tbmom = take((size_t)na1 * kTiles * kChebPMax * 8);
    // tiled backward / K5: sorted records; tiled K5: moments per (chunk CTA, antenna)
    L.cap_trs = (size_t)np * sizeof(Rec);
    L.off_trs = take(L.cap_trs);
    L.cap_tfp = (size_t)tile_fwd_blocks(n_q) * na1 * kChebPMax * 8;
    L.off_tfp = take(L.cap_tfp);
    L.off_tgeo = take((size_t)kTiles * na1 * 32);
  }
  {
    const int64_t np = std::max<int64_t>(std::max(n_s, n_q), 1);
    const int64_t na1 = std::max<int64_t>(n_a, 1);
    L.off_t2plan = take(256);
    L.off_t2boxp = take((size_t)kT2BoxBlocks * 6 * 4);
    L.off_t2tabs = take((size_t)(3 * kT2PMax * kT2PMax + 128) * 8);
    L.off_t2tbox = take((size_t)kT2Max * 6 * 4);
    L.off_t2lc = take((size_t)kT2Max * na1 * 8);
    L.off_t2lct = take((size_t)kT2Max * na1 * 8);
    L.off_t2geo = take((size_t)kT2Max * na1 * 32);
    L.off_t2geof = take((size_t)kT2Max * na1 * 32);
    L.off_t2lg = take((size_t)na1 * 3 * 8);
    L.off_t2acoef = take((size_t)2 * nf * kT2PgMax * 8);     // both layouts
    L.off_t2gexp = take((size_t)2 * na1 * kT2PgMax * 8);
    L.off_t2coef = take((size_t)2 * kT2TP * na1 * 8);
    L.off_t2mom = take((size_t)kT2TP * na1 * 8);
    L.off_t2tcimg = take(t2_tcimg_bytes(nf));
    L.off_t2mg = take((size_t)na1 * kT2PgMax * 8);
    // backward split partials [S][5][n_s] (compacted index), S <= 16 within 1 GiB
    const int64_t ns1 = std::max<int64_t>(n_s, 1);
    L.t2_bwd_splits = (int)std::max<int64_t>(1, std::min<int64_t>(16, (int64_t(1) << 30) / (ns1 * 20)));
    L.off_t2bwdp = take((size_t)L.t2_bwd_splits * 5 * ns1 * 4);
    // r2 filter split partials [S][n_q] complex (S from t2_flt_splits at the smallest chunk)
    L.t2_flt_cap = t2_flt_splits(np, kT2FltChunk, n_a, 16);
    L.off_t2fltp = take(L.t2_flt_cap > 1 ? (size_t)L.t2_flt_cap * np * 8 : 0);
    L.off_gsig = take((size_t)na1 * nf * 8);
    L.off_gant = take((size_t)3 * na1 * 4);
    const int64_t nb = (np + kT2SortBlock - 1) / kT2SortBlock;
    for (int v = 0; v < 2; ++v) {
      L.off_t2v[v][0] = take((size_t)(3 * (kT2Max + 1) + 1) * 4);
      L.off_t2v[v][1] = take((size_t)np * 4);
      L.off_t2v[v][2] = take((size_t)np * 16);
      L.off_t2v[v][3] = take((size_t)np * 16);
      L.off_t2v[v][4] = take((size_t)nb * kT2Max * 4);
    }
  }
  L.total = o;
  return true;
}

template <typename T>
T *at(const rfr_workspace *ws, size_t off) {
  return reinterpret_cast<T *>(static_cast<char *>(ws->ptr) + off);
}

// A call's workspace: planned for at least n_s samples, n_q queries, n_a antennas and n_f bins
// (every region is sized from the planning dimensions, so a call beyond any of them would write
// past its regions).  n_a = n_f = 0: the call touches no per-antenna / per-bin region.
rfr_status check_ws(const rfr_workspace *ws, int64_t n_s, int64_t n_q, Layout &L, int64_t n_a = 0,
                    int32_t n_f = 0) {
  if (!ws || !ws->ptr) return RFR_E_ARG;
  if (!make_layout(ws->n_samples, ws->n_ant, ws->n_freq, ws->n_query, L)) return RFR_E_SHAPE;
  if (ws->bytes < L.total || n_s > ws->n_samples || n_q > ws->n_query || n_a > ws->n_ant ||
      n_f > ws->n_freq)
    return RFR_E_SHAPE;
  return RFR_OK;
}

rfr_status check_samples(const rfr_samples *s) {
  if (!s || s->n_rays < 0) return RFR_E_ARG;
  if (s->n_rays > 0 && (!s->x || !s->y || !s->z || !s->sdf || !s->refl || !s->nx || !s->ny ||
                        !s->nz || !s->power))
    return RFR_E_ARG;
  if (s->n_per_ray <= 0) return RFR_E_SHAPE;
  return RFR_OK;
}

rfr_status check_ants(const rfr_antennas *a) {
  if (!a || a->n_ant < 0) return RFR_E_ARG;
  if (a->n_ant > 0 && (!a->tx_x || !a->tx_y || !a->tx_z)) return RFR_E_ARG;
  const int nrx = (a->rx_x != nullptr) + (a->rx_y != nullptr) + (a->rx_z != nullptr);
  if (nrx != 0 && nrx != 3) return RFR_E_ARG;
  if (a->phi_rx && !a->rx_x) return RFR_E_ARG;        // phi_rx only with a separate receiver
  return RFR_OK;
}

rfr_status check_grid(const rfr_freq_grid *g) {
  if (!g || g->n_freq <= 0 || !(g->df_hz > 0.0) || !(g->f0_hz >= 0.0) || !isfinite(g->f0_hz) ||
      !isfinite(g->df_hz))
    return RFR_E_ARG;
  if (g->n_freq > 8192) return RFR_E_SHAPE;
  return RFR_OK;
}

rfr_status cuda_status(cudaError_t e) { return e == cudaSuccess ? RFR_OK : RFR_E_CUDA; }

#define RFR_TRY(x) do { rfr_status _s = (x); if (_s != RFR_OK) return _s; } while (0)
#define RFR_CU(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return RFR_E_CUDA; } while (0)

rfr_status run_blend(const rfr_samples *s, float sharpness, uint32_t flags,
                     const rfr_workspace *ws, const Layout &L, cudaStream_t st) {
  if (flags & RFR_REUSE_BLEND) return RFR_OK;
  BlendArgs b;
  b.x = s->x; b.y = s->y; b.z = s->z; b.sdf = s->sdf; b.refl = s->refl;
  b.nx = s->nx; b.ny = s->ny; b.nz = s->nz; b.power = s->power; b.phi_origin = s->phi_origin;
  b.n_rays = s->n_rays; b.n_per_ray = s->n_per_ray; b.s = sharpness;
  b.rec = at<Rec>(ws, L.off_rec);
  b.aflag = at<unsigned char>(ws, L.off_aflag);
  b.flags = at<unsigned>(ws, 0);
  b.check_finite = (flags & RFR_CHECK_FINITE) != 0;
  return cuda_status(launch_blend(b, st));
}

bool has_corr(const rfr_samples *s, const rfr_antennas *a) {
  return s->phi_origin || a->phi_tx || a->phi_rx;
}

// K2 (trace) or K5 (matched-filter adjoint) over `rec` [n_pts] into out [n_a][n_f] (+ split sum)
// Chebyshev-moment arguments for a call over `rec` (n_pts points) and this antenna set
ChebArgs make_cheb(const Rec *rec, int64_t n_pts, const rfr_antennas *ants,
                   const rfr_freq_grid *grid, bool no_gain, const rfr_workspace *ws,
                   const Layout &L, int64_t per_split, bool direct = false) {
  ChebArgs c;
  memset(&c, 0, sizeof(c));
  c.rec = rec;
  c.n_s = n_pts;
  c.tx_x = ants->tx_x; c.tx_y = ants->tx_y; c.tx_z = ants->tx_z;
  c.rx_x = ants->rx_x; c.rx_y = ants->rx_y; c.rx_z = ants->rx_z;
  c.phi_tx = ants->phi_tx; c.phi_rx = ants->phi_rx;
  c.n_a = ants->n_ant;
  c.n_f = grid->n_freq;
  c.kd = grid->df_hz / kC;
  c.kc = (grid->f0_hz + (double)(grid->n_freq / 2) * grid->df_hz) / kC;
  c.samples_per_split = per_split;
  c.lc = at<double>(ws, L.off_clc);
  c.hdr = at<ChebHdr>(ws, kChebHdrOff);
  c.coef = at<float2>(ws, L.off_ccoef);
  c.pmax = kChebPMax;
  c.part = at<float2>(ws, L.off_cpart);
  c.flags = at<unsigned>(ws, 0);
  c.no_gain = no_gain;
  c.enable = cheb_enabled() && !direct;
  return c;
}

// tiled matched filter over n points at (qx, qy, qz) of the signal rows X into M partials `out`
TileArgs make_tile(const float *qx, const float *qy, const float *qz, int64_t n,
                   const rfr_antennas *ants, const rfr_freq_grid *grid, const ChebArgs &c,
                   const float2 *X, float2 *out, int64_t ants_per_split, const rfr_workspace *ws,
                   const Layout &L) {
  TileArgs t;
  memset(&t, 0, sizeof(t));
  t.qx = qx; t.qy = qy; t.qz = qz;
  t.n = n;
  t.tx_x = ants->tx_x; t.tx_y = ants->tx_y; t.tx_z = ants->tx_z;
  t.rx_x = ants->rx_x; t.rx_y = ants->rx_y; t.rx_z = ants->rx_z;
  t.phi_tx = ants->phi_tx; t.phi_rx = ants->phi_rx;
  t.n_a = ants->n_ant;
  t.n_f = grid->n_freq;
  t.kd = c.kd;
  t.kc = c.kc;
  t.ghdr = c.hdr;
  t.gbox = at<double>(ws, L.off_cbox) + (size_t)cheb_box_blocks() * 6;
  t.tile = at<unsigned char>(ws, L.off_ttile);
  t.bcnt = at<int>(ws, L.off_tbcnt);
  t.tstart = at<int>(ws, L.off_tstart);
  t.cstart = t.tstart + kTiles + 1;
  t.perm = at<int>(ws, L.off_tperm);
  t.qs = at<float4>(ws, L.off_tqs);
  t.tbox = at<double>(ws, L.off_tbox);
  t.lc = at<double>(ws, L.off_tlc);
  t.hdr = at<ChebHdr>(ws, L.off_thdr);
  t.dmax = reinterpret_cast<unsigned long long *>(at<char>(ws, L.off_thdr) + 32);
  t.coef = at<float2>(ws, L.off_tcoef);
  t.bmom = at<float2>(ws, L.off_tbmom);
  t.X = X;
  t.out = out;
  t.ants_per_split = ants_per_split;
  t.pub = at<int>(ws, kTilePOff);
  t.tgeo = at<float4>(ws, L.off_tgeo);
  return t;
}
// the tiled filter is on unless RFR_TILE=0 (A/B)
bool tile_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RFR_TILE");
    v = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

// the r2 tiled engine (rfr_tiled.cu) serves monostatic calls without the Eq. 7 correction unless
// RFR_V2=0 (A/B against the r1 kernels)
bool v2_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("RFR_V2");
    v = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}
bool use_v2(const rfr_antennas *a, bool corr, uint32_t flags) {
  return v2_enabled() && a->rx_x == nullptr && !corr && !(flags & (RFR_DIRECT | RFR_R1)) &&
         cheb_enabled();
}

T2Args make_t2(const rfr_antennas *ants, const rfr_freq_grid *grid, const rfr_workspace *ws,
               const Layout &L) {
  T2Args t;
  memset(&t, 0, sizeof(t));
  t.plan = at<T2Plan>(ws, L.off_t2plan);
  t.box_part = at<float>(ws, L.off_t2boxp);
  t.tx_x = ants->tx_x; t.tx_y = ants->tx_y; t.tx_z = ants->tx_z;
  t.n_a = ants->n_ant;
  t.n_f = grid->n_freq;
  t.kd = grid->df_hz / kC;
  t.kc = (grid->f0_hz + (double)(grid->n_freq / 2) * grid->df_hz) / kC;
  t.tbox = at<float>(ws, L.off_t2tbox);
  t.lc = at<double>(ws, L.off_t2lc);
  t.lct = at<double>(ws, L.off_t2lct);
  t.tgeo = at<float4>(ws, L.off_t2geo);
  t.tgeof = at<float4>(ws, L.off_t2geof);
  t.lg = at<double>(ws, L.off_t2lg);
  t.acoef = at<float2>(ws, L.off_t2acoef);
  t.tabs = at<double>(ws, L.off_t2tabs);
  t.gexp = at<float2>(ws, L.off_t2gexp);
  t.tcimg = at<unsigned char>(ws, L.off_t2tcimg);
  t.mg = at<float2>(ws, L.off_t2mg);
  t.coef = at<float2>(ws, L.off_t2coef);
  t.mom = at<float2>(ws, L.off_t2mom);
  t.skip = at<ChebHdr>(ws, kT2SkipOff);
  t.flags = at<unsigned>(ws, 0);
  return t;
}
T2Sorted make_view(const rfr_workspace *ws, const Layout &L, int v, int chunk) {
  T2Sorted s;
  memset(&s, 0, sizeof(s));
  s.tstart = at<int>(ws, L.off_t2v[v][0]);
  s.cstart = s.tstart + kT2Max + 1;
  s.n_items = s.cstart + kT2Max + 1;
  s.torder = s.n_items + 1;
  s.n_occ = s.torder + kT2Max;
  s.chunk = chunk;
  s.perm = at<int>(ws, L.off_t2v[v][1]);
  s.pos = at<float4>(ws, L.off_t2v[v][2]);
  s.aux = at<float4>(ws, L.off_t2v[v][3]);
  s.bcnt = at<int>(ws, L.off_t2v[v][4]);
  return s;
}
// antenna splits of a v2 adjoint sweep: enough work items for ~4 waves of the persistent grid
int t2_splits(int64_t n_pts, int chunk, int64_t n_a, int cap) {
  const int64_t items = std::max<int64_t>(1, cdiv(n_pts, chunk));
  int64_t s = cdiv((int64_t)device_sms() * 5 * 4, items);
  s = std::min<int64_t>(s, std::max<int64_t>(1, cdiv(n_a, 64)));
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, cap));
}

rfr_status run_fwd(const Rec *rec, int64_t n_pts, const rfr_antennas *ants,
                   const rfr_freq_grid *grid, bool no_gain, bool corr, int kind, float *out,
                   const rfr_workspace *ws, const Layout &L, cudaStream_t st,
                   const Rec *rec_c = nullptr, const int64_t *n_dev = nullptr,
                   bool direct = false, const ChebHdr *v2skip = nullptr) {
  FwdGeom g;
  if (!fwd_geom(grid->n_freq, g)) return RFR_E_SHAPE;
  const Split sp = fwd_split(n_pts, ants->n_ant, grid->n_freq, g, L.cap_fwdp);
  FwdArgs a;
  memset(&a, 0, sizeof(a));
  a.rec = rec;
  a.n_s = n_pts;
  a.tx_x = ants->tx_x; a.tx_y = ants->tx_y; a.tx_z = ants->tx_z;
  a.rx_x = ants->rx_x; a.rx_y = ants->rx_y; a.rx_z = ants->rx_z;
  a.phi_tx = ants->phi_tx; a.phi_rx = ants->phi_rx;
  a.n_a = ants->n_ant;
  a.n_f = grid->n_freq; a.nb = g.nb; a.nb_total = g.nb_total; a.taw = g.taw;
  a.warp_smem = fwd_warp_smem(g.B);
  a.k0 = grid->f0_hz / kC;
  a.kd = grid->df_hz / kC;
  a.kw = grid->df_hz * g.B / kC;
  a.kchunk = grid->df_hz * g.B * g.nb / kC;
  a.samples_per_split = sp.per_split;
  a.out = sp.splits > 1 ? at<float2>(ws, L.off_fwdp) : reinterpret_cast<float2 *>(out);
  a.flags = at<unsigned>(ws, 0);
  a.no_gain = no_gain;
  const bool mono = ants->rx_x == nullptr;
  if (v2skip) {
    // the r2 engine ran first: this is its direct fallback, a no-op when the plan applied
    a.skip = v2skip;
    RFR_CU(launch_trace_fwd(a, g.B, mono, corr, kind, sp.splits, st));
    if (sp.splits > 1)
      RFR_CU(launch_sum_splits(at<float>(ws, L.off_fwdp), sp.splits,
                               ants->n_ant * (int64_t)grid->n_freq * 2, out, device_sms(), st,
                               v2skip));
    return RFR_OK;
  }
  // Chebyshev-moment path (rfr_cheb.cu): chosen on the device from the delay spread; the direct
  // kernel and its split sum return at once when it runs, and vice versa
  ChebHdr *hdr = at<ChebHdr>(ws, kChebHdrOff);
  const Split cs = cheb_split(n_pts, ants->n_ant);
  const bool cheb = ants->n_ant > 0 && n_pts > 0 &&
                    (size_t)cs.splits * ants->n_ant * kChebPMax * 8 <= L.cap_cpart;
  ChebArgs c = make_cheb(rec_c ? rec_c : rec, n_pts, ants, grid, no_gain, ws, L, cs.per_split,
                         direct);
  c.n_dev = rec_c ? n_dev : nullptr;
  if (cheb) {
    RFR_CU(launch_cheb_prepare(c, at<double>(ws, L.off_cbox), st));
    a.skip = hdr;
  }
  RFR_CU(launch_trace_fwd(a, g.B, mono, corr, kind, sp.splits, st));
  if (sp.splits > 1)
    RFR_CU(launch_sum_splits(at<float>(ws, L.off_fwdp), sp.splits,
                             ants->n_ant * (int64_t)grid->n_freq * 2, out, device_sms(), st,
                             cheb ? hdr : nullptr));
  if (!cheb) return RFR_OK;
  // K5 tiled (DESIGN 6b): per-(antenna, tile) centres cut P to the tiles' spread
  if (kind == kFwdMFAdj && tile_enabled() && !rec_c && !direct &&
      (size_t)n_pts * sizeof(Rec) <= L.cap_trs &&
      (size_t)tile_fwd_blocks(n_pts) * ants->n_ant * kChebPMax * 8 <= L.cap_tfp) {
    TileArgs ta = make_tile(nullptr, nullptr, nullptr, n_pts, ants, grid, c, nullptr, nullptr, 0,
                            ws, L);
    ta.rec = rec;
    ta.rs = at<Rec>(ws, L.off_trs);
    ta.fpart = at<float2>(ws, L.off_tfp);
    RFR_CU(launch_tiled_mfadj(ta, mono, reinterpret_cast<float2 *>(out), st));
    return RFR_OK;
  }
  RFR_CU(launch_cheb_fwd(c, mono, corr, kind, cs.splits, reinterpret_cast<float2 *>(out), st));
  return RFR_OK;
}

}  // namespace

// Opaque communicator of the multi-GPU path: one NCCL communicator per rank, built from
// a unique id the caller distributes (e.g. a torch.distributed broadcast).
struct rfr_comm {
  ncclComm_t nccl;
  int nranks, rank;
};

namespace {
// In-place sum of n floats over the communicator's ranks on `st` (an identity for one rank; the
// call is still issued so the one-GPU tests exercise the NCCL path).
rfr_status allreduce_sum(const rfr_comm *c, float *buf, int64_t n, cudaStream_t st) {
  if (!c || n <= 0) return RFR_OK;
  if (ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, c->nccl, st) != ncclSuccess)
    return RFR_E_NCCL;
  return RFR_OK;
}
}  // namespace

extern "C" {

rfr_status rfr_comm_unique_id(void *id) {
  if (!id) return RFR_E_ARG;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return RFR_E_NCCL;
  memcpy(id, &u, sizeof(u));
  return RFR_OK;
}

rfr_status rfr_comm_init(const void *id, int nranks, int rank, rfr_comm **out) {
  if (!id || !out || nranks <= 0 || rank < 0 || rank >= nranks) return RFR_E_ARG;
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  rfr_comm *c = new (std::nothrow) rfr_comm;
  if (!c) return RFR_E_ARG;
  c->nranks = nranks;
  c->rank = rank;
  if (ncclCommInitRank(&c->nccl, nranks, u, rank) != ncclSuccess) {
    delete c;
    return RFR_E_NCCL;
  }
  *out = c;
  return RFR_OK;
}

rfr_status rfr_comm_destroy(rfr_comm *c) {
  if (!c) return RFR_E_ARG;
  ncclResult_t r = ncclCommDestroy(c->nccl);
  delete c;
  return r == ncclSuccess ? RFR_OK : RFR_E_NCCL;
}

int rfr_abi_version(void) { return RFR_ABI_VERSION; }

uint64_t rfr_launch_count(void) { return (uint64_t)launch_count(); }

const char *rfr_status_string(rfr_status s) {
  switch (s) {
    case RFR_OK: return "ok";
    case RFR_E_ARG: return "invalid argument";
    case RFR_E_SHAPE: return "shape mismatch or workspace too small";
    case RFR_E_DOMAIN: return "a pair closer than u_min contributed 0";
    case RFR_E_NUMERIC: return "non-finite input";
    case RFR_E_CUDA: return "CUDA launch failure";
    case RFR_E_UNSUPPORTED: return "unsupported configuration";
    case RFR_E_NCCL: return "NCCL failure";
  }
  return "unknown status";
}

rfr_status rfr_workspace_size(int64_t n_samples, int64_t n_ant, int32_t n_freq, int64_t n_query,
                              size_t *bytes) {
  if (!bytes) return RFR_E_ARG;
  Layout L;
  if (!make_layout(n_samples, n_ant, n_freq, n_query, L)) return RFR_E_SHAPE;
  *bytes = L.total;
  return RFR_OK;
}

rfr_status rfr_forward(const rfr_samples *samples, float sharpness, const rfr_antennas *ants,
                       const rfr_freq_grid *grid, const rfr_opts *opts, float *signal,
                       const rfr_workspace *ws, rfr_stream_t stream) {
  RFR_TRY(check_samples(samples));
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  if (!(sharpness > 0.f) || (!signal && ants->n_ant > 0)) return RFR_E_ARG;
  const uint32_t flags = opts ? opts->flags : 0u;
  const int64_t n_s = samples->n_rays * (int64_t)samples->n_per_ray;
  Layout L;
  RFR_TRY(check_ws(ws, n_s, 0, L, ants->n_ant, grid->n_freq));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (ants->n_ant == 0) return RFR_OK;
  RFR_TRY(run_blend(samples, sharpness, flags, ws, L, st));
  // empty-space skipping for the Chebyshev path: the records with a non-zero amplitude, compacted
  const bool corr = has_corr(samples, ants);
  Rec *rec_c = at<Rec>(ws, L.off_recc);
  int64_t *n_act = at<int64_t>(ws, kActiveOff);
  RFR_CU(launch_compact(at<Rec>(ws, L.off_rec), n_s, corr, at<int>(ws, L.off_ccnt), n_act, rec_c,
                        st));
  const bool no_gain = (flags & RFR_NO_GAIN) != 0;
  if (use_v2(ants, corr, flags)) {
    // r2 engine: plan over the active records, tiled moments, virtual sources -> bins
    const T2Args t = make_t2(ants, grid, ws, L);
    const T2Sorted v = make_view(ws, L, 0, kT2FltChunk);
    T2Points pts;
    memset(&pts, 0, sizeof(pts));
    pts.rec = rec_c; pts.n_dev = n_act; pts.n = n_s;
    RFR_CU(t2_plan(t, pts, v, kT2PlanForward, st));
    RFR_CU(t2_forward(t, v, kFwdTrace, no_gain, reinterpret_cast<float2 *>(signal), device_sms(),
                      st));
    return run_fwd(at<Rec>(ws, L.off_rec), n_s, ants, grid, no_gain, corr, kFwdTrace, signal, ws,
                   L, st, nullptr, nullptr, false, t.skip);
  }
  return run_fwd(at<Rec>(ws, L.off_rec), n_s, ants, grid, no_gain, corr,
                 kFwdTrace, signal, ws, L, st, rec_c, n_act, (flags & RFR_DIRECT) != 0);
}

rfr_status rfr_loss(const float *signal, const float *target, int64_t n_complex, float *grad_signal,
                    float *loss, const rfr_workspace *ws, rfr_stream_t stream) {
  if (!signal || !target || !grad_signal || !loss || n_complex < 0) return RFR_E_ARG;
  Layout L;
  RFR_TRY(check_ws(ws, 0, 0, L));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  RFR_CU(launch_loss(signal, target, n_complex, grad_signal, at<float>(ws, L.off_tmp), kTmpN, loss,
                     st));
  return RFR_OK;
}

static rfr_status filter_impl(const float *signal, const rfr_antennas *ants,
                              const rfr_freq_grid *grid, const float *qx, const float *qy,
                              const float *qz, int64_t n_query, float *power, float *mf,
                              const rfr_comm *comm, const rfr_workspace *ws, cudaStream_t st) {
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  if (n_query < 0 || (n_query > 0 && (!qx || !qy || !qz)) || (ants->n_ant > 0 && !signal))
    return RFR_E_ARG;
  Layout L;
  RFR_TRY(check_ws(ws, 0, n_query, L, ants->n_ant, grid->n_freq));
  if (n_query == 0) return RFR_OK;
  float *M = mf ? mf : at<float>(ws, L.off_fltm);
  const Split sp = adj_split(n_query, ants->n_ant, 2, L.cap_fltp);
  AdjArgs a;
  memset(&a, 0, sizeof(a));
  a.qx = qx; a.qy = qy; a.qz = qz;
  a.n_s = n_query;
  a.tx_x = ants->tx_x; a.tx_y = ants->tx_y; a.tx_z = ants->tx_z;
  a.rx_x = ants->rx_x; a.rx_y = ants->rx_y; a.rx_z = ants->rx_z;
  a.n_a = ants->n_ant;
  a.n_f = grid->n_freq;
  a.k0 = grid->f0_hz / kC;
  a.kd = grid->df_hz / kC;
  a.X = reinterpret_cast<const float2 *>(signal);
  a.bprep = at<unsigned char>(ws, L.off_bprep);
  a.bprep_cap = L.total - L.off_bprep;
  a.ants_per_split = sp.per_split;
  a.out = sp.splits > 1 ? at<float>(ws, L.off_fltp) : M;
  a.flags = at<unsigned>(ws, 0);
  a.no_gain = false;
  const bool mono = ants->rx_x == nullptr;
  if (ants->n_ant > 0 && use_v2(ants, false, 0)) {
    // r2 engine: plan over the queries, Horner coefficients of the signal, filter sweep
    const T2Args t = make_t2(ants, grid, ws, L);
    const T2Sorted v = make_view(ws, L, 0, t2_filter_chunk());
    T2Points pts;
    memset(&pts, 0, sizeof(pts));
    pts.qx = qx; pts.qy = qy; pts.qz = qz; pts.n = n_query;
    RFR_CU(t2_plan(t, pts, v, kT2PlanAdjoint, st));
    RFR_CU(t2_prep_adjoint(t, v.tstart, reinterpret_cast<const float2 *>(signal), nullptr, st));
    const int S = t2_flt_splits(n_query, t2_filter_chunk(), ants->n_ant, L.t2_flt_cap);
    const int64_t aps = cdiv(cdiv(ants->n_ant, S), 16) * 16;
    float2 *o = reinterpret_cast<float2 *>(S > 1 ? at<float>(ws, L.off_t2fltp) : M);
    RFR_CU(t2_filter(t, v, 0, o, n_query, S, aps, device_sms(), st));
    if (S > 1) RFR_CU(t2_sum_splits(t, at<float>(ws, L.off_t2fltp), S, n_query * 2, M, device_sms(), st));
    a.skip = t.skip;                                   // direct fallback: no-op when planned
    a.gated = true;                                    // ... on one short persistent wave
    RFR_CU(launch_adjoint(a, kModeFlt, mono, false, sp.splits, st));
    if (sp.splits > 1)
      RFR_CU(launch_sum_splits(at<float>(ws, L.off_fltp), sp.splits, n_query * 2, M,
                               device_sms(), st, t.skip));
    RFR_TRY(allreduce_sum(comm, M, 2 * n_query, st));
    if (power) RFR_CU(launch_abs(M, n_query, power, device_sms(), st));
    return RFR_OK;
  }
  // Chebyshev-moment filter: the query points are packed as records (for their bounding box)
  const bool cheb = ants->n_ant > 0;
  const ChebArgs c = make_cheb(at<Rec>(ws, L.off_qrec), n_query, ants, grid, false, ws, L, 0);
  if (cheb) {
    RFR_CU(launch_pack_points(qx, qy, qz, n_query, at<Rec>(ws, L.off_qrec), device_sms(), st));
    RFR_CU(launch_cheb_prepare(c, at<double>(ws, L.off_cbox), st));
    a.skip = c.hdr;
  }
  RFR_CU(launch_adjoint(a, kModeFlt, mono, false, sp.splits, st));
  if (cheb)
    if (tile_enabled()) {
      const TileArgs ta = make_tile(qx, qy, qz, n_query, ants, grid, c,
                                    reinterpret_cast<const float2 *>(signal),
                                    reinterpret_cast<float2 *>(a.out), sp.per_split, ws, L);
      RFR_CU(launch_tiled_filter(ta, mono, sp.splits, st));
    } else {
      RFR_CU(launch_cheb_flt(c, a, at<float2>(ws, L.off_cbadj), mono, sp.splits, st));
    }
  if (sp.splits > 1)
    RFR_CU(launch_sum_splits(at<float>(ws, L.off_fltp), sp.splits, n_query * 2, M, device_sms(),
                             st));
  RFR_TRY(allreduce_sum(comm, M, 2 * n_query, st));     // antenna shards -> full M (a4)
  if (power) RFR_CU(launch_abs(M, n_query, power, device_sms(), st));
  return RFR_OK;
}

rfr_status rfr_filter(const float *signal, const rfr_antennas *ants, const rfr_freq_grid *grid,
                      const float *qx, const float *qy, const float *qz, int64_t n_query,
                      float *power, float *mf, const rfr_comm *comm, const rfr_workspace *ws,
                      rfr_stream_t stream) {
  if (!power && n_query > 0) return RFR_E_ARG;
  return filter_impl(signal, ants, grid, qx, qy, qz, n_query, power, mf, comm, ws,
                     reinterpret_cast<cudaStream_t>(stream));
}

rfr_status rfr_filter_gather(const float *signal, const rfr_antennas *ants, int64_t n_ant_total,
                             const rfr_freq_grid *grid, const float *qx, const float *qy,
                             const float *qz, int64_t n_query, float *power, float *mf,
                             const rfr_comm *comm, const rfr_workspace *ws, rfr_stream_t stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!comm) {
    if (!power && n_query > 0) return RFR_E_ARG;
    return filter_impl(signal, ants, grid, qx, qy, qz, n_query, power, mf, nullptr, ws, st);
  }
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  if (ants->rx_x || ants->phi_tx || n_ant_total < 0 || n_query < 0) return RFR_E_ARG;
  const int N = comm->nranks, r = comm->rank;
  auto shard = [&](int64_t n, int k, int64_t &lo, int64_t &hi) {
    const int64_t base = n / N, rem = n % N;
    lo = k * base + std::min<int64_t>(k, rem);
    hi = lo + base + (k < rem ? 1 : 0);
  };
  int64_t alo, ahi;
  shard(n_ant_total, r, alo, ahi);
  if (ants->n_ant != ahi - alo) return RFR_E_SHAPE;
  Layout L;
  RFR_TRY(check_ws(ws, 0, n_query, L, n_ant_total, grid->n_freq));
  int64_t qlo, qhi;
  shard(n_query, r, qlo, qhi);
  if (qhi > qlo && !power) return RFR_E_ARG;
  float2 *gsig = at<float2>(ws, L.off_gsig);
  float *gant = at<float>(ws, L.off_gant);        // [3][n_ant_total]
  // all-gather by one broadcast per rank (exact, contiguous slices; concurrent in the group)
  if (ncclGroupStart() != ncclSuccess) return RFR_E_NCCL;
  for (int k = 0; k < N; ++k) {
    int64_t lo, hi;
    shard(n_ant_total, k, lo, hi);
    if (hi == lo) continue;
    const size_t nrow = (size_t)(hi - lo);
    const bool me = k == r;
    ncclBroadcast(me ? (const void *)signal : nullptr, gsig + lo * grid->n_freq,
                  nrow * grid->n_freq * 2, ncclFloat32, k, comm->nccl, st);
    const float *src[3] = {ants->tx_x, ants->tx_y, ants->tx_z};
    for (int c = 0; c < 3; ++c)
      ncclBroadcast(me ? (const void *)src[c] : nullptr, gant + c * n_ant_total + lo, nrow,
                    ncclFloat32, k, comm->nccl, st);
  }
  if (ncclGroupEnd() != ncclSuccess) return RFR_E_NCCL;
  if (qhi == qlo) return RFR_OK;
  rfr_antennas all;
  memset(&all, 0, sizeof(all));
  all.tx_x = gant; all.tx_y = gant + n_ant_total; all.tx_z = gant + 2 * n_ant_total;
  all.n_ant = n_ant_total;
  return filter_impl(reinterpret_cast<const float *>(gsig), &all, grid, qx + qlo, qy + qlo,
                     qz + qlo, qhi - qlo, power, mf, nullptr, ws, st);
}

rfr_status rfr_filter_partial(const float *signal, const rfr_antennas *ants,
                              const rfr_freq_grid *grid, const float *qx, const float *qy,
                              const float *qz, int64_t n_query, float *mf,
                              const rfr_workspace *ws, rfr_stream_t stream) {
  if (!mf && n_query > 0) return RFR_E_ARG;
  return filter_impl(signal, ants, grid, qx, qy, qz, n_query, nullptr, mf, nullptr, ws,
                     reinterpret_cast<cudaStream_t>(stream));
}

rfr_status rfr_filter_power(const float *mf, int64_t n_query, float *power, rfr_stream_t stream) {
  if (n_query < 0 || (n_query > 0 && (!mf || !power))) return RFR_E_ARG;
  if (n_query == 0) return RFR_OK;
  RFR_CU(launch_abs(mf, n_query, power, device_sms(), reinterpret_cast<cudaStream_t>(stream)));
  return RFR_OK;
}

rfr_status rfr_backward_partial(const float *grad_signal, const rfr_samples *samples,
                                float sharpness, const rfr_antennas *ants,
                                const rfr_freq_grid *grid, const rfr_opts *opts, float *partials,
                                const rfr_workspace *ws, rfr_stream_t stream) {
  RFR_TRY(check_samples(samples));
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  if (!(sharpness > 0.f) || !partials || (ants->n_ant > 0 && !grad_signal)) return RFR_E_ARG;
  const uint32_t flags = opts ? opts->flags : 0u;
  const int64_t n_s = samples->n_rays * (int64_t)samples->n_per_ray;
  Layout L;
  RFR_TRY(check_ws(ws, n_s, 0, L, ants->n_ant, grid->n_freq));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n_s == 0) return RFR_OK;
  RFR_TRY(run_blend(samples, sharpness, flags, ws, L, st));
  const Split sp = adj_split(n_s, ants->n_ant, 5, L.cap_bwdp);
  AdjArgs a;
  memset(&a, 0, sizeof(a));
  a.rec = at<Rec>(ws, L.off_rec);
  a.n_s = n_s;
  a.tx_x = ants->tx_x; a.tx_y = ants->tx_y; a.tx_z = ants->tx_z;
  a.rx_x = ants->rx_x; a.rx_y = ants->rx_y; a.rx_z = ants->rx_z;
  a.phi_tx = ants->phi_tx; a.phi_rx = ants->phi_rx;
  a.n_a = ants->n_ant;
  a.n_f = grid->n_freq;
  a.k0 = grid->f0_hz / kC;
  a.kd = grid->df_hz / kC;
  a.X = reinterpret_cast<const float2 *>(grad_signal);
  a.bprep = at<unsigned char>(ws, L.off_bprep);
  a.bprep_cap = L.total - L.off_bprep;
  a.ants_per_split = sp.per_split;
  a.out = sp.splits > 1 ? at<float>(ws, L.off_bwdp) : partials;
  a.flags = at<unsigned>(ws, 0);
  a.no_gain = (flags & RFR_NO_GAIN) != 0;
  const bool mono = ants->rx_x == nullptr;
  // Chebyshev-moment adjoint (rfr_cheb.cu), chosen on the device; the direct kernels return at
  // once when it runs
  // Chebyshev adjoint over the samples with alpha != 0 only (DESIGN 5c): the others' partials are
  // zero (their gradients vanish or carry sigma(-s f) factors below the fp32 range)
  const bool corr = has_corr(samples, ants);
  const bool cheb = ants->n_ant > 0;
  Rec *rec_c = at<Rec>(ws, L.off_recc);
  int *idx_c = at<int>(ws, L.off_idxc);
  int64_t *n_act = at<int64_t>(ws, kActiveBwdOff);
  if (cheb && use_v2(ants, corr, flags)) {
    // r2 engine: plan over the alpha != 0 samples, Horner coefficients of G, backward sweep
    RFR_CU(launch_compact(a.rec, n_s, corr, at<int>(ws, L.off_ccnt), n_act, rec_c, st,
                          at<unsigned char>(ws, L.off_aflag), idx_c));
    const T2Args t = make_t2(ants, grid, ws, L);
    const T2Sorted v = make_view(ws, L, 0, t2_backward_chunk());
    T2Points pts;
    memset(&pts, 0, sizeof(pts));
    pts.rec = rec_c; pts.n_dev = n_act; pts.n = n_s;
    RFR_CU(t2_plan(t, pts, v, kT2PlanAdjoint, st));
    RFR_CU(t2_prep_adjoint(t, v.tstart, a.X, nullptr, st));
    RFR_CU(cudaMemsetAsync(partials, 0, (size_t)5 * n_s * 4, st));
    const int S = std::max(1, std::min<int>(L.t2_bwd_splits, (int)cdiv(ants->n_ant, 1024)));
    const int64_t aps = cdiv(cdiv(ants->n_ant, S), 16) * 16;
    RFR_CU(t2_backward(t, v, 0, idx_c, n_act, n_s, at<float>(ws, L.off_t2bwdp), partials, n_s, S,
                       aps, a.no_gain, device_sms(), st));
    a.skip = t.skip;                                   // direct fallback: no-op when planned
    a.gated = true;                                    // ... on one short persistent wave
    RFR_CU(launch_adjoint(a, kModeBwd, mono, corr, sp.splits, st));
    if (sp.splits > 1)
      RFR_CU(launch_sum_splits(at<float>(ws, L.off_bwdp), sp.splits, 5 * n_s, partials,
                               device_sms(), st, t.skip));
    return RFR_OK;
  }
  ChebArgs c = make_cheb(rec_c, n_s, ants, grid, a.no_gain, ws, L, 0, (flags & RFR_DIRECT) != 0);
  c.n_dev = n_act;
  c.idx = idx_c;
  if (cheb) {
    RFR_CU(launch_compact(a.rec, n_s, corr, at<int>(ws, L.off_ccnt), n_act, rec_c, st,
                          at<unsigned char>(ws, L.off_aflag), idx_c));
    RFR_CU(launch_cheb_prepare(c, at<double>(ws, L.off_cbox), st));
    a.skip = c.hdr;
    RFR_CU(cudaMemsetAsync(a.out, 0, (size_t)sp.splits * 5 * n_s * 4, st));
  }
  RFR_CU(launch_adjoint(a, kModeBwd, mono, corr, sp.splits, st));
  if (cheb) {
    if (tile_enabled()) {
      TileArgs tb = make_tile(nullptr, nullptr, nullptr, n_s, ants, grid, c, a.X, nullptr,
                              sp.per_split, ws, L);
      tb.rec = rec_c;
      tb.n_dev = n_act;
      tb.idx = idx_c;
      tb.rs = at<Rec>(ws, L.off_trs);
      RFR_CU(launch_tiled_backward(tb, a, mono, corr, sp.splits, st));
    } else {
      AdjArgs ab = a;
      ab.rec = rec_c;
      RFR_CU(launch_cheb_adj(c, ab, at<float2>(ws, L.off_cbadj), kModeBwd, mono, corr,
                             sp.splits, st));
    }
  }
  if (sp.splits > 1)
    RFR_CU(launch_sum_splits(at<float>(ws, L.off_bwdp), sp.splits, 5 * n_s, partials,
                             device_sms(), st));
  return RFR_OK;
}

rfr_status rfr_backward_finish(const float *partials, const rfr_samples *samples, float sharpness,
                               const rfr_opts *opts, const rfr_sample_grads *out,
                               const rfr_workspace *ws, rfr_stream_t stream) {
  RFR_TRY(check_samples(samples));
  if (!(sharpness > 0.f) || !partials || !out || !out->sdf || !out->refl || !out->nx ||
      !out->ny || !out->nz || !out->power || !out->sharpness)
    return RFR_E_ARG;
  const uint32_t flags = opts ? opts->flags : 0u;
  const int64_t n_s = samples->n_rays * (int64_t)samples->n_per_ray;
  Layout L;
  RFR_TRY(check_ws(ws, n_s, 0, L));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  RFR_TRY(run_blend(samples, sharpness, flags, ws, L, st));
  BlendBwdArgs b;
  b.sdf = samples->sdf; b.refl = samples->refl; b.power = samples->power;
  b.rec = at<Rec>(ws, L.off_rec);
  b.partials = partials;
  b.n_rays = samples->n_rays; b.n_s = n_s; b.n_per_ray = samples->n_per_ray;
  b.s = sharpness;
  b.g_sdf = out->sdf; b.g_refl = out->refl; b.g_nx = out->nx; b.g_ny = out->ny; b.g_nz = out->nz;
  b.g_power = out->power;
  b.ds_part = at<float>(ws, L.off_ds);
  RFR_CU(launch_blend_bwd(b, st));
  RFR_CU(launch_reduce_sum(b.ds_part, samples->n_rays, at<float>(ws, L.off_tmp), kTmpN,
                           out->sharpness, st));
  return RFR_OK;
}

rfr_status rfr_backward(const float *grad_signal, const rfr_samples *samples, float sharpness,
                        const rfr_antennas *ants, const rfr_freq_grid *grid, const rfr_opts *opts,
                        const rfr_sample_grads *out, const rfr_comm *comm,
                        const rfr_workspace *ws, rfr_stream_t stream) {
  RFR_TRY(check_samples(samples));
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  const int64_t n_s = samples->n_rays * (int64_t)samples->n_per_ray;
  Layout L;
  RFR_TRY(check_ws(ws, n_s, 0, L));
  float *part = at<float>(ws, L.off_bwds);
  RFR_TRY(rfr_backward_partial(grad_signal, samples, sharpness, ants, grid, opts, part, ws,
                               stream));
  // a7: sum the per-sample partials over the antenna shards
  RFR_TRY(allreduce_sum(comm, part, 5 * n_s, reinterpret_cast<cudaStream_t>(stream)));
  rfr_opts o2;
  o2.flags = (opts ? opts->flags : 0u) | RFR_REUSE_BLEND;   // K1 ran in the partial call
  return rfr_backward_finish(part, samples, sharpness, &o2, out, ws, stream);
}

rfr_status rfr_backward_filter_partial(const float *grad_signal, const float *signal,
                                       const rfr_samples *samples, float sharpness,
                                       const rfr_antennas *ants, const rfr_freq_grid *grid,
                                       const rfr_opts *opts, float *partials, float *mf,
                                       const rfr_workspace *ws, rfr_stream_t stream) {
  RFR_TRY(check_samples(samples));
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  if (!(sharpness > 0.f) || (ants->n_ant > 0 && (!grad_signal || !signal))) return RFR_E_ARG;
  const uint32_t flags = opts ? opts->flags : 0u;
  const int64_t n_s = samples->n_rays * (int64_t)samples->n_per_ray;
  if (n_s > 0 && (!partials || !mf)) return RFR_E_ARG;
  Layout L;
  RFR_TRY(check_ws(ws, n_s, n_s, L, ants->n_ant, grid->n_freq));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n_s == 0) return RFR_OK;
  RFR_TRY(run_blend(samples, sharpness, flags, ws, L, st));
  // one split count for both partial sets: the backward's (5 floats per sample) is the tighter
  const Split sp = adj_split(n_s, ants->n_ant, 5, std::min(L.cap_bwdp, L.cap_fltp * 5 / 2));
  AdjArgs a;
  memset(&a, 0, sizeof(a));
  a.rec = at<Rec>(ws, L.off_rec);
  a.n_s = n_s;
  a.tx_x = ants->tx_x; a.tx_y = ants->tx_y; a.tx_z = ants->tx_z;
  a.rx_x = ants->rx_x; a.rx_y = ants->rx_y; a.rx_z = ants->rx_z;
  a.phi_tx = ants->phi_tx; a.phi_rx = ants->phi_rx;
  a.n_a = ants->n_ant;
  a.n_f = grid->n_freq;
  a.k0 = grid->f0_hz / kC;
  a.kd = grid->df_hz / kC;
  a.X = reinterpret_cast<const float2 *>(grad_signal);
  a.X2 = reinterpret_cast<const float2 *>(signal);
  a.qx = samples->x; a.qy = samples->y; a.qz = samples->z;   // SIMT fallback's filter queries
  a.bprep = at<unsigned char>(ws, L.off_bprep);
  a.bprep_cap = L.total - L.off_bprep;
  a.ants_per_split = sp.per_split;
  a.out = sp.splits > 1 ? at<float>(ws, L.off_bwdp) : partials;
  a.out2 = sp.splits > 1 ? at<float>(ws, L.off_fltp) : mf;
  a.flags = at<unsigned>(ws, 0);
  a.no_gain = (flags & RFR_NO_GAIN) != 0;
  const bool mono = ants->rx_x == nullptr;
  // Chebyshev path: the filter over every sample (row 1 of B = the signal), the backward over the
  // samples with alpha != 0 only (row 0 = G, compacted list, DESIGN 5c)
  const bool corr = has_corr(samples, ants);
  const bool cheb = ants->n_ant > 0;
  if (cheb && use_v2(ants, corr, flags)) {
    // r2 engine: one plan over every sample (the filter's queries), Horner coefficients of both
    // rows (G and s), the filter sweep over all samples and the backward sweep over the alpha != 0
    // samples sorted into the same tiles
    const T2Args t = make_t2(ants, grid, ws, L);
    const T2Sorted v0 = make_view(ws, L, 0, t2_filter_chunk()), v1 = make_view(ws, L, 1, t2_backward_chunk());
    T2Points all;
    memset(&all, 0, sizeof(all));
    all.qx = samples->x; all.qy = samples->y; all.qz = samples->z; all.n = n_s;
    RFR_CU(t2_plan(t, all, v0, kT2PlanAdjoint, st));
    // the alpha != 0 samples sorted into the plan's tiles first: row G's coefficients are prepared
    // only for the tiles that hold one
    Rec *rec_c = at<Rec>(ws, L.off_recc);
    int *idx_c = at<int>(ws, L.off_idxc);
    int64_t *n_act = at<int64_t>(ws, kActiveBwdOff);
    RFR_CU(launch_compact(a.rec, n_s, corr, at<int>(ws, L.off_ccnt), n_act, rec_c, st,
                          at<unsigned char>(ws, L.off_aflag), idx_c));
    T2Points act;
    memset(&act, 0, sizeof(act));
    act.rec = rec_c; act.n_dev = n_act; act.n = n_s;
    RFR_CU(t2_sort(t, act, v1, st));
    RFR_CU(t2_prep_adjoint(t, v0.tstart, a.X, a.X2, st, v1.tstart));
    const int Sf = t2_flt_splits(n_s, t2_filter_chunk(), ants->n_ant, L.t2_flt_cap);
    const int64_t apf = cdiv(cdiv(ants->n_ant, Sf), 16) * 16;
    float2 *o = reinterpret_cast<float2 *>(Sf > 1 ? at<float>(ws, L.off_t2fltp) : mf);
    RFR_CU(t2_filter(t, v0, 1, o, n_s, Sf, apf, device_sms(), st));
    if (Sf > 1) RFR_CU(t2_sum_splits(t, at<float>(ws, L.off_t2fltp), Sf, n_s * 2, mf, device_sms(), st));
    RFR_CU(cudaMemsetAsync(partials, 0, (size_t)5 * n_s * 4, st));
    const int Sb = std::max(1, std::min<int>(L.t2_bwd_splits, (int)cdiv(ants->n_ant, 1024)));
    const int64_t apb = cdiv(cdiv(ants->n_ant, Sb), 16) * 16;
    RFR_CU(t2_backward(t, v1, 0, idx_c, n_act, n_s, at<float>(ws, L.off_t2bwdp), partials, n_s,
                       Sb, apb, a.no_gain, device_sms(), st));
    a.skip = t.skip;                                   // direct fallback: no-op when planned
    a.gated = true;                                    // ... on one short persistent wave
    RFR_CU(launch_adjoint(a, kModeBoth, mono, corr, sp.splits, st));
    if (sp.splits > 1) {
      RFR_CU(launch_sum_splits(at<float>(ws, L.off_bwdp), sp.splits, 5 * n_s, partials,
                               device_sms(), st, t.skip));
      RFR_CU(launch_sum_splits(at<float>(ws, L.off_fltp), sp.splits, 2 * n_s, mf, device_sms(),
                               st, t.skip));
    }
    return RFR_OK;
  }
  const ChebArgs c = make_cheb(a.rec, n_s, ants, grid, a.no_gain, ws, L, 0,
                               (flags & RFR_DIRECT) != 0);
  if (cheb) {
    RFR_CU(launch_cheb_prepare(c, at<double>(ws, L.off_cbox), st));
    a.skip = c.hdr;
    // the compacted backward leaves the inactive samples' partials at zero (the direct sweep, if
    // the device chooses it, overwrites every entry)
    RFR_CU(cudaMemsetAsync(a.out, 0, (size_t)sp.splits * 5 * n_s * 4, st));
  }
  RFR_CU(launch_adjoint(a, kModeBoth, mono, corr, sp.splits, st));
  if (cheb) {
    float2 *bmom = at<float2>(ws, L.off_cbadj);
    ChebArgs cf = c;
    cf.row = 1;
    AdjArgs af = a;
    af.out = a.out2;
    const bool tiled = tile_enabled();
    if (tiled) {
      const TileArgs ta = make_tile(samples->x, samples->y, samples->z, n_s, ants, grid, c, a.X2,
                                    reinterpret_cast<float2 *>(a.out2), sp.per_split, ws, L);
      RFR_CU(launch_tiled_filter(ta, mono, sp.splits, st));
    } else {
      RFR_CU(launch_cheb_flt(cf, af, bmom, mono, sp.splits, st, 2));
    }
    Rec *rec_c = at<Rec>(ws, L.off_recc);
    int *idx_c = at<int>(ws, L.off_idxc);
    int64_t *n_act = at<int64_t>(ws, kActiveBwdOff);
    RFR_CU(launch_compact(a.rec, n_s, corr, at<int>(ws, L.off_ccnt), n_act, rec_c, st,
                          at<unsigned char>(ws, L.off_aflag), idx_c));
    if (tiled) {
      TileArgs tb = make_tile(nullptr, nullptr, nullptr, n_s, ants, grid, c, a.X, nullptr,
                              sp.per_split, ws, L);
      tb.rec = rec_c;
      tb.n_dev = n_act;
      tb.idx = idx_c;
      tb.rs = at<Rec>(ws, L.off_trs);
      RFR_CU(launch_tiled_backward(tb, a, mono, corr, sp.splits, st));
    } else {
      ChebArgs cb = c;
      cb.rec = rec_c;
      cb.n_dev = n_act;
      cb.idx = idx_c;
      cb.row = 0;
      AdjArgs ab = a;
      ab.rec = rec_c;
      RFR_CU(launch_cheb_adj(cb, ab, bmom, kModeBwd, mono, corr, sp.splits, st, -1));
    }
  }
  if (sp.splits > 1) {
    RFR_CU(launch_sum_splits(at<float>(ws, L.off_bwdp), sp.splits, 5 * n_s, partials,
                             device_sms(), st));
    RFR_CU(launch_sum_splits(at<float>(ws, L.off_fltp), sp.splits, 2 * n_s, mf, device_sms(),
                             st));
  }
  return RFR_OK;
}

rfr_status rfr_backward_filter(const float *grad_signal, const float *signal,
                               const rfr_samples *samples, float sharpness,
                               const rfr_antennas *ants, const rfr_freq_grid *grid,
                               const rfr_opts *opts, const rfr_sample_grads *out, float *power,
                               float *mf, const rfr_comm *comm, const rfr_workspace *ws,
                               rfr_stream_t stream) {
  RFR_TRY(check_samples(samples));
  if (!out) return RFR_E_ARG;
  const uint32_t flags = opts ? opts->flags : 0u;
  const int64_t n_s = samples->n_rays * (int64_t)samples->n_per_ray;
  if (n_s > 0 && !power) return RFR_E_ARG;
  Layout L;
  RFR_TRY(check_ws(ws, n_s, n_s, L));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  float *part = at<float>(ws, L.off_bwds);
  float *M = mf ? mf : at<float>(ws, L.off_fltm);
  RFR_TRY(rfr_backward_filter_partial(grad_signal, signal, samples, sharpness, ants, grid, opts,
                                      part, M, ws, stream));
  // a7 and the filter's shard sum
  RFR_TRY(allreduce_sum(comm, part, 5 * n_s, st));
  RFR_TRY(allreduce_sum(comm, M, 2 * n_s, st));
  if (n_s > 0) RFR_CU(launch_abs(M, n_s, power, device_sms(), st));
  rfr_opts o2;
  o2.flags = flags | RFR_REUSE_BLEND;                 // K1 ran in the partial call
  return rfr_backward_finish(part, samples, sharpness, &o2, out, ws, stream);
}

rfr_status rfr_filter_backward(const float *grad_power, const float *mf, const float *power,
                               float eps, const rfr_antennas *ants, const rfr_freq_grid *grid,
                               const float *qx, const float *qy, const float *qz, int64_t n_query,
                               float *grad_signal, const rfr_workspace *ws,
                               rfr_stream_t stream) {
  RFR_TRY(check_ants(ants));
  RFR_TRY(check_grid(grid));
  if (n_query < 0 || !(eps >= 0.f) || (ants->n_ant > 0 && !grad_signal) ||
      (n_query > 0 && (!grad_power || !mf || !qx || !qy || !qz)))
    return RFR_E_ARG;
  if (ants->phi_tx || ants->phi_rx) return RFR_E_ARG;      // the filter has no transmittance
  Layout L;
  RFR_TRY(check_ws(ws, 0, n_query, L, ants->n_ant, grid->n_freq));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (ants->n_ant == 0) return RFR_OK;
  Rec *qrec = at<Rec>(ws, L.off_qrec);
  RFR_CU(launch_mf_adj_pack(grad_power, mf, power, eps, qx, qy, qz, n_query, qrec, device_sms(),
                            st));
  if (use_v2(ants, false, 0)) {
    // r2 engine: plan over the queries, tiled moments of the K5 weights c_q -> bins
    const T2Args t = make_t2(ants, grid, ws, L);
    const T2Sorted v = make_view(ws, L, 0, kT2FltChunk);
    T2Points pts;
    memset(&pts, 0, sizeof(pts));
    pts.rec = qrec; pts.n = n_query;
    RFR_CU(t2_plan(t, pts, v, kT2PlanForward, st));
    RFR_CU(t2_forward(t, v, kFwdMFAdj, false, reinterpret_cast<float2 *>(grad_signal),
                      device_sms(), st));
    return run_fwd(qrec, n_query, ants, grid, false, false, kFwdMFAdj, grad_signal, ws, L, st,
                   nullptr, nullptr, false, t.skip);
  }
  return run_fwd(qrec, n_query, ants, grid, false, false, kFwdMFAdj, grad_signal, ws, L, st);
}

rfr_status rfr_heatmap_loss(const float *power, const float *power_gt, int64_t n_query,
                            const int32_t *cell, float *history, float thr_hi, float ratio,
                            float *grad_power, uint8_t *mask, float *loss,
                            const rfr_workspace *ws, rfr_stream_t stream) {
  if (n_query < 0 || !loss || (n_query > 0 && (!power || !power_gt || !grad_power)) ||
      ((history == nullptr) != (cell == nullptr)))
    return RFR_E_ARG;
  Layout L;
  RFR_TRY(check_ws(ws, 0, 0, L));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  RFR_CU(launch_heat_loss(power, power_gt, n_query, cell, history, thr_hi, ratio, grad_power, mask,
                          at<float>(ws, L.off_tmp), kTmpN, loss, st));
  return RFR_OK;
}

rfr_status rfr_plan_state(const rfr_workspace *ws, rfr_plan_info *out, rfr_stream_t stream) {
  if (!ws || !ws->ptr || !out) return RFR_E_ARG;
  Layout L;
  RFR_TRY(check_ws(ws, 0, 0, L));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  T2Plan pl;
  ChebHdr sk;
  if (cudaMemcpyAsync(&pl, at<T2Plan>(ws, L.off_t2plan), sizeof(pl), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(&sk, at<ChebHdr>(ws, kT2SkipOff), sizeof(sk), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return RFR_E_CUDA;
  out->applied = sk.sel ? 1 : 0;
  out->tiles = pl.T;
  out->lx = pl.L[0]; out->ly = pl.L[1]; out->lz = pl.L[2];
  out->P = pl.P;
  out->Pg = pl.Pg;
  out->n_points = pl.n_pts;
  out->delta_t = pl.delta_t;
  out->delta_g = pl.delta_g;
  return RFR_OK;
}

rfr_status rfr_profile_enable(int on) {
  t2_profile_enable(on != 0);
  return RFR_OK;
}

rfr_status rfr_profile_read(int32_t sweep, double *ms, uint64_t *launches) {
  if (!ms || !launches || sweep < 0 || sweep >= kT2ProfSlots) return RFR_E_ARG;
  unsigned long long n = 0;
  t2_profile_read(sweep, ms, &n);
  *launches = (uint64_t)n;
  return RFR_OK;
}

rfr_status rfr_poll_flags(const rfr_workspace *ws, uint32_t *flags, rfr_stream_t stream) {
  if (!ws || !ws->ptr || !flags) return RFR_E_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // read and clear on the caller's stream, after every kernel queued there before this call
  uint32_t v = 0;
  if (cudaMemcpyAsync(&v, ws->ptr, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) return RFR_E_CUDA;
  if (cudaMemsetAsync(ws->ptr, 0, 4, st) != cudaSuccess) return RFR_E_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return RFR_E_CUDA;
  *flags = v;
  return RFR_OK;
}

}  // extern "C"
