// rfr_tiled.cu -- the r2 tiled engine (see rfr_tiled.h).
//
// Every sweep of the hot path sums, per (point q, antenna i), a phasor over the N_f uniform bins
// (Eq. 3 P:L182-187 filter, Eq. 4 P:L231-234 forward, App. A.5 P:L725-728 adjoint).  With the delay
// in cycles per bin u = L df / c (L = 2 d monostatic), the centred bins m' = m - N/2 and the centre
// frequency f_c = f0 + (N/2) df, the adjoint bin sum is E * F_i(u) with E = e^{+j 2 pi f_c tau} and
//     F_i(u) = sum_m X_i[m] e^{+j 2 pi m' u},
// a band-limited function that varies by only a few cycles over the delays of one spatial tile.
// On a tile t (delay interval u_c,it +- delta_t, x = (u - u_c,it) / delta_t in [-1, 1]) it is a
// polynomial of degree P - 1 in x up to the Chebyshev interpolation error (<= 2 x the Jacobi-Anger
// tail, < 2e-7 of sum |X| by the P rule).  The filter / backward sweeps evaluate that polynomial by
// Horner from monomial coefficients (one FFMA2 per coefficient and point; the monomial form is
// well conditioned here because sum_j |c_j| <= e^{z} sum |X| with z = 2 pi (N/2 + 1) delta_t <= 4.8).
// The coefficients come from P values of F_i at the tile's Chebyshev nodes, evaluated through one
// global expansion per antenna, F_i(u) = sum_q G_i[q] T_q((u - u_g,i) / delta_g) (Jacobi-Anger,
// Pg <= 48 terms), so the per-(antenna, tile) preparation costs P * Pg instead of P * N_f.
// The forward runs the transpose: per-(antenna, tile) Chebyshev moments of the tile's points, P
// virtual sources per tile at the nodes (weights = Lagrange interpolation of the moments), their
// global moments and the bins a[m][q] Mg[q].  All sums are fixed-order (no float atomics).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "rfr_device.cuh"
#include "rfr_launch.h"
#include "rfr_tiled.h"

namespace rfr {

// ------------------------------------------------------------ per-sweep device-time profiling
// (rfr_profile_enable / rfr_profile_read): CUDA events recorded on the launching stream around
// each sweep launch while enabled; read back (synchronising on the stop events) on request.
namespace {
struct ProfPending {
  int id;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfPending> g_prof_pending;
std::vector<cudaEvent_t> g_prof_pool;
double g_prof_ms[kT2ProfSlots];
unsigned long long g_prof_n[kT2ProfSlots];
cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_drain() {                 // caller holds g_prof_mu
  for (auto &p : g_prof_pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      g_prof_ms[p.id] += ms;
      g_prof_n[p.id] += 1;
    }
    g_prof_pool.push_back(p.a);
    g_prof_pool.push_back(p.b);
  }
  g_prof_pending.clear();
}
}  // namespace

ProfScope::ProfScope(int id, cudaStream_t st) : st_(st), id_(-1), a_(nullptr) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  id_ = id;
  a_ = prof_event();
  cudaEventRecord(static_cast<cudaEvent_t>(a_), st_);
}
ProfScope::~ProfScope() {
  if (id_ < 0) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEvent_t b = prof_event();
  cudaEventRecord(b, st_);
  g_prof_pending.push_back({id_, static_cast<cudaEvent_t>(a_), b});
  if (g_prof_pending.size() > 4096) prof_drain();
}
void t2_profile_enable(bool on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  prof_drain();
  if (on)
    for (int k = 0; k < kT2ProfSlots; ++k) { g_prof_ms[k] = 0.0; g_prof_n[k] = 0; }
  g_prof_on = on;
}
void t2_profile_read(int id, double *ms, unsigned long long *n) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  prof_drain();
  *ms = (id >= 0 && id < kT2ProfSlots) ? g_prof_ms[id] : 0.0;
  *n = (id >= 0 && id < kT2ProfSlots) ? g_prof_n[id] : 0ull;
}

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr float kInv16Pi2f = 0.00633257759406206f;   // 1 / (4 pi)^2 (Q3)
constexpr float kSqrt2f = 1.41421356237309505f;

// ------------------------------------------------------------------ packed f32x2 helpers
__device__ __forceinline__ f2x bcv(float v) { return pk(v, v); }
__device__ __forceinline__ float rsq_ftz(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float rcp_ftz_(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ void sc_ftz(float v, float &s, float &c) {
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(v));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(v));
}
__device__ __forceinline__ float rni(float v) {
  float r;
  asm("cvt.rni.f32.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// per-tile expansions: truncation tail sum_{p >= P} eps_p |J_p(z)| < 1e-5 -- below the per-pair
// phase error of the sweeps' unreduced fp32 carrier angle (~2e-5 rad at c3, t2_geo1), so the
// truncation never dominates a pair's error (DESIGN 5e, Q28; tests/test_cheb_math.py pins the rule).
// z stays <= 4.812 (the round-1 limit): the fp32 rounding of the monomial (Horner) evaluation is
// bounded by eps e^z sum|X|.  The global expansion (t2_select_Pg) keeps the 1e-7 rule: its error
// enters every tile.
__host__ __device__ inline int t2_select_P(double z) {
  if (z <= 1.632) return 8;
  if (z <= 2.681) return 10;
  if (z <= 3.866) return 12;
  if (z <= 4.812) return 14;
  return 0;
}
__device__ inline int t2_select_Pg(double z) {
  if (z <= 4.812) return 16;
  if (z <= 7.33) return 20;
  if (z <= 10.061) return 24;
  if (z <= 12.946) return 28;
  if (z <= 15.948) return 32;
  if (z <= 28.6) return 48;
  return 0;
}

// distance range [dmin, dmax] from a point to an axis-aligned box (fp64)
__device__ __forceinline__ void t2_box_dist(const float *b, double px, double py, double pz,
                                            double &dmin, double &dmax) {
  const double p[3] = {px, py, pz};
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
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

__device__ __forceinline__ int64_t t2_count(const T2Points &p) { return p.n_dev ? *p.n_dev : p.n; }
__device__ __forceinline__ float3 t2_pos(const T2Points &p, int64_t j) {
  if (p.rec) {
    const Rec &r = p.rec[j];
    return make_float3((float)r.x, (float)r.y, (float)r.z);
  }
  return make_float3(p.qx[j], p.qy[j], p.qz[j]);
}

// tile of a position in the plan's grid
__device__ __forceinline__ int t2_tile_of(const T2Plan &pl, float3 q) {
  const float v[3] = {q.x, q.y, q.z};
  int id = 0;
#pragma unroll
  for (int c = 2; c >= 0; --c) {
    const float lo = pl.gbox[c], w = pl.gbox[3 + c] - lo;
    int k = w > 0.f ? (int)((v[c] - lo) / w * (float)pl.L[c]) : 0;
    k = min(max(k, 0), pl.L[c] - 1);
    id = id * pl.L[c] + k;
  }
  return id;
}

// fp32 centre of a tile's tight box (the same rounding wherever it is used)
__device__ __forceinline__ float t2_centre(const float *tb, int c) { return 0.5f * (tb[c] + tb[3 + c]); }

// ================================================================================= plan
__global__ void __launch_bounds__(256) k2_box(T2Points p, float *part, unsigned long long *cand) {
  if (blockIdx.x == 0 && threadIdx.x < 128) cand[threadIdx.x] = 0ull;   // k2_cand's maxima
  const int64_t n = t2_count(p);
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float3 q = t2_pos(p, j);
    lo[0] = fminf(lo[0], q.x); hi[0] = fmaxf(hi[0], q.x);
    lo[1] = fminf(lo[1], q.y); hi[1] = fmaxf(hi[1], q.y);
    lo[2] = fminf(lo[2], q.z); hi[2] = fmaxf(hi[2], q.z);
  }
  __shared__ float sh[6][256];
  for (int c = 0; c < 3; ++c) { sh[c][threadIdx.x] = lo[c]; sh[3 + c][threadIdx.x] = hi[c]; }
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int c = 0; c < 3; ++c) {
        sh[c][threadIdx.x] = fminf(sh[c][threadIdx.x], sh[c][threadIdx.x + s]);
        sh[3 + c][threadIdx.x] = fmaxf(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

// candidate grids: L_c in {1, 2, 4, 8, 16} per axis, T <= kT2Max
constexpr int kT2Cand = 125;
__device__ __forceinline__ void t2_cand(int c, int L[3]) {
  L[0] = 1 << (c % 5);
  L[1] = 1 << ((c / 5) % 5);
  L[2] = 1 << (c / 25);
}
constexpr int kT2SubAnts = 32;

// kT2CandSlices CTAs per candidate grid: max over its cells and a subsample of the antennas of the
// delay half-spread (cell boxes bound the tight boxes from above), combined over the slices by an
// order-independent atomicMax on the fp64 bits (non-negative); k2_pick turns it into P and a cost
constexpr int kT2CandSlices = 4;
__global__ void __launch_bounds__(256) k2_cand(const float *part, int nblk, T2Args a,
                                               unsigned long long *hmax_bits) {
  __shared__ float box[6];
  __shared__ double red[256];
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int b = 0; b < nblk; ++b) {
      const float u = part[b * 6 + threadIdx.x];
      v = threadIdx.x < 3 ? fminf(v, u) : fmaxf(v, u);
    }
    box[threadIdx.x] = v;
  }
  __syncthreads();
  const int cidx = blockIdx.x % kT2Cand, slice = blockIdx.x / kT2Cand;
  int L[3];
  t2_cand(cidx, L);
  const int T = L[0] * L[1] * L[2];
  double hmax = 0.0;
  if (T <= kT2Max && box[0] <= box[3]) {
    const int ns = (int)(a.n_a < kT2SubAnts ? a.n_a : kT2SubAnts);
    for (int w = slice * blockDim.x + threadIdx.x; w < T * ns; w += kT2CandSlices * blockDim.x) {
      const int t = w / ns, k = w % ns;
      const int64_t i = ns > 1 ? (int64_t)k * (a.n_a - 1) / (ns - 1) : 0;
      const int cx = t % L[0], cy = (t / L[0]) % L[1], cz = t / (L[0] * L[1]);
      const int cc[3] = {cx, cy, cz};
      float cb[6];
      for (int c = 0; c < 3; ++c) {
        const float lo = box[c], wd = (box[3 + c] - box[c]) / (float)L[c];
        cb[c] = lo + wd * (float)cc[c];
        cb[3 + c] = lo + wd * (float)(cc[c] + 1);
      }
      double dmin, dmax;
      t2_box_dist(cb, a.tx_x[i], a.tx_y[i], a.tx_z[i], dmin, dmax);
      hmax = fmax(hmax, dmax - dmin);            // half-spread of L = 2 d
    }
  }
  red[threadIdx.x] = hmax;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(hmax_bits + cidx, (unsigned long long)__double_as_longlong(red[0]));
}

// cost of a candidate grid from its delay half-spread: FMA-pipe cost per antenna (FFMA2 units).
// Adjoint sweeps (kind 0): per point P Horner steps + ~10 for the geometry, partially filled work
// items waste ~half a warp segment (chunk / 8) of lanes per tile (t2_item), plus the per-(tile,
// antenna) preparation; forward (kind 1):
// per record 1.5 P moment steps + ~12, plus per tile P virtual sources through ~32 global moments
// (k2_fout).  T P <= kT2TP (coefficient storage)
__device__ double t2_cand_cost(int T, double hmax, const T2Args &a, int64_t n, int kind,
                               int chunk) {
  const double z = 2.0 * kPi * (double)(a.n_f / 2 + 1) * hmax * a.kd * (1.0 + 1e-6);
  const int P = t2_select_P(z);
  if (P > 0 && T * P <= kT2TP)
    return kind == 0 ? (double)(P + 10) * ((double)n + (double)T * chunk * 0.125) + (double)T * P * 64.0
                     : (1.5 * P + 12.0) * (double)n + (double)T * P * 48.0;
  return 1e300;
}

// pick the cheapest candidate (ties: fewer tiles), write the box and the grid; reset scratch
__global__ void __launch_bounds__(128) k2_pick(const float *part, int nblk,
                                               const unsigned long long *hmax_bits, T2Args a,
                                               T2Plan *pl, int64_t n_pts_host,
                                               const int64_t *n_dev, int kind, int chunk) {
  __shared__ int best;
  __shared__ double cost[kT2Cand];
  __shared__ float bx[6];
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int b = 0; b < nblk; ++b) {
      const float u = part[b * 6 + threadIdx.x];
      v = threadIdx.x < 3 ? fminf(v, u) : fmaxf(v, u);
    }
    bx[threadIdx.x] = v;
  }
  __syncthreads();
  {
    const int64_t n = n_dev ? *n_dev : n_pts_host;
    for (int c = threadIdx.x; c < kT2Cand; c += blockDim.x) {
      int L[3];
      t2_cand(c, L);
      const int T = L[0] * L[1] * L[2];
      cost[c] = (T <= kT2Max && bx[0] <= bx[3])
                    ? t2_cand_cost(T, __longlong_as_double((long long)hmax_bits[c]), a, n, kind, chunk)
                    : 1e300;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = -1;
    double bc = 1e300;
    for (int c = 0; c < kT2Cand; ++c) {
      int L[3];
      t2_cand(c, L);
      const double v = cost[c];
      if (v < bc || (v == bc && b >= 0 && L[0] * L[1] * L[2] < pl->T)) { bc = v; b = c; pl->T = L[0] * L[1] * L[2]; }
    }
    best = b;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int b = 0; b < nblk; ++b) {
      const float u = part[b * 6 + threadIdx.x];
      v = threadIdx.x < 3 ? fminf(v, u) : fmaxf(v, u);
    }
    pl->gbox[threadIdx.x] = v;
  }
  const int64_t n = n_dev ? *n_dev : n_pts_host;
  if (n == 0 && threadIdx.x < 6) pl->gbox[threadIdx.x] = 0.f;   // empty set: a trivial plan
  if (threadIdx.x == 0) {
    int L[3] = {1, 1, 1};
    if (best >= 0) t2_cand(best, L);
    if (n == 0) best = 0;
    pl->L[0] = L[0]; pl->L[1] = L[1]; pl->L[2] = L[2];
    pl->T = L[0] * L[1] * L[2];
    pl->P = best >= 0 ? 1 : 0;              // provisional (k2_select decides)
    pl->n_pts = (int)n;
    pl->dmax_bits = 0ull;
    pl->gmax_bits = 0ull;
    pl->umin_bits = (unsigned long long)__double_as_longlong(1e300);
  }
}

// ------------------------------------------------------------- stable counting sort by tile
// per block of kT2SortBlock points: per-warp counts of each tile (match_any groups), so the order
// inside a tile is the source order (deterministic)
__device__ __forceinline__ void t2_block_counts(const T2Plan &pl, const T2Points &p, int64_t n,
                                                int *wc /* [32][T] */, int T, int &t_out,
                                                bool &ok_out, unsigned &peers_out) {
  const int64_t j = (int64_t)blockIdx.x * kT2SortBlock + threadIdx.x;
  const bool ok = j < n;
  const int t = ok ? t2_tile_of(pl, t2_pos(p, j)) : -1;
  for (int k = threadIdx.x; k < 32 * T; k += blockDim.x) wc[k] = 0;
  __syncthreads();
  const unsigned peers = __match_any_sync(0xffffffffu, t);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (ok && lane == __ffs(peers) - 1) wc[warp * T + t] = __popc(peers);
  __syncthreads();
  t_out = t;
  ok_out = ok;
  peers_out = peers;
}

__global__ void __launch_bounds__(kT2SortBlock) k2_count(const T2Plan *plp, T2Points p,
                                                         T2Sorted s) {
  extern __shared__ int wc[];
  const T2Plan pl = *plp;
  if (pl.P == 0) return;
  const int T = pl.T;
  const int64_t n = t2_count(p);
  if ((int64_t)blockIdx.x * kT2SortBlock >= n) return;
  int t;
  bool ok;
  unsigned peers;
  t2_block_counts(pl, p, n, wc, T, t, ok, peers);
  for (int q = threadIdx.x; q < T; q += blockDim.x) {
    int c = 0;
    for (int w = 0; w < kT2SortBlock / 32; ++w) c += wc[w * T + q];
    s.bcnt[(int64_t)blockIdx.x * kT2Max + q] = c;
  }
}

// thread per tile: exclusive offsets over the blocks, then tile starts and work-item starts
__global__ void __launch_bounds__(kT2Max) k2_scan(const T2Plan *plp, const int64_t *n_dev,
                                                  int64_t n_host, T2Sorted s) {
  __shared__ int tot[kT2Max];
  const T2Plan pl = *plp;
  const int T = pl.P ? pl.T : 0;
  const int64_t n = n_dev ? *n_dev : n_host;
  const int nb = (int)((n + kT2SortBlock - 1) / kT2SortBlock);
  const int q = threadIdx.x;
  if (q < T) {
    // 16 blocks' counts loaded before their offsets are stored: 16 loads in flight instead of a
    // load -> store chain per block (one CTA scans every block of the sort)
    int run = 0;
    int b = 0;
    for (; b + 16 <= nb; b += 16) {
      int c[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) c[u] = s.bcnt[(int64_t)(b + u) * kT2Max + q];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        s.bcnt[(int64_t)(b + u) * kT2Max + q] = run;
        run += c[u];
      }
    }
    for (; b < nb; ++b) {
      const int c = s.bcnt[(int64_t)b * kT2Max + q];
      s.bcnt[(int64_t)b * kT2Max + q] = run;
      run += c;
    }
    tot[q] = run;
  }
  // exclusive scans over the tiles of the point counts and the work-item counts (warp shuffles,
  // then the warp totals)
  __shared__ int wsum[2][kT2Max / 32];
  // work units of chunk / 2 points per tile (t2_item: an item = two units)
  const int unit = s.chunk / 2;
  const int cnt = q < T ? tot[q] : 0, items = (cnt + unit - 1) / unit;
  const int lane = q & 31, warp = q >> 5;
  int a0 = cnt, a1 = items;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int b0 = __shfl_up_sync(0xffffffffu, a0, o), b1 = __shfl_up_sync(0xffffffffu, a1, o);
    if (lane >= o) { a0 += b0; a1 += b1; }
  }
  if (lane == 31) { wsum[0][warp] = a0; wsum[1][warp] = a1; }
  __syncthreads();
  int o0 = 0, o1 = 0;
  for (int w = 0; w < warp; ++w) { o0 += wsum[0][w]; o1 += wsum[1][w]; }
  if (q < T) {
    s.tstart[q] = o0 + a0 - cnt;
    s.cstart[q] = o1 + a1 - items;
  }
  if (q == T - 1 || (T == 0 && q == 0)) {
    s.tstart[T] = T ? o0 + a0 : 0;
    s.cstart[T] = T ? o1 + a1 : 0;
    *s.n_items = T ? (o1 + a1 + 1) / 2 : 0;
  }
}

__global__ void __launch_bounds__(kT2SortBlock) k2_write(const T2Plan *plp, T2Points p,
                                                         T2Sorted s) {
  extern __shared__ int wc[];
  const T2Plan pl = *plp;
  if (pl.P == 0) return;
  const int T = pl.T;
  const int64_t n = t2_count(p);
  if ((int64_t)blockIdx.x * kT2SortBlock >= n) return;
  int t;
  bool ok;
  unsigned peers;
  t2_block_counts(pl, p, n, wc, T, t, ok, peers);
  // exclusive prefix over the warps, per tile
  for (int q = threadIdx.x; q < T; q += blockDim.x) {
    int run = 0;
    for (int w = 0; w < kT2SortBlock / 32; ++w) {
      const int c = wc[w * T + q];
      wc[w * T + q] = run;
      run += c;
    }
  }
  __syncthreads();
  if (!ok) return;
  const int64_t j = (int64_t)blockIdx.x * kT2SortBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pos = s.tstart[t] + s.bcnt[(int64_t)blockIdx.x * kT2Max + t] + wc[warp * T + t] +
                  __popc(peers & ((1u << lane) - 1u));
  s.perm[pos] = (int)j;
  if (p.rec) {
    const Rec r = p.rec[j];
    s.pos[pos] = make_float4((float)r.x, (float)r.y, (float)r.z, r.w);
    s.aux[pos] = make_float4(r.nx, r.ny, r.nz, r.T);
  } else {
    s.pos[pos] = make_float4(p.qx[j], p.qy[j], p.qz[j], 0.f);
  }
}

// tight box per tile from the sorted positions
__global__ void __launch_bounds__(256) k2_tbox(const T2Plan *plp, T2Sorted s, float *tbox) {
  const int t = blockIdx.x;
  if (plp->P == 0 || t >= plp->T) return;
  const int lo = s.tstart[t], hi = s.tstart[t + 1];
  float mn[3] = {3e38f, 3e38f, 3e38f}, mx[3] = {-3e38f, -3e38f, -3e38f};
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const float4 v = s.pos[k];
    mn[0] = fminf(mn[0], v.x); mx[0] = fmaxf(mx[0], v.x);
    mn[1] = fminf(mn[1], v.y); mx[1] = fmaxf(mx[1], v.y);
    mn[2] = fminf(mn[2], v.z); mx[2] = fmaxf(mx[2], v.z);
  }
  __shared__ float sh[6][256];
  for (int c = 0; c < 3; ++c) { sh[c][threadIdx.x] = mn[c]; sh[3 + c][threadIdx.x] = mx[c]; }
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st)
      for (int c = 0; c < 3; ++c) {
        sh[c][threadIdx.x] = fminf(sh[c][threadIdx.x], sh[c][threadIdx.x + st]);
        sh[3 + c][threadIdx.x] = fmaxf(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + st]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) tbox[t * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

// per (tile, antenna): centre path length L_c = dmin + dmax, half-spread dmax - dmin, and the
// tile-relative geometry around the fp32 tile centre c_t: g0 = (-2a', |a'|^2), g1 = (d_a,
// frac(2 d_a kc), 2 d_a - L_c, 1 / d_a^2) with a' = a - c_t, d_a = |a'| (fp64, rounded once).  Thread =
// (tile, antenna), antennas fastest; the per-antenna range of L_c and the global maxima by
// order-independent atomics on the fp64 bits (positive values), so the results are deterministic.
__global__ void __launch_bounds__(256) k2_tsetup(T2Args a, const int *tstart) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0) return;
  // task = (8 tiles, 32 antennas): warp = tile, lane = antenna (coalesced tile-major writes); the
  // antenna-major copy of L_c through shared memory (64-byte runs), the per-antenna L_c range over
  // the task's tiles reduced in shared memory before the atomics (one pair per antenna and task)
  __shared__ double Ls[8][33];
  const int tt = threadIdx.x >> 5, ii = threadIdx.x & 31;
  const int ntg = (pl.T + 7) / 8;
  const int64_t nag = (a.n_a + 31) / 32, ntask = (int64_t)ntg * nag;
  double hm = 0.0, umin = 1e300;
  for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int tg = (int)(task / nag);
    const int64_t ag = task % nag;
    const int t = tg * 8 + tt;
    const int64_t i = ag * 32 + ii;
    double Lc = -1.0;                                // marker: empty tile / no antenna
    if (t < pl.T && i < a.n_a && tstart[t + 1] > tstart[t]) {
      const double ax = a.tx_x[i], ay = a.tx_y[i], az = a.tx_z[i];
      const float *b = a.tbox + t * 6;
      double dmin, dmax;
      t2_box_dist(b, ax, ay, az, dmin, dmax);
      umin = fmin(umin, dmin);
      Lc = dmin + dmax;
      const int64_t w = (int64_t)t * a.n_a + i;
      a.lc[w] = Lc;
      hm = fmax(hm, dmax - dmin);
      const double px = ax - (double)t2_centre(b, 0), py = ay - (double)t2_centre(b, 1),
                   pz = az - (double)t2_centre(b, 2);
      const double D = px * px + py * py + pz * pz, da = sqrt(D);
      const double cyc = 2.0 * da * a.kc;
      float4 *g = a.tgeo + w * 2;
      g[0] = make_float4((float)(-2.0 * px), (float)(-2.0 * py), (float)(-2.0 * pz), (float)D);
      g[1] = make_float4((float)da, (float)(cyc - rint(cyc)), (float)(2.0 * da - Lc), (float)(1.0 / D));
    }
    Ls[tt][ii] = Lc;
    __syncthreads();
    {
      const int ka = threadIdx.x >> 3, kt = threadIdx.x & 7;
      const int64_t ia = ag * 32 + ka;
      const double v = Ls[kt][ka];
      if (v >= 0.0) a.lct[ia * kT2Max + tg * 8 + kt] = v;
    }
    if (threadIdx.x < 32) {
      double mn = 1e300, mx = -1.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double v = Ls[k][threadIdx.x];
        if (v >= 0.0) { mn = fmin(mn, v); mx = fmax(mx, v); }
      }
      if (mx >= 0.0) {
        unsigned long long *mm = reinterpret_cast<unsigned long long *>(a.lg + (ag * 32 + threadIdx.x) * 3);
        atomicMin(mm + 1, (unsigned long long)__double_as_longlong(mn));
        atomicMax(mm + 2, (unsigned long long)__double_as_longlong(mx));
      }
    }
    __syncthreads();
  }
  __shared__ double red[256];
  red[threadIdx.x] = hm;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + st]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(&a.plan->dmax_bits, (unsigned long long)__double_as_longlong(red[0]));
  __syncthreads();
  red[threadIdx.x] = umin;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + st]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMin(&a.plan->umin_bits, (unsigned long long)__double_as_longlong(red[0]));
}

// per antenna: reset the L_c range before k2_tsetup (min: +inf bits, max: 0)
__global__ void k2_lg_reset(T2Args a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_a;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long *mm = reinterpret_cast<unsigned long long *>(a.lg + i * 3);
    mm[1] = (unsigned long long)__double_as_longlong(1e300);
    mm[2] = 0ull;
  }
}

// per antenna: the global interval covering every tile's [L_c -+ h_t]
__global__ void __launch_bounds__(256) k2_gsetup(T2Args a) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0) return;
  const double ht = __longlong_as_double((long long)pl.dmax_bits);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double hg = 0.0;
  if (i < a.n_a) {
    const double lmin = a.lg[i * 3 + 1], lmax = a.lg[i * 3 + 2];
    const bool any = lmin <= lmax;                   // the antenna sees at least one tile
    a.lg[i * 3] = any ? 0.5 * (lmin + lmax) : 0.0;
    hg = any ? 0.5 * (lmax - lmin) + ht : 0.0;
  }
  __shared__ double red[256];
  red[threadIdx.x] = hg;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(&a.plan->gmax_bits, (unsigned long long)__double_as_longlong(red[0]));
}

__global__ void k2_select(T2Args a) {
  T2Plan *pl = a.plan;
  if (pl->P == 0) { a.skip->sel = 0u; return; }
  const double ht = __longlong_as_double((long long)pl->dmax_bits);
  const double hg = __longlong_as_double((long long)pl->gmax_bits);
  // spreads in cycles per bin, with a margin for the fp32 rounding of the positions
  const double dt = fmax(ht * a.kd * (1.0 + 1e-6), 1e-30);
  const double dg = fmax(hg * a.kd * (1.0 + 1e-6), 1e-30);
  const double zf = 2.0 * kPi * (double)(a.n_f / 2 + 1);
  int P = t2_select_P(zf * dt);
  if (pl->T * P > kT2TP) P = 0;
  // u_min guard (Q24): a tile box closer than 1 mm to an antenna -> the direct kernels, which
  // zero such pairs and raise RFR_FLAG_DOMAIN
  if (__longlong_as_double((long long)pl->umin_bits) < kUmin) P = 0;
  a.skip->sel = P ? 1u : 0u;
  a.skip->P = 0;
  pl->P = P;
  pl->Pg = t2_select_Pg(zf * dg);
  pl->delta_t = dt;
  pl->inv_t = a.kd / dt;
  pl->delta_g = dg;
  pl->inv_g = a.kd / dg;
}

// g1.z = (2 d_a - L_c) -> (2 d_a - L_c) inv_t: x at the antenna's tile distance (the sweeps read
// the geometry as stored; scaling it in the sweeps instead measured 2 % slower, r2v).  Adjoint
// plans also get the filter's own image tgeof of the geometry (t2_geo1): every per-(tile, antenna)
// product of the one-MUFU form precomputed in fp64 -- g0 = (-2a', kang = -2 pi kc d_a),
// g1 = (kx = -inv_t d_a, 2 pi frac(2 d_a kc), x at the tile distance, 1 / d_a^2) -- three FMULs
// per antenna iteration off the filter's FMA pipe.
__global__ void k2_geofix(T2Args a, const int *tstart, int kind) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0) return;
  const int64_t n = (int64_t)pl.T * a.n_a;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(w / a.n_a);
    if (tstart[t + 1] == tstart[t]) continue;
    float4 *g = a.tgeo + w * 2;
    const float4 g0 = g[0];
    float4 g1 = g[1];
    g1.z = (float)((double)g1.z * pl.inv_t);
    g[1].z = g1.z;
    if (kind == kT2PlanAdjoint) {
      const double da = (double)g1.x;
      float4 *f = a.tgeof + w * 2;
      f[0] = make_float4(g0.x, g0.y, g0.z, (float)(-2.0 * kPi * a.kc * da));
      f[1] = make_float4((float)(-pl.inv_t * da), (float)((double)g1.y * (2.0 * kPi)), g1.z, g1.w);
    }
  }
}

// ------------------------------------------------------------------ tables
// a[m][q] = eps_q (-j)^q J_q(2 pi m' delta_g) (Miller's backward recurrence in fp64), q < Pg;
// tabs[0][k] = node x_k = cos(pi (k + 1/2) / P); tabs[1][j][k] = W (node values -> monomial
// coefficients of the interpolant); tabs[2][k][p] = lambda (moments -> node weights)
__global__ void k2_tables(T2Args a) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0) return;
  const int P = pl.P;
  if (blockIdx.x == 0) {
    __shared__ double tp[kT2PMax][kT2PMax];          // t_{p, j}: monomial coefficients of T_p
    __shared__ double Tk[kT2PMax][kT2PMax];          // T_p(x_k)
    const int tid = threadIdx.x;
    if (tid == 0) {
      for (int p = 0; p < kT2PMax; ++p)
        for (int j = 0; j < kT2PMax; ++j) tp[p][j] = 0.0;
      tp[0][0] = 1.0;
      tp[1][1] = 1.0;
      for (int p = 1; p + 1 < kT2PMax; ++p)
        for (int j = 0; j < kT2PMax; ++j)
          tp[p + 1][j] = (j > 0 ? 2.0 * tp[p][j - 1] : 0.0) - tp[p - 1][j];
    }
    if (tid < P) {
      const double x = cos(kPi * (tid + 0.5) / P);
      a.tabs[tid] = x;
      double t0 = 1.0, t1 = x;
      Tk[0][tid] = 1.0;
      if (P > 1) Tk[1][tid] = x;
      for (int p = 2; p < P; ++p) {
        const double t2 = 2.0 * x * t1 - t0;
        Tk[p][tid] = t2;
        t0 = t1;
        t1 = t2;
      }
    }
    __syncthreads();
    for (int w = tid; w < P * P; w += blockDim.x) {
      const int j = w / P, k = w % P;
      double s = 0.0;
      for (int p = 0; p < P; ++p) s += tp[p][j] * (p ? 2.0 : 1.0) / P * Tk[p][k];
      a.tabs[kT2PMax * kT2PMax + j * kT2PMax + k] = s;                   // W[j][k]
      a.tabs[2 * kT2PMax * kT2PMax + k * kT2PMax + j] = (j ? 2.0 : 1.0) / P * Tk[j][k];  // lambda[k][p=j]
    }
    return;
  }
  // Bessel table, one thread per bin
  const int m = (blockIdx.x - 1) * blockDim.x + threadIdx.x;
  const int Pg = pl.Pg;
  if (m >= a.n_f || Pg == 0) return;
  const double z0 = 2.0 * kPi * (double)(m - a.n_f / 2) * pl.delta_g;
  const double z = fabs(z0);
  double J[kT2PgMax];
  if (z < 1e-12) {
    for (int p = 0; p < Pg; ++p) J[p] = p == 0 ? 1.0 : 0.0;
  } else {
    const int top = min(200, Pg + 24 + (int)z);
    double jp1 = 0.0, jp = 1e-30, norm = 0.0;
    for (int k = top; k >= 1; --k) {
      if (k < Pg) J[k] = jp;
      if ((k & 1) == 0) norm += 2.0 * jp;
      const double jm1 = (2.0 * k / z) * jp - jp1;
      jp1 = jp;
      jp = jm1;
      if (fabs(jp) > 1e200) {
        jp *= 1e-200; jp1 *= 1e-200; norm *= 1e-200;
        for (int q = k; q < Pg; ++q) J[q] *= 1e-200;
      }
    }
    J[0] = jp;
    norm += jp;
    for (int p = 0; p < Pg; ++p) J[p] /= norm;
  }
  for (int p = 0; p < Pg; ++p) {
    double v = (p == 0 ? 1.0 : 2.0) * J[p];
    if (z0 < 0.0 && (p & 1)) v = -v;
    const int q = p & 3;                              // (-j)^p = 1, -j, -1, j
    const float2 c = q == 0 ? make_float2((float)v, 0.f)
                   : q == 1 ? make_float2(0.f, (float)-v)
                   : q == 2 ? make_float2((float)-v, 0.f)
                            : make_float2(0.f, (float)v);
    a.acoef[(int64_t)p * a.n_f + m] = c;           // [q][m]: coalesced over bins (k2_fout)
    a.acoef[(int64_t)kT2PgMax * a.n_f + (int64_t)m * kT2PgMax + p] = c;   // [m][q] (k2_gexp)
  }
}

}  // namespace

cudaError_t t2_sort(const T2Args &a, const T2Points &pts, const T2Sorted &srt, cudaStream_t st) {
  ProfScope prof(kProfSort, st);
  const int nb = (int)std::max<int64_t>(1, (pts.n + kT2SortBlock - 1) / kT2SortBlock);
  const size_t sm = (size_t)32 * kT2Max * sizeof(int);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k2_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k2_write, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k2_count<<<nb, kT2SortBlock, sm, st>>>(a.plan, pts, srt);
  k2_scan<<<1, kT2Max, 0, st>>>(a.plan, pts.n_dev, pts.n, srt);
  k2_write<<<nb, kT2SortBlock, sm, st>>>(a.plan, pts, srt);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(3);
  return e;
}

cudaError_t t2_plan(const T2Args &a, const T2Points &pts, const T2Sorted &srt, int kind,
                    cudaStream_t st) {
  cudaError_t e;
  {
  ProfScope prof(kProfPlan, st);
  // per-candidate maxima (fp64 bits) in the tables' scratch tail (128 slots)
  unsigned long long *hb = reinterpret_cast<unsigned long long *>(a.tabs + 3 * kT2PMax * kT2PMax);
  k2_box<<<kT2BoxBlocks, 256, 0, st>>>(pts, a.box_part, hb);
  k2_cand<<<kT2Cand * kT2CandSlices, 256, 0, st>>>(a.box_part, kT2BoxBlocks, a, hb);
  k2_pick<<<1, 128, 0, st>>>(a.box_part, kT2BoxBlocks, hb, a, a.plan, pts.n, pts.n_dev, kind,
                             srt.chunk);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  add_launches(3);
  }
  if ((e = t2_sort(a, pts, srt, st)) != cudaSuccess) return e;
  ProfScope prof(kProfPlan, st);
  k2_tbox<<<kT2Max, 256, 0, st>>>(a.plan, srt, a.tbox);
  k2_lg_reset<<<(unsigned)std::min<int64_t>((a.n_a + 255) / 256, 1024), 256, 0, st>>>(a);
  k2_tsetup<<<(unsigned)std::min<int64_t>((int64_t)(kT2Max / 8) * ((a.n_a + 31) / 32), 148 * 16), 256, 0, st>>>(a, srt.tstart);
  k2_gsetup<<<(unsigned)((a.n_a + 255) / 256), 256, 0, st>>>(a);
  k2_select<<<1, 1, 0, st>>>(a);
  k2_geofix<<<(unsigned)std::min<int64_t>((kT2Max * a.n_a + 255) / 256, 148 * 16), 256, 0, st>>>(a, srt.tstart, kind);
  k2_tables<<<1 + (a.n_f + 127) / 128, 128, 0, st>>>(a);
  if ((e = cudaGetLastError()) == cudaSuccess) add_launches(7);
  else return e;
  return t2_tc_images(a, st);                        // fp16 images of the a table (tcgen05 GEMMs)
}

// ============================================================================ adjoint prep
namespace {

constexpr int kGexpThreads = 256;

// G[row][i][q] = sum_m X_row,i[m] e^{+j 2 pi m' u_g,i} conj(a[m][q]), q < Pg; one CTA per antenna
__global__ void __launch_bounds__(kGexpThreads) k2_gexp(T2Args a, const float2 *X0,
                                                        const float2 *X1) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0 || pl.Pg == 0) return;
  extern __shared__ float2 ys[];                    // [n_f] rotated row, then [4][64] partials
  const int Pg = pl.Pg;
  const int64_t i = blockIdx.x;
  const int N = a.n_f;
  const double ug = a.lg[i * 3] * a.kd;
  float2 *part = ys + N;
  const int nrow = X1 ? 2 : 1;
  for (int row = 0; row < nrow; ++row) {
    const float2 *X = (row == 0 ? X0 : X1) + i * N;
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
      const double c = (double)(m - N / 2) * ug;
      float ps, pc;                                  // e^{+j 2 pi m' u_g}
      sincospif(2.f * (float)(c - rint(c)), &ps, &pc);
      const float2 v = X[m];
      ys[m] = make_float2(fmaf(pc, v.x, -ps * v.y), fmaf(pc, v.y, ps * v.x));
    }
    __syncthreads();
    const int q = threadIdx.x & 63, r = threadIdx.x >> 6;    // 64 x 4
    float re = 0.f, im = 0.f;
    if (q < Pg)
      for (int m = r; m < N; m += 4) {
        const float2 c = a.acoef[(int64_t)kT2PgMax * N + (int64_t)m * kT2PgMax + q], y = ys[m];   // y conj(c)
        re = fmaf(y.x, c.x, fmaf(y.y, c.y, re));
        im = fmaf(y.y, c.x, fmaf(-y.x, c.y, im));
      }
    part[r * 64 + q] = make_float2(re, im);
    __syncthreads();
    if (threadIdx.x < Pg) {
      float2 v = part[threadIdx.x];
      for (int rr = 1; rr < 4; ++rr) {
        v.x += part[rr * 64 + threadIdx.x].x;
        v.y += part[rr * 64 + threadIdx.x].y;
      }
      a.gexp[((int64_t)row * a.n_a + i) * kT2PgMax + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

// per (tile, antenna): F at the tile's P Chebyshev nodes (global expansion; the direct bin sum when
// Pg == 0), then the monomial coefficients c_j = sum_k W[j][k] F_k accumulated in fp64, stored
// reversed (c_{P-1} first: the order the sweeps' Horner reads them).  Thread = (tile, antenna),
// antennas fastest (coalesced centre reads and coefficient writes).
// F(u) = sum_m X[m] e^{+j 2 pi m' u}, fp64 (the fallback when no global expansion applies)
__device__ __noinline__ float2 t2_direct_F(const float2 *X, int n_f, double u) {
  double sr = 0.0, si = 0.0;
  for (int m = 0; m < n_f; ++m) {
    const double c = (double)(m - n_f / 2) * u;
    double ps, pc;
    sincospi(2.0 * (c - rint(c)), &ps, &pc);
    const float2 v = X[m];
    sr += pc * v.x - ps * v.y;
    si += pc * v.y + ps * v.x;
  }
  return make_float2((float)sr, (float)si);
}

template <int P>
__device__ __forceinline__ void k2_cprep_one(const T2Args &a, const T2Plan &pl, int t, int64_t i,
                                             const float2 *X0, const float2 *X1,
                                             const double (*W)[kT2PMax], const double *xk,
                                             const float2 (*Gs)[kT2PgMax], unsigned rows) {
  const int Pg = pl.Pg, T = pl.T;
  const int nrow = X1 ? 2 : 1;
  const double uc = a.lct[i * kT2Max + t] * a.kd;
  const double ug = a.lg[i * 3] * a.kd;
  const double inv_dg = 1.0 / pl.delta_g;
  const double yc = (uc - ug) * inv_dg, yd = pl.delta_t * inv_dg;   // y_k = yc + yd x_k
  for (int row = 0; row < nrow; ++row) {
    if (!((rows >> row) & 1u)) continue;           // no point of this row's sweep in the tile
    float Fr[P], Fi[P];
    if (Pg) {
      // F_k = sum_q G_q T_q(y_k) with T_q by the forward three-term recurrence, two nodes per
      // packed register (one FFMA2 advances both) and the complex accumulation one FFMA2 per node:
      // 3 FFMA2 per (q, node pair) against Clenshaw's 4
      f2x y2[P / 2], t0[P / 2], t1[P / 2], acc[P];
#pragma unroll
      for (int kk = 0; kk < P / 2; ++kk) {
        const float ya = (float)fma(yd, xk[2 * kk], yc), yb = (float)fma(yd, xk[2 * kk + 1], yc);
        y2[kk] = pk(2.f * ya, 2.f * yb);
        t0[kk] = pk(1.f, 1.f);
        t1[kk] = pk(ya, yb);
      }
      {
        const float2 g0 = Gs[row][0];
        const f2x g = pk(g0.x, g0.y);
#pragma unroll
        for (int k = 0; k < P; ++k) acc[k] = g;            // T_0 = 1
      }
      for (int q = 1; q < Pg; ++q) {
        const float2 gq = Gs[row][q];                // broadcast: one antenna per CTA
        const f2x g = pk(gq.x, gq.y);
#pragma unroll
        for (int kk = 0; kk < P / 2; ++kk) {
          const float2 tv = upk(t1[kk]);
          acc[2 * kk] = ffma2(bcv(tv.x), g, acc[2 * kk]);
          acc[2 * kk + 1] = ffma2(bcv(tv.y), g, acc[2 * kk + 1]);
          const float2 pv = upk(t0[kk]);
          const f2x tn = ffma2(y2[kk], t1[kk], pk(-pv.x, -pv.y));
          t0[kk] = t1[kk];
          t1[kk] = tn;
        }
      }
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const float2 f = upk(acc[k]);
        Fr[k] = f.x;
        Fi[k] = f.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < P; ++k) {          // direct bin sums (wide global spread, Pg == 0)
        const float2 f = t2_direct_F((row == 0 ? X0 : X1) + i * a.n_f, a.n_f, uc + pl.delta_t * xk[k]);
        Fr[k] = f.x;
        Fi[k] = f.y;
      }
    }
    float2 *dst = a.coef + (((int64_t)row * T + t) * a.n_a + i) * P;
    // c_j = sum_k W[j][k] F_k in fp64, four j at a time with k inner: 8 independent DFMA chains
    // instead of 2 (the per-j chains were latency-bound), each still summed in k order
#pragma unroll 1
    for (int j0 = 0; j0 < P; j0 += 4) {
      double cr[4], ci[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) { cr[jj] = 0.0; ci[jj] = 0.0; }
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const double fr = (double)Fr[k], fi = (double)Fi[k];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          cr[jj] = fma(W[j0 + jj][k], fr, cr[jj]);
          ci[jj] = fma(W[j0 + jj][k], fi, ci[jj]);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)                // P = 10, 14: the last block is half used
        if (j0 + jj < P) dst[P - 1 - (j0 + jj)] = make_float2((float)cr[jj], (float)ci[jj]);
    }
  }
}

// CTA = (one antenna, 128 tiles): the antenna's global expansions staged in shared memory (every
// thread reads the same coefficient: broadcast), antenna-major centres (coalesced)
// tstart0 / tstart: tile occupancy of the point sets row 0 / row 1 are swept over (the fused call:
// row 0 = G over the alpha != 0 samples, row 1 = s over every sample -- at c3 61 of 256 tiles hold
// an active sample, so three quarters of row 0's coefficients are never read and not computed)
__global__ void __launch_bounds__(128) k2_cprep(T2Args a, const int *tstart0, const int *tstart,
                                                const float2 *X0, const float2 *X1) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0) return;
  __shared__ double W[kT2PMax][kT2PMax];
  __shared__ double xk[kT2PMax];
  __shared__ float2 Gs[2][kT2PgMax];
  const int64_t i = blockIdx.x;
  const int t = blockIdx.y * blockDim.x + threadIdx.x;
  if (blockIdx.y * blockDim.x >= pl.T) return;
  for (int w = threadIdx.x; w < kT2PMax * kT2PMax; w += blockDim.x)
    W[w / kT2PMax][w % kT2PMax] = a.tabs[kT2PMax * kT2PMax + w];
  if (threadIdx.x < kT2PMax) xk[threadIdx.x] = a.tabs[threadIdx.x];
  const int nrow = X1 ? 2 : 1;
  for (int w = threadIdx.x; w < nrow * kT2PgMax; w += blockDim.x)
    Gs[w / kT2PgMax][w % kT2PgMax] =
        pl.Pg ? a.gexp[((int64_t)(w / kT2PgMax) * a.n_a + i) * kT2PgMax + w % kT2PgMax]
              : make_float2(0.f, 0.f);
  __syncthreads();
  if (t >= pl.T) return;
  const unsigned rows = (tstart0[t + 1] != tstart0[t] ? 1u : 0u) |
                        (X1 && tstart[t + 1] != tstart[t] ? 2u : 0u);
  if (!rows) return;
  switch (pl.P) {
    case 8: k2_cprep_one<8>(a, pl, t, i, X0, X1, W, xk, Gs, rows); break;
    case 10: k2_cprep_one<10>(a, pl, t, i, X0, X1, W, xk, Gs, rows); break;
    case 12: k2_cprep_one<12>(a, pl, t, i, X0, X1, W, xk, Gs, rows); break;
    case 14: k2_cprep_one<14>(a, pl, t, i, X0, X1, W, xk, Gs, rows); break;
    default: break;
  }
}

}  // namespace

cudaError_t t2_prep_adjoint(const T2Args &a, const int *tstart, const float2 *X0, const float2 *X1,
                            cudaStream_t st, const int *tstart0) {
  if (a.n_a <= 0) return cudaSuccess;
  if (!tstart0) tstart0 = tstart;
  ProfScope prof(kProfPrep, st);
  const size_t sm = ((size_t)a.n_f + 4 * 64) * sizeof(float2);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k2_gexp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  if (t2_tc_enabled()) {
    cudaError_t e = t2_gexp_tc(a, X0, X1, st);     // tcgen05 (rfr_tc_gemm.cu)
    if (e != cudaSuccess) return e;
    add_launches(-1);
  } else {
    k2_gexp<<<(unsigned)a.n_a, kGexpThreads, sm, st>>>(a, X0, X1);
  }
  k2_cprep<<<dim3((unsigned)a.n_a, (unsigned)(kT2Max / 128)), 128, 0, st>>>(a, tstart0, tstart, X0, X1);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(2);
  return e;
}


// ================================================================================= sweeps
namespace {

// work item -> tile (binary search over the work-item starts)
__device__ __forceinline__ int t2_item_tile(const int *cstart, int T, int item) {
  int lo = 0, hi = T;                             // cstart[lo] <= item < cstart[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cstart[mid] <= item) lo = mid; else hi = mid;
  }
  return lo;
}

// per point pair: tile-relative geometry (DESIGN 5d): d - d_a = delta / (sqrt(D + delta) + d_a),
// delta = |q'|^2 - 2 a'.q'; centre phase cycles = frac(2 d_a kc) + 2 kc (d - d_a) reduced to
// [-1/2, 1/2]; x = (2 d_a - L_c) inv + 2 inv (d - d_a).  NEG: returns (cos, -sin).
struct Geo2 {
  f2x c, s, x, r;                                 // cos, sin of the centre phase, x, 1/d
  f2x dl;                                         // d - d_a (t2_geo2 only; x = g1.z + 2 inv_t dl)
};
// RED = false (the filter's default): no reduction of the cycle count before the MUFU (the angle
// dl 2 pi 2 kc + 2 pi frac(2 d_a kc) in one FFMA2): |angle| <= ~2 pi (2 kc x tile spread), and
// MUFU.SIN / COS take the fractional revolutions themselves; the phase error grows to
// ~|angle| 2^-22 rad (~2e-5 at c3), 5x the reduced form's and 20x inside the 1e-4 budget
// (A/B: RFR_T2RED=1)
template <bool NEG, bool RED = true>
__device__ __forceinline__ Geo2 t2_geo2(const float4 &g0, const float4 &g1, f2x qx, f2x qy, f2x qz,
                                        f2x qw, float kc2f, float inv2f) {
  const f2x del = ffma2(bcv(g0.x), qx, ffma2(bcv(g0.y), qy, ffma2(bcv(g0.z), qz, qw)));
  const f2x s2 = fadd2(bcv(g0.w), del);
  const float2 s2v = upk(s2);
  const f2x r = pk(rsq_ftz(s2v.x), rsq_ftz(s2v.y));
  const f2x dd = fmul2(s2, r);
  const float2 den = upk(fadd2(dd, bcv(g1.x)));
  const f2x dl = fmul2(del, pk(rcp_ftz_(den.x), rcp_ftz_(den.y)));
  f2x ang;
  if (RED) {
    const f2x cy = ffma2(dl, bcv(kc2f), bcv(g1.y));
    // reduce to [-1/2, 1/2] by round-to-nearest with the 1.5 * 2^23 magic constant on the FMA
    // pipe (|cy| < 2^22; the XU pipe is the other bound of this loop: 4 MUFU per pair)
    const f2x rn = fadd2(fadd2(cy, bcv(12582912.f)), bcv(-12582912.f));
    ang = fmul2(ffma2(rn, bcv(-1.f), cy), bcv(NEG ? -kTwoPi : kTwoPi));
  } else {
    const float sg = NEG ? -kTwoPi : kTwoPi;
    ang = ffma2(dl, bcv(kc2f * sg), bcv(g1.y * sg));
  }
  const float2 av = upk(ang);
  Geo2 o;
  float s0, c0, s1, c1;
  sc_ftz(av.x, s0, c0);
  sc_ftz(av.y, s1, c1);
  o.c = pk(c0, c1);
  o.s = pk(s0, s1);
  o.x = ffma2(dl, bcv(inv2f), bcv(g1.z));
  o.r = r;
  o.dl = dl;
  return o;
}

// One-MUFU form of the same geometry (the filter's default, RFR_T2GEO=2 selects t2_geo2): with
// e = delta / d_a^2 (g1.w = 1 / d_a^2) the path ratio is d / d_a = sqrt(1 + e).  y = rsqrt(1 + e)
// (MUFU), w = (1 + e) y, and one Newton step against the unrounded residual
// rho = (1 + e) - w^2 gives sqrt(1 + e) = w + rho y / 2 to ~fp32 rounding; returned as
// dln = (2 - 2w) - rho y = -2 (d - d_a) / d_a (2 - 2w is exact).  Replaces the rsqrt + rcp pair
// (2 MUFU per point) by 1 MUFU and 4 more FMA-pipe operations per point pair: the filter's XU
// load was ~0.9 of its FMA load.  Error: the residual's rounding, ~2^-26 d_a (~3e-9 m at c3,
// below the rcp form's) -- 1e-5 rad of carrier phase.  kang = -pi 2 kc d_a (times the sign),
// kx = -inv_t d_a: the angle and x are affine in dln.
// g0, g1: the filter's image of the geometry (k2_geofix): g0.w = kang, g1.x = kx, g1.y = the
// centre angle in radians.
__device__ __forceinline__ Geo2 t2_geo1(const float4 &g0, const float4 &g1, f2x qx, f2x qy, f2x qz,
                                        f2x qw) {
  const f2x del = ffma2(bcv(g0.x), qx, ffma2(bcv(g0.y), qy, ffma2(bcv(g0.z), qz, qw)));
  const f2x s = ffma2(del, bcv(g1.w), bcv(1.f));           // 1 + e (rsqrt input only)
  const f2x en = fmul2(del, bcv(-g1.w));                    // -e
  const float2 sv = upk(s);
  const f2x y = pk(rsq_ftz(sv.x), rsq_ftz(sv.y));
  const f2x w = fmul2(s, y);
  const f2x rn = fadd2(ffma2(w, w, bcv(-1.f)), en);         // w^2 - (1 + e) = -rho
  const f2x dln = ffma2(rn, y, ffma2(w, bcv(-2.f), bcv(2.f)));
  const f2x ang = ffma2(dln, bcv(g0.w), bcv(g1.y));
  const float2 av = upk(ang);
  Geo2 o;
  float s0, c0, s1, c1;
  sc_ftz(av.x, s0, c0);
  sc_ftz(av.y, s1, c1);
  o.c = pk(c0, c1);
  o.s = pk(s0, s1);
  o.x = ffma2(dln, bcv(g1.x), bcv(g1.z));
  o.r = y;                                          // d_a / d (not 1 / d)
  o.dl = dln;
  return o;
}

// the same on the shared geometry image tgeo, the per-antenna products formed in the loop (A/B:
// RFR_T2GEO=3)
__device__ __forceinline__ Geo2 t2_geo1m(const float4 &g0, const float4 &g1, f2x qx, f2x qy, f2x qz,
                                         f2x qw, float kang, float kx) {
  float4 h0 = g0, h1 = g1;
  h0.w = kang; h1.x = kx; h1.y = g1.y * kTwoPi;
  return t2_geo1(h0, h1, qx, qy, qz, qw);
}

constexpr int kT2GA = 32;                         // antennas per shared-memory stage

// shared-memory stages of the adjoint sweeps, double-buffered: per antenna its P coefficients
// (stored reversed by k2_cprep: c_{P-1} first) and its tile-relative geometry (g1.z already scaled
// by inv_t).  Both blocks are contiguous in HBM for a run of antennas, so one thread moves a stage
// with two bulk copies on the TMA engine (cp.async.bulk, completion on the buffer's mbarrier)
// while the CTA computes the previous stage.
template <int GA>
struct AdjStageT {
  static constexpr int kGA = GA;
  float2 cs[2][2][GA * kT2PMax];                  // [buffer][slot][antenna * P + k]
  float4 gs[2][2][GA][2];                         // [buffer][slot][antenna][g0, g1]
  unsigned long long bar[2];
};
using AdjStage = AdjStageT<kT2GA>;
template <class Stage>
__device__ __forceinline__ void t2_stage_init(Stage &sm) {
  if (threadIdx.x == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}
// work item = two UNITS of srt.chunk / 2 sorted points; a unit = two warps' segments of one tile
// (32 SPT points each, lane-contiguous) and every tile is padded to whole units (k2_scan:
// cstart = the first unit of each tile), so an item spans at most two tiles -- one stage slot per
// tile -- and a tile wastes on average half a warp segment of lanes instead of half a chunk
// (c3 backward: ~270 active samples per tile in chunks of 256).  A warp whose segment lies past
// its tile's end skips the antenna loop.
struct T2Item {
  int t0, t1;                                     // tiles of the item's units (-1: past the end)
  int tw, slot;                                   // this warp's tile (-1: idle) and stage slot
  int64_t base, end;                              // this warp's first sorted position, tile end
  bool two;                                       // the units' tiles differ (slot 1 staged)
};
__device__ __forceinline__ T2Item t2_item(const T2Sorted &s, int T, int item, int seg) {
  const int nu = s.cstart[T];
  T2Item it;
  it.t0 = t2_item_tile(s.cstart, T, 2 * item);
  it.t1 = 2 * item + 1 < nu ? t2_item_tile(s.cstart, T, 2 * item + 1) : -1;
  it.two = it.t1 >= 0 && it.t1 != it.t0;
  const int w = (int)(threadIdx.x >> 5), h = w >> 1;
  it.tw = h ? it.t1 : it.t0;
  it.slot = (h && it.two) ? 1 : 0;
  it.base = 0;
  it.end = 0;
  if (it.tw >= 0) {
    it.base = s.tstart[it.tw] + (int64_t)(2 * item + h - s.cstart[it.tw]) * (2 * seg) + (w & 1) * seg;
    it.end = s.tstart[it.tw + 1];
    if (it.base >= it.end) it.tw = -1;
  }
  return it;
}

template <int P, class Stage>
__device__ __forceinline__ void t2_stage_issue(const T2Args &a, const T2Plan &pl, int row,
                                               const T2Item &it, int64_t i0, int ga, Stage &sm,
                                               int b, const float4 *tgeo) {
  if (threadIdx.x != 0) return;
  const unsigned bc = (unsigned)(ga * P * 8), bg = (unsigned)(ga * 32);
  mbar_arrive_expect_tx(&sm.bar[b], (bc + bg) * (it.two ? 2u : 1u));
  bulk_g2s(&sm.cs[b][0][0], a.coef + (((int64_t)row * pl.T + it.t0) * a.n_a + i0) * P, bc, &sm.bar[b]);
  bulk_g2s(&sm.gs[b][0][0][0], tgeo + ((int64_t)it.t0 * a.n_a + i0) * 2, bg, &sm.bar[b]);
  if (it.two) {
    bulk_g2s(&sm.cs[b][1][0], a.coef + (((int64_t)row * pl.T + it.t1) * a.n_a + i0) * P, bc, &sm.bar[b]);
    bulk_g2s(&sm.gs[b][1][0][0], tgeo + ((int64_t)it.t1 * a.n_a + i0) * 2, bg, &sm.bar[b]);
  }
}

// the same, point-packed: hre = (Re h(x0), Re h(x1)), him = (Im h(x0), Im h(x1)) -- two FFMA2
// per coefficient and point pair with the coefficient's parts as broadcast operands; the results
// stay in the point-packed layout of the geometry (no re-pairing in the epilogue)
template <int P>
__device__ __forceinline__ void t2_horner_pp(const float2 *cs, f2x x, f2x &hre, f2x &him) {
  const float4 c01 = *reinterpret_cast<const float4 *>(cs);
  hre = ffma2(x, bcv(c01.x), bcv(c01.z));
  him = ffma2(x, bcv(c01.y), bcv(c01.w));
#pragma unroll
  for (int k = 2; k < P; k += 2) {
    const float4 c = *reinterpret_cast<const float4 *>(cs + k);
    hre = ffma2(x, ffma2(x, hre, bcv(c.x)), bcv(c.z));
    him = ffma2(x, ffma2(x, him, bcv(c.y)), bcv(c.w));
  }
}

template <int P>
__device__ __forceinline__ void t2_horner2(const float2 *cs, f2x x, f2x &h0, f2x &h1) {
  const float2 xv = upk(x);
  const f2x x0 = bcv(xv.x), x1 = bcv(xv.y);
  const float4 c01 = *reinterpret_cast<const float4 *>(cs);
  const f2x p0 = pk(c01.x, c01.y), p1 = pk(c01.z, c01.w);
  h0 = ffma2(x0, p0, p1);
  h1 = ffma2(x1, p0, p1);
#pragma unroll
  for (int k = 2; k < P; k += 2) {
    const float4 c = *reinterpret_cast<const float4 *>(cs + k);
    const f2x pa = pk(c.x, c.y), pb = pk(c.z, c.w);
    h0 = ffma2(x0, ffma2(x0, h0, pa), pb);
    h1 = ffma2(x1, ffma2(x1, h1, pa), pb);
  }
}

// ------------------------------------------------------------------------- filter sweep
// work item = (two units of kT2FltChunk / 2 tile-sorted points, antenna split, t2_item); thread =
// 4 points of its warp's segment (lane + 32 u)
// GM: geometry of the filter: 0 = t2_geo2 unreduced angle, 1 = t2_geo2 reduced, 2 = t2_geo1
template <int P, int GM, int NPAIR, int UNR, int GA, bool DYN>
__device__ __forceinline__ void k2_filter_body(const T2Args &a, const T2Plan &pl, const T2Sorted &s,
                                               int row, float2 *__restrict__ out, int64_t n_out,
                                               int n_splits, int64_t aps, AdjStageT<GA> &sm) {
  constexpr int SPT = 2 * NPAIR;                   // points per thread (chunk = SPT * 128)
  const int total = *s.n_items * n_splits;
  unsigned ph = 0u;                                // mbarrier phase bits of the stage buffers
  const float kc2f = (float)(2.0 * a.kc), inv2f = (float)(2.0 * pl.inv_t);
  const float4 *fgeo = GM == 2 ? a.tgeof : a.tgeo;  // t2_geo1 reads its own image (k2_geofix)
  const float kangf = (float)(-2.0 * kPi * a.kc), kxf = (float)(-pl.inv_t);   // t2_geo1m
  const int lane = (int)(threadIdx.x & 31);
  // DYN: work items fetched from a device counter (plan->ctr[0], zeroed before the launch) instead
  // of the static stride -- a CTA that runs ahead takes more items; every item still writes its
  // own outputs, so the result does not depend on who ran it
  __shared__ int w_next;
  int w = blockIdx.x;
  if (DYN) {
    if (threadIdx.x == 0) w_next = (int)atomicAdd(&a.plan->ctr[0], 1u);
    __syncthreads();
    w = w_next;
    __syncthreads();                               // read before thread 0 fetches the next item
  }
  while (w < total) {
    const int item = w / n_splits, split = w % n_splits;
    const T2Item it = t2_item(s, pl.T, item, 32 * SPT);
    const int64_t base = it.base + lane, end = it.end;
    const float *tb = a.tbox + max(it.tw, 0) * 6;
    const float cx = t2_centre(tb, 0), cy = t2_centre(tb, 1), cz = t2_centre(tb, 2);
    f2x qx[NPAIR], qy[NPAIR], qz[NPAIR], qw[NPAIR];
    bool valid[SPT];
#pragma unroll
    for (int pp = 0; pp < NPAIR; ++pp) {
      float v4[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = 2 * pp + h;
        const int64_t k = base + u * 32;
        valid[u] = k < end;
        const float4 v = valid[u] ? s.pos[k] : make_float4(cx, cy, cz, 0.f);
        v4[h][0] = v.x - cx; v4[h][1] = v.y - cy; v4[h][2] = v.z - cz;
        v4[h][3] = fmaf(v4[h][0], v4[h][0], fmaf(v4[h][1], v4[h][1], v4[h][2] * v4[h][2]));
      }
      qx[pp] = pk(v4[0][0], v4[1][0]); qy[pp] = pk(v4[0][1], v4[1][1]);
      qz[pp] = pk(v4[0][2], v4[1][2]); qw[pp] = pk(v4[0][3], v4[1][3]);
    }
    // per point M = A1 + j A2, A1 = sum cos h, A2 = sum sin h (complex h, one register pair)
    f2x A1[SPT], A2[SPT];
#pragma unroll
    for (int u = 0; u < SPT; ++u) { A1[u] = 0ull; A2[u] = 0ull; }
    const int64_t i_lo = (int64_t)split * aps, i_hi = min(a.n_a, i_lo + aps);
    if (DYN && threadIdx.x == 0) w_next = (int)atomicAdd(&a.plan->ctr[0], 1u);   // the next item
    __syncthreads();                               // the previous item's stages are consumed
    const int wn = DYN ? w_next : w + (int)gridDim.x;
    if (DYN && i_lo >= i_hi) __syncthreads();      // (no stage barrier below: order the read of w_next)
    if (i_lo < i_hi) t2_stage_issue<P>(a, pl, row, it, i_lo, (int)min((int64_t)GA, i_hi - i_lo), sm, 0, fgeo);
    int b = 0;
    for (int64_t i0 = i_lo; i0 < i_hi; i0 += GA, b ^= 1) {
      const int ga = (int)min((int64_t)GA, i_hi - i0);
      mbar_wait(&sm.bar[b], (ph >> b) & 1u);
      ph ^= 1u << b;
      __syncthreads();                             // every thread is done with buffer b ^ 1
      if (i0 + GA < i_hi)
        t2_stage_issue<P>(a, pl, row, it, i0 + GA, (int)min((int64_t)GA, i_hi - i0 - GA), sm, b ^ 1, fgeo);
      // the stage slot as a compile-time index in each of two copies of the antenna loop: a
      // per-warp shared-memory base would move the loop's addressing and control off the uniform
      // datapath (r3b: +9 instructions per antenna, filter 22.7 -> 23.2 ms)
      auto sweep = [&](const float2 *csb, const float4 (*gsb)[2]) {
      // UNR == 3 (A/B, RFR_T2FV=pf): the next antenna's geometry words are loaded into the same
      // registers as soon as this antenna's geometry has consumed them (before its Horner), so
      // the first FFMA2 of an iteration does not wait on its own LDS
      constexpr bool PF = UNR == 3;
      float4 g0n = gsb[0][0], g1n = gsb[0][1];
#pragma unroll (PF ? 1 : UNR)
      for (int aa = 0; aa < ga; ++aa) {
        // (issuing the next antenna's geometry ahead of this Horner -- software pipelining --
        // measured slower, r2p: 24.8 -> 25.1 ms)
        const float4 g0 = PF ? g0n : gsb[aa][0], g1 = PF ? g1n : gsb[aa][1];
        Geo2 cur[NPAIR];
        if (GM == 2) {
#pragma unroll
          for (int pp = 0; pp < NPAIR; ++pp)
            cur[pp] = t2_geo1(g0, g1, qx[pp], qy[pp], qz[pp], qw[pp]);
        } else if (GM == 3) {
          const float kang = g1.x * kangf, kx = g1.x * kxf;
#pragma unroll
          for (int pp = 0; pp < NPAIR; ++pp)
            cur[pp] = t2_geo1m(g0, g1, qx[pp], qy[pp], qz[pp], qw[pp], kang, kx);
        } else {
#pragma unroll
          for (int pp = 0; pp < NPAIR; ++pp)
            cur[pp] = t2_geo2<false, GM == 1>(g0, g1, qx[pp], qy[pp], qz[pp], qw[pp], kc2f, inv2f);
        }
        if (PF) {
          const int an = min(aa + 1, ga - 1);
          g0n = gsb[an][0]; g1n = gsb[an][1];
        }
#pragma unroll
        for (int pp = 0; pp < NPAIR; ++pp) {
          const Geo2 &e = cur[pp];
          // complex h per point: the coefficients' (re, im) pair times the broadcast x -- the
          // point-packed form (t2_horner_pp) needs the coefficient as a broadcast addend, which
          // FFMA2 cannot take (MOVs: r2m, filter 24.8 -> 26.8 ms)
          f2x h0, h1;
          t2_horner2<P>(&csb[aa * P], e.x, h0, h1);
          const float2 cv = upk(e.c), sv = upk(e.s);
          A1[2 * pp] = ffma2(bcv(cv.x), h0, A1[2 * pp]);
          A2[2 * pp] = ffma2(bcv(sv.x), h0, A2[2 * pp]);
          A1[2 * pp + 1] = ffma2(bcv(cv.y), h1, A1[2 * pp + 1]);
          A2[2 * pp + 1] = ffma2(bcv(sv.y), h1, A2[2 * pp + 1]);
        }
      }
      };
      if (it.tw < 0) continue;                     // idle warp (its segment is past the tile)
      if (it.slot) sweep(sm.cs[b][1], sm.gs[b][1]);
      else sweep(sm.cs[b][0], sm.gs[b][0]);
    }
    float2 *o = out + (int64_t)split * n_out;
#pragma unroll
    for (int u = 0; u < SPT; ++u)
      if (valid[u]) {
        const float2 p1 = upk(A1[u]), p2 = upk(A2[u]);   // M = A1 + j A2
        o[s.perm[base + u * 32]] = make_float2(p1.x - p2.y, p1.y + p2.x);
      }
    w = wn;
  }
}

template <int MINB, int GM, int NPAIR, int UNR = 1, int GA = kT2GA, bool DYN = false>
__global__ void __launch_bounds__(128, MINB) k2_filter(T2Args a, T2Sorted s, int row,
                                                       float2 *__restrict__ out, int64_t n_out,
                                                       int n_splits, int64_t aps) {
  const T2Plan pl = *a.plan;
  __shared__ __align__(16) AdjStageT<GA> sm;
  t2_stage_init(sm);
  switch (pl.P) {
    case 8: k2_filter_body<8, GM, NPAIR, UNR, GA, DYN>(a, pl, s, row, out, n_out, n_splits, aps, sm); break;
    case 10: k2_filter_body<10, GM, NPAIR, UNR, GA, DYN>(a, pl, s, row, out, n_out, n_splits, aps, sm); break;
    case 12: k2_filter_body<12, GM, NPAIR, UNR, GA, DYN>(a, pl, s, row, out, n_out, n_splits, aps, sm); break;
    case 14: k2_filter_body<14, GM, NPAIR, UNR, GA, DYN>(a, pl, s, row, out, n_out, n_splits, aps, sm); break;
    default: break;
  }
}

// ------------------------------------------------------------------------- backward sweep
// Monostatic, no Eq. 7 correction: T_t = T_r = T_j, chi = [T_j > 0], g = max(2 (n.w)^2 - 1, 0),
// dg/dn = 4 (n.w) w, gamma = 1 / (16 pi^2 d^2) (Eq. 5, gain P:L679-683), so per sample
//   S1 = T^2 U,  S2 = 2 T chi U,  S3 = T^2 V,  U = sum_i R g gamma,  V = sum_i R gamma dg/dn
// with R = Re(E h) (App. A.5).  Thread = 2 active samples (one packed pair).
template <int P, int NPAIR>
__device__ __forceinline__ void k2_bwd_body(const T2Args &a, const T2Plan &pl, const T2Sorted &s,
                                            int row, float *__restrict__ out, int64_t n_out,
                                            int n_splits, int64_t aps, bool no_gain,
                                            AdjStage &sm) {
  constexpr int SPT = 2 * NPAIR;
  const int total = *s.n_items * n_splits;
  unsigned ph = 0u;                                // mbarrier phase bits of the stage buffers
  const float kc2f = (float)(2.0 * a.kc), inv2f = (float)(2.0 * pl.inv_t);
  const int lane = (int)(threadIdx.x & 31);
  // work items from the device counter plan->ctr[2] (zeroed before the launch) when there are at
  // least a.dyn (2; RFR_T2BDYN, r4x) per CTA, else the static stride (as in the filter and the forward)
  const bool dynf = a.dyn > 0 && total >= a.dyn * (int)gridDim.x;
  __shared__ int w_next;
  int w = blockIdx.x;
  if (dynf) {
    if (threadIdx.x == 0) w_next = (int)atomicAdd(&a.plan->ctr[2], 1u);
    __syncthreads();
    w = w_next;
    __syncthreads();                               // read before thread 0 fetches the next item
  }
  while (w < total) {
    const int item = w / n_splits, split = w % n_splits;
    const T2Item it = t2_item(s, pl.T, item, 32 * SPT);
    const int64_t base = it.base + lane, end = it.end;
    const float *tb = a.tbox + max(it.tw, 0) * 6;
    const float cx = t2_centre(tb, 0), cy = t2_centre(tb, 1), cz = t2_centre(tb, 2);
    f2x qx[NPAIR], qy[NPAIR], qz[NPAIR], qw[NPAIR], nx[NPAIR], ny[NPAIR], nz[NPAIR], nq[NPAIR];
    bool valid[SPT];
#pragma unroll
    for (int pp = 0; pp < NPAIR; ++pp) {
      float v4[2][4], n3[2][3];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = 2 * pp + h;
        const int64_t k = base + u * 32;
        valid[u] = k < end;
        const float4 v = valid[u] ? s.pos[k] : make_float4(cx, cy, cz, 0.f);
        const float4 n4 = valid[u] ? s.aux[k] : make_float4(0.f, 0.f, 1.f, 0.f);
        v4[h][0] = v.x - cx; v4[h][1] = v.y - cy; v4[h][2] = v.z - cz;
        v4[h][3] = fmaf(v4[h][0], v4[h][0], fmaf(v4[h][1], v4[h][1], v4[h][2] * v4[h][2]));
        // the normal scaled by sqrt 2: g = 2 (n.w)^2 - 1 = (s n.w)(s n.w) - 1 without a doubling in
        // the pair loop; F, and with it sum F and W, carry the factor sqrt 2 (removed at the store).
        // Halved as well: n.(-a') = (n / 2).g0 with g0 = -2a' as staged (no per-antenna 0.5 g0)
        n3[h][0] = (0.5f * kSqrt2f) * n4.x; n3[h][1] = (0.5f * kSqrt2f) * n4.y;
        n3[h][2] = (0.5f * kSqrt2f) * n4.z;
      }
      qx[pp] = pk(v4[0][0], v4[1][0]); qy[pp] = pk(v4[0][1], v4[1][1]);
      qz[pp] = pk(v4[0][2], v4[1][2]); qw[pp] = pk(v4[0][3], v4[1][3]);
      nx[pp] = pk(n3[0][0], n3[1][0]); ny[pp] = pk(n3[0][1], n3[1][1]); nz[pp] = pk(n3[0][2], n3[1][2]);
      const f2x nqh = ffma2(nx[pp], qx[pp], ffma2(ny[pp], qy[pp], fmul2(nz[pp], qz[pp])));
      nq[pp] = fadd2(nqh, nqh);                                    // sqrt 2 n . q'
    }
    f2x U[NPAIR], SF[NPAIR], Wx[NPAIR], Wy[NPAIR], Wz[NPAIR];
#pragma unroll
    for (int pp = 0; pp < NPAIR; ++pp) { U[pp] = SF[pp] = Wx[pp] = Wy[pp] = Wz[pp] = 0ull; }
    const int64_t i_lo = (int64_t)split * aps, i_hi = min(a.n_a, i_lo + aps);
    if (dynf && threadIdx.x == 0) w_next = (int)atomicAdd(&a.plan->ctr[2], 1u);   // the next item
    __syncthreads();                               // the previous item's stages are consumed
    const int wn = dynf ? w_next : w + (int)gridDim.x;
    if (dynf && i_lo >= i_hi) __syncthreads();     // (no stage barrier below: order the read of w_next)
    if (i_lo < i_hi) t2_stage_issue<P>(a, pl, row, it, i_lo, (int)min((int64_t)kT2GA, i_hi - i_lo), sm, 0, a.tgeo);
    int b = 0;
    for (int64_t i0 = i_lo; i0 < i_hi; i0 += kT2GA, b ^= 1) {
      const int ga = (int)min((int64_t)kT2GA, i_hi - i0);
      mbar_wait(&sm.bar[b], (ph >> b) & 1u);
      ph ^= 1u << b;
      __syncthreads();                             // every thread is done with buffer b ^ 1
      if (i0 + kT2GA < i_hi)
        t2_stage_issue<P>(a, pl, row, it, i0 + kT2GA, (int)min((int64_t)kT2GA, i_hi - i0 - kT2GA), sm, b ^ 1, a.tgeo);
      // (as in the filter; no_gain as a compile-time flag keeps its test out of the loop)
      auto sweep = [&](auto ng, const float2 *csb, const float4 (*gsb)[2]) {
        constexpr bool kNoGain = decltype(ng)::value;
#pragma unroll 1
      for (int aa = 0; aa < ga; ++aa) {
        const float4 g0 = gsb[aa][0], g1 = gsb[aa][1];
        // -a' = g0.xyz / 2:  n.(q' - a') = n.q' + (n/2).g0; W accumulates F g0 = 2 F (-a')
        const f2x h0x = bcv(g0.x), h0y = bcv(g0.y), h0z = bcv(g0.z);
#pragma unroll
        for (int pp = 0; pp < NPAIR; ++pp) {
          const Geo2 e = t2_geo2<true, false>(g0, g1, qx[pp], qy[pp], qz[pp], qw[pp], kc2f, inv2f);  // (cos, -sin)
          f2x hre, him;
          t2_horner_pp<P>(&csb[aa * P], e.x, hre, him);
          const f2x R = ffma2(e.c, hre, fmul2(e.s, him));          // Re(E h) = c hr - s hi
          const f2x r2 = fmul2(e.r, e.r);
          const f2x Rr2 = fmul2(R, r2);
          if (kNoGain) {                               // E11 ablation: g = 1, dg/dn = 0
            U[pp] = fadd2(U[pp], Rr2);
            continue;
          }
          const f2x nd = ffma2(nx[pp], h0x, ffma2(ny[pp], h0y, ffma2(nz[pp], h0z, nq[pp])));
          const f2x ndr2 = fmul2(nd, r2);              // sqrt 2 (n.w) / d
          const f2x g = ffma2(nd, ndr2, bcv(-1.f));    // 2 (n.w)^2 - 1
          const float2 gv = upk(g);
          const f2x gpos = pk(fmaxf(gv.x, 0.f), fmaxf(gv.y, 0.f));
          U[pp] = ffma2(Rr2, gpos, U[pp]);
          // sqrt 2 R gamma 4 (n.w) / d without 4 / (4 pi)^2, zero where the gain is clamped (selects
          // on the ALU pipe, no mask multiply)
          const float2 Fm = upk(fmul2(Rr2, ndr2));
          const f2x F = pk(gv.x > 0.f ? Fm.x : 0.f, gv.y > 0.f ? Fm.y : 0.f);
          SF[pp] = fadd2(SF[pp], F);
          Wx[pp] = ffma2(F, h0x, Wx[pp]);
          Wy[pp] = ffma2(F, h0y, Wy[pp]);
          Wz[pp] = ffma2(F, h0z, Wz[pp]);
        }
      }
      };
      if (it.tw < 0) continue;                     // idle warp (its segment is past the tile)
      if (no_gain) {
        if (it.slot) sweep(std::true_type{}, sm.cs[b][1], sm.gs[b][1]);
        else sweep(std::true_type{}, sm.cs[b][0], sm.gs[b][0]);
      } else {
        if (it.slot) sweep(std::false_type{}, sm.cs[b][1], sm.gs[b][1]);
        else sweep(std::false_type{}, sm.cs[b][0], sm.gs[b][0]);
      }
    }
    float *o = out + (int64_t)split * 5 * n_out;
#pragma unroll
    for (int pp = 0; pp < NPAIR; ++pp) {
      const float2 Uv = upk(U[pp]), SFv = upk(SF[pp]), Wxv = upk(Wx[pp]), Wyv = upk(Wy[pp]),
                   Wzv = upk(Wz[pp]), qxv = upk(qx[pp]), qyv = upk(qy[pp]), qzv = upk(qz[pp]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = 2 * pp + h;
        if (!valid[u]) continue;
        const int k = (int)(base + u * 32);
        const int64_t j = s.perm[k];                            // compacted index
        const float T = s.aux[k].w, TT = T * T;
        const float Uu = h ? Uv.y : Uv.x, SFu = h ? SFv.y : SFv.x;
        const float u16 = Uu * kInv16Pi2f;
        const float f4 = (4.f * kInv16Pi2f / kSqrt2f) * TT;
        o[j] = TT * u16;                                        // S1
        o[n_out + j] = T > 0.f ? 2.f * T * u16 : 0.f;           // S2
        // S3 = T^2 sum F (q' - a')
        o[2 * n_out + j] = f4 * fmaf(h ? qxv.y : qxv.x, SFu, 0.5f * (h ? Wxv.y : Wxv.x));
        o[3 * n_out + j] = f4 * fmaf(h ? qyv.y : qyv.x, SFu, 0.5f * (h ? Wyv.y : Wyv.x));
        o[4 * n_out + j] = f4 * fmaf(h ? qzv.y : qzv.x, SFu, 0.5f * (h ? Wzv.y : Wzv.x));
      }
    }
    w = wn;
  }
}

template <int MINB, int NPAIR>
__global__ void __launch_bounds__(128, MINB) k2_bwd(T2Args a, T2Sorted s, int row,
                                                    float *__restrict__ out, int64_t n_out,
                                                    int n_splits, int64_t aps, bool no_gain) {
  const T2Plan pl = *a.plan;
  __shared__ __align__(16) AdjStage sm;
  t2_stage_init(sm);
  switch (pl.P) {
    case 8: k2_bwd_body<8, NPAIR>(a, pl, s, row, out, n_out, n_splits, aps, no_gain, sm); break;
    case 10: k2_bwd_body<10, NPAIR>(a, pl, s, row, out, n_out, n_splits, aps, no_gain, sm); break;
    case 12: k2_bwd_body<12, NPAIR>(a, pl, s, row, out, n_out, n_splits, aps, no_gain, sm); break;
    case 14: k2_bwd_body<14, NPAIR>(a, pl, s, row, out, n_out, n_splits, aps, no_gain, sm); break;
    default: break;
  }
}

// fixed-order sum of the split partials [S][5][n_c] of the compacted list, scattered to the
// sample index: out[r][idx[c]] (idx NULL: c itself)
__global__ void k2_bsum(const T2Plan *plp, const float *__restrict__ part, int S, int64_t n_c,
                        const int64_t *n_dev, const int *__restrict__ idx, float *__restrict__ out,
                        int64_t n_s) {
  if (plp->P == 0) return;
  const int64_t n = n_dev ? *n_dev : n_c;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx ? (int64_t)idx[c] : c;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      float v = 0.f;
      for (int sp = 0; sp < S; ++sp) v += part[((int64_t)sp * 5 + r) * n_c + c];
      out[(int64_t)r * n_s + j] = v;
    }
  }
}

// ------------------------------------------------------------------------- forward sweep
// work item = (tile, block of kT2FwdAnts antennas); thread = antenna, the tile's sorted records
// staged through shared memory; Chebyshev moments M[t][i][p] = sum_j c_ij T_p(x_ij) with
// c_ij = A_ij e^{-j 2 pi f_c tau_ij} (trace: A = w g gamma T^2, Eq. 5) or the K5 weight c_q.
constexpr int kT2FwdTJ = kT2FwdAnts;             // records per shared-memory stage (one per thread)

// staged records, one float per component (SoA) so that a float2 load yields a record pair:
// 0-2 q' = q - c_t, 3 |q'|^2, 4 w T^2 (trace) / Re c (K5), 5 n.q' (trace) / Im c (K5), 6-8 n
struct FwdStage {
  float v[2][9][kT2FwdTJ];
};
__device__ __forceinline__ f2x ld2(const float *p) {
  const float2 v = *reinterpret_cast<const float2 *>(p);
  return pk(v.x, v.y);
}

// occupied tiles by record count, largest first (ties by tile index): the order the forward's
// dynamic scheduler hands tiles out in (longest items first, so the sweep's tail is made of the
// smallest tiles); 1 CTA of kT2Max threads, rank by counting
__global__ void __launch_bounds__(kT2Max) k2_order(const T2Plan *plp, T2Sorted s) {
  __shared__ int cnt[kT2Max];
  const int T = plp->T, t = (int)threadIdx.x;
  const int n = (plp->P != 0 && t < T) ? s.tstart[t + 1] - s.tstart[t] : 0;
  cnt[t] = n;
  __syncthreads();
  if (n > 0) {
    int r = 0;
    for (int u = 0; u < T; ++u) {
      const int m = cnt[u];
      r += (m > n) || (m == n && u < t);
    }
    s.torder[r] = t;
  }
  const int occ = __syncthreads_count(n > 0);
  if (t == 0) *s.n_occ = occ;
}

// DYN: work items (occupied tile in k2_order's order, antenna block) fetched from the device
// counter plan->ctr[1] (zeroed before the launch); else the static stride over (tile, block)
template <int P, int KIND, int RP, bool DYN>
__device__ __forceinline__ void k2_fwd_body(const T2Args &a, const T2Plan &pl, const T2Sorted &s,
                                            bool no_gain, FwdStage &sm) {
  const int nab = (int)((a.n_a + kT2FwdAnts - 1) / kT2FwdAnts);
  // (with few items per CTA the static stride in tile order balances better -- one rank's share at
  // N = 8, r4s: 0.51 vs 0.60 ms -- so the counter is used from 8 items per CTA on)
  const int n_dyn = DYN ? *s.n_occ * nab : 0;
  const bool dynf = DYN && n_dyn >= 8 * (int)gridDim.x;
  const int total = dynf ? n_dyn : pl.T * nab;
  const float kc2f = (float)(2.0 * a.kc), inv2f = (float)(2.0 * pl.inv_t);
  __shared__ int w_next;
  int w = blockIdx.x;
  if (dynf) {
    if (threadIdx.x == 0) w_next = (int)atomicAdd(&a.plan->ctr[1], 1u);
    __syncthreads();
    w = w_next;
    __syncthreads();                                // read before thread 0 fetches the next item
  }
  while (w < total) {
    if (dynf && threadIdx.x == 0) w_next = (int)atomicAdd(&a.plan->ctr[1], 1u);   // the next item
    int wn = w + (int)gridDim.x;
    const int t = dynf ? s.torder[w / nab] : w / nab, ab = w % nab;
    const int64_t j_lo = s.tstart[t], j_hi = s.tstart[t + 1];
    if (j_hi == j_lo) {                             // (static stride only: DYN lists occupied tiles)
      if (dynf) __syncthreads();
      w = dynf ? w_next : wn;
      if (dynf) __syncthreads();
      continue;
    }
    const int64_t i = (int64_t)ab * kT2FwdAnts + threadIdx.x;
    const bool ok = i < a.n_a;
    const float *tb = a.tbox + t * 6;
    const float cx = t2_centre(tb, 0), cy = t2_centre(tb, 1), cz = t2_centre(tb, 2);
    float4 g0 = make_float4(0.f, 0.f, 0.f, 1.f), g1 = make_float4(1.f, 0.f, 0.f, 0.f);
    if (ok) {
      const float4 *g = a.tgeo + ((int64_t)t * a.n_a + i) * 2;
      g0 = g[0];
      g1 = g[1];
    }
    const f2x h0x = bcv(0.5f * g0.x), h0y = bcv(0.5f * g0.y), h0z = bcv(0.5f * g0.z);
    f2x Mre[P], Mim[P];
#pragma unroll
    for (int p = 0; p < P; ++p) { Mre[p] = 0ull; Mim[p] = 0ull; }
    // this thread's record of the next stage, prefetched into registers
    float4 pv = make_float4(cx, cy, cz, 0.f), pn = make_float4(0.f, 0.f, 1.f, 0.f);
    if (j_lo + threadIdx.x < j_hi) { pv = s.pos[j_lo + threadIdx.x]; pn = s.aux[j_lo + threadIdx.x]; }
    int b = 0;
    for (int64_t jt = j_lo; jt < j_hi; jt += kT2FwdTJ, b ^= 1) {
      {
        const float x = pv.x - cx, y = pv.y - cy, z = pv.z - cz;
        float(*v)[kT2FwdTJ] = sm.v[b];
        const int k = threadIdx.x;
        v[0][k] = x; v[1][k] = y; v[2][k] = z; v[3][k] = fmaf(x, x, fmaf(y, y, z * z));
        if (KIND == kFwdTrace) {
          // the constant of gamma folded into the weight; the normal scaled by sqrt 2 so that
          // g = 2 (n.w)^2 - 1 = (s n.w)(s n.w) - 1 needs no doubling in the pair loop
          v[4][k] = pv.w * pn.w * pn.w * kInv16Pi2f;
          const float sx = kSqrt2f * pn.x, sy = kSqrt2f * pn.y, sz = kSqrt2f * pn.z;
          v[5][k] = fmaf(sx, x, fmaf(sy, y, sz * z));
          v[6][k] = sx; v[7][k] = sy; v[8][k] = sz;
        } else {
          v[4][k] = pv.w;                                   // K5 records: w = Re c_q, T = Im c_q
          v[5][k] = pn.w;
          v[6][k] = -pn.w;                                  // -Im c_q (no negation in the pair loop)
        }
      }
      __syncthreads();
      if (dynf && jt == j_lo) wn = w_next;                   // (ordered by this barrier and the item's last)
      const int64_t jn = jt + kT2FwdTJ + threadIdx.x;       // prefetch the next stage
      pv = make_float4(cx, cy, cz, 0.f);
      pn = make_float4(0.f, 0.f, 1.f, 0.f);
      if (jn < j_hi) { pv = s.pos[jn]; pn = s.aux[jn]; }
      const int nv = (int)min((int64_t)kT2FwdTJ, j_hi - jt);
#pragma unroll 1
      for (int jj = 0; jj < nv; jj += 2 * RP) {
        const float(*v)[kT2FwdTJ] = sm.v[b];
        // RP record pairs per iteration: independent geometry chains in flight (staged slots past
        // nv hold zero-weight records)
        f2x cre[RP], cim[RP], xp[RP], xn[RP];       // c and +-2x
#pragma unroll
        for (int rp = 0; rp < RP; ++rp) {
          const int j2 = jj + 2 * rp;
          const Geo2 e = t2_geo2<true, false>(g0, g1, ld2(&v[0][j2]), ld2(&v[1][j2]), ld2(&v[2][j2]),
                                              ld2(&v[3][j2]), kc2f, inv2f);    // (cos, -sin)
          if (KIND == kFwdTrace) {
            const f2x r2 = fmul2(e.r, e.r);
            f2x gg;
            if (no_gain) {
              gg = bcv(1.f);
            } else {
              const f2x nd = ffma2(ld2(&v[6][j2]), h0x,
                                   ffma2(ld2(&v[7][j2]), h0y, ffma2(ld2(&v[8][j2]), h0z, ld2(&v[5][j2]))));
              const f2x ndr2 = fmul2(nd, r2);          // nd = sqrt 2 (n.(q - a))
              const float2 gv = upk(ffma2(nd, ndr2, bcv(-1.f)));
              gg = pk(fmaxf(gv.x, 0.f), fmaxf(gv.y, 0.f));
            }
            // A = w T^2 g gamma; c = A e^{-j theta} = (A cos, A (-sin))
            const f2x A = fmul2(fmul2(ld2(&v[4][j2]), gg), r2);
            cre[rp] = fmul2(A, e.c);
            cim[rp] = fmul2(A, e.s);
          } else {
            // c = (Ar + j Ai) e^{-j theta} = (Ar cos - Ai (-sin), Ai cos + Ar (-sin))
            const f2x Ar = ld2(&v[4][j2]), Ai = ld2(&v[5][j2]);
            cre[rp] = ffma2(Ar, e.c, fmul2(ld2(&v[6][j2]), e.s));
            cim[rp] = ffma2(Ai, e.c, fmul2(Ar, e.s));
          }
          // +-2x straight from the path difference (x itself is not needed: the recurrence
          // below runs on the doubled polynomials)
          xp[rp] = ffma2(e.dl, bcv(2.f * inv2f), bcv(2.f * g1.z));
          xn[rp] = ffma2(e.dl, bcv(-2.f * inv2f), bcv(-2.f * g1.z));
        }
#pragma unroll
        for (int rp = 0; rp < RP; ++rp) {
          // moments in record-packed pairs (lane = record): Mre[p] += v_p(x) cre, Mim[p] += v_p(x)
          // cim, v_p = s_p T_p(x) by the plain recurrence, s = (+ + - -); no re-pairing
          // (w_p = 2 v_p for p >= 1: w_1 = 2x, w_2 = (-2x)(2x) + 2, then the same recurrence;
          // doubling is exact, the moments p >= 1 are halved when stored)
          const f2x tp = xp[rp], tn = xn[rp];
          Mre[0] = fadd2(Mre[0], cre[rp]);
          Mim[0] = fadd2(Mim[0], cim[rp]);
          Mre[1] = ffma2(tp, cre[rp], Mre[1]);
          Mim[1] = ffma2(tp, cim[rp], Mim[1]);
          f2x v2 = bcv(2.f), v1 = tp;
#pragma unroll
          for (int p = 2; p < P; ++p) {
            const f2x vv = ffma2((p & 1) ? tp : tn, v1, v2);
            v2 = v1;
            v1 = vv;
            Mre[p] = ffma2(vv, cre[rp], Mre[p]);
            Mim[p] = ffma2(vv, cim[rp], Mim[p]);
          }
        }
      }
    }
    __syncthreads();                                  // the stage buffers are reused by the next item
    if (ok) {
      float2 *dst = a.mom + ((int64_t)i * pl.T + t) * P;     // antenna-major (k2_fout)
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float2 r = upk(Mre[p]), i2 = upk(Mim[p]);
        float2 v = make_float2(r.x + r.y, i2.x + i2.y);
        if (p) { v.x *= 0.5f; v.y *= 0.5f; }
        if ((p >> 1) & 1) { v.x = -v.x; v.y = -v.y; }
        dst[p] = v;
      }
    }
    w = wn;
  }
}

template <int KIND, int RP, int MINB, bool DYN = false>
__global__ void __launch_bounds__(kT2FwdAnts, MINB) k2_fwd(T2Args a, T2Sorted s, bool no_gain) {
  const T2Plan pl = *a.plan;
  __shared__ FwdStage sm;
  switch (pl.P) {
    case 8: k2_fwd_body<8, KIND, RP, DYN>(a, pl, s, no_gain, sm); break;
    case 10: k2_fwd_body<10, KIND, RP, DYN>(a, pl, s, no_gain, sm); break;
    case 12: k2_fwd_body<12, KIND, RP, DYN>(a, pl, s, no_gain, sm); break;
    case 14: k2_fwd_body<14, KIND, RP, DYN>(a, pl, s, no_gain, sm); break;
    default: break;
  }
}

// ------------------------------------------------------------------------- forward output
// per antenna: tile t's moments -> P virtual sources at the nodes u_tk = u_c,it + delta_t x_k with
// weights W_tk = sum_p lambda[k][p] M_t[p] (Chebyshev interpolation of e^{-j z x}); global moments
// Mg[q] = sum_{t,k} W_tk T_q(y_tk), y = (u - u_g) / delta_g; bins
// s[m] = e^{-j 2 pi m' u_g} sum_q a[m][q] Mg[q] (or, Pg == 0, the direct sum over the sources).
// CTA = one antenna; thread = a strided set of sources with all (<= 32 per pass) global moments in
// registers; fixed-order reduction: warp shuffles, then the 8 warps in order.
constexpr int kT2OutThreads = 256;
constexpr int kT2OutQ = 32;

template <int P, int QN>
__device__ __forceinline__ void t2_fout_tiles(int T, const float2 *Ms, const double *Lt,
                                              const float (*lam)[kT2PMax], const float *xk,
                                              double kd, double dt, double ug, double inv_dg,
                                              int q0, f2x (&acc)[kT2OutQ]) {
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    float2 M[P];
#pragma unroll
    for (int p = 0; p < P; ++p) M[p] = Ms[t * P + p];
    const double yc = (Lt[t] * kd - ug) * inv_dg, yd = dt * inv_dg;
#pragma unroll 1
    for (int k = 0; k < P; k += 2) {                // two nodes per pass: independent recurrences
      f2x wp[2];
      float y2[2], t0[2], t1[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float wr = 0.f, wi = 0.f;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          wr = fmaf(lam[k + h][p], M[p].x, wr);
          wi = fmaf(lam[k + h][p], M[p].y, wi);
        }
        wp[h] = pk(wr, wi);
        const float y = (float)fma(yd, (double)xk[k + h], yc);
        y2[h] = 2.f * y;
        t0[h] = 1.f;
        t1[h] = y;
      }
      for (int q = 0; q < q0; ++q) {                 // advance to T_q0 (second pass only)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float t2 = fmaf(y2[h], t1[h], -t0[h]);
          t0[h] = t1[h];
          t1[h] = t2;
        }
      }
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        acc[q] = ffma2(bcv(t0[1]), wp[1], ffma2(bcv(t0[0]), wp[0], acc[q]));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float t2 = fmaf(y2[h], t1[h], -t0[h]);
          t0[h] = t1[h];
          t1[h] = t2;
        }
      }
    }
  }
}

// sum of acc[0..32) over the warp's lanes, transposed: lane L returns the sum of acc[L] (a
// butterfly that halves the values at every step: 31 shuffles per component instead of 160)
__device__ __forceinline__ float2 t2_warp_sum_transpose(f2x (&acc)[kT2OutQ], int lane) {
  float vx[kT2OutQ], vy[kT2OutQ];
#pragma unroll
  for (int q = 0; q < kT2OutQ; ++q) {
    const float2 v = upk(acc[q]);
    vx[q] = v.x;
    vy[q] = v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {               // n = 2 o values left; keep o of them
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const float sx = up ? vx[k] : vx[k + o], sy = up ? vy[k] : vy[k + o];
      const float kx = up ? vx[k + o] : vx[k], ky = up ? vy[k + o] : vy[k];
      vx[k] = kx + __shfl_xor_sync(0xffffffffu, sx, o);
      vy[k] = ky + __shfl_xor_sync(0xffffffffu, sy, o);
    }
  }
  return make_float2(vx[0], vy[0]);
}

// mg != NULL (the tensor-core bins, t2_bins_tc): the global moments M_g go to mg[i][q] instead
// of the bins (when a global expansion applies)
__global__ void __launch_bounds__(kT2OutThreads, 2) k2_fout(T2Args a, const int *tstart,
                                                         float2 *__restrict__ out,
                                                         float2 *__restrict__ mg) {
  const T2Plan pl = *a.plan;
  if (pl.P == 0) return;
  extern __shared__ unsigned char smraw[];
  const int P = pl.P, T = pl.T, Pg = pl.Pg;
  const int nv = T * P;
  float2 *Ms = reinterpret_cast<float2 *>(smraw);                     // [T][P] this antenna's moments
  double *Lt = reinterpret_cast<double *>(smraw + (size_t)nv * 8);     // [T] tile centres (m)
  __shared__ float lam[kT2PMax][kT2PMax];
  __shared__ float xk[kT2PMax];
  __shared__ float2 red[kT2OutThreads / 32][kT2OutQ];
  __shared__ float2 Mg[kT2PgMax];
  __shared__ unsigned char full[kT2Max];
  __shared__ __align__(8) unsigned long long mbar;
  const int64_t i = blockIdx.x;
  // the antenna's moments [T][P] (one contiguous row) by one bulk copy on the TMA engine, while the
  // threads stage the tables, the tiles' occupancy and centres (coalesced)
  const float2 *Mi = a.mom + (int64_t)i * nv;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(&mbar, (unsigned)(nv * 8));
    bulk_g2s(Ms, Mi, (unsigned)(nv * 8), &mbar);
  }
  for (int w = threadIdx.x; w < kT2PMax * kT2PMax; w += blockDim.x)
    lam[w / kT2PMax][w % kT2PMax] = (float)a.tabs[2 * kT2PMax * kT2PMax + w];
  if (threadIdx.x < kT2PMax) xk[threadIdx.x] = (float)a.tabs[threadIdx.x];
  const double lg0 = a.lg[i * 3];
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const bool f = tstart[t + 1] > tstart[t];
    full[t] = f;
    Lt[t] = f ? a.lct[i * kT2Max + t] : lg0;
  }
  __syncthreads();
  mbar_wait(&mbar, 0u);
  // empty tiles: k2_fwd never wrote their moments -- zero them (the row may hold stale values)
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    if (!full[t])
      for (int p = 0; p < P; ++p) Ms[t * P + p] = make_float2(0.f, 0.f);
  __syncthreads();
  const double ug = a.lg[i * 3] * a.kd;
  const double dt = pl.delta_t;
  // source v = (tile t, node k): u = u_c,it + delta_t x_k, weight W = sum_p lambda[k][p] M_t[p]
  // (lambda is a well-conditioned interpolation transpose: |lambda| <= 2 / P, fp32)
  auto source = [&](int v, float &y, float2 &wv) {
    const int t = v / P, k = v % P;
    float wr = 0.f, wi = 0.f;
    for (int p = 0; p < P; ++p) {
      const float2 mv = Ms[t * P + p];
      wr = fmaf(lam[k][p], mv.x, wr);
      wi = fmaf(lam[k][p], mv.y, wi);
    }
    wv = make_float2(wr, wi);
    const double u = Lt[t] * a.kd + dt * (double)xk[k];
    y = Pg ? (float)((u - ug) / pl.delta_g) : (float)(u - ug);
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (Pg) {
    const double inv_dg = 1.0 / pl.delta_g;
    for (int q0 = 0; q0 < Pg; q0 += kT2OutQ) {
      f2x acc[kT2OutQ];
#pragma unroll
      for (int q = 0; q < kT2OutQ; ++q) acc[q] = 0ull;
      // thread = whole tiles (P and the pass's moment count compile-time); per tile its P node
      // weights from the P moments, then every source through the Chebyshev recurrence in y
      const int qn = min(kT2OutQ, (Pg - q0 + 7) & ~7);
#define RFR_FOUT_P(PP)                                                                          \
  switch (qn) {                                                                                 \
    case 8: t2_fout_tiles<PP, 8>(T, Ms, Lt, lam, xk, a.kd, dt, ug, inv_dg, q0, acc); break;     \
    case 16: t2_fout_tiles<PP, 16>(T, Ms, Lt, lam, xk, a.kd, dt, ug, inv_dg, q0, acc); break;   \
    case 24: t2_fout_tiles<PP, 24>(T, Ms, Lt, lam, xk, a.kd, dt, ug, inv_dg, q0, acc); break;   \
    default: t2_fout_tiles<PP, 32>(T, Ms, Lt, lam, xk, a.kd, dt, ug, inv_dg, q0, acc); break;   \
  }
      switch (P) {
        case 8: RFR_FOUT_P(8) break;
        case 10: RFR_FOUT_P(10) break;
        case 12: RFR_FOUT_P(12) break;
        default: RFR_FOUT_P(14) break;
      }
#undef RFR_FOUT_P
      // transposed warp reduction (lane q holds moment q0 + q), then the warps in order
      const float2 wsum = t2_warp_sum_transpose(acc, lane);
      red[warp][lane] = wsum;
      __syncthreads();
      if (threadIdx.x < kT2OutQ && q0 + (int)threadIdx.x < Pg) {
        float2 v = red[0][threadIdx.x];
        for (int wq = 1; wq < kT2OutThreads / 32; ++wq) {
          v.x += red[wq][threadIdx.x].x;
          v.y += red[wq][threadIdx.x].y;
        }
        Mg[q0 + threadIdx.x] = v;
      }
      __syncthreads();
    }
    if (mg) {
      if (threadIdx.x < Pg) mg[i * kT2PgMax + threadIdx.x] = Mg[threadIdx.x];
      return;
    }
    for (int m = threadIdx.x; m < a.n_f; m += blockDim.x) {
      const float2 *cf = a.acoef + m;                // [q][m] layout: stride n_f over q
      float re = 0.f, im = 0.f;
      for (int q = 0; q < Pg; ++q) {
        const float2 c = cf[(int64_t)q * a.n_f], v = Mg[q];
        re = fmaf(c.x, v.x, fmaf(-c.y, v.y, re));
        im = fmaf(c.x, v.y, fmaf(c.y, v.x, im));
      }
      const double c = (double)(m - a.n_f / 2) * ug;
      float ps, pc;                                   // e^{-j 2 pi m' u_g}
      sincospif(2.f * (float)(c - rint(c)), &ps, &pc);
      out[i * a.n_f + m] = make_float2(fmaf(pc, re, ps * im), fmaf(pc, im, -ps * re));
    }
  } else {
    // direct (no global expansion applies): s[m] = sum_v W_v e^{-j 2 pi m' u_v}, u_v = u_g + y_v
    for (int m = threadIdx.x; m < a.n_f; m += blockDim.x) {
      const double mc = (double)(m - a.n_f / 2);
      double re = 0.0, im = 0.0;
      for (int v = 0; v < nv; ++v) {
        float y;
        float2 wv;
        source(v, y, wv);
        const double c = mc * (ug + (double)y);
        double ps, pc;
        sincospi(2.0 * (c - rint(c)), &ps, &pc);
        re += pc * wv.x + ps * wv.y;
        im += pc * wv.y - ps * wv.x;
      }
      out[i * a.n_f + m] = make_float2((float)re, (float)im);
    }
  }
}

// fixed-order sum of [S][n] split partials into out (only when the plan applies)
__global__ void k2_ssum(const T2Plan *plp, const float *__restrict__ part, int S, int64_t n,
                        float *__restrict__ out) {
  if (plp->P == 0) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int sp = 0; sp < S; ++sp) v += part[(int64_t)sp * n + k];
    out[k] = v;
  }
}

int occ_blocks(const void *k, int threads) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, 0) != cudaSuccess || n < 1) n = 1;
  return n;
}

}  // namespace

int t2_backward_chunk() {
  static int c = 0;
  if (!c) { const char *e = getenv("RFR_T2BPT"); c = (e && atoi(e) == 4) ? 4 * 128 : kT2BwdChunk; }
  return c;
}

int t2_filter_chunk() {
  static int c = 0;
  if (!c) {
    const char *e = getenv("RFR_T2SPT");
    c = (e && atoi(e) == 8) ? 8 * 128 : (e && atoi(e) == 6) ? 6 * 128
      : (e && atoi(e) == 2) ? 2 * 128 : kT2FltChunk;
  }
  return c;
}

cudaError_t t2_sum_splits(const T2Args &a, const float *part, int S, int64_t n, float *out,
                          int n_sms, cudaStream_t st) {
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)n_sms * 8);
  k2_ssum<<<g, 256, 0, st>>>(a.plan, part, S, n, out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

cudaError_t t2_filter(const T2Args &a, const T2Sorted &srt, int row, float2 *out, int64_t n_out,
                      int n_splits, int64_t ants_per_split, int n_sms, cudaStream_t st) {
  if (a.n_a <= 0 || n_out <= 0) return cudaSuccess;
  ProfScope prof(kProfFilter, st);
  // default: no reduction before the MUFU (r2l: filter 26.3 -> 24.8 ms at c3, rel-L2(M) 3.1e-6 ->
  // 4.5e-6 on 2048 sampled queries); RFR_T2RED=1 reduces the cycle count first
  // geometry (RFR_T2GEO): 2 = one MUFU per point (t2_geo1, default); 0 = rsqrt + rcp with the
  // unreduced angle; 1 = rsqrt + rcp, angle reduced first (RFR_T2RED=1 is the same)
  static int gm = -1;
  if (gm < 0) {
    const char *e = getenv("RFR_T2GEO"), *r = getenv("RFR_T2RED");
    gm = e ? atoi(e) : 2;
    if (r && r[0] == '1') gm = 1;
    if (gm < 0 || gm > 3) gm = 2;
  }
  // launch-shape variants (RFR_T2FV).  Default dyn = pf64 with the work items fetched from a device
  // counter instead of the static stride (r4q: 22.22 -> 21.71 ms).  pf64: stages of 64 antennas (half the per-stage CTA
  // barriers) and the next antenna's geometry words loaded before this antenna's Horner (r4c/r4d at
  // c3: base 22.96 ms, g64 22.8, pf 22.3, pf64 22.17).  A/B: base, g64, pf; m4 = 4 CTAs per SM (128
  // registers), u2 = the antenna loop unrolled by 2 (two antennas' independent work in one
  // scheduling window), m6 = 6 CTAs per SM
  static int fv = -1;
  if (fv < 0) {
    const char *e = getenv("RFR_T2FV");
    fv = !e ? 8 : !strcmp(e, "base") ? 0 : !strcmp(e, "m4") ? 1 : !strcmp(e, "u2") ? 2 : !strcmp(e, "m4u2") ? 3
       : !strcmp(e, "m6") ? 4 : !strcmp(e, "g64") ? 5 : !strcmp(e, "pf") ? 6 : !strcmp(e, "pf64") ? 7 : !strcmp(e, "dyn") ? 8 : 0;
  }
  const unsigned g5 = (unsigned)(n_sms * 5), g4 = (unsigned)(n_sms * 4), g3 = (unsigned)(n_sms * 3);
  if (srt.chunk == 8 * 128) {
    if (gm == 2) k2_filter<3, 2, 4><<<g3, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
    else if (gm == 1) k2_filter<3, 1, 4><<<g3, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
    else k2_filter<3, 0, 4><<<g3, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (srt.chunk == 6 * 128) {
    k2_filter<4, 2, 3><<<g4, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (srt.chunk == 2 * 128) {
    k2_filter<8, 2, 1><<<(unsigned)(n_sms * 8), 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 1) {
    k2_filter<4, 2, 2><<<g4, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 2) {
    k2_filter<5, 2, 2, 2><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 4) {
    k2_filter<6, 2, 2><<<(unsigned)(n_sms * 6), 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 5) {
    // stages of 64 antennas (half the per-stage CTA barriers; 40 KB of shared memory per CTA)
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(k2_filter<5, 2, 2, 1, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      once = true;
    }
    k2_filter<5, 2, 2, 1, 64><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 6) {
    k2_filter<5, 2, 2, 3><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 8) {
    // pf64 with the work items fetched from a device counter (A/B: RFR_T2FV=dyn)
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(k2_filter<5, 2, 2, 3, 64, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      once = true;
    }
    cudaMemsetAsync(reinterpret_cast<char *>(a.plan) + offsetof(T2Plan, ctr), 0, sizeof(unsigned), st);
    static int cps = -1;                           // CTAs per SM of the grid (A/B: RFR_T2CPS)
    if (cps < 0) { const char *e = getenv("RFR_T2CPS"); cps = e ? std::max(1, atoi(e)) : 5; }
    k2_filter<5, 2, 2, 3, 64, true><<<(unsigned)(n_sms * cps), 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 7) {
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(k2_filter<5, 2, 2, 3, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      once = true;
    }
    k2_filter<5, 2, 2, 3, 64><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 3 && fv == 7) {
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(k2_filter<5, 3, 2, 3, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      once = true;
    }
    k2_filter<5, 3, 2, 3, 64><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 3) {
    k2_filter<5, 3, 2><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else if (gm == 2 && fv == 3) {
    k2_filter<4, 2, 2, 2><<<g4, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  } else {
    if (gm == 2) k2_filter<5, 2, 2><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
    else if (gm == 1) k2_filter<5, 1, 2><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
    else k2_filter<5, 0, 2><<<g5, 128, 0, st>>>(a, srt, row, out, n_out, n_splits, ants_per_split);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(1);
  return e;
}

cudaError_t t2_backward(const T2Args &a_in, const T2Sorted &srt, int row, const int *idx,
                        const int64_t *n_dev, int64_t n_c, float *part, float *out, int64_t n_s,
                        int n_splits, int64_t ants_per_split, bool no_gain, int n_sms,
                        cudaStream_t st) {
  T2Args a = a_in;
  a.dyn = 0;
  if (a.n_a <= 0 || n_c <= 0) return cudaSuccess;
  {
    ProfScope prof(kProfBackward, st);
    // CTAs per SM of the 2-points-per-thread form (RFR_T2BV = 4 / 5 / 6; r2w at c3: 2.63 / 2.62 /
    // 2.56 ms, dense 15.89 / 15.59 / 15.56)
    static int bv = -1;
    if (bv < 0) { const char *e = getenv("RFR_T2BV"); bv = e ? atoi(e) : 6; }   // r2w: 6 fastest
    static int dyn = -1;                           // RFR_T2BDYN=0: static stride
    if (dyn < 0) { const char *e = getenv("RFR_T2BDYN"); dyn = e ? std::max(0, atoi(e)) : 2; }
    a.dyn = dyn;
    if (dyn)
      cudaMemsetAsync(reinterpret_cast<char *>(a.plan) + offsetof(T2Plan, ctr) + 2 * sizeof(unsigned),
                      0, sizeof(unsigned), st);
    if (srt.chunk == 4 * 128)
      k2_bwd<3, 2><<<(unsigned)(n_sms * 3), 128, 0, st>>>(a, srt, row, part, n_c, n_splits,
                                                          ants_per_split, no_gain);
    else if (bv == 5)
      k2_bwd<5, 1><<<(unsigned)(n_sms * 5), 128, 0, st>>>(a, srt, row, part, n_c, n_splits,
                                                          ants_per_split, no_gain);
    else if (bv == 6)
      k2_bwd<6, 1><<<(unsigned)(n_sms * 6), 128, 0, st>>>(a, srt, row, part, n_c, n_splits,
                                                          ants_per_split, no_gain);
    else
      k2_bwd<4, 1><<<(unsigned)(n_sms * 4), 128, 0, st>>>(a, srt, row, part, n_c, n_splits,
                                                          ants_per_split, no_gain);
  }
  const unsigned g = (unsigned)std::min<int64_t>((n_c + 255) / 256, (int64_t)n_sms * 8);
  k2_bsum<<<g, 256, 0, st>>>(a.plan, part, n_splits, n_c, n_dev, idx, out, n_s);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(2);
  return e;
}

cudaError_t t2_forward(const T2Args &a, const T2Sorted &srt, int kind, bool no_gain, float2 *out,
                       int n_sms, cudaStream_t st) {
  if (a.n_a <= 0) return cudaSuccess;
  {
  ProfScope prof(kProfForward, st);
  static int rp = -1;
  // two record pairs per iteration (r2q: forward 2.79 -> 2.67 ms at c3); RFR_T2FRP=1: one
  if (rp < 0) { const char *e = getenv("RFR_T2FRP"); rp = (e && atoi(e) == 1) ? 1 : 2; }
  // CTAs per SM (RFR_T2FWM = 3 / 4; r2w at c3: 2.674 / 2.643 ms, dense 17.41 / 17.25); 5 / 6: one
  // record pair per iteration at 5 / 6 CTAs per SM (A/B)
  static int fm = -1;
  if (fm < 0) { const char *e = getenv("RFR_T2FWM"); fm = e ? atoi(e) : 4; }
  // dynamic scheduling (default; RFR_T2FDYN=0: the static stride): occupied tiles largest first,
  // (tile, antenna block) items fetched from a device counter
  static int dyn = -1;
  if (dyn < 0) { const char *e = getenv("RFR_T2FDYN"); dyn = (e && e[0] == '0') ? 0 : 1; }
  // (from 64 antenna blocks on: with fewer -- a rank's share at N = 4, 8 -- the items per CTA are too
  // few for the counter to pay, and the plain static kernel is the faster one, r4t)
  if (dyn && rp == 2 && fm == 4 && a.n_a >= 64 * kT2FwdAnts) {
    k2_order<<<1, kT2Max, 0, st>>>(a.plan, srt);
    cudaMemsetAsync(reinterpret_cast<char *>(a.plan) + offsetof(T2Plan, ctr) + sizeof(unsigned), 0,
                    sizeof(unsigned), st);
    if (kind == kFwdTrace)
      k2_fwd<kFwdTrace, 2, 4, true><<<(unsigned)(n_sms * 4), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else
      k2_fwd<kFwdMFAdj, 2, 4, true><<<(unsigned)(n_sms * 4), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    add_launches(1);
  } else if (kind == kFwdTrace) {
    if (fm == 5) k2_fwd<kFwdTrace, 1, 5><<<(unsigned)(n_sms * 5), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else if (fm == 6) k2_fwd<kFwdTrace, 1, 6><<<(unsigned)(n_sms * 6), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else if (rp == 2 && fm == 4) k2_fwd<kFwdTrace, 2, 4><<<(unsigned)(n_sms * 4), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else if (rp == 2) k2_fwd<kFwdTrace, 2, 3><<<(unsigned)(n_sms * 3), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else k2_fwd<kFwdTrace, 1, 4><<<(unsigned)(n_sms * 4), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
  } else {
    if (fm == 5) k2_fwd<kFwdMFAdj, 1, 5><<<(unsigned)(n_sms * 5), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else if (fm == 6) k2_fwd<kFwdMFAdj, 1, 6><<<(unsigned)(n_sms * 6), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else if (rp == 2 && fm == 4) k2_fwd<kFwdMFAdj, 2, 4><<<(unsigned)(n_sms * 4), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else if (rp == 2) k2_fwd<kFwdMFAdj, 2, 3><<<(unsigned)(n_sms * 3), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
    else k2_fwd<kFwdMFAdj, 1, 4><<<(unsigned)(n_sms * 4), kT2FwdAnts, 0, st>>>(a, srt, no_gain);
  }
  }
  ProfScope prof(kProfForwardOut, st);
  const size_t sm = (size_t)kT2TP * 8 + (size_t)kT2Max * 8;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k2_fout, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const bool tc = t2_tc_enabled();
  k2_fout<<<(unsigned)a.n_a, kT2OutThreads, sm, st>>>(a, srt.tstart, out, tc ? a.mg : nullptr);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) add_launches(2);
  if (e == cudaSuccess && tc) e = t2_bins_tc(a, out, st);   // M_g -> bins on tcgen05
  return e;
}

}  // namespace rfr
