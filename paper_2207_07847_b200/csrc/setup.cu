// setup.cu -- GPU setup phase of the PEGP/MSP solver (sm_100a).
//
// Builds, entirely with device kernels (CUB for sort / scan / run-length):
//  1. the MWM aggregation hierarchy (§2.2, l.59-70), level by level,
//     with a parallel "mutual best edge" matching that reproduces the paper's
//     sequential random-order visit exactly;
//  2. the Galerkin coarse graphs (the coarse blocks of Eq. def:L_ell);
//  3. a nested numbering of all levels (every aggregate a contiguous range),
//     the GPU layout of the expanded vector x~ (n~ = sum n_k entries);
//  4. the MSP T~ (§3.3) in factored block-tree form: per aggregate the
//     core-pair 2x2 inverse and per leftover member its elimination
//     coefficients, subtree sizes, and the dense pseudo-inverse of the top
//     level -- everything apply_R needs for an exact L_T~^+ solve.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>

#include "internal.cuh"

namespace msp {

namespace {

constexpr int TPB = 256;

inline unsigned grid_for(int64_t n, int tpb = TPB) {
  int64_t g = (n + tpb - 1) / tpb;
  return (unsigned)std::max<int64_t>(g, 1);
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  // splitmix64 finaliser -- the counter-based generator of reading R1
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

constexpr int64_t HEAVY_DEG = 512;  // rows longer than this get a CTA in the matching

// ------------------------------------------------------------------ MWM
// Sequential rule: visit vertices in random order; an
// unmatched vertex takes its heaviest unmatched neighbour (ties: lowest index).
// Equivalent edge-greedy form: edge {v,u} has key (rank(first), -w, id(second))
// with first = the endpoint visited first; the sequential rule adds edges in
// increasing key order when both ends are free.  A round here matches every
// edge that is the minimum-key free edge of BOTH its endpoints (a local
// minimum); repeating gives the same matching (lexicographically-first
// maximal matching).  mate: -1 free, -2 free with no free neighbour, >=0 mate.
__global__ void k_mwm_propose(int64_t n, const int64_t* __restrict__ rowptr,
                              const int32_t* __restrict__ col, const double* __restrict__ w,
                              int32_t* __restrict__ mate, int32_t* __restrict__ best,
                              uint64_t base, unsigned int* __restrict__ nactive) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int found = 0;
  if (v < n && rowptr[v + 1] - rowptr[v] > HEAVY_DEG) {
    found = best[v] >= 0;  // a heavy vertex: k_mwm_propose_heavy's (same round, launched before)
  } else if (v < n) {
    int32_t b = -1;
    if (mate[v] == -1) {
      const uint64_t pv = mix64(base ^ (uint64_t)v);
      uint64_t bp = 0;
      int64_t bf = 0, bs = 0;
      double bw = 0.0;
      for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
        const int32_t u = col[e];
        if (u == v || mate[u] >= 0) continue;
        const uint64_t pu = mix64(base ^ (uint64_t)u);
        const bool vfirst = (pv < pu) || (pv == pu && v < u);
        const uint64_t kp = vfirst ? pv : pu;
        const int64_t kf = vfirst ? v : (int64_t)u;
        const int64_t ks = vfirst ? (int64_t)u : v;
        const double kw = w[e];
        const bool better =
            b < 0 || kp < bp ||
            (kp == bp && (kf < bf || (kf == bf && (kw > bw || (kw == bw && ks < bs)))));
        if (better) { b = u; bp = kp; bf = kf; bs = ks; bw = kw; }
      }
      if (b < 0) mate[v] = -2;  // no free neighbour now or later: a leftover
    }
    best[v] = b;
    found = b >= 0;
  }
  unsigned m = __ballot_sync(0xffffffffu, found);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(nactive, (unsigned)__popc(m));
}

// The same proposal for a vertex of degree > HEAVY_DEG, a CTA per vertex: each
// thread scans a strided share of the row, then the strict total order of
// the keys picks one winner (the result equals the sequential scan's).
struct MwmKey {
  int32_t b;
  uint64_t kp;
  int64_t kf, ks;
  double kw;
};

__device__ __forceinline__ bool mwm_better(const MwmKey& a, const MwmKey& c) {  // a better than c
  if (a.b < 0) return false;
  if (c.b < 0) return true;
  return a.kp < c.kp ||
         (a.kp == c.kp && (a.kf < c.kf || (a.kf == c.kf && (a.kw > c.kw || (a.kw == c.kw && a.ks < c.ks)))));
}

__device__ __forceinline__ MwmKey mwm_shfl(const MwmKey& k, int o) {
  MwmKey r;
  r.b = __shfl_xor_sync(0xffffffffu, k.b, o);
  r.kp = __shfl_xor_sync(0xffffffffu, k.kp, o);
  r.kf = __shfl_xor_sync(0xffffffffu, k.kf, o);
  r.ks = __shfl_xor_sync(0xffffffffu, k.ks, o);
  r.kw = __shfl_xor_sync(0xffffffffu, k.kw, o);
  return r;
}

constexpr int HEAVY_TPB = 256;

__global__ void __launch_bounds__(HEAVY_TPB) k_mwm_propose_heavy(const int32_t* __restrict__ heavy,
                                                                 const int64_t* __restrict__ rowptr,
                                                                 const int32_t* __restrict__ col,
                                                                 const double* __restrict__ w,
                                                                 int32_t* __restrict__ mate,
                                                                 int32_t* __restrict__ best, uint64_t base) {
  const int64_t v = heavy[blockIdx.x];
  __shared__ MwmKey sk[HEAVY_TPB / 32];
  if (mate[v] != -1) {  // matched or a known leftover: no proposal (as the thread kernel)
    if (threadIdx.x == 0) best[v] = -1;
    return;
  }
  const uint64_t pv = mix64(base ^ (uint64_t)v);
  MwmKey k{-1, 0, 0, 0, 0.0};
  for (int64_t e = rowptr[v] + threadIdx.x; e < rowptr[v + 1]; e += HEAVY_TPB) {
    const int32_t u = col[e];
    if (u == v || mate[u] >= 0) continue;
    const uint64_t pu = mix64(base ^ (uint64_t)u);
    const bool vfirst = (pv < pu) || (pv == pu && v < u);
    MwmKey c{u, vfirst ? pv : pu, vfirst ? v : (int64_t)u, vfirst ? (int64_t)u : v, w[e]};
    if (mwm_better(c, k)) k = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const MwmKey c = mwm_shfl(k, o);
    if (mwm_better(c, k)) k = c;
  }
  if ((threadIdx.x & 31) == 0) sk[threadIdx.x >> 5] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    MwmKey t = sk[0];
    for (int i = 1; i < HEAVY_TPB / 32; ++i)
      if (mwm_better(sk[i], t)) t = sk[i];
    if (t.b < 0) mate[v] = -2;
    best[v] = t.b;
  }
}

__global__ void k_flag_deg(int64_t n, const int64_t* __restrict__ rowptr, int64_t dmin, int32_t* __restrict__ f) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < n) f[v] = (rowptr[v + 1] - rowptr[v] > dmin) ? 1 : 0;
}

__global__ void k_mwm_match(int64_t n, const int32_t* __restrict__ best, int32_t* __restrict__ mate) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n || mate[v] != -1) return;
  const int32_t b = best[v];
  if (b >= 0 && best[b] == (int32_t)v) mate[v] = b;
}

// pair numbering (reading R3): flag the smaller endpoint of each matched pair
__global__ void k_pair_flag(int64_t n, const int32_t* __restrict__ mate, int32_t* __restrict__ flag) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < n) flag[v] = (mate[v] > (int32_t)v) ? 1 : 0;
}

__global__ void k_pair_assign(int64_t n, const int32_t* __restrict__ mate,
                              const int32_t* __restrict__ scan, int32_t* __restrict__ agg) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t m = mate[v];
  agg[v] = (m >= 0) ? scan[min((int32_t)v, m)] : -1;
}

// leftovers join the aggregate of their heaviest neighbour
__global__ void k_leftover(int64_t n, const int64_t* __restrict__ rowptr,
                           const int32_t* __restrict__ col, const double* __restrict__ w,
                           const int32_t* __restrict__ mate, int32_t* __restrict__ agg,
                           int* __restrict__ err) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n || mate[v] >= 0) return;
  int32_t b = -1;
  double bw = 0.0;
  for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
    const int32_t u = col[e];
    if (u == v) continue;
    if (b < 0 || w[e] > bw) { b = u; bw = w[e]; }  // ascending columns: lowest index on ties
  }
  if (b < 0) { atomicExch(err, 1); return; }
  agg[v] = agg[b];  // b is matched (maximality), numbered by k_pair_assign
}

// --------------------------------------------------------------- coarse graph
__global__ void k_coarse_count(int64_t n, const int64_t* __restrict__ rowptr,
                               const int32_t* __restrict__ col, const int32_t* __restrict__ agg,
                               int64_t* __restrict__ cnt) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int32_t a = agg[u];
  int64_t c = 0;
  for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) c += (agg[col[e]] != a);
  cnt[u] = c;
}

__global__ void k_coarse_emit(int64_t n, const int64_t* __restrict__ rowptr,
                              const int32_t* __restrict__ col, const int32_t* __restrict__ agg,
                              const int64_t* __restrict__ pos, int64_t nc,
                              uint64_t* __restrict__ keys, int64_t* __restrict__ vals) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int32_t a = agg[u];
  int64_t p = pos[u];
  for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
    const int32_t b = agg[col[e]];
    if (b == a) continue;
    keys[p] = (uint64_t)a * (uint64_t)nc + (uint64_t)b;
    vals[p] = e;  // fine entries enumerated in (u, v) order; stable sort keeps it (R4)
    ++p;
  }
}

__global__ void k_coarse_sum(int64_t nruns, const uint64_t* __restrict__ ukeys,
                             const int64_t* __restrict__ roff, const int64_t* __restrict__ svals,
                             const double* __restrict__ w, int64_t nc, int32_t* __restrict__ ccol,
                             double* __restrict__ cw) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  double acc = 0.0;
  for (int64_t j = roff[r]; j < roff[r + 1]; ++j) acc += w[svals[j]];  // left to right (R4)
  cw[r] = acc;
  ccol[r] = (int32_t)(ukeys[r] % (uint64_t)nc);
}

__global__ void k_rowptr_from_keys(int64_t nc, int64_t nruns, const uint64_t* __restrict__ ukeys,
                                   int64_t* __restrict__ crowptr) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a > nc) return;
  const uint64_t target = (uint64_t)a * (uint64_t)nc;
  int64_t lo = 0, hi = nruns;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (ukeys[mid] < target) lo = mid + 1; else hi = mid;
  }
  crowptr[a] = (a == nc) ? nruns : lo;
}

// ------------------------------------------------------------ nested order
__global__ void k_nest_keys(int64_t n, const int32_t* __restrict__ agg, const int32_t* __restrict__ mate,
                            const int32_t* __restrict__ parent_nested, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ ids) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t m = mate[v];
  const uint64_t role = (m >= 0) ? ((int32_t)v < m ? 0u : 1u) : 2u;  // core lo, core hi, leftover
  keys[v] = (uint64_t)parent_nested[agg[v]] * 3u + role;
  ids[v] = (int32_t)v;
}

__global__ void k_scatter_pos(int64_t n, const int32_t* __restrict__ order, int32_t* __restrict__ pos_of) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) pos_of[order[p]] = (int32_t)p;
}

__global__ void k_cptr(int64_t nparent, int64_t n, const uint64_t* __restrict__ skeys,
                       int32_t* __restrict__ cptr) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b > nparent) return;
  if (b == nparent) { cptr[b] = (int32_t)n; return; }
  const uint64_t target = (uint64_t)b * 3u;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (skeys[mid] < target) lo = mid + 1; else hi = mid;
  }
  cptr[b] = (int32_t)lo;
}

__global__ void k_iota32(int64_t n, int32_t* __restrict__ a) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

// level-1 adjacency in nested numbering (int32 offsets for the solve phase)
__global__ void k_deg_nested(int64_t n, const int32_t* __restrict__ perm, const int64_t* __restrict__ rowptr,
                             int32_t* __restrict__ deg) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) { const int32_t v = perm[i]; deg[i] = (int32_t)(rowptr[v + 1] - rowptr[v]); }
}

__global__ void k_fill_nested(int64_t n, const int32_t* __restrict__ perm, const int64_t* __restrict__ rowptr,
                              const int32_t* __restrict__ col, const double* __restrict__ w,
                              const int32_t* __restrict__ nested_of, const int32_t* __restrict__ rp1,
                              int32_t* __restrict__ col1, double* __restrict__ w1) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t v = perm[i];
  int32_t p = rp1[i];
  for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e, ++p) {
    col1[p] = nested_of[col[e]];
    w1[p] = w[e];
  }
}

// ------------------------------------------------------------- MSP factors
// Per level-k node (canonical): parent-edge weight a = mu^{2k-1} * cut, with
// cut = weight to nodes outside its aggregate (the L_G~ entry of block
// (k,k+1), Eq. def:L_ell), the matched-edge weight and, for leftovers, the
// weights to the two core vertices of their aggregate.
__global__ void k_node_weights(int64_t n, const int64_t* __restrict__ rowptr,
                               const int32_t* __restrict__ col, const double* __restrict__ w,
                               const int32_t* __restrict__ agg, const int32_t* __restrict__ mate,
                               const int32_t* __restrict__ core_lo, const int32_t* __restrict__ core_hi,
                               double mu_2km1, double* __restrict__ apar, double* __restrict__ wa,
                               double* __restrict__ wb) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t a = agg[v];
  const int32_t lo = core_lo[a], hi = core_hi[a];
  const int32_t m = mate[v];
  double cut = 0.0, x = 0.0, y = 0.0;
  for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
    const int32_t u = col[e];
    if (agg[u] != a) cut += w[e];
    else if (m >= 0) { if (u == m) x = w[e]; }
    else { if (u == lo) x = w[e]; else if (u == hi) y = w[e]; }
  }
  apar[v] = mu_2km1 * cut;
  wa[v] = x;  // core: weight to mate;   leftover: weight to core lo
  wb[v] = y;  // leftover: weight to core hi
}

__global__ void k_core_ids(int64_t n, const int32_t* __restrict__ mate, const int32_t* __restrict__ agg,
                           int32_t* __restrict__ core_lo, int32_t* __restrict__ core_hi) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t m = mate[v];
  if (m > (int32_t)v) { core_lo[agg[v]] = (int32_t)v; core_hi[agg[v]] = m; }
}

// One thread per aggregate B (nested position at level k+1); its children S
// are the level-k nested positions [cptr[B], cptr[B+1]): S[0], S[1] the matched
// pair (u, v), S[2..] leftovers x (each adjacent only to u / v inside S).
// K_S = sigma L_intra(S) + diag(a_S), sigma = mu^{2(k-1)}.  Eliminating the
// leftovers into the pair gives  K' = [[q+e_u, -q], [-q, q+e_v]]  with
//   d_x = a_x + sigma (w_xu + w_xv),  q = sigma w_uv + sum sigma^2 w_xu w_xv / d_x,
//   e_u = a_u + sum sigma w_xu a_x / d_x,  e_v likewise
// (all terms positive: no cancellation).  Stored packed:
//   kinv[3 (off_{k+1} - n + B) + (0,1,2)] = K'^{-1} (uu, uv, vv)
//   lof[3 (lo_k + x - 2B - 2) + (0,1,2)]  = (sigma w_xu / d_x, sigma w_xv / d_x, 1 / d_x)
// Also N_B = 1 + sum N_c (subtree sizes in T~) and g_S = K_S^{-1} N_S.
__global__ void k_msp_factor(int64_t nparent, const int32_t* __restrict__ cptr,
                             const int32_t* __restrict__ order_k,   // nested pos -> canonical (level k)
                             const double* __restrict__ apar, const double* __restrict__ wa,
                             const double* __restrict__ wb, double sigma, int64_t off_k,
                             int64_t off_k1, int64_t n1, int64_t lo_k, double* __restrict__ kinv,
                             double* __restrict__ lof, double* __restrict__ Nsub,
                             double* __restrict__ gvec, double* __restrict__ gN_part, int first_level) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nparent) return;
  const int32_t s0 = cptr[B], s1 = cptr[B + 1];
  const int32_t cu = order_k[s0], cv = order_k[s0 + 1];
  const double au = apar[cu], av = apar[cv];
  const double wuv = wa[cu];
  double q = sigma * wuv, eu = au, ev = av;
  const int64_t lb = 3 * (lo_k - 2 * B - 2);  // lof[lb + 3 x + j] for leftover child x
  for (int32_t p = s0 + 2; p < s1; ++p) {
    const int32_t x = order_k[p];
    const double ax = apar[x], wxu = sigma * wa[x], wxv = sigma * wb[x];
    const double d = ax + wxu + wxv;
    q += wxu * wxv / d;
    eu += wxu * ax / d;
    ev += wxv * ax / d;
    lof[lb + 3 * (int64_t)p + 0] = wxu / d;
    lof[lb + 3 * (int64_t)p + 1] = wxv / d;
    lof[lb + 3 * (int64_t)p + 2] = 1.0 / d;
  }
  const double det = q * (eu + ev) + eu * ev;
  const double kuu = (q + ev) / det, kuv = q / det, kvv = (q + eu) / det;
  double* ki = kinv + 3 * (off_k1 - n1 + B);
  ki[0] = kuu; ki[1] = kuv; ki[2] = kvv;
  // subtree sizes
  double NB = 1.0;
  for (int32_t p = s0; p < s1; ++p) {
    const double nc = first_level ? 1.0 : Nsub[off_k + p];
    if (first_level) Nsub[off_k + p] = 1.0;
    NB += nc;
  }
  Nsub[off_k1 + B] = NB;
  // g_S = K_S^{-1} N_S (same elimination as apply_R)
  const double Nu = Nsub[off_k + s0], Nv = Nsub[off_k + s0 + 1];
  double tu = Nu, tv = Nv;
  for (int32_t p = s0 + 2; p < s1; ++p) {
    const double t = Nsub[off_k + p];
    tu += lof[lb + 3 * (int64_t)p + 0] * t;
    tv += lof[lb + 3 * (int64_t)p + 1] * t;
  }
  const double zu = kuu * tu + kuv * tv, zv = kuv * tu + kvv * tv;
  gvec[off_k + s0] = zu;
  gvec[off_k + s0 + 1] = zv;
  double gN = zu * Nu + zv * Nv;
  for (int32_t p = s0 + 2; p < s1; ++p) {
    const double t = Nsub[off_k + p];
    const double zx = lof[lb + 3 * (int64_t)p + 2] * t + lof[lb + 3 * (int64_t)p + 0] * zu + lof[lb + 3 * (int64_t)p + 1] * zv;
    gvec[off_k + p] = zx;
    gN += zx * t;
  }
  gN_part[B] = gN;
}

// gdot weights, top-down: G_k[c] = c(k) g_k[c] + G_{k+1}[parent(c)] (G_L = 0);
// then sum_{non-top i} g_i s_i = sum_i g_i c(lev i) y_i = (r, G_1)
__global__ void k_hvec(int64_t nB, const int32_t* __restrict__ cptr, const double* __restrict__ gk, double ckk,
                       const double* __restrict__ Gpar, double* __restrict__ Gk) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  const double gp = Gpar ? Gpar[B] : 0.0;
  for (int32_t c = cptr[B]; c < cptr[B + 1]; ++c) Gk[c] = ckk * gk[c] + gp;
}

// (rowptr[r], rowptr[r + 1]) of rows[0..m)
__global__ void k_row_bounds(int64_t m, const int32_t* __restrict__ rows, const int32_t* __restrict__ rowptr,
                             int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) { out[2 * i] = rowptr[rows[i]]; out[2 * i + 1] = rowptr[rows[i] + 1]; }
}

// ------------------------------------------------------------ SELL-32
__global__ void k_fill_uniform_ptr(int64_t ns, int64_t stride, int64_t* __restrict__ sptr) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s <= ns) sptr[s] = s * stride;
}

// islong: 1 for a long row (warp per row in the SpMV), 2 for a huge one
// (degree > hcap: a CTA per row)
__global__ void k_sell_width(int64_t n, int64_t nslices, const int32_t* __restrict__ rowptr, int lcap, int hcap,
                             int64_t* __restrict__ width, uint32_t* __restrict__ mask, int32_t* __restrict__ islong,
                             int* __restrict__ maxw) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;  // warp-uniform
  const int64_t r = s * 32 + lane;
  int deg = 0;
  if (r < n) deg = rowptr[r + 1] - rowptr[r];
  const bool lng = deg > lcap;
  // 1: medium (lcap < deg <= MED_ROW: 8 lanes per row), 3: long (a warp),
  // 2: huge (CTA segments)
  if (r < n) islong[r] = lng ? (deg > hcap ? 2 : (deg > MED_ROW ? 3 : 1)) : 0;
  int w = lng ? 0 : deg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
  const uint32_t m = __ballot_sync(0xffffffffu, lng);
  if (lane == 0) { width[s] = 32 * (int64_t)w; mask[s] = m; atomicMax(maxw, w); }
}

__global__ void k_flag_heavy(int64_t nB, const int32_t* __restrict__ cptr, int32_t* __restrict__ f) {
  const int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B < nB) f[B] = (cptr[B + 1] - cptr[B] > HEAVY_AGG) ? 1 : 0;
}

__global__ void k_max_degree(int64_t n, const int32_t* __restrict__ rowptr, int* __restrict__ md) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int d = (i < n) ? rowptr[i + 1] - rowptr[i] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
  if ((threadIdx.x & 31) == 0 && d > 0) atomicMax(md, d);
}

__global__ void k_flag_eq(int64_t n, const int32_t* __restrict__ v, int32_t want, int32_t* __restrict__ f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) f[i] = (v[i] == want) ? 1 : 0;
}

__global__ void k_sell_fill(int64_t n, int64_t nslices, const int64_t* __restrict__ sptr,
                            const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const double* __restrict__ w, const uint32_t* __restrict__ mask,
                            int32_t* __restrict__ scol, double* __restrict__ sw) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int64_t r = s * 32 + lane;
  const int64_t base = sptr[s];
  const int64_t width = (sptr[s + 1] - base) / 32;
  const bool lng = (mask[s] >> lane) & 1u;
  int32_t e0 = 0, deg = 0;
  if (r < n && !lng) { e0 = rowptr[r]; deg = rowptr[r + 1] - e0; }
  for (int64_t k = 0; k < width; ++k) {
    const int64_t idx = base + k * 32 + lane;
    if (k < deg) { scol[idx] = col[e0 + k]; sw[idx] = w[e0 + k]; }
    else { scol[idx] = (r < n) ? (int32_t)r : 0; sw[idx] = 0.0; }
  }
}

// dense top-level Laplacian sigma_l L_l (top nested order == canonical order)
__global__ void k_top_dense(int64_t nt, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const double* __restrict__ w, double sigma, double* __restrict__ M) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  double d = 0.0;
  for (int64_t j = 0; j < nt; ++j) M[i * nt + j] = 0.0;
  for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
    M[i * nt + col[e]] = -sigma * w[e];
    d += sigma * w[e];
  }
  M[i * nt + i] = d;
}

// L^+ = Pi G Pi, G = inverse of the grounded (last node removed) SPD block,
// Pi = I - 11^T/n.  One block, Gauss-Jordan without pivoting (SPD), nt <= 256.
__global__ void k_top_pinv(int nt, const double* __restrict__ M, double* __restrict__ A,
                           double* __restrict__ out) {
  __shared__ double fac[256];
  __shared__ double rmean[256];
  __shared__ double cmean[256];
  __shared__ double gmean;
  const int m = nt - 1;
  const int W = 2 * m;
  for (int idx = threadIdx.x; idx < m * W; idx += blockDim.x) {  // A = [M_g | I]
    const int i = idx / W, j = idx % W;
    A[idx] = (j < m) ? M[i * nt + j] : (j - m == i ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int piv = 0; piv < m; ++piv) {
    const double inv = 1.0 / A[piv * W + piv];
    __syncthreads();
    for (int j = threadIdx.x; j < W; j += blockDim.x) A[piv * W + j] *= inv;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) fac[i] = (i == piv) ? 0.0 : A[i * W + piv];
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * W; idx += blockDim.x) {
      const int i = idx / W, j = idx % W;
      if (i != piv) A[idx] -= fac[i] * A[piv * W + j];
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    double s = 0.0;
    if (i < m) for (int j = 0; j < m; ++j) s += A[i * W + m + j];
    rmean[i] = s / nt;
  }
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    double s = 0.0;
    if (j < m) for (int i = 0; i < m; ++i) s += A[i * W + m + j];
    cmean[j] = s / nt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nt; ++i) s += rmean[i];
    gmean = s / nt;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nt * nt; idx += blockDim.x) {
    const int i = idx / nt, j = idx % nt;
    const double g = (i < m && j < m) ? A[i * W + m + j] : 0.0;
    out[idx] = g - rmean[i] - cmean[j] + gmean;
  }
}


// ------------------------------------------------------------ solve schedule
// first1_{k+1}[B] = first level-1 descendant of level-(k+1) node B (B <= n_{k+1})
__global__ void k_first1(int64_t nB, const int32_t* __restrict__ cptr, const int32_t* __restrict__ f_in,
                         int32_t* __restrict__ f_out, int* __restrict__ maxsz) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B > nB) return;
  f_out[B] = f_in[cptr[B]];
  if (B < nB) atomicMax(maxsz, f_in[cptr[B + 1]] - f_in[cptr[B]]);
}

// tile j starts at the first level-Kt node whose subtree starts at or after j*T
__global__ void k_tile_bounds(int64_t ntiles, int64_t nK, int64_t T, const int32_t* __restrict__ first1,
                              int32_t* __restrict__ bnd) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > ntiles) return;
  if (j == ntiles) { bnd[j] = (int32_t)nK; return; }
  const int64_t target = j * T;
  int64_t lo = 0, hi = nK;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (first1[mid] < target) lo = mid + 1; else hi = mid;
  }
  bnd[j] = (int32_t)lo;
}

__global__ void k_tile_descend(int64_t cnt, const int32_t* __restrict__ cptr, const int32_t* __restrict__ above,
                               int32_t* __restrict__ below) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < cnt) below[j] = cptr[above[j]];
}

// ------------------------------------------------------------ validation
__global__ void k_validate(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           const double* __restrict__ w, int* __restrict__ err) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t prev = -1;
  const int64_t e0 = rowptr[v], e1 = rowptr[v + 1];
  if (e0 == e1) { atomicOr(err, 1); return; }            // isolated vertex
  for (int64_t e = e0; e < e1; ++e) {
    const int64_t c = col[e];
    if (c < 0 || c >= n || c == v || c <= prev) { atomicOr(err, 2); return; }
    if (!(w[e] > 0.0)) { atomicOr(err, 4); return; }
    prev = c;
  }
}

// ------------------------------------------------------------ CUB helpers
struct Temp {
  DBuf<unsigned char> buf;
  void* get(size_t bytes) {
    if (bytes > buf.n) buf.alloc(std::max<size_t>(bytes, 1 << 20));
    return buf.p;
  }
};

template <typename T>
void exclusive_scan(Temp& tmp, const T* in, T* out, int64_t n, cudaStream_t st) {
  size_t bytes = 0;
  MSP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st));
  MSP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, in, out, n, st));
}

template <typename K, typename V>
void sort_pairs(Temp& tmp, const K* kin, K* kout, const V* vin, V* vout, int64_t n, int end_bit,
                cudaStream_t st) {
  size_t bytes = 0;
  MSP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit, st));
  MSP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, kin, kout, vin, vout, n, 0, end_bit, st));
}

int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

template <typename T>
T d2h_scalar(const T* d, cudaStream_t st) {
  T v;
  MSP_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  MSP_CUDA(cudaStreamSynchronize(st));
  return v;
}

double reduce_sum(Temp& tmp, const double* in, int64_t n, cudaStream_t st) {
  DBuf<double> out;
  out.alloc(1);
  size_t bytes = 0;
  MSP_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, in, out.p, n, st));
  MSP_CUDA(cub::DeviceReduce::Sum(tmp.get(bytes), bytes, in, out.p, n, st));
  return d2h_scalar(out.p, st);
}

}  // namespace

void validate_csr(Handle& h, const int64_t* rowptr, const int32_t* col, const double* w, cudaStream_t st) {
  DBuf<int> err;
  err.alloc(1);
  MSP_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), st));
  k_validate<<<grid_for(h.n), TPB, 0, st>>>(h.n, rowptr, col, w, err.p);
  MSP_LAUNCH_CHECK();
  const int e = d2h_scalar(err.p, st);
  if (e & 1) throw Error{MSP_ERR_GRAPH, "isolated vertex (graph must be connected)"};
  if (e & 2) throw Error{MSP_ERR_GRAPH, "CSR columns out of range, self loop, or not strictly increasing"};
  if (e & 4) throw Error{MSP_ERR_GRAPH, "edge weights must be > 0"};
}

// ------------------------------------------------------------------ driver
// MSP_SETUP_TIMING=1: per-phase setup times on stderr (synchronises the stream)
struct SetupClock {
  bool on = std::getenv("MSP_SETUP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(cudaStream_t st, const char* what, int k = -1) {
    if (!on) return;
    MSP_CUDA(cudaStreamSynchronize(st));
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - t).count();
    if (k >= 0) std::fprintf(stderr, "[setup] %-22s level %2d %9.2f ms\n", what, k, ms);
    else std::fprintf(stderr, "[setup] %-31s %9.2f ms\n", what, ms);
    t = now;
  }
};

void build_setup(Handle& h, const int64_t* rowptr_d, const int32_t* col_d, const double* w_d,
                 cudaStream_t st) {
  Temp tmp;
  SetupClock clk;
  cudaEvent_t e0, e1;
  MSP_CUDA(cudaEventCreate(&e0));
  MSP_CUDA(cudaEventCreate(&e1));
  MSP_CUDA(cudaEventRecord(e0, st));

  const int64_t n = h.n;
  // ---- level 1 canonical CSR (copy of the input)
  h.canon_rowptr.emplace_back(); h.canon_rowptr.back().alloc(n + 1);
  h.canon_col.emplace_back(); h.canon_col.back().alloc(h.nnz_adj);
  h.canon_w.emplace_back(); h.canon_w.back().alloc(h.nnz_adj);
  MSP_CUDA(cudaMemcpyAsync(h.canon_rowptr[0].p, rowptr_d, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  MSP_CUDA(cudaMemcpyAsync(h.canon_col[0].p, col_d, h.nnz_adj * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  MSP_CUDA(cudaMemcpyAsync(h.canon_w[0].p, w_d, h.nnz_adj * sizeof(double), cudaMemcpyDeviceToDevice, st));
  h.lv.clear();
  h.lv.push_back(LevelHost{n, h.nnz_adj, 0});

  std::vector<DBuf<int32_t>> mates;
  DBuf<int32_t> best, flag, scan;
  DBuf<unsigned int> cnt_d;
  cnt_d.alloc(1);
  DBuf<int> err_d;
  err_d.alloc(1);
  h.mwm_rounds = 0;

  // ---- hierarchy (§2.2; reading R5 for "level = max")
  for (int k = 1;; ++k) {
    if (h.levels_req > 0 && (int)h.lv.size() >= h.levels_req) break;
    const int64_t nk = h.lv.back().n;
    if (nk <= 2) break;
    const int64_t* rp = h.canon_rowptr.back().p;
    const int32_t* cl = h.canon_col.back().p;
    const double* ww = h.canon_w.back().p;
    DBuf<int32_t> mate;
    mate.alloc(nk);
    best.alloc(nk);
    MSP_CUDA(cudaMemsetAsync(mate.p, 0xff, nk * sizeof(int32_t), st));  // -1
    const uint64_t base = mix64(h.seed + 0x9E3779B97F4A7C15ULL * (uint64_t)(k + 1));
    // heavy vertices of this level (a CTA each in the proposal)
    DBuf<int32_t> hv;
    int64_t nhv = 0;
    {
      DBuf<int32_t> ids, fl, nsel;
      ids.alloc(nk); fl.alloc(nk); nsel.alloc(1); hv.alloc(nk);
      k_iota32<<<grid_for(nk), TPB, 0, st>>>(nk, ids.p);
      k_flag_deg<<<grid_for(nk), TPB, 0, st>>>(nk, rp, HEAVY_DEG, fl.p);
      size_t bytes = 0;
      MSP_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ids.p, fl.p, hv.p, nsel.p, nk, st));
      MSP_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, ids.p, fl.p, hv.p, nsel.p, nk, st));
      nhv = d2h_scalar(nsel.p, st);
    }
    // rounds run in batches between host checks: a round after the last
    // productive one proposes nothing and matches nothing
    for (int batch = 1;; batch = std::min(batch * 2, 32)) {
      for (int i = 0; i < batch; ++i) {
        MSP_CUDA(cudaMemsetAsync(cnt_d.p, 0, sizeof(unsigned), st));
        if (nhv) k_mwm_propose_heavy<<<(unsigned)nhv, HEAVY_TPB, 0, st>>>(hv.p, rp, cl, ww, mate.p, best.p, base);
        k_mwm_propose<<<grid_for(nk), TPB, 0, st>>>(nk, rp, cl, ww, mate.p, best.p, base, cnt_d.p);
        k_mwm_match<<<grid_for(nk), TPB, 0, st>>>(nk, best.p, mate.p);
      }
      MSP_LAUNCH_CHECK();
      h.mwm_rounds += batch;
      if (d2h_scalar(cnt_d.p, st) == 0) break;
    }
    clk.mark(st, "matching", k);
    // numbering
    flag.alloc(nk);
    scan.alloc(nk);
    k_pair_flag<<<grid_for(nk), TPB, 0, st>>>(nk, mate.p, flag.p);
    exclusive_scan(tmp, flag.p, scan.p, nk, st);
    const int32_t last_scan = d2h_scalar(scan.p + nk - 1, st);
    const int32_t last_flag = d2h_scalar(flag.p + nk - 1, st);
    const int64_t nc = (int64_t)last_scan + last_flag;
    if (nc < 2) break;  // reading R5: keep >= 2 nodes on top
    DBuf<int32_t> agg;
    agg.alloc(nk);
    k_pair_assign<<<grid_for(nk), TPB, 0, st>>>(nk, mate.p, scan.p, agg.p);
    MSP_CUDA(cudaMemsetAsync(err_d.p, 0, sizeof(int), st));
    k_leftover<<<grid_for(nk), TPB, 0, st>>>(nk, rp, cl, ww, mate.p, agg.p, err_d.p);
    MSP_LAUNCH_CHECK();
    if (d2h_scalar(err_d.p, st)) throw Error{MSP_ERR_GRAPH, "isolated vertex: graph not connected"};
    clk.mark(st, "leftovers", k);

    // ---- coarse graph (Galerkin weights, reading R4 summation order)
    DBuf<int64_t> cnt, pos;
    cnt.alloc(nk + 1);
    pos.alloc(nk + 1);
    k_coarse_count<<<grid_for(nk), TPB, 0, st>>>(nk, rp, cl, agg.p, cnt.p);
    MSP_CUDA(cudaMemsetAsync(cnt.p + nk, 0, sizeof(int64_t), st));
    exclusive_scan(tmp, cnt.p, pos.p, nk + 1, st);
    const int64_t ne = d2h_scalar(pos.p + nk, st);
    DBuf<uint64_t> keys, skeys, ukeys;
    DBuf<int64_t> vals, svals, rcnt, roff;
    keys.alloc(ne); skeys.alloc(ne); vals.alloc(ne); svals.alloc(ne);
    k_coarse_emit<<<grid_for(nk), TPB, 0, st>>>(nk, rp, cl, agg.p, pos.p, nc, keys.p, vals.p);
    MSP_LAUNCH_CHECK();
    sort_pairs(tmp, keys.p, skeys.p, vals.p, svals.p, ne, bits_for((uint64_t)nc * (uint64_t)nc), st);
    ukeys.alloc(ne); rcnt.alloc(ne + 1); roff.alloc(ne + 1);
    DBuf<int64_t> nruns_d;
    nruns_d.alloc(1);
    {
      size_t bytes = 0;
      MSP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, skeys.p, ukeys.p, rcnt.p, nruns_d.p, ne, st));
      MSP_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(bytes), bytes, skeys.p, ukeys.p, rcnt.p, nruns_d.p, ne, st));
    }
    const int64_t nruns = d2h_scalar(nruns_d.p, st);
    MSP_CUDA(cudaMemsetAsync(rcnt.p + nruns, 0, sizeof(int64_t), st));
    exclusive_scan(tmp, rcnt.p, roff.p, nruns + 1, st);
    DBuf<int64_t> crp;
    DBuf<int32_t> ccol;
    DBuf<double> cw;
    crp.alloc(nc + 1); ccol.alloc(nruns); cw.alloc(nruns);
    k_coarse_sum<<<grid_for(nruns), TPB, 0, st>>>(nruns, ukeys.p, roff.p, svals.p, ww, nc, ccol.p, cw.p);
    k_rowptr_from_keys<<<grid_for(nc + 1), TPB, 0, st>>>(nc, nruns, ukeys.p, crp.p);
    MSP_LAUNCH_CHECK();

    mates.push_back(std::move(mate));
    h.agg_canon.push_back(std::move(agg));
    h.canon_rowptr.push_back(std::move(crp));
    h.canon_col.push_back(std::move(ccol));
    h.canon_w.push_back(std::move(cw));
    h.lv.push_back(LevelHost{nc, nruns, 0});
    clk.mark(st, "coarse graph", k);
  }
  h.levels = (int32_t)h.lv.size();
  const int L = h.levels;
  int64_t off = 0;
  for (auto& l : h.lv) { l.off = off; off += l.n; }
  h.n_tilde = off;
  const int64_t ntop = h.lv[L - 1].n;
  if (ntop > h.top_max)
    throw Error{MSP_ERR_UNSUPPORTED, "top level has " + std::to_string(ntop) +
                                         " nodes > top_max " + std::to_string(h.top_max)};

  // ---- powers of mu
  h.neg_mu_pow.assign(2 * L + 2, 1.0);
  std::vector<double> mu_pow(2 * L + 2, 1.0);
  for (int j = 1; j < 2 * L + 2; ++j) {
    mu_pow[j] = mu_pow[j - 1] * h.mu;
    h.neg_mu_pow[j] = h.neg_mu_pow[j - 1] * (-h.mu);
  }
  h.c_sum = 0.0;
  for (int k = 1; k <= L; ++k) h.c_sum += h.neg_mu_pow[k - 1];

  // ---- nested numbering, top-down
  h.nested_of_canon.clear();
  h.nested_of_canon.resize(L);
  std::vector<DBuf<int32_t>> order(L);  // nested pos -> canonical id
  h.nested_of_canon[L - 1].alloc(ntop);
  order[L - 1].alloc(ntop);
  k_iota32<<<grid_for(ntop), TPB, 0, st>>>(ntop, h.nested_of_canon[L - 1].p);
  k_iota32<<<grid_for(ntop), TPB, 0, st>>>(ntop, order[L - 1].p);
  h.cptr_off.assign(L, 0);
  int64_t cptr_total = 0;
  for (int k = 1; k < L; ++k) { h.cptr_off[k - 1] = cptr_total; cptr_total += h.lv[k].n + 1; }
  h.cptr.alloc(cptr_total + 8);  // + padding: TMA windows are rounded to 16 B
  MSP_CUDA(cudaMemsetAsync(h.cptr.p, 0, (cptr_total + 8) * sizeof(int32_t), st));
  for (int k = L - 1; k >= 1; --k) {
    const int64_t nk = h.lv[k - 1].n;
    DBuf<uint64_t> keys, skeys;
    DBuf<int32_t> ids;
    keys.alloc(nk); skeys.alloc(nk); ids.alloc(nk);
    order[k - 1].alloc(nk);
    h.nested_of_canon[k - 1].alloc(nk);
    k_nest_keys<<<grid_for(nk), TPB, 0, st>>>(nk, h.agg_canon[k - 1].p, mates[k - 1].p,
                                              h.nested_of_canon[k].p, keys.p, ids.p);
    sort_pairs(tmp, keys.p, skeys.p, ids.p, order[k - 1].p, nk, bits_for((uint64_t)h.lv[k].n * 3u), st);
    k_scatter_pos<<<grid_for(nk), TPB, 0, st>>>(nk, order[k - 1].p, h.nested_of_canon[k - 1].p);
    k_cptr<<<grid_for(h.lv[k].n + 1), TPB, 0, st>>>(h.lv[k].n, nk, skeys.p, h.cptr.p + h.cptr_off[k - 1]);
    MSP_LAUNCH_CHECK();
  }

  // heavy aggregates per parent level
  {
    h.heavy_off.assign(L, 0);
    int64_t maxB = 1;
    for (int k = 1; k < L; ++k) maxB = std::max<int64_t>(maxB, h.lv[k].n);
    DBuf<int32_t> ids, fl, sel, nsel;
    ids.alloc(maxB); fl.alloc(maxB); sel.alloc(maxB); nsel.alloc(1);
    k_iota32<<<grid_for(maxB), TPB, 0, st>>>(maxB, ids.p);
    std::vector<std::vector<int32_t>> lists(L);
    int64_t tot = 0;
    for (int k = 1; k < L; ++k) {
      const int64_t nB = h.lv[k].n;
      k_flag_heavy<<<grid_for(nB), TPB, 0, st>>>(nB, h.cptr.p + h.cptr_off[k - 1], fl.p);
      size_t bytes = 0;
      MSP_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ids.p, fl.p, sel.p, nsel.p, nB, st));
      MSP_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, ids.p, fl.p, sel.p, nsel.p, nB, st));
      const int64_t c = d2h_scalar(nsel.p, st);
      lists[k - 1].resize(c);
      if (c) MSP_CUDA(cudaMemcpyAsync(lists[k - 1].data(), sel.p, c * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
      h.heavy_off[k - 1] = tot;
      tot += c;
    }
    h.heavy_off[L - 1] = tot;
    h.heavy.alloc(std::max<int64_t>(tot, 1));
    for (int k = 1; k < L; ++k)
      if (!lists[k - 1].empty())
        MSP_CUDA(cudaMemcpyAsync(h.heavy.p + h.heavy_off[k - 1], lists[k - 1].data(),
                                 lists[k - 1].size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    MSP_CUDA(cudaStreamSynchronize(st));
  }
  clk.mark(st, "nested numbering");
  // ---- level-1 adjacency in nested numbering
  if (h.nnz_adj >= (int64_t)INT32_MAX) throw Error{MSP_ERR_UNSUPPORTED, "nnz >= 2^31"};
  h.perm.alloc(n);
  MSP_CUDA(cudaMemcpyAsync(h.perm.p, order[0].p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  {
    DBuf<int32_t> deg;
    deg.alloc(n + 1);
    h.rowptr1.alloc(n + 1);
    k_deg_nested<<<grid_for(n), TPB, 0, st>>>(n, h.perm.p, h.canon_rowptr[0].p, deg.p);
    MSP_CUDA(cudaMemsetAsync(deg.p + n, 0, sizeof(int32_t), st));
    exclusive_scan(tmp, deg.p, h.rowptr1.p, n + 1, st);
    h.col1.alloc(h.nnz_adj);
    h.w1.alloc(h.nnz_adj);
    k_fill_nested<<<grid_for(n), TPB, 0, st>>>(n, h.perm.p, h.canon_rowptr[0].p, h.canon_col[0].p,
                                               h.canon_w[0].p, h.nested_of_canon[0].p, h.rowptr1.p,
                                               h.col1.p, h.w1.p);
    MSP_LAUNCH_CHECK();
  }

  clk.mark(st, "nested adjacency");
  // ---- MSP block-tree factors, bottom-up
  const int64_t nt = h.n_tilde;
  h.lo_off.assign(L, 0);
  {
    int64_t lo = 0;
    for (int k = 1; k < L; ++k) { h.lo_off[k - 1] = lo; lo += h.lv[k - 1].n - 2 * h.lv[k].n; }
    h.lo_off[L - 1] = lo;
    h.lof.alloc(3 * lo + 8);
    MSP_CUDA(cudaMemsetAsync(h.lof.p, 0, (3 * lo + 8) * sizeof(double), st));
  }
  h.kinv.alloc(3 * (nt - n) + 8);
  MSP_CUDA(cudaMemsetAsync(h.kinv.p, 0, (3 * (nt - n) + 8) * sizeof(double), st));
  h.Nsub.alloc(nt + 8); h.gvec.alloc(nt + 8);
  MSP_CUDA(cudaMemsetAsync(h.Nsub.p, 0, (nt + 8) * sizeof(double), st));
  MSP_CUDA(cudaMemsetAsync(h.gvec.p, 0, (nt + 8) * sizeof(double), st));
  h.apar_canon.clear();
  h.apar_canon.resize(L > 1 ? L - 1 : 0);
  double GN = 0.0;
  for (int k = 1; k < L; ++k) {
    const int64_t nk = h.lv[k - 1].n, nk1 = h.lv[k].n;
    DBuf<int32_t> clo, chi;
    DBuf<double> wa, wb, gpart;
    clo.alloc(nk1); chi.alloc(nk1);
    h.apar_canon[k - 1].alloc(nk);
    wa.alloc(nk); wb.alloc(nk); gpart.alloc(nk1);
    k_core_ids<<<grid_for(nk), TPB, 0, st>>>(nk, mates[k - 1].p, h.agg_canon[k - 1].p, clo.p, chi.p);
    k_node_weights<<<grid_for(nk), TPB, 0, st>>>(nk, h.canon_rowptr[k - 1].p, h.canon_col[k - 1].p,
                                                 h.canon_w[k - 1].p, h.agg_canon[k - 1].p, mates[k - 1].p,
                                                 clo.p, chi.p, mu_pow[2 * k - 1], h.apar_canon[k - 1].p,
                                                 wa.p, wb.p);
    k_msp_factor<<<grid_for(nk1), TPB, 0, st>>>(nk1, h.cptr.p + h.cptr_off[k - 1], order[k - 1].p,
                                                h.apar_canon[k - 1].p, wa.p, wb.p, mu_pow[2 * (k - 1)],
                                                h.lv[k - 1].off, h.lv[k].off, n, h.lo_off[k - 1], h.kinv.p,
                                                h.lof.p, h.Nsub.p, h.gvec.p, gpart.p, k == 1 ? 1 : 0);
    MSP_LAUNCH_CHECK();
    GN += reduce_sum(tmp, gpart.p, nk1, st);
  }
  h.GN = GN;
  build_heavy_chunks(h, st);
  clk.mark(st, "factors");

  // ---- gdot weights H = G_1 (top-down over the hierarchy)
  {
    std::vector<double> ckv(L + 1, 0.0);
    double c = 0.0, pw = 1.0;
    for (int k = 1; k <= L; ++k) { c += pw; pw *= -h.mu; ckv[k] = c; }
    DBuf<double> G;
    G.alloc(nt);
    MSP_CUDA(cudaMemsetAsync(G.p, 0, nt * sizeof(double), st));
    for (int k = L - 1; k >= 1; --k)
      k_hvec<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.gvec.p + h.lv[k - 1].off,
                                                   ckv[k], (k + 1 < L) ? G.p + h.lv[k].off : nullptr,
                                                   G.p + h.lv[k - 1].off);
    MSP_LAUNCH_CHECK();
    h.Hvec.alloc(n + 8);
    MSP_CUDA(cudaMemsetAsync(h.Hvec.p, 0, (n + 8) * sizeof(double), st));
    MSP_CUDA(cudaMemcpyAsync(h.Hvec.p, G.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    MSP_CUDA(cudaStreamSynchronize(st));
  }

  clk.mark(st, "gdot weights");
  // ---- level-1 Laplacian in SELL-32 for the solve
  {
    // rows above lcap leave the SELL slices: 64 by default; 8 for a
    // heavy-tailed degree distribution (max degree > 64 x mean), whose
    // nested order mixes row lengths within a slice (SELL padding at
    // configs[4] scale 0.1: 2.6x of the entries at lcap 8, 3.0x at 16, 4.8x
    // at 64); rows of lcap+1 .. MED_ROW entries take 8 lanes each
    int lcap = 64;
    {
      DBuf<int> md;
      md.alloc(1);
      MSP_CUDA(cudaMemsetAsync(md.p, 0, sizeof(int), st));
      k_max_degree<<<grid_for(n), TPB, 0, st>>>(n, h.rowptr1.p, md.p);
      MSP_LAUNCH_CHECK();
      const int maxdeg = d2h_scalar(md.p, st);
      if ((double)maxdeg > 64.0 * (double)h.nnz_adj / (double)n) lcap = 8;
    }
    if (const char* e = std::getenv("MSP_SELL_LCAP")) lcap = std::max(1, std::atoi(e));
    const int64_t ns = (n + 31) / 32;
    h.nslices = ns;
    DBuf<int64_t> width;
    DBuf<int32_t> islong;
    width.alloc(ns + 1);
    islong.alloc(n);
    h.sell_mask.alloc(ns);
    h.sell_ptr.alloc(ns + 1);
    MSP_CUDA(cudaMemsetAsync(width.p + ns, 0, sizeof(int64_t), st));
    DBuf<int> mw;
    mw.alloc(1);
    MSP_CUDA(cudaMemsetAsync(mw.p, 0, sizeof(int), st));
    int hcap = 2048;
    if (const char* e = std::getenv("MSP_SELL_HUGE")) hcap = std::max(lcap, std::atoi(e));
    k_sell_width<<<grid_for(ns * 32), TPB, 0, st>>>(n, ns, h.rowptr1.p, lcap, hcap, width.p, h.sell_mask.p,
                                                    islong.p, mw.p);
    h.sell_maxw = d2h_scalar(mw.p, st);
    MSP_LAUNCH_CHECK();
    exclusive_scan(tmp, width.p, h.sell_ptr.p, ns + 1, st);
    int64_t tot = d2h_scalar(h.sell_ptr.p + ns, st);
    // uniform slices (every slice padded to the widest) when that costs
    // < 10% padding: the SpMV then needs no slice pointers at all
    h.sell_uniform = std::getenv("MSP_SELL_NONUNIFORM") == nullptr && h.sell_maxw > 0 &&
                     (double)ns * 32 * h.sell_maxw <= 1.1 * (double)tot;
    if (h.sell_uniform) {
      k_fill_uniform_ptr<<<grid_for(ns + 1), TPB, 0, st>>>(ns, 32 * (int64_t)h.sell_maxw, h.sell_ptr.p);
      MSP_LAUNCH_CHECK();
      tot = ns * 32 * (int64_t)h.sell_maxw;
    }
    h.sell_col.alloc(std::max<int64_t>(tot, 1));
    h.sell_w.alloc(std::max<int64_t>(tot, 1));
    k_sell_fill<<<grid_for(ns * 32), TPB, 0, st>>>(n, ns, h.sell_ptr.p, h.rowptr1.p, h.col1.p, h.w1.p,
                                                   h.sell_mask.p, h.sell_col.p, h.sell_w.p);
    MSP_LAUNCH_CHECK();
    // medium, long and huge rows, each class in increasing order (deterministic)
    DBuf<int32_t> ids, nsel;
    ids.alloc(n);
    nsel.alloc(1);
    k_iota32<<<grid_for(n), TPB, 0, st>>>(n, ids.p);
    h.long_rows.alloc(n);
    DBuf<int32_t> fl;
    fl.alloc(n);
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ids.p, fl.p, h.long_rows.p, nsel.p, n, st));
    // medium rows first, then the long ones (both "long" for the SpMV
    // kernels that take a warp per row: nlong counts both)
    k_flag_eq<<<grid_for(n), TPB, 0, st>>>(n, islong.p, 1, fl.p);
    MSP_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, ids.p, fl.p, h.long_rows.p, nsel.p, n, st));
    h.nmed = d2h_scalar(nsel.p, st);
    k_flag_eq<<<grid_for(n), TPB, 0, st>>>(n, islong.p, 3, fl.p);
    MSP_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, ids.p, fl.p, h.long_rows.p + h.nmed, nsel.p, n, st));
    h.nlong = h.nmed + d2h_scalar(nsel.p, st);
    k_flag_eq<<<grid_for(n), TPB, 0, st>>>(n, islong.p, 2, fl.p);  // huge rows follow the long ones
    MSP_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, ids.p, fl.p, h.long_rows.p + h.nlong, nsel.p, n, st));
    h.nhuge = d2h_scalar(nsel.p, st);
    // huge rows cut into segments of <= HUGE_SEG entries (sched.cuh)
    {
      std::vector<int32_t> hr(std::max<int64_t>(h.nhuge, 1)), hp(std::max<int64_t>(2 * h.nhuge, 1));
      if (h.nhuge > 0)
        MSP_CUDA(cudaMemcpyAsync(hr.data(), h.long_rows.p + h.nlong, h.nhuge * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
      if (h.nhuge > 0) {
        DBuf<int32_t> bnd;
        bnd.alloc(2 * h.nhuge);
        k_row_bounds<<<grid_for(h.nhuge), TPB, 0, st>>>(h.nhuge, h.long_rows.p + h.nlong, h.rowptr1.p, bnd.p);
        MSP_LAUNCH_CHECK();
        MSP_CUDA(cudaMemcpyAsync(hp.data(), bnd.p, 2 * h.nhuge * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        MSP_CUDA(cudaStreamSynchronize(st));
      }
      std::vector<int4> segs;
      std::vector<int32_t> first(h.nhuge + 1, 0);
      int64_t hseg = HUGE_SEG;  // MSP_HUGE_SEG: shorter segments for tests of the multi-segment path
      if (const char* e = std::getenv("MSP_HUGE_SEG")) hseg = std::max<int64_t>(32, std::atoll(e));
      for (int64_t i = 0; i < h.nhuge; ++i) {
        first[i] = (int32_t)segs.size();
        for (int64_t e = hp[2 * i]; e < hp[2 * i + 1]; e += hseg)
          segs.push_back(make_int4((int)i, (int)e, (int)std::min<int64_t>(e + hseg, hp[2 * i + 1]), 0));
      }
      first[h.nhuge] = (int32_t)segs.size();
      h.nhseg = (int64_t)segs.size();
      if (std::getenv("MSP_VERBOSE"))
        fprintf(stderr, "[msp] SELL: n=%lld slices=%lld maxw=%d uniform=%d entries=%lld (adjacency %lld) lcap=%d "
                "long=%lld huge=%lld huge segments=%lld\n", (long long)n, (long long)ns, h.sell_maxw,
                (int)h.sell_uniform, (long long)tot, (long long)h.nnz_adj, lcap, (long long)h.nlong,
                (long long)h.nhuge, (long long)h.nhseg);
      h.hseg.alloc(std::max<size_t>(segs.size(), 1));
      h.hfirst.alloc(h.nhuge + 1);
      h.hcnt.alloc(std::max<int64_t>(h.nhuge, 1));
      h.hpart.alloc(std::max<size_t>(segs.size(), 1));
      h.hdot.alloc(std::max<int64_t>(h.nhuge, 1));
      if (!segs.empty())
        MSP_CUDA(cudaMemcpyAsync(h.hseg.p, segs.data(), segs.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
      MSP_CUDA(cudaMemcpyAsync(h.hfirst.p, first.data(), first.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      MSP_CUDA(cudaMemsetAsync(h.hcnt.p, 0, std::max<int64_t>(h.nhuge, 1) * sizeof(unsigned), st));
      MSP_CUDA(cudaStreamSynchronize(st));
    }
  }

  build_hot_cache(h, st);
  clk.mark(st, "SELL");
  // ---- top level: dense pseudo-inverse of sigma_l L_l
  {
    DBuf<double> M, A;
    M.alloc(ntop * ntop);
    A.alloc(std::max<int64_t>((ntop - 1) * 2 * (ntop - 1), 1));
    h.top_pinv.alloc(ntop * ntop);
    k_top_dense<<<grid_for(ntop), TPB, 0, st>>>(ntop, h.canon_rowptr[L - 1].p, h.canon_col[L - 1].p,
                                                h.canon_w[L - 1].p, mu_pow[2 * (L - 1)], M.p);
    k_top_pinv<<<1, 256, 0, st>>>((int)ntop, M.p, A.p, h.top_pinv.p);
    MSP_LAUNCH_CHECK();
    if (L == 1) {  // no hierarchy (n <= 2): N = 1 for all top nodes
      std::vector<double> ones(ntop, 1.0);
      MSP_CUDA(cudaMemcpyAsync(h.Nsub.p, ones.data(), ntop * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    MSP_CUDA(cudaStreamSynchronize(st));
  }

  clk.mark(st, "top pseudo-inverse");
  {
    const char* e = std::getenv("MSP_WDOWN");
    h.wdown = e ? std::atoi(e) != 0 : false;
  }
  build_schedule(h, st);
  clk.mark(st, "schedule");
  MSP_CUDA(cudaEventRecord(e1, st));
  MSP_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  MSP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  h.setup_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  h.mates_canon = std::move(mates);
  h.order_nested = std::move(order);
}


Lv make_level_table(const Handle& h) {
  Lv lv{};
  lv.L = h.levels;
  lv.Kc = h.Kc;
  for (int k = 1; k <= h.levels; ++k) {
    lv.n[k - 1] = h.lv[k - 1].n;
    lv.off[k - 1] = h.lv[k - 1].off;
    lv.cpo[k - 1] = (k < h.levels) ? h.cptr_off[k - 1] : 0;
    lv.lo[k - 1] = h.lo_off.empty() ? 0 : h.lo_off[k - 1];
    lv.ck[k] = h.ck.empty() ? 0.0 : h.ck[k];
  }
  lv.negmu = -h.mu;
  lv.c_sum = h.c_sum;
  lv.n_tilde = (double)h.n_tilde;
  lv.GN = h.GN;
  return lv;
}

namespace {
inline int a16(int64_t b) { return (int)((b + 15) & ~(int64_t)15); }

// per-tier shared-memory layout from the largest per-level tile ranges
// cap[t] (nodes) and caplo[t] (leftovers among level-(k0+t) children);
// the up kernel's segments come first (smem_up is their end)
TierDesc tier_layout(int k0, int nl, int64_t ntiles, const std::vector<int64_t>& cap,
                     const std::vector<int64_t>& caplo, int64_t gemv_n) {
  TierDesc d{};
  d.k0 = k0;
  d.nl = nl;
  d.ntiles = (int)ntiles;
  d.gemv_n = (int)gemv_n;
  d.o_v = -1;
  int64_t cur = 0;
  auto take = [&](int64_t bytes) { const int o = a16(cur); cur = o + bytes; return o; };
  d.o_uf = take((cap[nl - 1] + 1 + 8) * 4);
  d.o_uy0 = take((cap[0] + 2) * 8);
  d.smem_up = a16(cur);
  cur = 0;
  for (int t = 1; t < nl; ++t) d.o_cp[t] = take((cap[t] + 1 + 8) * 4);
  d.o_y[0] = take((cap[0] + 2) * 8);
  for (int t = 1; t + 1 < nl; ++t) d.o_y[t] = take(cap[t] * 8);
  for (int t = 1; t < nl; ++t) d.o_ki[t] = take((3 * cap[t] + 2) * 8);
  for (int t = 0; t + 1 < nl; ++t) d.o_lo[t] = take((3 * caplo[t] + 2) * 8);
  d.o_n[0] = (k0 > 1) ? take((cap[0] + 2) * 8) : 0;
  // z, w of an intermediate level overwrite its y, N: the down step of level
  // k reads y_p, N_p of a child before it writes z_p, w_p (block_solve)
  for (int t = 1; t + 1 < nl; ++t) {
    d.o_n[t] = take(cap[t] * 8);
    d.o_z[t] = d.o_y[t];
    d.o_w[t] = d.o_n[t];
  }
  d.o_z[nl - 1] = take((cap[nl - 1] + 2) * 8);
  d.o_w[nl - 1] = take((cap[nl - 1] + 2) * 8);
  if (gemv_n > 0) d.o_v = take((gemv_n + 1) * 8);
  d.smem_down = a16(cur);
  return d;
}

}  // namespace

static inline int a16c(int64_t b) { return (int)((b + 15) & ~(int64_t)15); }
CoarseDesc coarse_desc(const Handle& h, int Kc, bool stage_pinv) {
  CoarseDesc d{};
  const int L = h.levels, nl = L - Kc + 1;
  d.nl = nl;
  d.stage_pinv = stage_pinv ? 1 : 0;
  int64_t cur = 0;
  auto take = [&](int64_t bytes) { const int o = a16c(cur); cur = o + bytes; return o; };
  auto nk = [&](int t) { return h.lv[Kc + t - 1].n; };
  for (int t = 1; t < nl; ++t) {
    d.o_cp[t] = take((nk(t) + 1 + 8) * 4);
    d.o_ki[t] = take((3 * nk(t) + 2) * 8);
  }
  for (int t = 0; t + 1 < nl; ++t) d.o_lo[t] = take((3 * (nk(t) - 2 * nk(t + 1)) + 2) * 8);
  for (int t = 0; t < nl; ++t) d.o_n[t] = take((nk(t) + 2) * 8);
  d.o_y[0] = take((nk(0) + 2) * 8);
  for (int t = 1; t < nl; ++t) d.o_y[t] = take(nk(t) * 8);
  for (int t = 0; t < nl; ++t) {
    d.o_z[t] = take(nk(t) * 8);
    d.o_w[t] = take(nk(t) * 8);
  }
  const int64_t ntop = h.lv[L - 1].n;
  d.o_pinv = stage_pinv ? take((ntop * ntop + 2) * 8) : 0;
  d.o_tt = take(ntop * 8);
  d.smem = a16c(cur);
  return d;
}


// Static TMA segments (sched.cuh) of tiles whose starts per level are
// ts[u * (ntiles + 1) + j] (host copy), for the down kernel of tier k0.. with
// nl levels and layout d: the kernel stages them without computing windows.
std::vector<int4> make_tile_segs(const Handle& h, int k0_, int nl, const TierDesc& d, const std::vector<int32_t>& ts,
                                 int64_t ntiles) {
  const int S = 3 * (nl - 1) + (k0_ > 1 ? 1 : 0);
  const int64_t nt1 = ntiles + 1;
  std::vector<int4> segs((size_t)ntiles * S);
  const int64_t n1 = h.lv[0].n;
  for (int64_t j = 0; j < ntiles; ++j) {
    auto sa = [&](int u) { return (int64_t)ts[(size_t)u * nt1 + j]; };
    auto sn = [&](int u) { return (int64_t)ts[(size_t)u * nt1 + j + 1] - sa(u); };
    int g = 0;
    auto put = [&](int kind, int tt, int dst, int es, int64_t lo, int64_t hi) {
      const int64_t m = (es == 4) ? 3 : 1;
      const int64_t a0 = lo & ~m;
      const int64_t e0 = (hi + m) & ~m;
      const int64_t bytes = (hi > lo) ? (e0 - a0) * es : 0;
      if (a0 > INT32_MAX || bytes > INT32_MAX) throw Error{MSP_ERR_UNSUPPORTED, "segment offset >= 2^31"};
      segs[(size_t)j * S + g++] = make_int4(kind | (tt << 2) | (dst << 8), (int)bytes, (int)a0, (int)(lo - a0));
    };
    for (int u = 1; u < nl; ++u) {
      const int64_t base = h.cptr_off[k0_ + u - 2];
      put(SEG_CP, u, d.o_cp[u], 4, base + sa(u), base + sa(u) + sn(u) + 1);
    }
    for (int u = 1; u < nl; ++u) {
      const int64_t base = 3 * (h.lv[k0_ + u - 1].off - n1 + sa(u));
      put(SEG_KI, u, d.o_ki[u], 8, base, base + 3 * sn(u));
    }
    for (int u = 0; u + 1 < nl; ++u) {
      const int64_t lo0 = sa(u) - 2 * sa(u + 1);
      const int64_t lo1 = (sa(u) + sn(u)) - 2 * (sa(u + 1) + sn(u + 1));
      const int64_t base = 3 * h.lo_off[k0_ + u - 1];
      put(SEG_LO, u, d.o_lo[u], 8, base + 3 * lo0, base + 3 * lo1);
    }
    if (k0_ > 1) {
      const int64_t base = h.lv[k0_ - 1].off;
      put(SEG_N0, 0, d.o_n[0], 8, base + sa(0), base + sa(0) + sn(0));
    }
  }
  return segs;
}

__global__ void k_deg_key(int64_t n, const int32_t* __restrict__ rowptr, int32_t maxdeg, int32_t* __restrict__ key) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) key[i] = maxdeg - (rowptr[i + 1] - rowptr[i]);  // ascending key = decreasing degree
}

__global__ void k_hot_rank(int64_t nhot, const int32_t* __restrict__ rows, int32_t* __restrict__ rank) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nhot) rank[rows[k]] = (int32_t)k;
}

__global__ void k_remap_cols(int64_t m, const int32_t* __restrict__ col, const int32_t* __restrict__ rank,
                             int32_t* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < m) {
    const int32_t j = col[e];
    const int32_t r = rank[j];
    out[e] = (r >= 0) ? (HOT_BIT | r) : j;
  }
}

// Hot-vertex gather cache of a heavy-tailed graph (long rows present, n
// large): in a Chung-Lu graph of exponent 2.1 the few highest-degree
// vertices are the endpoints of most edges, but the nested numbering
// scatters them over the whole (z, p) array, so at configs[4]'s full size
// (47M vertices, a 757 MB pair array) the SpMV's gathers missed L2 83 % of
// the time (57.7 GB of DRAM reads per SpMV for 10 GB of streams).  Their
// pairs are copied each iteration into one compact array (16 B each) that
// stays in L2, and the SpMV's column copies address it directly.  The
// copied values are the same doubles: the SpMV result is unchanged bit for
// bit.  MSP_HOT_K sets the count (0: off).
void build_hot_cache(Handle& h, cudaStream_t st) {
  h.nhot = 0;
  const int64_t n = h.n;
  int64_t K = 0;
  if (h.nlong + h.nhuge > 0 && n >= (int64_t(1) << 23)) K = int64_t(1) << 22;  // 64 MB of pairs
  if (const char* e = std::getenv("MSP_HOT_K")) K = std::atoll(e);
  K = std::min<int64_t>(K, n);
  if (K <= 0) return;
  Temp tmp;
  DBuf<int> md;
  md.alloc(1);
  MSP_CUDA(cudaMemsetAsync(md.p, 0, sizeof(int), st));
  k_max_degree<<<grid_for(n), TPB, 0, st>>>(n, h.rowptr1.p, md.p);
  const int maxdeg = d2h_scalar(md.p, st);
  DBuf<int32_t> key, skey, ids, sids, rank;
  key.alloc(n); skey.alloc(n); ids.alloc(n); sids.alloc(n); rank.alloc(n);
  k_deg_key<<<grid_for(n), TPB, 0, st>>>(n, h.rowptr1.p, maxdeg, key.p);
  k_iota32<<<grid_for(n), TPB, 0, st>>>(n, ids.p);
  sort_pairs(tmp, key.p, skey.p, ids.p, sids.p, n, bits_for((uint64_t)maxdeg + 1), st);  // stable: ties by id
  h.nhot = K;
  h.hot_rows.alloc(K);
  MSP_CUDA(cudaMemcpyAsync(h.hot_rows.p, sids.p, K * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  MSP_CUDA(cudaMemsetAsync(rank.p, 0xff, n * sizeof(int32_t), st));
  k_hot_rank<<<grid_for(K), TPB, 0, st>>>(K, h.hot_rows.p, rank.p);
  const int64_t ms = h.sell_ptr.n ? d2h_scalar(h.sell_ptr.p + h.nslices, st) : 0;
  h.sell_colh.alloc(std::max<int64_t>(ms, 1));
  if (ms) k_remap_cols<<<grid_for(ms), TPB, 0, st>>>(ms, h.sell_col.p, rank.p, h.sell_colh.p);
  h.col1h.alloc(std::max<int64_t>(h.nnz_adj, 1));
  k_remap_cols<<<grid_for(h.nnz_adj), TPB, 0, st>>>(h.nnz_adj, h.col1.p, rank.p, h.col1h.p);
  h.hot_pairs.alloc(2 * K + 8);
  MSP_CUDA(cudaMemsetAsync(h.hot_pairs.p, 0, (2 * K + 8) * sizeof(double), st));
  MSP_LAUNCH_CHECK();
  MSP_CUDA(cudaStreamSynchronize(st));
}

// K_j = sum over the leftovers x of heavy aggregate h of C(x, j) N_x (one
// CTA per heavy aggregate, fixed-order block sum; setup only)
__global__ void k_heavy_const(int64_t nh, const int32_t* __restrict__ heavy, const int32_t* __restrict__ cp,
                              const double* __restrict__ lof, const double* __restrict__ Nk, int64_t lo_k,
                              double* __restrict__ cst) {
  const int64_t B = heavy[blockIdx.x];
  const int64_t s0 = cp[B], s1 = cp[B + 1];
  const int64_t lb = 3 * (lo_k - 2 * B - 2);
  double a = 0.0, b = 0.0;
  for (int64_t p = s0 + 2 + threadIdx.x; p < s1; p += blockDim.x) {
    a += lof[lb + 3 * p + 0] * Nk[p];
    b += lof[lb + 3 * p + 1] * Nk[p];
  }
  __shared__ double sa[256], sb[256];
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) { ta += sa[i]; tb += sb[i]; }
    cst[2 * blockIdx.x] = ta;
    cst[2 * blockIdx.x + 1] = tb;
  }
}

// Chunks of the heavy aggregates (sched.cuh HeavyChunks)
void build_heavy_chunks(Handle& h, cudaStream_t st) {
  const int L = h.levels;
  h.hch_off.assign(L, 0);
  const int64_t nh = h.heavy_off.empty() ? 0 : h.heavy_off[L - 1];
  if (nh == 0 || std::getenv("MSP_NO_HEAVY_CHUNKS")) { h.hch_off.clear(); return; }  // off: a CTA per heavy aggregate
  int64_t CH = HEAVY_CHUNK;  // MSP_HEAVY_CHUNK: smaller chunks for tests of the multi-chunk path
  if (const char* e = std::getenv("MSP_HEAVY_CHUNK")) CH = std::max<int64_t>(2, std::atoll(e));
  std::vector<int4> segs;
  std::vector<int32_t> first(nh + 1, 0);
  for (int k = 1; k < L; ++k) {
    h.hch_off[k - 1] = (int64_t)segs.size();
    const int64_t a = h.heavy_off[k - 1], b = h.heavy_off[k];
    if (b == a) continue;
    std::vector<int32_t> ids(b - a);
    MSP_CUDA(cudaMemcpyAsync(ids.data(), h.heavy.p + a, (b - a) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    const int64_t nB = h.lv[k].n;
    std::vector<int32_t> cp(nB + 1);
    MSP_CUDA(cudaMemcpyAsync(cp.data(), h.cptr.p + h.cptr_off[k - 1], (nB + 1) * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < b - a; ++i) {
      const int32_t B = ids[i];
      first[a + i] = (int32_t)segs.size();
      for (int64_t c = cp[B]; c < cp[B + 1]; c += CH)
        segs.push_back(make_int4(B, (int)c, (int)std::min<int64_t>(c + CH, cp[B + 1]), (int)(a + i)));
    }
    h.hch_off[k] = (int64_t)segs.size();
  }
  h.hch_off[L - 1] = (int64_t)segs.size();
  for (int k = 1; k < L; ++k) h.hch_off[k] = std::max(h.hch_off[k], h.hch_off[k - 1]);
  first[nh] = (int32_t)segs.size();
  h.hch_seg.alloc(segs.size());
  MSP_CUDA(cudaMemcpyAsync(h.hch_seg.p, segs.data(), segs.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  h.hch_first.alloc(nh + 1);
  MSP_CUDA(cudaMemcpyAsync(h.hch_first.p, first.data(), (nh + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  h.hch_cnt.alloc(nh);
  MSP_CUDA(cudaMemsetAsync(h.hch_cnt.p, 0, nh * sizeof(unsigned), st));
  h.hch_part.alloc(3 * segs.size());
  h.hch_sum.alloc(2 * nh);
  MSP_CUDA(cudaMemsetAsync(h.hch_sum.p, 0, 2 * nh * sizeof(double), st));
  h.hch_cst.alloc(2 * nh);
  for (int k = 1; k < L; ++k) {
    const int64_t a = h.heavy_off[k - 1], b = h.heavy_off[k];
    if (b == a) continue;
    k_heavy_const<<<(unsigned)(b - a), 256, 0, st>>>(b - a, h.heavy.p + a, h.cptr.p + h.cptr_off[k - 1], h.lof.p,
                                                     h.Nsub.p + h.lv[k - 1].off, h.lo_off[k - 1],
                                                     h.hch_cst.p + 2 * a);
  }
  MSP_LAUNCH_CHECK();
  MSP_CUDA(cudaStreamSynchronize(st));
}

// Tiers and tiles of the solve schedule.
void build_schedule(Handle& h, cudaStream_t st) {
  const int L = h.levels;
  if (L >= MAXL) throw Error{MSP_ERR_UNSUPPORTED, "more than 39 levels"};
  h.ck.assign(L + 1, 0.0);
  {
    double c = 0.0, pw = 1.0;
    for (int k = 1; k <= L; ++k) { c += pw; pw *= -h.mu; h.ck[k] = c; }
  }
  int64_t T = 512, SUB = 256, CMAX = 512;   // CMAX: measured best over configs[1..3]
  if (const char* e = std::getenv("MSP_TILE_T")) T = std::max<int64_t>(16, std::atoll(e));
  SUB = T / 2;
  if (const char* e = std::getenv("MSP_TILE_SUB")) SUB = std::max<int64_t>(2, std::atoll(e));
  // the first tier's tiles and subtree cap (its down kernel runs a warp per
  // tile, k_wtile_down: smaller tiles, more independent warps per SM)
  int64_t T1 = T, SUB1 = SUB;
  if (h.wdown) { T1 = 128; SUB1 = 128; }
  if (const char* e = std::getenv("MSP_WTILE")) T1 = std::max<int64_t>(16, std::atoll(e));
  if (const char* e = std::getenv("MSP_WSUB")) SUB1 = std::max<int64_t>(2, std::atoll(e));
  if (const char* e = std::getenv("MSP_COARSE_MAX")) CMAX = std::max<int64_t>(2, std::atoll(e));
  const size_t SMEM_CAP = 200 * 1024;
  const Lv lv = make_level_table(h);

  // coarse level: smallest Kc whose levels Kc..L fit the single-CTA kernel
  // (and, in GEMV mode, whose n_Kc <= GEMV_MAX)
  int64_t GEMV_MAX = 0;  // off: see DESIGN.md "Coarse GEMV" (3e-12 vs 1e-14 accuracy, no faster)
  if (const char* e = std::getenv("MSP_GEMV_MAX")) GEMV_MAX = std::atoll(e);
  const bool stage_pinv = h.lv[L - 1].n <= 32;
  {
    int Kc = L;
    int64_t tail = 0;
    for (int k = L; k >= 1; --k) {
      tail += h.lv[k - 1].n;
      if (tail > CMAX || L - k + 1 > MAXT + 8) break;
      if ((size_t)coarse_desc(h, k, stage_pinv).smem > SMEM_CAP) break;
      if (GEMV_MAX > 0 && k > 1 && h.lv[k - 1].n > GEMV_MAX) break;
      Kc = k;
    }
    h.Kc = Kc;
  }
  // GEMV mode needs Kc > 1 and a tiled top tier (checked below)
  bool gemv_ok = GEMV_MAX > 0 && h.Kc > 1;
  h.cdesc = coarse_desc(h, h.Kc, stage_pinv);
  h.coarse_smem = (size_t)h.cdesc.smem;

  // tiers over levels 1..Kc
  h.tiers.clear();
  int k0 = 1;
  const int64_t T0 = T;
  auto add_tiles = [&](int k0_, int k1_, DBuf<int32_t>* first_k1) {
    Handle::Tier t;
    t.k0 = k0_;
    t.k1 = k1_;
    const int nl = k1_ - k0_ + 1;
    const int64_t n0 = h.lv[k0_ - 1].n;
    const int64_t T = (k0_ == 1) ? T1 : T0;
    t.ntiles = std::max<int64_t>(1, (n0 + T - 1) / T);
    const int64_t nt1 = t.ntiles + 1;
    t.tstart.alloc((size_t)nl * nt1);
    if (nl == 1) {
      DBuf<int32_t> id;
      id.alloc(n0 + 1);
      k_iota32<<<grid_for(n0 + 1), TPB, 0, st>>>(n0 + 1, id.p);
      k_tile_bounds<<<grid_for(nt1), TPB, 0, st>>>(t.ntiles, n0, T, id.p, t.tstart.p);
      MSP_LAUNCH_CHECK();
      MSP_CUDA(cudaStreamSynchronize(st));
      // level 1 only: the r, q, H windows of one tile of T rows
      t.desc.o_uf = 0;
      t.desc.o_uy0 = 16;
      t.desc.o_uq = a16(t.desc.o_uy0 + (T + 2) * 8);
      t.desc.o_uh = a16(t.desc.o_uq + (T + 2) * 8);
      t.desc.smem_up = a16(t.desc.o_uh + (T + 2) * 8);
      t.smem_up = t.desc.smem_up;
      t.desc.k0 = 1;
      t.desc.nl = 1;
      t.desc.ntiles = (int)t.ntiles;
      t.desc.up_group = 1;
      t.up_group = 1;
    } else {
      k_tile_bounds<<<grid_for(nt1), TPB, 0, st>>>(t.ntiles, h.lv[k1_ - 1].n, T, first_k1->p,
                                                    t.tstart.p + (int64_t)(nl - 1) * nt1);
      for (int u = nl - 2; u >= 0; --u) {
        const int kc = k0_ + u;  // child level
        k_tile_descend<<<grid_for(nt1), TPB, 0, st>>>(nt1, h.cptr.p + h.cptr_off[kc - 1],
                                                       t.tstart.p + (int64_t)(u + 1) * nt1,
                                                       t.tstart.p + (int64_t)u * nt1);
      }
      MSP_LAUNCH_CHECK();
      std::vector<int32_t> ts((size_t)nl * nt1);
      MSP_CUDA(cudaMemcpyAsync(ts.data(), t.tstart.p, ts.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
      std::vector<int64_t> cap(nl, 0), caplo(nl, 0);
      for (int64_t j = 0; j < t.ntiles; ++j) {
        for (int u = 0; u < nl; ++u) {
          const int64_t a = ts[(size_t)u * nt1 + j], b = ts[(size_t)u * nt1 + j + 1];
          cap[u] = std::max(cap[u], b - a);
          if (u + 1 < nl) {
            const int64_t a2 = ts[(size_t)(u + 1) * nt1 + j], b2 = ts[(size_t)(u + 1) * nt1 + j + 1];
            caplo[u] = std::max(caplo[u], (b - 2 * b2) - (a - 2 * a2));
          }
        }
      }
      const bool top = (k1_ == h.Kc) && gemv_ok;
      t.desc = tier_layout(k0_, nl, t.ntiles, cap, caplo, top ? h.lv[h.Kc - 1].n : 0);
      t.desc.tpc = 1;  // first tier: set in alloc_solve_workspace (needs the occupancy)
      // static TMA segments of every tile of the down kernel (sched.cuh)
      {
        t.desc.nseg = 3 * (nl - 1) + (k0_ > 1 ? 1 : 0);
        const std::vector<int4> segs = make_tile_segs(h, k0_, nl, t.desc, ts, t.ntiles);
        t.segs.alloc(std::max<size_t>(segs.size(), 1));
        MSP_CUDA(cudaMemcpyAsync(t.segs.p, segs.data(), segs.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
        MSP_CUDA(cudaStreamSynchronize(st));
      }
      // the up kernel takes `up_group` consecutive tiles per CTA (its level-1
      // pass is a plain stream; more work per CTA amortises the fixed cost)
      {
        int G = (k0_ == 1) ? 8 : 1;  // 1 / 2 / 4 / 6 / 8 / 16 measured on configs[1..3]: 8 best
        if (const char* e = std::getenv("MSP_UP_GROUP")) G = (k0_ == 1) ? std::max(1, std::atoi(e)) : 1;
        int64_t c0 = 0, c1 = 0;
        for (int64_t j = 0; j < t.ntiles; j += G) {
          const int64_t je = std::min<int64_t>(j + G, t.ntiles);
          c0 = std::max<int64_t>(c0, ts[je] - ts[j]);
          c1 = std::max<int64_t>(c1, ts[(size_t)(nl - 1) * nt1 + je] - ts[(size_t)(nl - 1) * nt1 + j]);
        }
        t.up_group = G;
        t.desc.o_uf = 0;
        t.desc.o_uy0 = a16((c1 + 1 + 8) * 4);            // r (FIRST: staged, updated in place) or y_k0
        t.desc.o_uq = a16(t.desc.o_uy0 + (c0 + 2) * 8);  // q (FIRST)
        t.desc.o_uh = a16(t.desc.o_uq + (c0 + 2) * 8);   // H (FIRST)
        t.desc.smem_up = (k0_ == 1) ? a16(t.desc.o_uh + (c0 + 2) * 8) : a16(t.desc.o_uy0 + (c0 + 2) * 8);
        t.desc.up_group = G;
      }
      const int64_t nk1 = h.lv[k1_ - 1].n;
      t.firstk0.alloc(nk1 + 1 + 8);
      MSP_CUDA(cudaMemsetAsync(t.firstk0.p, 0, (nk1 + 1 + 8) * sizeof(int32_t), st));
      MSP_CUDA(cudaMemcpyAsync(t.firstk0.p, first_k1->p, (nk1 + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      t.smem_up = t.desc.smem_up;
      t.smem_down = t.desc.smem_down;
    }
    h.tiers.push_back(std::move(t));
  };
  if (h.Kc == 1) {
    add_tiles(1, 1, nullptr);  // the PCG update only; everything else in the coarse kernel
  }
  while (k0 < h.Kc) {
    // first level-k0 descendants of the levels above, and the largest subtree
    const int kmax = std::min(h.Kc, k0 + MAXT - 1);  // tier depth <= MAXT levels
    std::vector<DBuf<int32_t>> first(kmax - k0 + 1);
    first[0].alloc(h.lv[k0 - 1].n + 1);
    k_iota32<<<grid_for(h.lv[k0 - 1].n + 1), TPB, 0, st>>>(h.lv[k0 - 1].n + 1, first[0].p);
    DBuf<int> mx;
    mx.alloc(kmax - k0 + 1);
    MSP_CUDA(cudaMemsetAsync(mx.p, 0, (kmax - k0 + 1) * sizeof(int), st));
    for (int k = k0 + 1; k <= kmax; ++k) {
      const int u = k - k0;
      first[u].alloc(h.lv[k - 1].n + 1);
      k_first1<<<grid_for(h.lv[k - 1].n + 1), TPB, 0, st>>>(h.lv[k - 1].n, h.cptr.p + h.cptr_off[k - 2],
                                                           first[u - 1].p, first[u].p, mx.p + u);
    }
    MSP_LAUNCH_CHECK();
    std::vector<int> maxsz(kmax - k0 + 1);
    MSP_CUDA(cudaMemcpyAsync(maxsz.data(), mx.p, maxsz.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    int k1 = k0;
    for (int k = k0 + 1; k <= kmax; ++k) {
      if (maxsz[k - k0] <= (k0 == 1 ? SUB1 : SUB)) k1 = k;
      else break;
    }
    if (k1 == k0) {  // an aggregate with more than SUB children: one generic level
      Handle::Tier t;
      t.k0 = k0;
      t.k1 = k0 + 1;
      t.generic = true;
      h.tiers.push_back(std::move(t));
      if (k0 == 1) {  // the PCG update still needs a tile pass over level 1
        add_tiles(1, 1, nullptr);
        std::swap(h.tiers[h.tiers.size() - 1], h.tiers[h.tiers.size() - 2]);
      }
      k0 += 1;
      continue;
    }
    for (;;) {  // shrink the tier until its tiles fit in shared memory
      add_tiles(k0, k1, &first[k1 - k0]);
      if (h.tiers.back().smem_down <= SMEM_CAP || k1 == k0 + 1) break;
      h.tiers.pop_back();
      --k1;
    }
    if (h.tiers.back().smem_down > SMEM_CAP)
      throw Error{MSP_ERR_UNSUPPORTED, "a tile does not fit in shared memory"};
    k0 = k1;
  }
  h.gemv = gemv_ok && !h.tiers.empty() && !h.tiers.back().generic && h.tiers.back().k1 == h.Kc &&
           h.tiers.back().desc.gemv_n > 0;
}

}  // namespace msp
