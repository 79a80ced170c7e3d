// pegp.cu -- the PEGP preconditioner R = P(mu) L_H~^+ P(mu)^T (§3.2)
// on the GPU, and the expanded-space pieces it needs (sm_100a).
//
// H~ (readings R6/R7) is assembled once, at the first PEGP call, as an
// explicit symmetric CSR of its edge weights over the nested expanded
// numbering.  Its edges are enumerated from the per-level graphs (Eq.
// def:L_ell written blockwise: block (k, j) = (-mu)^{k-1} (-mu)^{j-1} L_k P_k^j,
// with P_k^j the 0/1 aggregation from level k to level j):
//   * k = j:   every level-k edge, weight mu^{2(k-1)} w_k(i, m);
//   * j > k, j - k odd:  node i -> its level-j ancestor A_j(i), weight
//     mu^{k+j-2} cut_kj(i), cut_kj(i) = weight from i to level-k neighbours m
//     whose level-j ancestor differs from i's;
//   * j > k, j - k even: node i -> A_j(m) for every level-k neighbour m with
//     A_j(m) != A_j(i), weight mu^{k+j-2} w_k(i, m).
// These are exactly the negative off-diagonal entries of L_G~ (the positive
// edges of G~); walking the two ancestor chains from (i, m) upwards until they
// meet enumerates them.  Every (row, column, weight) triple is emitted in both
// directions, sorted by (row, column) and merged (duplicates summed in sorted
// order: the CSR is bit-identical run to run).  L_H~ x is then applied in the
// difference form sum_j w_ij (x_i - x_j) -- the exact diagonal of R7, never
// rounded into an assembled diagonal.
//
// L_H~^+ r~ (minimum norm) is computed by CG in the expanded space,
// preconditioned by the exact MSP solve L_T~^+ (T~ is a spanning subgraph of
// H~, §3.3), to a relative residual of `pegp_rtol` (default 1e-13), optionally
// followed by `pegp_refine` steps of iterative refinement whose residual is
// formed in double-double arithmetic (reading R13).  One inner iteration is
//   k_h_spmv   p = z + beta p and q = L_H~ p fused, (p, q) by a ticketed
//              block reduction that also forms alpha;
//   k_e_up     per level above 1 while the level is large: x += alpha p,
//              r -= alpha q, T~ subtree sums s, block partials of (r, r),
//              sum r and (g, s);
//   k_e_coarse one CTA: the small levels' up sweep, the partial sums, the
//              convergence test, the top solve and the small levels' down
//              sweep;
//   k_e_down   per large level, top-down: z of the children from the block-
//              tree factors of T~, (r, z) partials; the last CTA of the
//              level-1 sweep forms (r, z) and beta.
// Iterations run in captured CUDA graphs of 8; the host reads the converged
// flag once per graph.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace msp {

namespace {

constexpr int TPB = 256;
constexpr int CO_T = 1024;   // threads of the coarse CTA (one node per thread per level at most CO_MAX)
constexpr int CO_MAX = 1024; // levels of at most this many nodes go to the coarse CTA
constexpr int H_G0 = 8;      // lanes per row of the short-row class
constexpr int H_D0 = 32;     // short rows: degree <= H_D0
constexpr int H_D1 = 512;    // warp rows: degree <= H_D1; longer rows: segments
constexpr int H_SEG = 2048;  // entries per long-row segment (a CTA)
constexpr int H_U = 4;       // short rows per 8-lane group and step

inline unsigned grid_for(int64_t n, int tpb = TPB) {
  int64_t g = (n + tpb - 1) / tpb;
  return (unsigned)std::max<int64_t>(g, 1);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-tree block sum (deterministic); every thread gets the total
template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[NT / 32];
  __shared__ double tot;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = (lane < NT / 32) ? ws[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) tot = t;
  }
  __syncthreads();
  return tot;
}

// last-CTA ticket: true in exactly one CTA, after every CTA's writes are visible
__device__ __forceinline__ bool last_cta(unsigned* cnt) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(cnt, 1u) == gridDim.x - 1;
    if (last) *cnt = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// device scalar slots of the inner CG
struct S {
  enum { ALPHA = 0, BETA, RZ, RZ_OLD, PQ, RR, SUMR, GDOT, RHO, TOL2, FROZEN, ITS, BB, N };
};
// ticket counters
enum { T_SPMV = 0, T_DOWN, T_N };

// ------------------------------------------------------------ setup kernels
__global__ void k_parent(int64_t nB, const int32_t* __restrict__ cptr, int64_t off_k, int64_t off_k1,
                         int32_t* __restrict__ parent) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  for (int32_t c = cptr[B]; c < cptr[B + 1]; ++c) parent[off_k + c] = (int32_t)(off_k1 + B);
}

// nested CSR of level k from its canonical CSR: degree pass, then fill with
// columns mapped to absolute nested expanded indices
__global__ void k_ldeg(int64_t nk, const int32_t* __restrict__ order, const int64_t* __restrict__ crow,
                       int64_t* __restrict__ deg) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nk) return;
  const int32_t a = order[p];
  deg[p] = crow[a + 1] - crow[a];
}

__global__ void k_lfill(int64_t nk, const int32_t* __restrict__ order, const int64_t* __restrict__ crow,
                        const int32_t* __restrict__ ccol, const double* __restrict__ cw,
                        const int32_t* __restrict__ nested_of, int64_t off_k, const int64_t* __restrict__ lrow,
                        int32_t* __restrict__ lcol, double* __restrict__ lw) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nk) return;
  const int32_t a = order[p];
  int64_t q = lrow[off_k + p];
  for (int64_t e = crow[a]; e < crow[a + 1]; ++e, ++q) {
    lcol[q] = (int32_t)(off_k + nested_of[ccol[e]]);
    lw[q] = cw[e];
  }
}

// The H~ edges of a level-k node gi (header): FILL = false counts the
// directed triples, FILL = true writes them at pos (key = row * nt + col).
template <bool FILL>
__global__ void __launch_bounds__(TPB) k_hedges(int64_t nk, int64_t off_k, int k, int L, double mu, uint64_t nt,
                                                const int64_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                                                const double* __restrict__ lw, const int32_t* __restrict__ parent,
                                                int64_t* __restrict__ count, uint64_t* __restrict__ key,
                                                double* __restrict__ wout) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nk) return;
  const int64_t gi = off_k + i;
  int64_t pos = FILL ? count[gi] : 0;
  auto emit = [&](int64_t r, int64_t c, double w) {
    if (FILL) {
      key[pos] = (uint64_t)r * nt + (uint64_t)c;
      wout[pos] = w;
    }
    ++pos;
  };
  double sig = 1.0;
  for (int j = 1; j < k; ++j) sig *= mu * mu;  // mu^{2(k-1)}
  double cut[MAXL];
  for (int j = 0; j < L; ++j) cut[j] = 0.0;
  for (int64_t e = lrow[gi]; e < lrow[gi + 1]; ++e) {
    const int32_t gm = lcol[e];
    const double w = lw[e];
    emit(gi, gm, sig * w);                   // same-level edge (block (k, k)); gm emits the reverse
    int32_t ai = (int32_t)gi, am = gm;
    double pw = sig * mu;                    // mu^{k+j-2} at j = k+1 is mu^{2k-1}
    for (int j = k + 1; j <= L; ++j) {
      ai = parent[ai];
      am = parent[am];
      if (ai == am) break;
      if (((j - k) & 1) == 0) {              // i -> A_j(m), non-ancestor
        emit(gi, am, pw * w);
        emit(am, gi, pw * w);
      } else {
        cut[j - 1] += pw * w;                // i -> A_j(i), summed over m
      }
      pw *= mu;
    }
  }
  int32_t aj = (int32_t)gi;
  for (int j = k + 1; j <= L; ++j) {
    aj = parent[aj];
    const double c = cut[j - 1];
    if (c != 0.0) {
      emit(gi, aj, c);
      emit(aj, gi, c);
    }
  }
  if (!FILL) count[gi] = pos;
}

// merged entries: w = sum of the run (in sorted order), column, row count
__global__ void k_hmerge(int64_t nu, uint64_t nt, const uint64_t* __restrict__ ukey, const int32_t* __restrict__ rcnt,
                         const int64_t* __restrict__ rstart, const double* __restrict__ sw, int32_t* __restrict__ hcol,
                         double* __restrict__ hw, int32_t* __restrict__ rowcnt) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= nu) return;
  double w = 0.0;
  const int64_t s0 = rstart[u];
  for (int32_t t = 0; t < rcnt[u]; ++t) w += sw[s0 + t];
  const uint64_t kk = ukey[u];
  hcol[u] = (int32_t)(kk % nt);
  hw[u] = w;
  atomicAdd(&rowcnt[kk / nt], 1);
}

__global__ void k_i32_to_i64(int64_t n, const int32_t* __restrict__ a, int64_t* __restrict__ b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_class_flags(int64_t n, const int64_t* __restrict__ hrow, int cls, char* __restrict__ fl,
                              int32_t* __restrict__ ids) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t d = hrow[i + 1] - hrow[i];
  const int c = d <= H_D0 ? 0 : (d <= H_D1 ? 1 : 2);
  fl[i] = c == cls;
  ids[i] = (int32_t)i;
}

// ------------------------------------------------------------ L_H~ products
// Rows by degree class: short rows (<= H_D0) on 8 lanes, warp rows
// (<= H_D1) on a warp, long rows cut into segments of H_SEG entries, a CTA
// each; a long row's segment sums are added in segment order by the CTA
// that finishes the row last (per-row ticket), so the result does not depend
// on which CTA that is.
struct HMat {
  const int64_t* row;
  const int32_t* col;
  const double* w;
  const int32_t* rows;  // rows by class: [0, n0) short, [n0, n0+n1) warp, then long rows
  int64_t n0, n1, n2;
  unsigned b0, b1, b2;  // CTAs per class (b2 = long-row segments)
  const int4* seg;      // [b2]: (long-row index, first entry, end entry, first segment of the row)
  const int32_t* lnseg; // [n2]: segments of long row j
  double* segpart;      // [b2]
  unsigned* ltick;      // [n2] (zero between launches)
  double* lpq;          // [n2]: the long rows' p_i q_i (fixed slots of the (p, q) sum)
};

__device__ __forceinline__ double group_sum(double v, int gsz) {
  for (int o = gsz / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_{e in [e0, e1) step gsz} f(e), four loads in flight per thread
template <typename F>
__device__ __forceinline__ double h_sum(int64_t e0, int64_t e1, int gsz, F&& f) {
  double a0 = 0.0, a1 = 0.0;
  int64_t e = e0;
  for (; e + 3 * gsz < e1; e += 4 * gsz) {
    const double t0 = f(e), t1 = f(e + gsz), t2 = f(e + 2 * gsz), t3 = f(e + 3 * gsz);
    a0 += t0 + t1;
    a1 += t2 + t3;
  }
  for (; e < e1; e += gsz) a0 += f(e);
  return a0 + a1;
}

// The row product of this thread's group, by class.  fv(i) -> value of the
// own entry, term(vi, e) -> w_e (vi - v_col(e)).  done(i, vi, acc) is called
// once per row, by one thread, with the finished row sum.  Returns nothing;
// CTA-uniform control flow (long-row CTAs use block reductions).
template <typename FV, typename TERM, typename DONE>
__device__ __forceinline__ void h_rows(const HMat& H, FV&& fv, TERM&& term, DONE&& done) {
  const unsigned b = blockIdx.x;
  if (b < H.b0) {
    // short rows (degree <= H_D0 = 4 x 8 lanes): every 8-lane group takes
    // H_U rows at once so the index, row-pointer, column and gather loads of
    // H_U rows are in flight together (the product is load-latency bound)
    const int lane = threadIdx.x & (H_G0 - 1);
    const int64_t per = TPB / H_G0;
    const int64_t stride = (int64_t)H.b0 * per * H_U;
    for (int64_t base = (int64_t)b * per * H_U; base < H.n0; base += stride) {
      int64_t i[H_U], e0[H_U], e1[H_U];
      double vi[H_U], acc[H_U];
#pragma unroll
      for (int u = 0; u < H_U; ++u) {
        const int64_t t = base + u * per + threadIdx.x / H_G0;
        i[u] = t < H.n0 ? H.rows[t] : -1;
      }
#pragma unroll
      for (int u = 0; u < H_U; ++u) {
        e0[u] = i[u] >= 0 ? H.row[i[u]] : 0;
        e1[u] = i[u] >= 0 ? H.row[i[u] + 1] : 0;
        vi[u] = i[u] >= 0 ? fv(i[u]) : 0.0;
        acc[u] = 0.0;
      }
#pragma unroll
      for (int s2 = 0; s2 < H_D0 / H_G0; ++s2) {
#pragma unroll
        for (int u = 0; u < H_U; ++u) {
          const int64_t e = e0[u] + lane + s2 * H_G0;
          if (e < e1[u]) acc[u] += term(vi[u], e);
        }
      }
#pragma unroll
      for (int u = 0; u < H_U; ++u) {
        const double a = group_sum(acc[u], H_G0);
        if (i[u] >= 0 && lane == 0) done(i[u], vi[u], a, -1);
      }
    }
    return;
  }
  if (b < H.b0 + H.b1) {  // grid-stride over row groups (warp-uniform trip count)
    const bool shortc = b < H.b0;
    const int gsz = shortc ? H_G0 : 32;
    const int lane = threadIdx.x & (gsz - 1);
    const int64_t per = TPB / gsz, ncls = shortc ? H.n0 : H.n1, first = shortc ? 0 : H.n0;
    const int64_t stride = (int64_t)(shortc ? H.b0 : H.b1) * per;
    for (int64_t base = (int64_t)(shortc ? b : b - H.b0) * per; base < ncls; base += stride) {
      const int64_t t = base + threadIdx.x / gsz;
      const bool ok = t < ncls;
      const int64_t i = ok ? H.rows[first + t] : -1;
      double acc = 0.0, vi = 0.0;
      if (ok) {
        vi = fv(i);
        acc = h_sum(H.row[i] + lane, H.row[i + 1], gsz, [&](int64_t e) { return term(vi, e); });
      }
      acc = group_sum(acc, gsz);
      if (ok && lane == 0) done(i, vi, acc, -1);
    }
    return;
  }
  // a segment of a long row
  const int4 sd = H.seg[b - H.b0 - H.b1];
  const int64_t i = H.rows[H.n0 + H.n1 + sd.x];
  const int64_t base = H.row[i];
  const double vi = fv(i);
  double acc = h_sum(base + sd.y + threadIdx.x, base + sd.z, TPB, [&](int64_t e) { return term(vi, e); });
  acc = block_sum<TPB>(acc);
  __shared__ bool fin;
  if (threadIdx.x == 0) {
    H.segpart[b - H.b0 - H.b1] = acc;
    __threadfence();
    const int ns = H.lnseg[sd.x];
    fin = atomicAdd(&H.ltick[sd.x], 1u) == (unsigned)(ns - 1);
    if (fin) {
      __threadfence();
      H.ltick[sd.x] = 0u;
      double t = 0.0;
      for (int k = 0; k < ns; ++k) t += H.segpart[sd.w + k];
      done(i, vi, t, sd.x);
    }
  }
  __syncthreads();
}

// y = L_H~ x (difference form)
__global__ void __launch_bounds__(TPB) k_h_apply(HMat H, const double* __restrict__ x, double* __restrict__ y) {
  h_rows(
      H, [&](int64_t i) { return x[i]; },
      [&](double xi, int64_t e) { return H.w[e] * (xi - x[H.col[e]]); },
      [&](int64_t i, double, double acc, int) { y[i] = acc; });
}

// double-double helpers (Knuth TwoSum, fma TwoProd)
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void dd_add(double& hi, double& lo, double a, double ae) {
  double s, e;
  two_sum(hi, a, s, e);
  e += lo + ae;
  two_sum(s, e, hi, lo);
}

// res = b - L_H~ x with every difference, product and sum in double-double
// (the residual of the refinement steps, reading R13); one thread per row
__global__ void __launch_bounds__(TPB) k_h_resid_dd(int64_t nt, const int64_t* __restrict__ row,
                                                    const int32_t* __restrict__ col, const double* __restrict__ w,
                                                    const double* __restrict__ x, const double* __restrict__ b,
                                                    double* __restrict__ res) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const double xi = x[i];
  double hi = b[i], lo = 0.0;
  for (int64_t e = row[i]; e < row[i + 1]; ++e) {
    double d, de;
    two_sum(xi, -x[col[e]], d, de);       // xi - xj = d + de exactly
    const double p = w[e] * d;
    const double pe = fma(w[e], d, -p) + w[e] * de;
    dd_add(hi, lo, -p, -pe);
  }
  res[i] = hi + lo;
}

// the inner CG's product: p_i = z_i + beta p_i (on the fly for every gathered
// column), q = L_H~ p, (p, q) by ticket (CTA partials in CTA order, then the
// long rows' slots in row order); the last CTA forms alpha = rz / pq
__global__ void __launch_bounds__(TPB) k_h_spmv(HMat H, const double2* __restrict__ zp_old, double2* __restrict__ zp_new,
                                                double* __restrict__ q, double* __restrict__ sc,
                                                double* __restrict__ part, unsigned* __restrict__ tick) {
  if (sc[S::FROZEN] != 0.0) return;
  const double beta = sc[S::BETA];
  double pq = 0.0;
  h_rows(
      H,
      [&](int64_t i) {
        const double2 a = zp_old[i];
        return a.x + beta * a.y;
      },
      [&](double pi, int64_t e) {
        const double2 c = zp_old[H.col[e]];
        return H.w[e] * (pi - (c.x + beta * c.y));
      },
      [&](int64_t i, double pi, double acc, int lr) {
        q[i] = acc;
        zp_new[i].y = pi;
        if (lr < 0) pq += pi * acc;
        else H.lpq[lr] = pi * acc;
      });
  pq = block_sum<TPB>(pq);
  if (threadIdx.x == 0) part[blockIdx.x] = pq;
  if (last_cta(tick)) {
    double t = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += TPB) t += part[b];
    t = block_sum<TPB>(t);
    double u = 0.0;
    for (int64_t j = threadIdx.x; j < H.n2; j += TPB) u += H.lpq[j];
    u = block_sum<TPB>(u);
    if (threadIdx.x == 0) {
      sc[S::PQ] = t + u;
      sc[S::ALPHA] = sc[S::RZ] / (t + u);
    }
  }
}

// ------------------------------------------------- expanded MSP: L_T~^+ r~
struct ELv {
  int L, Kc;
  int64_t n[MAXL], off[MAXL], cpo[MAXL], lo[MAXL];
  int64_t n1;
  double nt, GN;
};

struct EVec {
  double* x;           // inner CG iterate (the solution z~)
  double* r;           // residual
  const double* q;     // L_H~ p
  double2* zp;         // (z, p) pairs of this iteration: p read, z written
  double* s;           // T~ subtree sums (levels >= 2; level 1 is r)
  const int32_t* cptr;
  const double* kinv;
  const double* lof;
  const double* Nsub;
  const double* g;
  const double* pinv;
  double* sc;
  double* upart;       // up-sweep partials, 3 per CTA: (r, r), sum r, (g, s)
  double* zpart;       // (r, z) partials
};

// one aggregate B at level k+1 (children at level k): update (x, r) of B
// (and of the children when k == 1), s_B = r_B + sum_c s_c; accumulates the
// partial sums (g, s over non-top nodes)
__device__ __forceinline__ void up_node(const ELv& lv, const EVec& v, int k, int64_t B, bool init, double alpha,
                                        double& rr, double& sr, double& gs) {
  const int64_t ok = lv.off[k - 1], ok1 = lv.off[k];
  const int32_t* cp = v.cptr + lv.cpo[k - 1];
  const bool top = (k + 1 == lv.L);
  double sB = 0.0;
  for (int32_t c = cp[B]; c < cp[B + 1]; ++c) {
    const int64_t gc = ok + c;
    double sc;
    if (k == 1) {
      double rc = v.r[gc];
      if (!init) {
        v.x[gc] += alpha * v.zp[gc].y;
        rc -= alpha * v.q[gc];
        v.r[gc] = rc;
      }
      rr += rc * rc;
      sr += rc;
      sc = rc;
      gs += v.g[gc] * rc;
    } else {
      sc = v.s[gc];
    }
    sB += sc;
  }
  const int64_t gB = ok1 + B;
  double rB = v.r[gB];
  if (!init) {
    v.x[gB] += alpha * v.zp[gB].y;
    rB -= alpha * v.q[gB];
    v.r[gB] = rB;
  }
  rr += rB * rB;
  sr += rB;
  sB += rB;
  v.s[gB] = sB;
  if (!top) gs += v.g[gB] * sB;
}

// one aggregate B at level k+1: z of its children from z_B (block-tree
// factors of T~), t_c = s_c - rho N_c
__device__ __forceinline__ double down_node(const ELv& lv, const EVec& v, int k, int64_t B, double rho) {
  const int64_t ok = lv.off[k - 1], ok1 = lv.off[k];
  const int32_t* cp = v.cptr + lv.cpo[k - 1];
  const int32_t s0 = cp[B], s1 = cp[B + 1];
  const double* ki = v.kinv + 3 * (ok1 - lv.n1 + B);
  const int64_t lb = 3 * (lv.lo[k - 1] - 2 * B - 2);
  auto sv = [&](int64_t p) { return (k == 1 ? v.r[ok + p] : v.s[ok + p]) - rho * v.Nsub[ok + p]; };
  const double zb = v.zp[ok1 + B].x;
  const double tu = sv(s0), tv = sv(s0 + 1);
  double au = tu, av = tv;
  for (int32_t p = s0 + 2; p < s1; ++p) {
    const double tx = sv(p);
    au += v.lof[lb + 3 * p] * tx;
    av += v.lof[lb + 3 * p + 1] * tx;
  }
  const double zu = ki[0] * au + ki[1] * av, zv = ki[1] * au + ki[2] * av;
  double rz = 0.0;
  auto put = [&](int64_t p, double z) {
    v.zp[ok + p].x = z;
    rz += v.r[ok + p] * z;
  };
  put(s0, zb + zu);
  put(s0 + 1, zb + zv);
  for (int32_t p = s0 + 2; p < s1; ++p)
    put(p, zb + v.lof[lb + 3 * p + 2] * sv(p) + v.lof[lb + 3 * p] * zu + v.lof[lb + 3 * p + 1] * zv);
  return rz;
}

// one step of the up sweep: a tile tier (tstart != nullptr: a CTA per tile,
// levels k0+1..k1 of the tile's subtree, block barriers between levels --
// the nested numbering makes every tile a contiguous subtree, DESIGN.md "Data
// layout") or one level (aggregates of level k0+1, a thread each)
__global__ void __launch_bounds__(TPB) k_e_up(ELv lv, EVec v, int k0, int k1, const int32_t* __restrict__ tstart,
                                              int64_t ntiles, int init, int64_t slot) {
  const double* sc = v.sc;
  if (sc[S::FROZEN] != 0.0) return;
  const double alpha = init ? 0.0 : sc[S::ALPHA];
  double rr = 0.0, sr = 0.0, gs = 0.0;
  if (!tstart) {
    const int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (B < lv.n[k0]) up_node(lv, v, k0, B, init, alpha, rr, sr, gs);
  } else {
    const int64_t j = blockIdx.x;
    for (int t = 1; t <= k1 - k0; ++t) {
      const int32_t* ts = tstart + (int64_t)t * (ntiles + 1);
      const int64_t e = ts[j + 1];
      for (int64_t B = ts[j] + threadIdx.x; B < e; B += TPB) up_node(lv, v, k0 + t - 1, B, init, alpha, rr, sr, gs);
      __syncthreads();
    }
  }
  rr = block_sum<TPB>(rr);
  sr = block_sum<TPB>(sr);
  gs = block_sum<TPB>(gs);
  if (threadIdx.x == 0) {
    double* p = v.upart + 3 * (slot + blockIdx.x);
    p[0] = rr;
    p[1] = sr;
    p[2] = gs;
  }
}

// (r, z) over all slots -> RZ, BETA (run by one CTA)
__device__ void finish_rz(EVec& v, int64_t nslots, int init) {
  double t = 0.0;
  for (int64_t b = threadIdx.x; b < nslots; b += blockDim.x) t += v.zpart[b];
  t = (blockDim.x == TPB) ? block_sum<TPB>(t) : block_sum<CO_T>(t);
  if (threadIdx.x == 0) {
    double* sc = v.sc;
    if (init) {
      sc[S::RZ] = t;
      sc[S::BETA] = 0.0;
    } else {
      sc[S::RZ_OLD] = sc[S::RZ];
      sc[S::RZ] = t;
      sc[S::BETA] = t / sc[S::RZ_OLD];
    }
  }
}

// the small levels (Kc..L): up sweep, the sums, the convergence test, the
// top solve rho / z_top / shift (k_e_top of round 1), the down sweep
__global__ void __launch_bounds__(CO_T) k_e_coarse(ELv lv, EVec v, int init, int64_t nup_slots, int64_t zslot,
                                                   int64_t nz_slots) {
  double* sc = v.sc;
  if (sc[S::FROZEN] != 0.0) return;
  const double alpha = init ? 0.0 : sc[S::ALPHA];
  const int L = lv.L, Kc = lv.Kc;
  double rr = 0.0, sr = 0.0, gs = 0.0;
  for (int k = Kc; k < L; ++k) {  // aggregates of level k+1
    for (int64_t B = threadIdx.x; B < lv.n[k]; B += CO_T) up_node(lv, v, k, B, init, alpha, rr, sr, gs);
    __syncthreads();
  }
  if (L == 1) {  // single level: the top is level 1 itself
    for (int64_t i = threadIdx.x; i < lv.n[0]; i += CO_T) {
      double ri = v.r[i];
      if (!init) {
        v.x[i] += alpha * v.zp[i].y;
        ri -= alpha * v.q[i];
        v.r[i] = ri;
      }
      rr += ri * ri;
      sr += ri;
      v.s[i] = ri;
    }
    __syncthreads();
  }
  for (int64_t b = threadIdx.x; b < nup_slots; b += CO_T) {
    rr += v.upart[3 * b];
    sr += v.upart[3 * b + 1];
    gs += v.upart[3 * b + 2];
  }
  rr = block_sum<CO_T>(rr);
  sr = block_sum<CO_T>(sr);
  gs = block_sum<CO_T>(gs);
  __shared__ bool stop;
  if (threadIdx.x == 0) {
    sc[S::RR] = rr;
    stop = false;
    if (!init) {
      sc[S::ITS] += 1.0;
      if (rr <= sc[S::TOL2]) {
        sc[S::FROZEN] = 1.0;
        stop = true;
      }
    }
  }
  __syncthreads();
  if (stop) return;
  // top: rho = sum(r~)/n~, z_top = (sigma L_l)^+ (s - rho N), shift m
  const double rho = sr / lv.nt;
  const int64_t ot = lv.off[L - 1];
  const int ntop = (int)lv.n[L - 1];
  __shared__ double t[256];
  __shared__ double sh_m;
  for (int i = threadIdx.x; i < ntop; i += CO_T) t[i] = v.s[ot + i] - rho * v.Nsub[ot + i];
  __syncthreads();
  double zi = 0.0, nz = 0.0;
  if ((int)threadIdx.x < ntop) {
    for (int j = 0; j < ntop; ++j) zi += v.pinv[threadIdx.x * ntop + j] * t[j];
    nz = v.Nsub[ot + threadIdx.x] * zi;
  }
  nz = block_sum<CO_T>(nz);
  if (threadIdx.x == 0) {
    sh_m = (nz + gs - rho * lv.GN) / lv.nt;
    sc[S::RHO] = rho;
  }
  __syncthreads();
  double rz = 0.0;
  if ((int)threadIdx.x < ntop) {
    const double z = zi - sh_m;
    v.zp[ot + threadIdx.x].x = z;
    rz += v.r[ot + threadIdx.x] * z;
  }
  __syncthreads();
  for (int k = L - 1; k >= Kc; --k) {
    for (int64_t B = threadIdx.x; B < lv.n[k]; B += CO_T) rz += down_node(lv, v, k, B, rho);
    __syncthreads();
  }
  rz = block_sum<CO_T>(rz);
  if (threadIdx.x == 0) v.zpart[zslot] = rz;
  if (Kc == 1) {  // no large levels: this CTA finishes (r, z)
    __syncthreads();
    __threadfence_block();
    finish_rz(v, nz_slots, init);
  }
}

// one step of the down sweep (tile tier or one level, as k_e_up), top-down;
// the step that ends at level 1 finishes (r, z) in its last CTA
__global__ void __launch_bounds__(TPB) k_e_down(ELv lv, EVec v, int k0, int k1, const int32_t* __restrict__ tstart,
                                                int64_t ntiles, int init, int64_t slot, int64_t nz_slots,
                                                unsigned* __restrict__ tick) {
  if (v.sc[S::FROZEN] != 0.0) return;
  const double rho = v.sc[S::RHO];
  double rz = 0.0;
  if (!tstart) {
    const int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (B < lv.n[k0]) rz = down_node(lv, v, k0, B, rho);
  } else {
    const int64_t j = blockIdx.x;
    for (int t = k1 - k0; t >= 1; --t) {
      const int32_t* ts = tstart + (int64_t)t * (ntiles + 1);
      const int64_t e = ts[j + 1];
      for (int64_t B = ts[j] + threadIdx.x; B < e; B += TPB) rz += down_node(lv, v, k0 + t - 1, B, rho);
      __syncthreads();
    }
  }
  rz = block_sum<TPB>(rz);
  if (threadIdx.x == 0) v.zpart[slot + blockIdx.x] = rz;
  if (k0 == 1 && last_cta(tick)) finish_rz(v, nz_slots, init);
}

// ------------------------------------------------------------ small kernels
__global__ void k_copy(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_add(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] += a[i];
}

// fixed-order dot over [0, n): block partials, then one block
__global__ void __launch_bounds__(TPB) k_dot_part(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                                  double* __restrict__ part) {
  double d = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d += b ? a[i] * b[i] : a[i];
  d = block_sum<TPB>(d);
  if (threadIdx.x == 0) part[blockIdx.x] = d;
}

__global__ void __launch_bounds__(TPB) k_dot_final(int np, const double* __restrict__ part, double* __restrict__ out) {
  double d = 0.0;
  for (int i = threadIdx.x; i < np; i += TPB) d += part[i];
  d = block_sum<TPB>(d);
  if (threadIdx.x == 0) *out = d;
}

__global__ void k_shift(int64_t n, double* __restrict__ a, const double* __restrict__ sum, double inv_n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] -= *sum * inv_n;
}

// r~_k = (-mu)^{k-1} (P^k)^T r, level by level (y_{k+1} = P^T y_k)
__global__ void k_restrict(int64_t nB, const int32_t* __restrict__ cptr, int64_t off_k, int64_t off_k1, double scale,
                           const double* __restrict__ yk, double* __restrict__ yk1, double* __restrict__ rt) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  double v = 0.0;
  for (int32_t c = cptr[B]; c < cptr[B + 1]; ++c) v += yk[c];
  yk1[B] = v;
  rt[off_k1 + B] = scale * v;
}

// w_k = z_k + (-mu) P w_{k+1} (Horner form of z = P(mu) z~), top-down
__global__ void k_prolong(int64_t nB, const int32_t* __restrict__ cptr, int64_t off_k, int64_t off_k1, double negmu,
                          const double* __restrict__ zt, double* __restrict__ w) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  const double wb = negmu * w[off_k1 + B];
  for (int32_t c = cptr[B]; c < cptr[B + 1]; ++c) w[off_k + c] = zt[off_k + c] + wb;
}

__global__ void k_gather_canon(int64_t nk, const int32_t* __restrict__ order, int64_t off, const double* __restrict__ src,
                               double* __restrict__ dst, int to_nested) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nk) return;
  if (to_nested) dst[off + p] = src[off + order[p]];
  else dst[off + order[p]] = src[off + p];
}

struct Temp {
  DBuf<char> buf;
  void* get(size_t bytes) {
    if (bytes > buf.n) buf.alloc(std::max<size_t>(bytes, 1 << 20));
    return buf.p;
  }
};

template <typename T>
T d2h(const T* d, cudaStream_t st) {
  T v;
  MSP_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  MSP_CUDA(cudaStreamSynchronize(st));
  return v;
}

// the sweep steps of the expanded MSP below the coarse CTA: the solve
// schedule's tile tiers (generic tiers level by
// level), else one step per level up to pegp_Kc
struct EStep {
  int k0, k1;
  const int32_t* tstart;
  int64_t ntiles;
  unsigned grid;
};

std::vector<EStep> e_steps(const Handle& h, int& Kc) {
  std::vector<EStep> out;
  const bool tiles = !h.tiers.empty() && std::getenv("MSP_PEGP_NOTILE") == nullptr;
  int k = 1;
  if (tiles) {
    for (const auto& t : h.tiers) {
      if (t.k0 != k) break;
      if (t.generic || t.k1 - t.k0 < 1) {
        for (int kk = t.k0; kk < t.k1; ++kk) out.push_back({kk, kk + 1, nullptr, 0, grid_for(h.lv[kk].n)});
      } else {
        out.push_back({t.k0, t.k1, t.tstart.p, t.ntiles, (unsigned)t.ntiles});
      }
      k = t.k1;
    }
  }
  const int target = tiles ? std::max(k, h.Kc) : h.pegp_Kc;
  for (; k < target; ++k) out.push_back({k, k + 1, nullptr, 0, grid_for(h.lv[k].n)});
  Kc = k;
  return out;
}

}  // namespace

// ------------------------------------------------------------ host side
void pegp_build(Handle& h, cudaStream_t st) {
  if (h.pegp_ready) return;
  const int L = h.levels;
  const int64_t nt = h.n_tilde;
  Temp tmp;
  cudaEvent_t e0, e1;
  MSP_CUDA(cudaEventCreate(&e0));
  MSP_CUDA(cudaEventCreate(&e1));
  MSP_CUDA(cudaEventRecord(e0, st));
  // parent pointers
  h.parent.alloc(nt);
  MSP_CUDA(cudaMemsetAsync(h.parent.p, 0xff, nt * sizeof(int32_t), st));
  for (int k = 1; k < L; ++k)
    k_parent<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.lv[k - 1].off,
                                                  h.lv[k].off, h.parent.p);
  // per-level adjacency, nested, in one CSR over n~ (absolute columns)
  DBuf<int64_t> deg, lrow;
  DBuf<int32_t> lcol;
  DBuf<double> lw;
  deg.alloc(nt + 1);
  MSP_CUDA(cudaMemsetAsync(deg.p, 0, (nt + 1) * sizeof(int64_t), st));
  for (int k = 1; k <= L; ++k)
    k_ldeg<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.order_nested[k - 1].p, h.canon_rowptr[k - 1].p,
                                                    deg.p + h.lv[k - 1].off);
  MSP_LAUNCH_CHECK();
  lrow.alloc(nt + 1);
  {
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg.p, lrow.p, nt + 1, st));
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, deg.p, lrow.p, nt + 1, st));
  }
  const int64_t lnnz = d2h(lrow.p + nt, st);
  lcol.alloc(std::max<int64_t>(lnnz, 1));
  lw.alloc(std::max<int64_t>(lnnz, 1));
  for (int k = 1; k <= L; ++k)
    k_lfill<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.order_nested[k - 1].p, h.canon_rowptr[k - 1].p,
                                                     h.canon_col[k - 1].p, h.canon_w[k - 1].p,
                                                     h.nested_of_canon[k - 1].p, h.lv[k - 1].off, lrow.p, lcol.p,
                                                     lw.p);
  MSP_LAUNCH_CHECK();
  // H~ triples: count, scan, fill
  DBuf<int64_t> cnt, pos;
  cnt.alloc(nt + 1);
  pos.alloc(nt + 1);
  MSP_CUDA(cudaMemsetAsync(cnt.p, 0, (nt + 1) * sizeof(int64_t), st));
  for (int k = 1; k <= L; ++k)
    k_hedges<false><<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.lv[k - 1].off, k, L, h.mu,
                                                             (uint64_t)nt, lrow.p, lcol.p, lw.p, h.parent.p, cnt.p,
                                                             nullptr, nullptr);
  MSP_LAUNCH_CHECK();
  {
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, pos.p, nt + 1, st));
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, cnt.p, pos.p, nt + 1, st));
  }
  const int64_t ne = d2h(pos.p + nt, st);
  DBuf<uint64_t> key, skey;
  DBuf<double> w, sw;
  key.alloc(std::max<int64_t>(ne, 1));
  skey.alloc(std::max<int64_t>(ne, 1));
  w.alloc(std::max<int64_t>(ne, 1));
  sw.alloc(std::max<int64_t>(ne, 1));
  for (int k = 1; k <= L; ++k)
    k_hedges<true><<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.lv[k - 1].off, k, L, h.mu,
                                                            (uint64_t)nt, lrow.p, lcol.p, lw.p, h.parent.p, pos.p,
                                                            key.p, w.p);
  MSP_LAUNCH_CHECK();
  int end_bit = 1;
  while (end_bit < 64 && (((uint64_t)nt * (uint64_t)nt) >> end_bit) != 0) ++end_bit;
  {
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, skey.p, w.p, sw.p, ne, 0, end_bit, st));
    MSP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, key.p, skey.p, w.p, sw.p, ne, 0, end_bit, st));
  }
  // runs of equal (row, column): unique keys and lengths
  DBuf<int32_t> rcnt;
  DBuf<int64_t> nruns_d, rstart, rcnt64;
  rcnt.alloc(std::max<int64_t>(ne, 1));
  nruns_d.alloc(1);
  {
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, skey.p, key.p, rcnt.p, nruns_d.p, ne, st));
    MSP_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(bytes), bytes, skey.p, key.p, rcnt.p, nruns_d.p, ne, st));
  }
  const int64_t nu = d2h(nruns_d.p, st);
  rcnt64.alloc(nu + 1);
  rstart.alloc(nu + 1);
  k_i32_to_i64<<<grid_for(nu), TPB, 0, st>>>(nu, rcnt.p, rcnt64.p);
  {
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, rcnt64.p, rstart.p, nu, st));
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, rcnt64.p, rstart.p, nu, st));
  }
  h.hnnz = nu;
  h.hcol.alloc(std::max<int64_t>(nu, 1));
  h.hw.alloc(std::max<int64_t>(nu, 1));
  DBuf<int32_t> rowcnt;
  DBuf<int64_t> rowcnt64;
  rowcnt.alloc(nt + 1);
  rowcnt64.alloc(nt + 1);
  MSP_CUDA(cudaMemsetAsync(rowcnt.p, 0, (nt + 1) * sizeof(int32_t), st));
  k_hmerge<<<grid_for(nu), TPB, 0, st>>>(nu, (uint64_t)nt, key.p, rcnt.p, rstart.p, sw.p, h.hcol.p, h.hw.p,
                                         rowcnt.p);
  k_i32_to_i64<<<grid_for(nt + 1), TPB, 0, st>>>(nt + 1, rowcnt.p, rowcnt64.p);
  h.hrow.alloc(nt + 1);
  {
    size_t bytes = 0;
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, rowcnt64.p, h.hrow.p, nt + 1, st));
    MSP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, rowcnt64.p, h.hrow.p, nt + 1, st));
  }
  MSP_LAUNCH_CHECK();
  // rows by degree class (each class in nested order)
  h.hrows.alloc(nt);
  {
    DBuf<char> fl;
    DBuf<int32_t> ids;
    DBuf<int64_t> nsel;
    fl.alloc(nt);
    ids.alloc(nt);
    nsel.alloc(1);
    int64_t at = 0;
    for (int c = 0; c < 3; ++c) {
      k_class_flags<<<grid_for(nt), TPB, 0, st>>>(nt, h.hrow.p, c, fl.p, ids.p);
      size_t bytes = 0;
      MSP_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ids.p, fl.p, h.hrows.p + at, nsel.p, nt, st));
      MSP_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, ids.p, fl.p, h.hrows.p + at, nsel.p, nt, st));
      h.hclass[c] = d2h(nsel.p, st);
      at += h.hclass[c];
    }
  }
  // long rows: segments of H_SEG entries
  {
    const int64_t n2 = h.hclass[2];
    std::vector<int32_t> lr(n2);
    std::vector<int64_t> hr(nt + 1);
    if (n2) MSP_CUDA(cudaMemcpyAsync(lr.data(), h.hrows.p + h.hclass[0] + h.hclass[1], n2 * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaMemcpyAsync(hr.data(), h.hrow.p, (nt + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    std::vector<int4> seg;
    std::vector<int32_t> ns(std::max<int64_t>(n2, 1), 0);
    for (int64_t j = 0; j < n2; ++j) {
      const int64_t d = hr[lr[j] + 1] - hr[lr[j]];
      const int first = (int)seg.size();
      for (int64_t e = 0; e < d; e += H_SEG)
        seg.push_back(make_int4((int)j, (int)e, (int)std::min<int64_t>(d, e + H_SEG), first));
      ns[j] = (int32_t)(seg.size() - first);
    }
    h.hnseg = (int64_t)seg.size();
    h.hseg2.alloc(std::max<int64_t>(h.hnseg, 1));
    h.hlnseg.alloc(ns.size());
    h.hsegpart.alloc(std::max<int64_t>(h.hnseg, 1));
    h.hlpq.alloc(std::max<int64_t>(n2, 1));
    h.hltick.alloc(std::max<int64_t>(n2, 1));
    if (h.hnseg) MSP_CUDA(cudaMemcpyAsync(h.hseg2.p, seg.data(), seg.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    MSP_CUDA(cudaMemcpyAsync(h.hlnseg.p, ns.data(), ns.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    MSP_CUDA(cudaMemsetAsync(h.hltick.p, 0, std::max<int64_t>(n2, 1) * sizeof(unsigned), st));
    MSP_CUDA(cudaStreamSynchronize(st));
  }
  // inner-CG workspace: vectors, pair arrays, partial slots
  for (auto* v : {&h.ex, &h.er, &h.eq, &h.es, &h.ey, &h.eres, &h.ecor}) v->alloc(nt + 8);
  h.ezp[0].alloc(2 * (nt + 8));
  h.ezp[1].alloc(2 * (nt + 8));
  h.edots.alloc(S::N);
  h.epart.alloc(1024);
  h.etick.alloc(T_N);
  MSP_CUDA(cudaMemsetAsync(h.etick.p, 0, T_N * sizeof(unsigned), st));
  // large levels: k + 1 <= Kc with n_{k+1} > CO_MAX (the coarse CTA takes the rest)
  int Kc = 1;
  while (Kc < L - 1 && h.lv[Kc].n > CO_MAX) ++Kc;  // lv[Kc] is level Kc+1
  h.pegp_Kc = Kc;
  int64_t nup = 0, nz = 1;  // coarse CTA's (r, z) slot first
  {
    int kc = 1;
    for (const auto& sp : e_steps(h, kc)) {
      nup += sp.grid;
      nz += sp.grid;
    }
    h.pegp_Kc = kc;
  }
  h.eup.alloc(3 * std::max<int64_t>(nup, 1));
  h.ezs.alloc(nz);
  const int64_t sp = (int64_t)grid_for(h.hclass[0], TPB / H_G0) + grid_for(h.hclass[1], TPB / 32) + h.hnseg;
  h.espmv_part.alloc(std::max<int64_t>(sp, 1));
  MSP_CUDA(cudaEventRecord(e1, st));
  MSP_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  MSP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  h.pegp_build_ms = ms;
  h.pegp_ready = true;
}

namespace {

HMat hmat(const Handle& h) {
  HMat H;
  H.row = h.hrow.p;
  H.col = h.hcol.p;
  H.w = h.hw.p;
  H.rows = h.hrows.p;
  H.n0 = h.hclass[0];
  H.n1 = h.hclass[1];
  H.n2 = h.hclass[2];
  // short and warp rows: persistent grid-stride CTAs (a few per SM), so the
  // (p, q) ticket is taken by ~1k CTAs, not one per 32 rows
  // (MSP_PEGP_B0 / MSP_PEGP_B1: CTAs per SM of the two classes, for sweeps)
  static const int per_sm0 = std::getenv("MSP_PEGP_B0") ? std::max(1, std::atoi(std::getenv("MSP_PEGP_B0"))) : 3;
  static const int per_sm1 = std::getenv("MSP_PEGP_B1") ? std::max(1, std::atoi(std::getenv("MSP_PEGP_B1"))) : 2;
  H.b0 = (unsigned)std::min<int64_t>((H.n0 + H_U * TPB / H_G0 - 1) / (H_U * TPB / H_G0), 148 * per_sm0);
  H.b1 = (unsigned)std::min<int64_t>((H.n1 + TPB / 32 - 1) / (TPB / 32), 148 * per_sm1);
  H.b2 = (unsigned)h.hnseg;
  H.seg = h.hseg2.p;
  H.lnseg = h.hlnseg.p;
  H.segpart = h.hsegpart.p;
  H.ltick = h.hltick.p;
  H.lpq = h.hlpq.p;
  return H;
}

ELv elv(const Handle& h) {
  ELv lv{};
  lv.L = h.levels;
  e_steps(h, lv.Kc);
  for (int k = 1; k <= h.levels; ++k) {
    lv.n[k - 1] = h.lv[k - 1].n;
    lv.off[k - 1] = h.lv[k - 1].off;
    lv.cpo[k - 1] = k < h.levels ? h.cptr_off[k - 1] : 0;
    lv.lo[k - 1] = k < h.levels ? h.lo_off[k - 1] : 0;
  }
  lv.n1 = h.n;
  lv.nt = (double)h.n_tilde;
  lv.GN = h.GN;
  return lv;
}

void dot(Handle& h, int64_t n, const double* a, const double* b, double* out, cudaStream_t st) {
  const unsigned g = std::min<unsigned>(grid_for(n), 1024u);
  k_dot_part<<<g, TPB, 0, st>>>(n, a, b, h.epart.p);
  k_dot_final<<<1, TPB, 0, st>>>((int)g, h.epart.p, out);
  h.launches += 2;
}

// the preconditioner pass of one inner iteration (init: z0 = L_T~^+ r0 only)
// on pair array zp (p read from .y, z written to .x)
void e_sweeps(Handle& h, const ELv& lv, EVec v, int init, cudaStream_t st) {
  int Kc = 1;
  const std::vector<EStep> steps = e_steps(h, Kc);
  int64_t slot = 0;
  for (const auto& sp : steps) {
    k_e_up<<<sp.grid, TPB, 0, st>>>(lv, v, sp.k0, sp.k1, sp.tstart, sp.ntiles, init, slot);
    slot += sp.grid;
  }
  const int64_t nup = slot;
  int64_t nz = 1;
  for (const auto& sp : steps) nz += sp.grid;
  k_e_coarse<<<1, CO_T, 0, st>>>(lv, v, init, nup, 0, nz);
  int64_t zs = nz;
  for (auto it = steps.rbegin(); it != steps.rend(); ++it) {
    zs -= it->grid;
    k_e_down<<<it->grid, TPB, 0, st>>>(lv, v, it->k0, it->k1, it->tstart, it->ntiles, init, zs, nz,
                                       h.etick.p + T_DOWN);
  }
  h.launches += 2 * (int64_t)steps.size() + 1;
}

EVec evec(Handle& h, double* x, int which) {
  EVec v;
  v.x = x;
  v.r = h.er.p;
  v.q = h.eq.p;
  v.zp = reinterpret_cast<double2*>(h.ezp[which].p);
  v.s = h.es.p;
  v.cptr = h.cptr.p;
  v.kinv = h.kinv.p;
  v.lof = h.lof.p;
  v.Nsub = h.Nsub.p;
  v.g = h.gvec.p;
  v.pinv = h.top_pinv.p;
  v.sc = h.edots.p;
  v.upart = h.eup.p;
  v.zpart = h.ezs.p;
  return v;
}

// CG on L_H~ x = b - mean(b) (x0 = 0), preconditioned by L_T~^+, to
// ||r|| <= rtol ||b - mean(b)||; returns the iteration count
int inner_cg(Handle& h, const double* b, double* x, double rtol, cudaStream_t st) {
  const int64_t nt = h.n_tilde;
  const unsigned gn = grid_for(nt);
  double* d = h.edots.p;
  const ELv lv = elv(h);
  const HMat H = hmat(h);
  k_copy<<<gn, TPB, 0, st>>>(nt, b, h.er.p);
  dot(h, nt, h.er.p, nullptr, d + S::SUMR, st);
  k_shift<<<gn, TPB, 0, st>>>(nt, h.er.p, d + S::SUMR, 1.0 / (double)nt);
  MSP_CUDA(cudaMemsetAsync(x, 0, nt * sizeof(double), st));
  MSP_CUDA(cudaMemsetAsync(h.ezp[0].p, 0, 2 * nt * sizeof(double), st));
  MSP_CUDA(cudaMemsetAsync(h.ezp[1].p, 0, 2 * nt * sizeof(double), st));
  dot(h, nt, h.er.p, h.er.p, d + S::BB, st);
  const double bb = d2h(d + S::BB, st);
  if (bb == 0.0) return 0;
  {
    double init[S::N] = {0};
    init[S::TOL2] = rtol * rtol * bb;
    MSP_CUDA(cudaMemcpyAsync(d, init, S::N * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  // z0 = L_T~^+ r0 into pair array 0, (r0, z0), beta = 0
  e_sweeps(h, lv, evec(h, x, 0), 1, st);
  MSP_LAUNCH_CHECK();
  const unsigned gs = H.b0 + H.b1 + H.b2;
  // msp_set_profiling: events around the product (category 6) and the
  // sweeps (category 7) of every iteration, no graphs
  std::vector<cudaEvent_t> ev;
  std::vector<int> evcat;
  auto mark = [&](cudaStream_t s2) {
    cudaEvent_t e;
    MSP_CUDA(cudaEventCreate(&e));
    MSP_CUDA(cudaEventRecord(e, s2));
    ev.push_back(e);
  };
  auto prof_flush = [&]() {
    if (ev.empty()) return;
    MSP_CUDA(cudaEventSynchronize(ev.back()));
    for (size_t i = 0; i < evcat.size(); ++i) {
      float ms = 0.f;
      MSP_CUDA(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
      h.prof_ms[evcat[i]] += ms;
      h.prof_cnt[evcat[i]] += 1;
    }
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    evcat.clear();
  };
  auto one_iteration = [&](int cur, cudaStream_t s2) {
    const int nxt = cur ^ 1;
    if (h.profile) mark(s2);
    k_h_spmv<<<gs, TPB, 0, s2>>>(H, reinterpret_cast<const double2*>(h.ezp[cur].p),
                                 reinterpret_cast<double2*>(h.ezp[nxt].p), h.eq.p, d, h.espmv_part.p,
                                 h.etick.p + T_SPMV);
    ++h.launches;
    if (h.profile) {
      mark(s2);
      evcat.push_back(6);
      mark(s2);
    }
    e_sweeps(h, lv, evec(h, x, nxt), 0, s2);
    if (h.profile) {
      mark(s2);
      evcat.push_back(7);
    }
  };
  const int kb = 8;  // iterations per captured batch (even: the pair ping-pong is periodic)
  const bool use_graph = !h.profile && std::getenv("MSP_NO_GRAPH") == nullptr;
  if (use_graph && !h.own_stream) {
    MSP_CUDA(cudaStreamCreateWithFlags(&h.own_stream, cudaStreamNonBlocking));
    MSP_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    MSP_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
  }
  for (int it = 0; it < h.pegp_maxit; it += kb) {
    if (use_graph) {
      cudaStream_t gs2 = h.own_stream;
      MSP_CUDA(cudaEventRecord(h.ev_fork, st));
      MSP_CUDA(cudaStreamWaitEvent(gs2, h.ev_fork, 0));
      if (h.pegp_graph && h.pegp_graph_z != x) {
        cudaGraphExecDestroy(h.pegp_graph);
        h.pegp_graph = nullptr;
      }
      if (!h.pegp_graph) {
        h.pegp_graph_z = x;
        const int64_t l0 = h.launches;
        cudaGraph_t g;
        MSP_CUDA(cudaStreamBeginCapture(gs2, cudaStreamCaptureModeThreadLocal));
        for (int b2 = 0; b2 < kb; ++b2) one_iteration(b2 & 1, gs2);
        MSP_CUDA(cudaStreamEndCapture(gs2, &g));
        MSP_CUDA(cudaGraphInstantiate(&h.pegp_graph, g, 0));
        cudaGraphDestroy(g);
        h.pegp_graph_launches = h.launches - l0;
      } else {
        h.launches += h.pegp_graph_launches;
      }
      MSP_CUDA(cudaGraphLaunch(h.pegp_graph, gs2));
      MSP_CUDA(cudaEventRecord(h.ev_join, gs2));
      MSP_CUDA(cudaStreamWaitEvent(st, h.ev_join, 0));
    } else {
      for (int b2 = 0; b2 < kb; ++b2) one_iteration(b2 & 1, st);
      prof_flush();
    }
    MSP_LAUNCH_CHECK();
    if (d2h(d + S::FROZEN, st) != 0.0) break;
  }
  return (int)d2h(d + S::ITS, st);
}

}  // namespace

// y~ = L_H~ x~ (nested expanded vectors)
void apply_LH_nested(Handle& h, const double* x, double* y, cudaStream_t st) {
  pegp_build(h, st);
  const HMat H = hmat(h);
  k_h_apply<<<H.b0 + H.b1 + H.b2, TPB, 0, st>>>(H, x, y);
  ++h.launches;
  MSP_LAUNCH_CHECK();
}

// z~ = L_H~^+ r~: inner CG, then pegp_refine refinement steps (residual in
// double-double from the edge weights, correction by the same inner CG)
int solve_LH_nested(Handle& h, const double* rt_in, double* z, cudaStream_t st) {
  pegp_build(h, st);
  const int64_t nt = h.n_tilde;
  int its = inner_cg(h, rt_in, z, h.pegp_rtol, st);
  for (int s = 0; s < h.pegp_refine; ++s) {
    // the residual of the projected right-hand side: b - mean(b) - L_H~ z
    k_copy<<<grid_for(nt), TPB, 0, st>>>(nt, rt_in, h.ey.p);
    dot(h, nt, h.ey.p, nullptr, h.edots.p + S::SUMR, st);
    k_shift<<<grid_for(nt), TPB, 0, st>>>(nt, h.ey.p, h.edots.p + S::SUMR, 1.0 / (double)nt);
    k_h_resid_dd<<<grid_for(nt), TPB, 0, st>>>(nt, h.hrow.p, h.hcol.p, h.hw.p, z, h.ey.p, h.eres.p);
    h.launches += 3;
    its += inner_cg(h, h.eres.p, h.ecor.p, h.pegp_rtol, st);
    k_add<<<grid_for(nt), TPB, 0, st>>>(nt, h.ecor.p, z);
    ++h.launches;
  }
  MSP_LAUNCH_CHECK();
  h.pegp_last_inner = its;
  return its;
}

// z~ = L_T~^+ r~ (exact; nested expanded vectors): the init pass of the inner CG
void apply_LT_pinv_nested(Handle& h, const double* rt, double* z, cudaStream_t st) {
  pegp_build(h, st);
  const int64_t nt = h.n_tilde;
  double* d = h.edots.p;
  k_copy<<<grid_for(nt), TPB, 0, st>>>(nt, rt, h.er.p);
  MSP_CUDA(cudaMemsetAsync(h.ezp[0].p, 0, 2 * nt * sizeof(double), st));
  MSP_CUDA(cudaMemsetAsync(d, 0, S::N * sizeof(double), st));
  e_sweeps(h, elv(h), evec(h, h.ex.p, 0), 1, st);
  // z = the .x lanes of the pair array
  MSP_CUDA(cudaMemcpy2DAsync(z, sizeof(double), h.ezp[0].p, 2 * sizeof(double), sizeof(double), nt,
                             cudaMemcpyDeviceToDevice, st));
  MSP_LAUNCH_CHECK();
}

// z = P(mu) L_H~^+ P(mu)^T r on nested level-1 vectors
void apply_R_pegp_nested(Handle& h, const double* r, double* z, cudaStream_t st) {
  pegp_build(h, st);
  const int L = h.levels;
  double* rt = h.Y.p;   // r~ (Y is free outside the MSP sweeps)
  double* y = h.ex.p;   // y_k = (P^k)^T r (scratch in the level layout)
  k_copy<<<grid_for(h.n), TPB, 0, st>>>(h.n, r, rt);
  k_copy<<<grid_for(h.n), TPB, 0, st>>>(h.n, r, y);
  double scale = 1.0;
  for (int k = 1; k < L; ++k) {
    scale *= -h.mu;
    k_restrict<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.lv[k - 1].off,
                                                    h.lv[k].off, scale, y + h.lv[k - 1].off, y + h.lv[k].off, rt);
  }
  double* zt = h.W.p;   // z~ (W is free outside the MSP sweeps)
  solve_LH_nested(h, rt, zt, st);
  // w = P(mu) z~ (Horner, top-down), output level 1
  double* w = h.Z.p;
  const int64_t ot = h.lv[L - 1].off;
  k_copy<<<grid_for(h.lv[L - 1].n), TPB, 0, st>>>(h.lv[L - 1].n, zt + ot, w + ot);
  for (int k = L - 1; k >= 1; --k)
    k_prolong<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.lv[k - 1].off,
                                                   h.lv[k].off, -h.mu, zt, w);
  k_copy<<<grid_for(h.n), TPB, 0, st>>>(h.n, w, z);
  h.launches += 4 + 2 * (L - 1);
  MSP_LAUNCH_CHECK();
}

// canonical <-> nested expanded vectors (for the C ABI of the expanded-space calls)
void expanded_to_nested(Handle& h, const double* src, double* dst, cudaStream_t st) {
  for (int k = 1; k <= h.levels; ++k)
    k_gather_canon<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.order_nested[k - 1].p, h.lv[k - 1].off,
                                                            src, dst, 1);
  MSP_LAUNCH_CHECK();
}

void nested_to_expanded(Handle& h, const double* src, double* dst, cudaStream_t st) {
  for (int k = 1; k <= h.levels; ++k)
    k_gather_canon<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.order_nested[k - 1].p, h.lv[k - 1].off,
                                                            src, dst, 0);
  MSP_LAUNCH_CHECK();
}

}  // namespace msp
