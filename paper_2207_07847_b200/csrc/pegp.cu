// pegp.cu -- the PEGP preconditioner R = P(mu) L_H~^+ P(mu)^T (§3.2)
// on the GPU, and the expanded-space pieces it needs (sm_100a).
//
// H~ (reading R6/R7) is never assembled.  Its Laplacian is applied
// matrix-free from the per-level graphs (Eq. def:L_ell written blockwise:
// block (k, j) = (-mu)^{k-1} (-mu)^{j-1} L_k P_k^j, with P_k^j the 0/1
// aggregation from level k to level j):
//   * k = j:   every level-k edge, weight mu^{2(k-1)} w_k(i, m);
//   * j > k, j - k odd:  node i -> its level-j ancestor A_j(i), weight
//     mu^{k+j-2} cut_kj(i), cut_kj(i) = weight from i to level-k neighbours m
//     whose level-j ancestor differs from i's;
//   * j > k, j - k even: node i -> A_j(m) for every level-k neighbour m with
//     A_j(m) != A_j(i), weight mu^{k+j-2} w_k(i, m).
// These are exactly the negative off-diagonal entries of L_G~ (the positive
// edges of G~); walking the two ancestor chains from (i, m) upwards until they
// meet enumerates them.  Each edge is visited once, from its lower endpoint;
// the contribution to the upper endpoint is an fp64 atomic add.
//
// L_H~^+ r~ (minimum norm) is computed by CG in the expanded space,
// preconditioned by the exact MSP solve L_T~^+ (T~ is a spanning subgraph of
// H~, §3.3), to a relative residual of `pegp_rtol` (default 1e-13): the PEGP
// apply is inexact by construction; reading R13.
#include <algorithm>
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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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

// ------------------------------------------------------------ setup kernels
__global__ void k_parent(int64_t nB, const int32_t* __restrict__ cptr, int64_t off_k, int64_t off_k1,
                         int32_t* __restrict__ parent) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  for (int32_t c = cptr[B]; c < cptr[B + 1]; ++c) parent[off_k + c] = (int32_t)(off_k1 + B);
}

// nested CSR of level k from its canonical CSR: degree pass, then fill with
// columns mapped to absolute nested expanded indices
__global__ void k_hdeg(int64_t nk, const int32_t* __restrict__ order, const int64_t* __restrict__ crow,
                       int64_t* __restrict__ deg) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nk) return;
  const int32_t a = order[p];
  deg[p] = crow[a + 1] - crow[a];
}

__global__ void k_hfill(int64_t nk, const int32_t* __restrict__ order, const int64_t* __restrict__ crow,
                        const int32_t* __restrict__ ccol, const double* __restrict__ cw,
                        const int32_t* __restrict__ nested_of, int64_t off_k, const int64_t* __restrict__ hrow,
                        int32_t* __restrict__ hcol, double* __restrict__ hw) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nk) return;
  const int32_t a = order[p];
  int64_t q = hrow[off_k + p];
  for (int64_t e = crow[a]; e < crow[a + 1]; ++e, ++q) {
    hcol[q] = (int32_t)(off_k + nested_of[ccol[e]]);
    hw[q] = cw[e];
  }
}

// ------------------------------------------------------------ L_H~ x~
// One thread per level-k node (grid over level k); y must be zeroed first.
__global__ void __launch_bounds__(TPB) k_lh_apply(int64_t nk, int64_t off_k, int k, int L, double mu,
                                                  const int64_t* __restrict__ hrow, const int32_t* __restrict__ hcol,
                                                  const double* __restrict__ hw, const int32_t* __restrict__ parent,
                                                  const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nk) return;
  const int64_t gi = off_k + i;
  const double xi = x[gi];
  double sig = 1.0;
  for (int j = 1; j < k; ++j) sig *= mu * mu;  // mu^{2(k-1)}
  double cut[MAXL];
  for (int j = 0; j < L; ++j) cut[j] = 0.0;
  double acc = 0.0;
  for (int64_t e = hrow[gi]; e < hrow[gi + 1]; ++e) {
    const int32_t gm = hcol[e];
    const double w = hw[e];
    acc += sig * w * (xi - x[gm]);           // same-level edge (block (k, k))
    int32_t ai = (int32_t)gi, am = gm;
    double pw = sig * mu;                    // mu^{k+j-2} at j = k+1 is mu^{2k-1}
    for (int j = k + 1; j <= L; ++j) {
      ai = parent[ai];
      am = parent[am];
      if (ai == am) break;
      const double wt = pw * w;
      if (((j - k) & 1) == 0) {              // i -> A_j(m), non-ancestor
        const double xa = x[am];
        acc += wt * (xi - xa);
        atomicAdd(&y[am], wt * (xa - xi));
      } else {
        cut[j - 1] += wt;                    // i -> A_j(i), summed over m
      }
      pw *= mu;
    }
  }
  int32_t aj = (int32_t)gi;
  for (int j = k + 1; j <= L; ++j) {
    aj = parent[aj];
    const double c = cut[j - 1];
    if (c != 0.0) {
      const double xa = x[aj];
      acc += c * (xi - xa);
      atomicAdd(&y[aj], c * (xa - xi));
    }
  }
  atomicAdd(&y[gi], acc);
}

// ------------------------------------------------- expanded MSP: L_T~^+ r~
// s = subtree sums of r~ in T~ (s_B = r~_B + sum_children s_c)
__global__ void k_exp_up(int64_t nB, const int32_t* __restrict__ cptr, int64_t off_k, int64_t off_k1,
                         const double* __restrict__ rt, double* __restrict__ s) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  double v = rt[off_k1 + B];
  for (int32_t c = cptr[B]; c < cptr[B + 1]; ++c) v += s[off_k + c];
  s[off_k1 + B] = v;
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

// top of the expanded MSP solve: rho = sum(r~)/n~, z_top = (sigma L_l)^+ (s - rho N),
// shift m = (N.z_top + gdot - rho GN)/n~ (sc: [0] sum r~, [1] gdot)
__global__ void k_exp_top(int ntop, int64_t off_t, const double* __restrict__ s, const double* __restrict__ Nsub,
                          const double* __restrict__ pinv, const double* __restrict__ sc, double n_tilde, double GN,
                          double* __restrict__ z, double* __restrict__ rho_out) {
  __shared__ double t[256];
  __shared__ double sh_m;
  const double rho = sc[0] / n_tilde;
  for (int i = threadIdx.x; i < ntop; i += blockDim.x) t[i] = s[off_t + i] - rho * Nsub[off_t + i];
  __syncthreads();
  double zi = 0.0, nz = 0.0;
  if (threadIdx.x < ntop) {
    for (int j = 0; j < ntop; ++j) zi += pinv[threadIdx.x * ntop + j] * t[j];
    nz = Nsub[off_t + threadIdx.x] * zi;
  }
  nz = block_sum<256>(nz);
  if (threadIdx.x == 0) { sh_m = (nz + sc[1] - rho * GN) / n_tilde; *rho_out = rho; }
  __syncthreads();
  if (threadIdx.x < ntop) z[off_t + threadIdx.x] = zi - sh_m;
}

__global__ void k_exp_down(int64_t nB, const int32_t* __restrict__ cptr, int64_t off_k, int64_t off_k1, int64_t n1,
                           int64_t lo_k, const double* __restrict__ kinv, const double* __restrict__ lof,
                           const double* __restrict__ s, const double* __restrict__ Nsub,
                           const double* __restrict__ rho_p, double* __restrict__ z) {
  int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (B >= nB) return;
  const double rho = *rho_p;
  const int32_t s0 = cptr[B], s1 = cptr[B + 1];
  const double* ki = kinv + 3 * (off_k1 - n1 + B);
  const int64_t lb = 3 * (lo_k - 2 * B - 2);
  auto tf = [&](int64_t p) { return s[off_k + p] - rho * Nsub[off_k + p]; };
  const double zb = z[off_k1 + B];
  const double tu = tf(s0), tv = tf(s0 + 1);
  double au = tu, av = tv;
  for (int32_t p = s0 + 2; p < s1; ++p) {
    const double tx = tf(p);
    au += lof[lb + 3 * p] * tx;
    av += lof[lb + 3 * p + 1] * tx;
  }
  const double zu = ki[0] * au + ki[1] * av, zv = ki[1] * au + ki[2] * av;
  z[off_k + s0] = zb + zu;
  z[off_k + s0 + 1] = zb + zv;
  for (int32_t p = s0 + 2; p < s1; ++p) {
    const double tx = tf(p);
    z[off_k + p] = zb + lof[lb + 3 * p + 2] * tx + lof[lb + 3 * p] * zu + lof[lb + 3 * p + 1] * zv;
  }
}

// ------------------------------------------------------------ restrict / prolong
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

__global__ void k_copy(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_shift(int64_t n, double* __restrict__ a, const double* __restrict__ sum, double inv_n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] -= *sum * inv_n;
}

// CG vector updates with device scalars
// frozen (optional): once the inner CG has converged the updates stop, so a
// captured batch may run past convergence; its (optional) counts iterations
__global__ void k_axpy2(int64_t n, const double* __restrict__ num, const double* __restrict__ den,
                        double* __restrict__ x, const double* __restrict__ p, double* __restrict__ r,
                        const double* __restrict__ q, const double* __restrict__ frozen = nullptr,
                        double* __restrict__ its = nullptr) {
  if (frozen && *frozen != 0.0) return;
  if (its && blockIdx.x == 0 && threadIdx.x == 0) *its += 1.0;
  const double a = *num / *den;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) { x[i] += a * p[i]; r[i] -= a * q[i]; }
}

__global__ void k_pupd(int64_t n, const double* __restrict__ num, const double* __restrict__ den,
                       const double* __restrict__ z, double* __restrict__ p,
                       const double* __restrict__ frozen = nullptr) {
  if (frozen && *frozen != 0.0) return;
  const double b = *num / *den;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = z[i] + b * p[i];
}

// the convergence test of the inner CG on the device: (r, r) <= tol^2 (b, b)
__global__ void k_freeze(const double* __restrict__ rr, const double* __restrict__ tol2, double* __restrict__ frozen) {
  if (*frozen == 0.0 && *rr <= *tol2) *frozen = 1.0;
}

__global__ void k_gather_canon(int64_t nk, const int32_t* __restrict__ order, int64_t off, const double* __restrict__ src,
                               double* __restrict__ dst, int to_nested) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nk) return;
  if (to_nested) dst[off + p] = src[off + order[p]];
  else dst[off + order[p]] = src[off + p];
}

struct Dots {  // device scalar slots of the PEGP inner CG
  enum { SUMR = 0, GDOT, RHO, RZ, RZ_OLD, PQ, RR, BB, TOL2, FROZEN, ITS, N };
};

}  // namespace

// ------------------------------------------------------------ host side
void pegp_build(Handle& h, cudaStream_t st) {
  if (h.pegp_ready) return;
  const int L = h.levels;
  const int64_t nt = h.n_tilde;
  // parent pointers
  h.parent.alloc(nt);
  MSP_CUDA(cudaMemsetAsync(h.parent.p, 0xff, nt * sizeof(int32_t), st));
  for (int k = 1; k < L; ++k)
    k_parent<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.lv[k - 1].off,
                                                  h.lv[k].off, h.parent.p);
  // per-level adjacency, nested, in one CSR over n~
  DBuf<int64_t> deg;
  deg.alloc(nt + 1);
  MSP_CUDA(cudaMemsetAsync(deg.p, 0, (nt + 1) * sizeof(int64_t), st));
  for (int k = 1; k <= L; ++k)
    k_hdeg<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.order_nested[k - 1].p, h.canon_rowptr[k - 1].p,
                                                    deg.p + h.lv[k - 1].off);
  MSP_LAUNCH_CHECK();
  h.hrow.alloc(nt + 1);
  {
    std::vector<int64_t> dh(nt + 1);
    MSP_CUDA(cudaMemcpyAsync(dh.data(), deg.p, (nt + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    int64_t acc = 0;
    for (int64_t i = 0; i <= nt; ++i) { const int64_t d = dh[i]; dh[i] = acc; acc += d; }
    MSP_CUDA(cudaMemcpyAsync(h.hrow.p, dh.data(), (nt + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    h.hnnz = dh[nt];
    MSP_CUDA(cudaStreamSynchronize(st));
  }
  h.hcol.alloc(std::max<int64_t>(h.hnnz, 1));
  h.hw.alloc(std::max<int64_t>(h.hnnz, 1));
  for (int k = 1; k <= L; ++k)
    k_hfill<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.order_nested[k - 1].p, h.canon_rowptr[k - 1].p,
                                                     h.canon_col[k - 1].p, h.canon_w[k - 1].p,
                                                     h.nested_of_canon[k - 1].p, h.lv[k - 1].off, h.hrow.p, h.hcol.p,
                                                     h.hw.p);
  MSP_LAUNCH_CHECK();
  for (auto* v : {&h.ex, &h.er, &h.ep, &h.eq, &h.ez, &h.es, &h.ey}) v->alloc(nt + 8);
  h.edots.alloc(Dots::N);
  h.epart.alloc(1024);
  MSP_CUDA(cudaStreamSynchronize(st));
  h.pegp_ready = true;
}

namespace {

void dot(Handle& h, int64_t n, const double* a, const double* b, double* out, cudaStream_t st) {
  const unsigned g = std::min<unsigned>(grid_for(n), 1024u);
  k_dot_part<<<g, TPB, 0, st>>>(n, a, b, h.epart.p);
  k_dot_final<<<1, TPB, 0, st>>>((int)g, h.epart.p, out);
  h.launches += 2;
}

double read_slot(Handle& h, int i, cudaStream_t st) {
  double v = 0.0;
  MSP_CUDA(cudaMemcpyAsync(&v, h.edots.p + i, sizeof(double), cudaMemcpyDeviceToHost, st));
  MSP_CUDA(cudaStreamSynchronize(st));
  return v;
}

}  // namespace

// y~ = L_H~ x~ (nested expanded vectors)
void apply_LH_nested(Handle& h, const double* x, double* y, cudaStream_t st) {
  pegp_build(h, st);
  MSP_CUDA(cudaMemsetAsync(y, 0, h.n_tilde * sizeof(double), st));
  for (int k = 1; k <= h.levels; ++k) {
    k_lh_apply<<<grid_for(h.lv[k - 1].n), TPB, 0, st>>>(h.lv[k - 1].n, h.lv[k - 1].off, k, h.levels, h.mu, h.hrow.p,
                                                        h.hcol.p, h.hw.p, h.parent.p, x, y);
    ++h.launches;
  }
  MSP_LAUNCH_CHECK();
}

// z~ = L_T~^+ r~ (exact; nested expanded vectors; uses h.es as workspace)
void apply_LT_pinv_nested(Handle& h, const double* rt, double* z, cudaStream_t st) {
  const int L = h.levels;
  const int64_t nt = h.n_tilde;
  double* s = h.es.p;
  // level-1 subtree sums are r~ itself
  k_copy<<<grid_for(h.lv[0].n), TPB, 0, st>>>(h.lv[0].n, rt, s);
  for (int k = 1; k < L; ++k)
    k_exp_up<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.lv[k - 1].off,
                                                  h.lv[k].off, rt, s);
  dot(h, nt, rt, nullptr, h.edots.p + Dots::SUMR, st);
  dot(h, h.lv[L - 1].off, h.gvec.p, s, h.edots.p + Dots::GDOT, st);
  k_exp_top<<<1, 256, 0, st>>>((int)h.lv[L - 1].n, h.lv[L - 1].off, s, h.Nsub.p, h.top_pinv.p, h.edots.p, (double)nt,
                               h.GN, z, h.edots.p + Dots::RHO);
  for (int k = L - 1; k >= 1; --k)
    k_exp_down<<<grid_for(h.lv[k].n), TPB, 0, st>>>(h.lv[k].n, h.cptr.p + h.cptr_off[k - 1], h.lv[k - 1].off,
                                                    h.lv[k].off, h.n, h.lo_off[k - 1], h.kinv.p, h.lof.p, s, h.Nsub.p,
                                                    h.edots.p + Dots::RHO, z);
  h.launches += 2 + 2 * (L - 1);
  MSP_LAUNCH_CHECK();
}

// z~ = L_H~^+ r~ by MSP-preconditioned CG in the expanded space (r~ is first
// projected off the ones vector; x0 = 0 keeps the iterates mean-zero)
int solve_LH_nested(Handle& h, const double* rt_in, double* z, cudaStream_t st) {
  pegp_build(h, st);
  const int64_t nt = h.n_tilde;
  const unsigned gn = grid_for(nt);
  double* d = h.edots.p;
  k_copy<<<gn, TPB, 0, st>>>(nt, rt_in, h.er.p);
  dot(h, nt, h.er.p, nullptr, d + Dots::SUMR, st);
  k_shift<<<gn, TPB, 0, st>>>(nt, h.er.p, d + Dots::SUMR, 1.0 / (double)nt);
  MSP_CUDA(cudaMemsetAsync(z, 0, nt * sizeof(double), st));
  dot(h, nt, h.er.p, h.er.p, d + Dots::BB, st);
  const double bb = read_slot(h, Dots::BB, st);
  if (bb == 0.0) return 0;
  const double tol2 = h.pegp_rtol * h.pegp_rtol * bb;
  apply_LT_pinv_nested(h, h.er.p, h.ez.p, st);
  dot(h, nt, h.er.p, h.ez.p, d + Dots::RZ, st);
  k_copy<<<gn, TPB, 0, st>>>(nt, h.ez.p, h.ep.p);
  // inner iterations in captured batches (the graph is fixed per handle: every
  // vector is a handle buffer); the convergence test runs on the device after
  // every iteration and freezes the updates, the host reads it per batch
  {
    const double init[3] = {tol2, 0.0, 0.0};  // TOL2, FROZEN, ITS
    MSP_CUDA(cudaMemcpyAsync(d + Dots::TOL2, init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  auto one_iteration = [&](cudaStream_t s2) {
    apply_LH_nested(h, h.ep.p, h.eq.p, s2);
    dot(h, nt, h.ep.p, h.eq.p, d + Dots::PQ, s2);
    k_axpy2<<<gn, TPB, 0, s2>>>(nt, d + Dots::RZ, d + Dots::PQ, z, h.ep.p, h.er.p, h.eq.p, d + Dots::FROZEN,
                                d + Dots::ITS);
    dot(h, nt, h.er.p, h.er.p, d + Dots::RR, s2);
    k_freeze<<<1, 1, 0, s2>>>(d + Dots::RR, d + Dots::TOL2, d + Dots::FROZEN);
    apply_LT_pinv_nested(h, h.er.p, h.ez.p, s2);
    MSP_CUDA(cudaMemcpyAsync(d + Dots::RZ_OLD, d + Dots::RZ, sizeof(double), cudaMemcpyDeviceToDevice, s2));
    dot(h, nt, h.er.p, h.ez.p, d + Dots::RZ, s2);
    k_pupd<<<gn, TPB, 0, s2>>>(nt, d + Dots::RZ, d + Dots::RZ_OLD, h.ez.p, h.ep.p, d + Dots::FROZEN);
    h.launches += 4;
  };
  const int kb = 8;  // iterations per captured batch
  const bool use_graph = std::getenv("MSP_NO_GRAPH") == nullptr;
  if (use_graph && !h.own_stream) {
    MSP_CUDA(cudaStreamCreateWithFlags(&h.own_stream, cudaStreamNonBlocking));
    MSP_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    MSP_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
  }
  int it = 0;
  for (int done_b = 0; it < h.pegp_maxit && !done_b; it += kb) {
    if (use_graph) {
      cudaStream_t gs = h.own_stream;
      MSP_CUDA(cudaEventRecord(h.ev_fork, st));
      MSP_CUDA(cudaStreamWaitEvent(gs, h.ev_fork, 0));
      if (h.pegp_graph && h.pegp_graph_z != z) {
        cudaGraphExecDestroy(h.pegp_graph);
        h.pegp_graph = nullptr;
      }
      if (!h.pegp_graph) {
        h.pegp_graph_z = z;
        const int64_t l0 = h.launches;
        cudaGraph_t g;
        MSP_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        for (int b = 0; b < kb; ++b) one_iteration(gs);
        MSP_CUDA(cudaStreamEndCapture(gs, &g));
        MSP_CUDA(cudaGraphInstantiate(&h.pegp_graph, g, 0));
        cudaGraphDestroy(g);
        h.pegp_graph_launches = h.launches - l0;
      } else {
        h.launches += h.pegp_graph_launches;
      }
      MSP_CUDA(cudaGraphLaunch(h.pegp_graph, gs));
      MSP_CUDA(cudaEventRecord(h.ev_join, gs));
      MSP_CUDA(cudaStreamWaitEvent(st, h.ev_join, 0));
    } else {
      for (int b = 0; b < kb; ++b) one_iteration(st);
    }
    done_b = read_slot(h, Dots::FROZEN, st) != 0.0;
  }
  it = (int)read_slot(h, Dots::ITS, st);
  MSP_LAUNCH_CHECK();
  h.pegp_last_inner = it;
  return it;
}

// z = P(mu) L_H~^+ P(mu)^T r on nested level-1 vectors
void apply_R_pegp_nested(Handle& h, const double* r, double* z, cudaStream_t st) {
  pegp_build(h, st);
  const int L = h.levels;
  double* rt = h.ey.p;  // r~
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
