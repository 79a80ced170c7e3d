// solve.cu -- solve phase of the PEGP/MSP solver (sm_100a): apply_L, the
// exact MSP apply R = P(mu) L_T~^+ P(mu)^T as level-ordered restrict /
// prolong sweeps over the nested aggregate hierarchy, and fused PCG.
//
// Layout (nested numbering): level-k node i of the
// expanded graph lives at index off_k + i of every n~-vector; the children of
// level-(k+1) node B are level-k nodes cptr_k[B] .. cptr_k[B+1]-1, the first
// two being the matched pair, the rest leftovers.
#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace msp {

namespace {

constexpr int TPB = 256;

// device scalar slots
enum { S_RHO = 0, S_PQ, S_ALPHA, S_RR, S_BETA, S_TOL2, S_BB, S_SHIFT, S_NSCAL };
// counter slots
enum { C_SPMV = 0, C_UPD, C_DOWN, C_DONE, C_IT, C_NCNT };

inline unsigned grid_for(int64_t n, int tpb = TPB) {
  int64_t g = (n + tpb - 1) / tpb;
  return (unsigned)std::max<int64_t>(g, 1);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; result valid in thread 0
template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[NT / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = (lane < NT / 32) ? ws[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// deterministic sum of partials[0..n) by one block; result in thread 0
template <int NT>
__device__ __forceinline__ double block_sum_array(const double* part, int64_t n) {
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += NT) v += part[i];
  return block_sum<NT>(v);
}

// "last block done" ticket: returns true in every thread of the last block
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// ----------------------------------------------------------------- permute
__global__ void k_gather(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ src,
                         double* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

__global__ void k_scatter(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ src,
                          double* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[perm[i]] = src[i];
}

// ------------------------------------------------------------------ L_G x
// y_i = sum_j w_ij (x_i - x_j)   (L_G = B^T W B, §2.1)
// LANES threads per row; optional fused dot (x, y) -> alpha = rho / (p, Lp).
template <int LANES, bool DOT>
__global__ void __launch_bounds__(TPB) k_spmv(int64_t n, const int32_t* __restrict__ rowptr,
                                              const int32_t* __restrict__ col,
                                              const double* __restrict__ w,
                                              const double* __restrict__ x, double* __restrict__ y,
                                              double* __restrict__ part, double* __restrict__ scal,
                                              unsigned int* __restrict__ cnt) {
  if (DOT && cnt[C_DONE]) return;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid / LANES;
  const int lane = threadIdx.x % LANES;
  double acc = 0.0, xi = 0.0;
  if (row < n) {
    xi = x[row];
    const int32_t e0 = rowptr[row], e1 = rowptr[row + 1];
    for (int32_t e = e0 + lane; e < e1; e += LANES) acc += w[e] * (xi - x[col[e]]);
  }
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  double d = 0.0;
  if (row < n && lane == 0) {
    y[row] = acc;
    d = xi * acc;
  }
  if (DOT) {
    const double bs = block_sum<TPB>(d);
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (last_block(&cnt[C_SPMV])) {
      const double pq = block_sum_array<TPB>(part, gridDim.x);
      if (threadIdx.x == 0) {
        scal[S_PQ] = pq;
        scal[S_ALPHA] = scal[S_RHO] / pq;
        cnt[C_SPMV] = 0;
      }
    }
  }
}

// x += alpha p ; r -= alpha q ; rr = (r, r) -> convergence flag
__global__ void __launch_bounds__(TPB) k_update(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                const double* __restrict__ p, const double* __restrict__ q,
                                                double* __restrict__ part, double* __restrict__ scal,
                                                unsigned int* __restrict__ cnt) {
  if (cnt[C_DONE]) return;
  const double alpha = scal[S_ALPHA];
  double d = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    d += ri * ri;
  }
  const double bs = block_sum<TPB>(d);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
  if (last_block(&cnt[C_UPD])) {
    const double rr = block_sum_array<TPB>(part, gridDim.x);
    if (threadIdx.x == 0) {
      scal[S_RR] = rr;
      cnt[C_IT] += 1;
      if (rr <= scal[S_TOL2]) cnt[C_DONE] = 1;
      cnt[C_UPD] = 0;
    }
  }
}

// ----------------------------------------------------------- MSP up-sweep
// Restriction by P(mu)^T fused with the forward elimination of the block tree
// T~: for level-(k+1) node B with children S,
//   y_B = sum_{c in S} y_c              (P^T, unscaled)
//   s_B = (-mu)^k y_B + sum_{c in S} s_c  (subtree sum of r~ = P(mu)^T r)
//   gdot += sum_c g_c s_c               (for the mean of z~, see k_top)
__global__ void __launch_bounds__(TPB) k_up(int64_t nB, const int32_t* __restrict__ cptr,
                                            const double* __restrict__ yin, const double* __restrict__ sin,
                                            const double* __restrict__ g, double* __restrict__ yout,
                                            double* __restrict__ sout, double negmu_k,
                                            double* __restrict__ part, const unsigned int* __restrict__ cnt,
                                            int check_done) {
  if (check_done && cnt[C_DONE]) return;
  const int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double gs = 0.0;
  if (B < nB) {
    const int32_t c0 = cptr[B], c1 = cptr[B + 1];
    double y = 0.0, s = 0.0;
    for (int32_t c = c0; c < c1; ++c) {
      const double sc = sin[c];
      y += yin[c];
      s += sc;
      gs += g[c] * sc;
    }
    yout[B] = y;
    sout[B] = negmu_k * y + s;
  }
  const double bs = block_sum<TPB>(gs);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
}

// ------------------------------------------------------------- top solve
// rho = c sum(r) / n~ makes the right-hand side compatible (r~ - rho 1 is the
// projection of r~ = P^T r off the ones vector); z_top = (sigma_l L_l)^+ s'_top;
// then shift so that the whole z~ has zero mean (z~ = L_T~^+ r~, minimum norm):
//   sum z~ = sum_T N_T z_T + sum_{non-top} g_i (s_i - rho N_i).
template <int NT>
__global__ void __launch_bounds__(NT) k_top(int ntop, const double* __restrict__ ytop,
                                            const double* __restrict__ stop,
                                            const double* __restrict__ Ntop,
                                            const double* __restrict__ pinv, const double* __restrict__ part,
                                            int64_t npart, double c_sum, double n_tilde, double GN,
                                            double* __restrict__ ztop, double* __restrict__ wtop,
                                            double* __restrict__ scal, const unsigned int* __restrict__ cnt,
                                            int check_done) {
  if (check_done && cnt[C_DONE]) return;
  __shared__ double t[256];
  __shared__ double sh_rho, sh_m;
  const double gdot = block_sum_array<NT>(part, npart);
  double ys = 0.0;
  for (int i = threadIdx.x; i < ntop; i += NT) ys += ytop[i];
  ys = block_sum<NT>(ys);
  if (threadIdx.x == 0) sh_rho = c_sum * ys / n_tilde;
  __syncthreads();
  const double rho = sh_rho;
  for (int i = threadIdx.x; i < ntop; i += NT) t[i] = stop[i] - rho * Ntop[i];
  __syncthreads();
  double zi = 0.0, nz = 0.0;
  if (threadIdx.x < ntop) {
    const int i = threadIdx.x;
    for (int j = 0; j < ntop; ++j) zi += pinv[(int64_t)i * ntop + j] * t[j];
    nz = Ntop[i] * zi;
  }
  nz = block_sum<NT>(nz);
  if (threadIdx.x == 0) {
    sh_m = (nz + gdot - rho * GN) / n_tilde;
    scal[S_SHIFT] = rho;
  }
  __syncthreads();
  if (threadIdx.x < ntop) {
    ztop[threadIdx.x] = zi - sh_m;
    wtop[threadIdx.x] = zi - sh_m;
  }
}

// ----------------------------------------------------------- MSP down-sweep
// Back substitution of T~ fused with the prolongation P(mu) (Horner form):
// for children S of B:  t = s_S - rho N_S,  zeta = K_S^{-1} t (pair + leftover
// elimination with the factors of k_msp_factor),  z_c = z_B + zeta_c,
// w_c = z_c + (-mu) w_B.  At level 1, w_c is the output R r; mode 1/2 also
// reduce (r, z) for PCG (1: rho = rz; 2: beta = rz / rho, rho = rz).
template <bool LEVEL1>
__global__ void __launch_bounds__(TPB) k_down(int64_t nB, const int32_t* __restrict__ cptr,
                                              const double* __restrict__ sin, const double* __restrict__ Nk,
                                              const double* __restrict__ c0, const double* __restrict__ c1,
                                              const double* __restrict__ c2, const double* __restrict__ zB,
                                              const double* __restrict__ wB, double* __restrict__ zout,
                                              double* __restrict__ wout, double negmu,
                                              double* __restrict__ part, double* __restrict__ scal,
                                              unsigned int* __restrict__ cnt, int mode) {
  if (mode >= 2 && cnt[C_DONE]) return;
  const int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double rho = scal[S_SHIFT];
  double rz = 0.0;
  if (B < nB) {
    const int32_t s0 = cptr[B], s1 = cptr[B + 1];
    const double zb = zB[B], wb = negmu * wB[B];
    const double tu = sin[s0] - rho * (LEVEL1 ? 1.0 : Nk[s0]);
    const double tv = sin[s0 + 1] - rho * (LEVEL1 ? 1.0 : Nk[s0 + 1]);
    double au = tu, av = tv;
    for (int32_t p = s0 + 2; p < s1; ++p) {
      const double tx = sin[p] - rho * (LEVEL1 ? 1.0 : Nk[p]);
      au += c0[p] * tx;
      av += c1[p] * tx;
    }
    const double kuu = c0[s0], kuv = c1[s0], kvv = c2[s0];
    const double zu = kuu * au + kuv * av, zv = kuv * au + kvv * av;
    {
      const double z = zb + zu, ww = z + wb;
      if (!LEVEL1) zout[s0] = z;
      wout[s0] = ww;
      if (LEVEL1) rz += sin[s0] * ww;
    }
    {
      const double z = zb + zv, ww = z + wb;
      if (!LEVEL1) zout[s0 + 1] = z;
      wout[s0 + 1] = ww;
      if (LEVEL1) rz += sin[s0 + 1] * ww;
    }
    for (int32_t p = s0 + 2; p < s1; ++p) {
      const double tx = sin[p] - rho * (LEVEL1 ? 1.0 : Nk[p]);
      const double zx = c2[p] * tx + c0[p] * zu + c1[p] * zv;
      const double z = zb + zx, ww = z + wb;
      if (!LEVEL1) zout[p] = z;
      wout[p] = ww;
      if (LEVEL1) rz += sin[p] * ww;
    }
  }
  if (LEVEL1 && mode >= 1) {
    const double bs = block_sum<TPB>(rz);
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (last_block(&cnt[C_DOWN])) {
      const double tot = block_sum_array<TPB>(part, gridDim.x);
      if (threadIdx.x == 0) {
        if (mode == 2) scal[S_BETA] = tot / scal[S_RHO];
        else scal[S_BETA] = 0.0;
        scal[S_RHO] = tot;
        cnt[C_DOWN] = 0;
      }
    }
  }
}

// p = z + beta p
__global__ void __launch_bounds__(TPB) k_pupdate(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                                                 const double* __restrict__ scal,
                                                 const unsigned int* __restrict__ cnt, int check_done) {
  if (check_done && cnt[C_DONE]) return;
  const double beta = scal[S_BETA];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// unpreconditioned CG: z = r, rho = (r, r)
__global__ void __launch_bounds__(TPB) k_copy_dot(int64_t n, const double* __restrict__ r, double* __restrict__ z,
                                                  double* __restrict__ part, double* __restrict__ scal,
                                                  unsigned int* __restrict__ cnt, int mode) {
  if (mode >= 2 && cnt[C_DONE]) return;
  double d = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i];
    z[i] = ri;
    d += ri * ri;
  }
  const double bs = block_sum<TPB>(d);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
  if (last_block(&cnt[C_DOWN])) {
    const double tot = block_sum_array<TPB>(part, gridDim.x);
    if (threadIdx.x == 0) {
      scal[S_BETA] = (mode == 2) ? tot / scal[S_RHO] : 0.0;
      scal[S_RHO] = tot;
      cnt[C_DOWN] = 0;
    }
  }
}

__global__ void k_init_state(double* scal, unsigned int* cnt, double tol2, const double* bb) {
  for (int i = 0; i < S_NSCAL; ++i) scal[i] = 0.0;
  for (int i = 0; i < C_NCNT; ++i) cnt[i] = 0;
  scal[S_BB] = *bb;
  scal[S_TOL2] = tol2 * (*bb);
  if (*bb == 0.0) cnt[C_DONE] = 1;
}

__global__ void __launch_bounds__(TPB) k_dot_part(int64_t n, const double* __restrict__ a,
                                                  const double* __restrict__ b, double* __restrict__ part,
                                                  double* __restrict__ out, unsigned int* __restrict__ cnt) {
  double d = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d += a[i] * b[i];
  const double bs = block_sum<TPB>(d);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
  if (last_block(&cnt[C_UPD])) {
    const double tot = block_sum_array<TPB>(part, gridDim.x);
    if (threadIdx.x == 0) { *out = tot; cnt[C_UPD] = 0; }
  }
}

// dense top-only apply when the hierarchy has a single level (n <= 2, or a
// graph that aggregates to one node): z = (L_G)^+ r, plus the PCG scalars.
__global__ void __launch_bounds__(256) k_top_only(int nt, const double* __restrict__ pinv,
                                                  const double* __restrict__ r, double* __restrict__ z,
                                                  double* __restrict__ scal, unsigned int* __restrict__ cnt,
                                                  int mode) {
  if (mode >= 2 && cnt[C_DONE]) return;
  __shared__ double rs[256];
  for (int i = threadIdx.x; i < nt; i += 256) rs[i] = r[i];
  __syncthreads();
  double zi = 0.0, rz = 0.0;
  if (threadIdx.x < nt) {
    for (int j = 0; j < nt; ++j) zi += pinv[threadIdx.x * nt + j] * rs[j];  // pinv kills the mean
    z[threadIdx.x] = zi;
    rz = rs[threadIdx.x] * zi;
  }
  rz = block_sum<256>(rz);
  if (threadIdx.x == 0 && mode >= 1) {
    scal[S_BETA] = (mode == 2) ? rz / scal[S_RHO] : 0.0;
    scal[S_RHO] = rz;
  }
}

int lanes_for(double mean_deg) {
  if (mean_deg <= 3.0) return 2;
  if (mean_deg <= 6.0) return 4;
  if (mean_deg <= 12.0) return 8;
  if (mean_deg <= 24.0) return 16;
  return 32;
}

template <bool DOT>
void launch_spmv(Handle& h, const double* x, double* y, cudaStream_t st) {
  const double md = (double)h.nnz_adj / (double)h.n;
  const int lanes = lanes_for(md);
  const int64_t threads = h.n * lanes;
  const unsigned g = grid_for(threads);
  double* part = h.red.p;
  double* scal = h.scal.p;
  unsigned* cnt = h.counters.p;
#define SPMV_CASE(L)                                                                              \
  case L:                                                                                         \
    k_spmv<L, DOT><<<g, TPB, 0, st>>>(h.n, h.rowptr1.p, h.col1.p, h.w1.p, x, y, part, scal, cnt); \
    break;
  switch (lanes) {
    SPMV_CASE(2)
    SPMV_CASE(4)
    SPMV_CASE(8)
    SPMV_CASE(16)
    SPMV_CASE(32)
  }
#undef SPMV_CASE
  MSP_LAUNCH_CHECK();
  ++h.launches;
}

// ----------------------------------------------------------- profiling
// When h.profile is set, every launch of the solve is bracketed by CUDA
// events on the launching stream; per-category device time is accumulated
// (msp_get_profile).  Off by default: the timed bench steps run unbracketed.
struct Prof {
  Handle& h;
  cudaStream_t st;
  std::vector<cudaEvent_t> ev;
  std::vector<int> cat;
  explicit Prof(Handle& hh, cudaStream_t s) : h(hh), st(s) {}
  ~Prof() { flush(); }
  void begin() {
    if (!h.profile) return;
    cudaEvent_t e;
    MSP_CUDA(cudaEventCreate(&e));
    MSP_CUDA(cudaEventRecord(e, st));
    ev.push_back(e);
  }
  void end(int c) {
    if (!h.profile) return;
    cudaEvent_t e;
    MSP_CUDA(cudaEventCreate(&e));
    MSP_CUDA(cudaEventRecord(e, st));
    ev.push_back(e);
    cat.push_back(c);
  }
  void flush() {
    if (ev.empty()) return;
    cudaEventSynchronize(ev.back());
    for (size_t i = 0; i < cat.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      h.prof_ms[cat[i]] += ms;
      h.prof_cnt[cat[i]] += 1;
    }
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    cat.clear();
  }
};

// partial-sum region of the up-sweep of level k (children at level k)
int64_t up_part_off(const Handle& h, int k) {
  int64_t o = 0;
  for (int j = 1; j < k; ++j) o += grid_for(h.lv[j].n);
  return o;
}

// R r for the MSP, nested numbering; mode 0: plain apply, 1: PCG init, 2: PCG iteration
void msp_sweeps(Handle& h, const double* r, double* z, cudaStream_t st, int mode, Prof* pf = nullptr) {
  Prof local(h, st);
  Prof& P = pf ? *pf : local;
  const int L = h.levels;
  const int check = mode >= 2 ? 1 : 0;
  double* part = h.red.p;
  double* part_up = h.red.p + h.red_cap / 2;  // up-sweep partials live in the upper half
  if (L == 1) {
    k_top_only<<<1, 256, 0, st>>>((int)h.lv[0].n, h.top_pinv.p, r, z, h.scal.p, h.counters.p, mode);
    MSP_LAUNCH_CHECK();
    ++h.launches;
    return;
  }
  for (int k = 1; k < L; ++k) {
    const LevelHost& lk = h.lv[k - 1];
    const LevelHost& lk1 = h.lv[k];
    const double* yin = (k == 1) ? r : h.Y.p + lk.off;
    const double* sin = (k == 1) ? r : h.S.p + lk.off;
    P.begin();
    k_up<<<grid_for(lk1.n), TPB, 0, st>>>(lk1.n, h.cptr.p + h.cptr_off[k - 1], yin, sin, h.gvec.p + lk.off,
                                          h.Y.p + lk1.off, h.S.p + lk1.off, h.neg_mu_pow[k],
                                          part_up + up_part_off(h, k), h.counters.p, check);
    MSP_LAUNCH_CHECK();
    P.end(k == 1 ? PC_UP1 : PC_UPC);
    ++h.launches;
  }
  const LevelHost& lt = h.lv[L - 1];
  const int64_t npart = up_part_off(h, L);
  P.begin();
  k_top<256><<<1, 256, 0, st>>>((int)lt.n, h.Y.p + lt.off, h.S.p + lt.off, h.Nsub.p + lt.off, h.top_pinv.p,
                                part_up, npart, h.c_sum, (double)h.n_tilde, h.GN, h.Z.p + lt.off,
                                h.W.p + lt.off, h.scal.p, h.counters.p, check);
  MSP_LAUNCH_CHECK();
  P.end(PC_TOP);
  ++h.launches;
  for (int k = L - 1; k >= 1; --k) {
    const LevelHost& lk = h.lv[k - 1];
    const LevelHost& lk1 = h.lv[k];
    P.begin();
    if (k >= 2) {
      k_down<false><<<grid_for(lk1.n), TPB, 0, st>>>(
          lk1.n, h.cptr.p + h.cptr_off[k - 1], h.S.p + lk.off, h.Nsub.p + lk.off, h.c0.p + lk.off,
          h.c1.p + lk.off, h.c2.p + lk.off, h.Z.p + lk1.off, h.W.p + lk1.off, h.Z.p + lk.off,
          h.W.p + lk.off, -h.mu, part, h.scal.p, h.counters.p, mode >= 2 ? 2 : 0);
    } else {
      k_down<true><<<grid_for(lk1.n), TPB, 0, st>>>(
          lk1.n, h.cptr.p + h.cptr_off[0], r, nullptr, h.c0.p, h.c1.p, h.c2.p, h.Z.p + lk1.off,
          h.W.p + lk1.off, nullptr, z, -h.mu, part, h.scal.p, h.counters.p, mode);
    }
    MSP_LAUNCH_CHECK();
    P.end(k == 1 ? PC_DOWN1 : PC_DOWNC);
    ++h.launches;
  }
}

}  // namespace

void alloc_solve_workspace(Handle& h) {
  const int64_t nt = h.n_tilde;
  h.Y.alloc(nt); h.S.alloc(nt); h.Z.alloc(nt); h.W.alloc(nt);
  // partials: the SpMV grid is the largest per-launch grid; the up-sweep
  // partials of all levels go to the upper half
  const double md = (double)h.nnz_adj / (double)h.n;
  int64_t need = grid_for(h.n * lanes_for(md));
  need = std::max<int64_t>(need, grid_for(h.n));
  int64_t upn = 0;
  for (int k = 1; k < h.levels; ++k) upn += grid_for(h.lv[k].n);
  h.red_cap = 2 * std::max<int64_t>(need, upn) + 64;
  h.red.alloc(h.red_cap);
  h.vx.alloc(h.n); h.vr.alloc(h.n); h.vp.alloc(h.n); h.vq.alloc(h.n); h.vz.alloc(h.n); h.vb.alloc(h.n);
  h.counters.alloc(C_NCNT);
  h.scal.alloc(S_NSCAL);
  MSP_CUDA(cudaMemset(h.counters.p, 0, C_NCNT * sizeof(unsigned)));
  MSP_CUDA(cudaMemset(h.scal.p, 0, S_NSCAL * sizeof(double)));
}

void gather_to_nested(Handle& h, const double* src, double* dst, cudaStream_t st) {
  k_gather<<<grid_for(h.n), TPB, 0, st>>>(h.n, h.perm.p, src, dst);
  MSP_LAUNCH_CHECK();
  ++h.launches;
}

void scatter_from_nested(Handle& h, const double* src, double* dst, cudaStream_t st) {
  k_scatter<<<grid_for(h.n), TPB, 0, st>>>(h.n, h.perm.p, src, dst);
  MSP_LAUNCH_CHECK();
  ++h.launches;
}

void apply_L_nested(Handle& h, const double* x, double* y, cudaStream_t st) {
  launch_spmv<false>(h, x, y, st);
}

void apply_R_msp_nested(Handle& h, const double* r, double* z, cudaStream_t st) {
  msp_sweeps(h, r, z, st, 0);
}

// PCG (reading R10) on nested-numbered vectors b -> x.
void pcg_nested(Handle& h, int precond, const double* b, double* x, double rtol, int maxit,
                cudaStream_t st, msp_report* rep) {
  const int64_t n = h.n;
  const unsigned gv = std::min<unsigned>(grid_for(n), 148u * 8u);
  cudaEvent_t e0, e1;
  MSP_CUDA(cudaEventCreate(&e0));
  MSP_CUDA(cudaEventCreate(&e1));
  const int64_t launches0 = h.launches;
  MSP_CUDA(cudaEventRecord(e0, st));
  // x = 0, r = b, bb = (b, b)
  MSP_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  MSP_CUDA(cudaMemcpyAsync(h.vr.p, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  MSP_CUDA(cudaMemsetAsync(h.counters.p, 0, C_NCNT * sizeof(unsigned), st));
  double* bb = h.red.p + h.red_cap - 1;
  k_dot_part<<<gv, TPB, 0, st>>>(n, b, b, h.red.p, bb, h.counters.p);
  k_init_state<<<1, 1, 0, st>>>(h.scal.p, h.counters.p, rtol * rtol, bb);
  h.launches += 2;
  MSP_LAUNCH_CHECK();
  // z = R r, rho = (r, z), p = z
  if (precond == MSP_PRECOND_MSP) msp_sweeps(h, h.vr.p, h.vz.p, st, 1);
  else { k_copy_dot<<<gv, TPB, 0, st>>>(n, h.vr.p, h.vz.p, h.red.p, h.scal.p, h.counters.p, 1); ++h.launches; }
  k_pupdate<<<gv, TPB, 0, st>>>(n, h.vz.p, h.vp.p, h.scal.p, h.counters.p, 0);  // beta = 0
  ++h.launches;
  MSP_LAUNCH_CHECK();

  unsigned host_cnt[C_NCNT];
  const int check_every = h.profile ? 1 : 16;
  Prof P(h, st);
  int it = 0;
  while (it < maxit) {
    const int batch = std::min(check_every, maxit - it);
    for (int b2 = 0; b2 < batch; ++b2) {
      P.begin();
      launch_spmv<true>(h, h.vp.p, h.vq.p, st);                 // q = L p, alpha
      P.end(PC_SPMV);
      P.begin();
      k_update<<<gv, TPB, 0, st>>>(n, x, h.vr.p, h.vp.p, h.vq.p, h.red.p, h.scal.p, h.counters.p);
      P.end(PC_UPDATE);
      ++h.launches;
      if (precond == MSP_PRECOND_MSP) msp_sweeps(h, h.vr.p, h.vz.p, st, 2, &P);  // z = R r, beta
      else { k_copy_dot<<<gv, TPB, 0, st>>>(n, h.vr.p, h.vz.p, h.red.p, h.scal.p, h.counters.p, 2); ++h.launches; }
      P.begin();
      k_pupdate<<<gv, TPB, 0, st>>>(n, h.vz.p, h.vp.p, h.scal.p, h.counters.p, 1);
      P.end(PC_PUPD);
      ++h.launches;
      MSP_LAUNCH_CHECK();
    }
    it += batch;
    P.flush();
    MSP_CUDA(cudaMemcpyAsync(host_cnt, h.counters.p, sizeof(host_cnt), cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    if (host_cnt[C_DONE]) break;
  }
  MSP_CUDA(cudaEventRecord(e1, st));
  MSP_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  MSP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  double hs[S_NSCAL];
  MSP_CUDA(cudaMemcpy(hs, h.scal.p, sizeof(hs), cudaMemcpyDeviceToHost));
  MSP_CUDA(cudaMemcpy(host_cnt, h.counters.p, sizeof(host_cnt), cudaMemcpyDeviceToHost));
  if (rep) {
    rep->iterations = (int32_t)host_cnt[C_IT];
    rep->converged = host_cnt[C_DONE] ? 1 : 0;
    rep->relres = hs[S_BB] > 0 ? std::sqrt(hs[S_RR] / hs[S_BB]) : 0.0;
    if (hs[S_BB] == 0.0) rep->relres = 0.0;
    rep->solve_ms = ms;
    rep->kernel_launches = h.launches - launches0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace msp
