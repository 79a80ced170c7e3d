// solve.cu -- solve phase of the PEGP/MSP solver (sm_100a): apply_L, the
// exact MSP apply R = P(mu) L_T~^+ P(mu)^T, and fused PCG.
//
// Layout (nested numbering): level-k node i of the
// expanded graph lives at index off_k + i of every n~-vector; the children of
// level-(k+1) node B are level-k nodes cptr_k[B] .. cptr_k[B+1]-1, the first
// two being the matched pair, the rest leftovers.  Every aggregate of every
// level is a contiguous range of the level below, and so is every subtree:
// the MSP sweeps run as tiers of tile kernels (one CTA per tile of whole
// subtrees; all intermediate levels in shared memory, staged with TMA bulk
// copies), then one single-CTA kernel for the coarse levels Kc..L.
//
// Arithmetic of R r, with y_1 = r, y_{k+1} = P^T y_k
// (sums over children) and c(k) = sum_{j<k} (-mu)^j:
//   r~ = P(mu)^T r has level-k block (-mu)^{k-1} y_k, and its subtree sums in
//   T~ are s_k = c(k) y_k;
//   rho = c(L) sum(r) / n~ projects r~ off the ones vector;
//   top:   z_L = (sigma_L L_L)^+ (s_L - rho N_L), then shifted so that z~ has
//          zero mean: m = (N_L . z_L + gdot - rho GN) / n~ with
//          gdot = sum_{non-top} g_i s_i = (r, H);
//   down:  per aggregate, zeta = K_S^{-1} (s_S - rho N_S) (pair + leftover
//          elimination), z_c = z_B + zeta_c;
//   out:   w_L = z_L, w_k = z_k + (-mu) P w_{k+1}; R r = w_1.
//
// Every kernel of an iteration is launched with programmatic dependent launch
// (PDL): its prologue (tile ranges, shared-memory layout, TMA of constant
// data) overlaps the tail of the previous kernel; griddepcontrol.wait guards
// the first read of anything the previous kernel wrote.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include <nccl.h>

#include "internal.cuh"

namespace msp {

namespace {

constexpr int TPB = 256;      // SpMV and per-node kernels
#ifndef MSP_TT
#define MSP_TT 128
#endif
constexpr int TT = MSP_TT;
#ifndef MSP_UT
#define MSP_UT 256  // 128 / 256 / 512 measured on configs[1]: 65.2 / 64.2 / 64.7 us per iteration
#endif
constexpr int UT = MSP_UT;   // tile up kernels (threads per CTA)    // tile kernels (threads per CTA)
#ifndef MSP_PF_DIST
#define MSP_PF_DIST 1
#endif
#ifndef MSP_SPMV_LB
#define MSP_SPMV_LB 4  // min CTAs/SM of the pipelined SpMV (register budget)
#endif
#ifndef MSP_EARLY
#define MSP_EARLY 17  // measured: bit 1 (tier-2 up) -1.6 us, bit 16 (SpMV) -0.5 us; bits 2, 4, 8 neutral or worse
#endif
#ifndef MSP_FLAT_G
#define MSP_FLAT_G 8  // lanes per level-k1 node in the up kernels (2 / 4 / 8 / 16 / 32 measured; 8 best)
#endif
#ifndef MSP_CT
#define MSP_CT 1024
#endif
constexpr int CT = MSP_CT;    // coarse kernel (single CTA)

// device scalar slots
enum { S_RHO = 0, S_PQ, S_ALPHA, S_RR, S_GD, S_BETA, S_TOL2, S_BB, S_SHIFT, S_RTOL2, S_RZ, S_NSCAL };
// counter slots
enum { C_SPMV = 0, C_UPD, C_DOWN, C_DONE, C_IT, C_NCNT };
// sweep modes
enum { M_APPLY = 0, M_INIT = 1, M_ITER = 2, M_COLUMN = 3 };
// multi-GPU: local totals only (the caller all-reduces, k_dist_finish derives)
constexpr int M_DIST = 16;
// level-1 output z interleaved with p ([z_i, p_i] pairs, index 2i): the
// fused SpMV then gathers one 16-byte pair per neighbour
constexpr int M_ZS2 = 32;

// phase timestamps for kernel-structure work (build with -DMSP_TRACE; the
// in-tree library never defines it)
#ifdef MSP_TRACE
__device__ unsigned long long g_trace[8][16];
#define TRACE(tag)                                                                                  \
  do {                                                                                              \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                                                      \
      if ((tag) == 0) {                                                                             \
        unsigned long long t_;                                                                      \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
        g_trace[TRACE_KID][0] = t_;                                                                 \
        g_trace[TRACE_KID][14] = clock64();                                                         \
      } else {                                                                                      \
        g_trace[TRACE_KID][tag] = clock64(); /* SM cycles; slot 14 = cycles at tag 0 */            \
      }                                                                                             \
    }                                                                                               \
  } while (0)
// latest end over all CTAs (slot 15)
#define TRACE_END()                                                                                 \
  do {                                                                                              \
    if (threadIdx.x == 0) {                                                                         \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      atomicMax(&g_trace[TRACE_KID][15], t_);                                                       \
    }                                                                                               \
  } while (0)
// per-phase SM cycles summed over every CTA (thread 0): PHASE(k) adds the
// cycles since the previous PHASE call (or PHASE_START) to slot k
__device__ unsigned long long g_phase[8][16];
#define PHASE_START() long long ph_t_ = clock64()
#define PHASE(k)                                                                                    \
  do {                                                                                              \
    if (threadIdx.x == 0) {                                                                         \
      const long long t_ = clock64();                                                               \
      atomicAdd(&g_phase[TRACE_KID][k], (unsigned long long)(t_ - ph_t_));                          \
      ph_t_ = t_;                                                                                   \
    }                                                                                               \
  } while (0)
#else
#define TRACE(tag) do {} while (0)
#define TRACE_END() do {} while (0)
#define PHASE_START() do {} while (0)
#define PHASE(k) do {} while (0)
#endif
#define TRACE_KID 0

inline unsigned grid_for(int64_t n, int tpb = TPB) {
  int64_t g = (n + tpb - 1) / tpb;
  return (unsigned)std::max<int64_t>(g, 1);
}

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void tma_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// the same with an L2 evict-last policy: the solve's constant arrays
// (hierarchy pointers, factors) are re-read every iteration and should stay
// resident in the 126 MB L2 while the streamed vectors pass through it
__device__ __forceinline__ void tma_1d_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#ifndef MSP_NO_L2KEEP
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  tma_1d(dst, src, bytes, bar);
#endif
}

// bulk L2 prefetch of a 16-byte aligned range (no registers, no completion)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum, result valid in every thread
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

// block-wide sum of two values at once
template <int NT>
__device__ __forceinline__ double2 block_sum2(double2 v) {
  __shared__ double2 ws2[NT / 32];
  __shared__ double2 tot2;
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) ws2[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double2 t = (lane < NT / 32) ? ws2[lane] : make_double2(0.0, 0.0);
    t.x = warp_sum(t.x);
    t.y = warp_sum(t.y);
    if (lane == 0) tot2 = t;
  }
  __syncthreads();
  return tot2;
}

// deterministic sum of partials[0..n) written by other blocks (L2 reads)
template <int NT>
__device__ __forceinline__ double block_sum_partials(const double* part, int64_t n) {
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += NT) v += __ldcg(part + i);
  return block_sum<NT>(v);
}

// "last block done" ticket after thread 0 wrote this block's partial(s)
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
    if (is_last) __threadfence();
  }
  __syncthreads();
  return is_last;
}

// Warp-level ticket: lane 0 publishes this block's partial (already stored)
// and takes a ticket; true in every lane of the warp that arrives last.
__device__ __forceinline__ bool warp_last_block(unsigned int* counter) {
  unsigned last = 0;
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1) ? 1u : 0u;
    if (last) __threadfence();
  }
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

// fixed-order sum of partials[0..n) by one warp (all lanes get the result);
// four independent chains so the L2 loads overlap
__device__ __forceinline__ double warp_sum_partials(const double* part, int64_t n) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = threadIdx.x & 31;
  for (; i + 96 < n; i += 128) {
    a0 += __ldcg(part + i);
    a1 += __ldcg(part + i + 32);
    a2 += __ldcg(part + i + 64);
    a3 += __ldcg(part + i + 96);
  }
  for (; i < n; i += 32) a0 += __ldcg(part + i);
  return warp_sum((a0 + a1) + (a2 + a3));
}

// the same for two partial arrays at once (loads of both in flight together)
__device__ __forceinline__ double2 warp_sum_partials2(const double* pa, const double* pb, int64_t n) {
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  int64_t i = threadIdx.x & 31;
  for (; i + 32 < n; i += 64) {
    a0 += __ldcg(pa + i);
    b0 += __ldcg(pb + i);
    a1 += __ldcg(pa + i + 32);
    b1 += __ldcg(pb + i + 32);
  }
  for (; i < n; i += 32) { a0 += __ldcg(pa + i); b0 += __ldcg(pb + i); }
  return make_double2(warp_sum(a0 + a1), warp_sum(b0 + b1));
}

// Exact solve of one aggregate of T~: children [s0, s1) (matched pair s0,
// s0+1, leftovers s0+2..), K(j) the packed K'^{-1} (uu, uv, vv), C(p, j) the
// leftover coefficients (sigma w_xu / d, sigma w_xv / d, 1 / d):
// zeta = K_S^{-1} t, emitted as ef(p, z_B + zeta_p, z_B + zeta_p + wbm).
template <int UNR = 1, typename I, typename TF, typename KF, typename CF, typename EF>
__device__ __forceinline__ void block_solve(I s0, I s1, KF K, CF C, double zb, double wbm, TF tf, EF ef) {
  const double kuu = K(0), kuv = K(1), kvv = K(2);
  const double tu = tf(s0), tv = tf(s0 + 1);
  // (one code path for plain pairs and pairs with leftovers measured slower:
  // configs[2] tile_down 312 -> 342 us)
#ifndef MSP_BS_NO1
  if (s1 <= s0 + 3) {
    // a matched pair with at most one leftover (grids: ~99.5 % of the
    // aggregates; those with a leftover have one in ~95 % of the cases): one
    // straight-line path, the absent leftover's terms zero (tu + 0 * 0 = tu:
    // the same doubles as the separate pair branch), so a warp mixing the
    // two shapes does not serialize two paths
    const bool hx = s1 == s0 + 3;
    const double tx = hx ? tf(s0 + 2) : 0.0;
    const double c0 = hx ? C(s0 + 2, 0) : 0.0, c1 = hx ? C(s0 + 2, 1) : 0.0;
    const double au = tu + c0 * tx, av = tv + c1 * tx;
    const double zu = kuu * au + kuv * av, zv = kuv * au + kvv * av;
    { const double z = zb + zu; ef(s0, z, z + wbm); }
    { const double z = zb + zv; ef(s0 + 1, z, z + wbm); }
    if (hx) {
      const double zx = C(s0 + 2, 2) * tx + c0 * zu + c1 * zv;
      const double z = zb + zx;
      ef(s0 + 2, z, z + wbm);
    }
    return;
  }
#endif
  if (s1 == s0 + 2) {  // a matched pair without leftovers (the common case)
    const double zu = kuu * tu + kuv * tv, zv = kuv * tu + kvv * tv;
    { const double z = zb + zu; ef(s0, z, z + wbm); }
    { const double z = zb + zv; ef(s0 + 1, z, z + wbm); }
    return;
  }
  double au = tu, av = tv;
  #pragma unroll UNR
  for (I p = s0 + 2; p < s1; ++p) {
    const double tx = tf(p);
    au += C(p, 0) * tx;
    av += C(p, 1) * tx;
  }
  const double zu = kuu * au + kuv * av, zv = kuv * au + kvv * av;
  { const double z = zb + zu; ef(s0, z, z + wbm); }
  { const double z = zb + zv; ef(s0 + 1, z, z + wbm); }
  #pragma unroll UNR
  for (I p = s0 + 2; p < s1; ++p) {
    const double tx = tf(p);
    const double zx = C(p, 2) * tx + C(p, 0) * zu + C(p, 1) * zv;
    const double z = zb + zx;
    ef(p, z, z + wbm);
  }
}

// sum_e w_e (pi - p(col_e)) over e = e0 + sub, e0 + sub + S, ... < e1 with
// four independent chains (the column and gather loads of four entries are
// in flight together: long rows are latency bound otherwise).  (A
// predicated last group instead of the scalar tail measured no faster on
// configs[4].)
template <int S, typename PJ>
__device__ __forceinline__ double row_dot(const int32_t* __restrict__ col, const double* __restrict__ w, int32_t e0,
                                          int32_t e1, int sub, double pi, PJ pj) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  // the row's columns and weights are streamed once per product: evict-first,
  // so the gathered vectors (and the hot-vertex cache) keep the L2
  int32_t e = e0 + sub;
  for (; e + 3 * S < e1; e += 4 * S) {
    const int32_t j0 = __ldcs(col + e), j1 = __ldcs(col + e + S), j2 = __ldcs(col + e + 2 * S),
                  j3 = __ldcs(col + e + 3 * S);
    const double w0 = __ldcs(w + e), w1 = __ldcs(w + e + S), w2 = __ldcs(w + e + 2 * S), w3 = __ldcs(w + e + 3 * S);
    a0 += w0 * (pi - pj(j0));
    a1 += w1 * (pi - pj(j1));
    a2 += w2 * (pi - pj(j2));
    a3 += w3 * (pi - pj(j3));
  }
  for (; e < e1; e += S) a0 += __ldcs(w + e) * (pi - pj(__ldcs(col + e)));
  return (a0 + a1) + (a2 + a3);
}

// Huge-row segment s of huge row hr done with block sum acc (thread 0): true
// in the CTA that completes the row, with the row total (partials summed in
// segment order, so the result does not depend on arrival order)
__device__ __forceinline__ bool huge_last(const HugeDesc& hd, int hr, int64_t s, double acc, double* tot) {
  hd.part[s] = acc;
  __threadfence();
  const int f0 = hd.first[hr], f1 = hd.first[hr + 1];
  const unsigned t = atomicAdd(&hd.cnt[hr], 1u);
  if (t != (unsigned)(f1 - f0 - 1)) return false;
  __threadfence();
  double a = 0.0;
  for (int k = f0; k < f1; ++k) a += __ldcg(hd.part + k);
  hd.cnt[hr] = 0;
  *tot = a;
  return true;
}

// (p, q) terms of the huge rows (one warp, fixed row order; a distributed
// rank's own rows only)
__device__ __forceinline__ double huge_dot_sum(const HugeDesc& hd, const int32_t* __restrict__ long_rows,
                                              int64_t nlong, int64_t row0, int64_t row1) {
  double a = 0.0;
  for (int64_t i = threadIdx.x & 31; i < hd.nhuge; i += 32) {
    const int64_t r = long_rows[nlong + i];
    if (r >= row0 && r < row1) a += __ldcg(hd.dot + i);
  }
  return warp_sum(a);
}

// PCG scalars after the level-1 output: rz = (r, R r)
__device__ __forceinline__ void finish_rz(double rz, double* scal, int mode) {
  if (mode == M_ITER) scal[S_BETA] = rz / scal[S_RHO];
  else scal[S_BETA] = 0.0;
  scal[S_RHO] = rz;
}

// (r, r) and the convergence test (reading R10)
__device__ __forceinline__ void finish_rr(double rr, double* scal, unsigned* cnt, int mode) {
  scal[S_RR] = rr;
  if (mode == M_INIT) {
    scal[S_BB] = rr;
    scal[S_TOL2] = scal[S_RTOL2] * rr;
  } else {
    cnt[C_IT] += 1;
  }
  if (rr <= scal[S_TOL2]) cnt[C_DONE] = 1;
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
// y_i = sum_j w_ij (x_i - x_j)   (L_G = B^T W B, §2.1), SELL-32.
// PCG: p = z + beta p_old (rows and gathered neighbours alike), q = L_G p,
// (p, q) -> alpha = rho / (p, q); and the deferred x += alpha_prev p_old.
#ifndef MSP_SPMV_MINB
#define MSP_SPMV_MINB 8
#endif
template <bool PCG>
__global__ void __launch_bounds__(TPB, MSP_SPMV_MINB) k_spmv(int64_t n, int64_t nslices, const int64_t* __restrict__ sptr,
                                              const int32_t* __restrict__ scol, const double* __restrict__ sw,
                                              const uint32_t* __restrict__ smask, int64_t nlong, const HugeDesc hd,
                                              const int32_t* __restrict__ long_rows,
                                              const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                              const double* __restrict__ w, const double* __restrict__ z,
                                              const double* __restrict__ pold, double* __restrict__ pnew,
                                              double* __restrict__ q, double* __restrict__ x,
                                              double* __restrict__ part, double* __restrict__ scal,
                                              unsigned int* __restrict__ cnt, int64_t row0, int64_t row1) {
  pdl_wait();
  if (PCG && cnt[C_DONE]) return;
  const double beta = PCG ? scal[S_BETA] : 0.0;
  const double alpha = PCG ? scal[S_ALPHA] : 0.0;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)TPB + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * TPB) >> 5;
  double d = 0.0;
  const int64_t s_begin = row0 >> 5, s_end = (row1 + 31) >> 5;
  for (int64_t s = s_begin + warp; s < s_end; s += nwarps) {
    const int64_t r = s * 32 + lane;
    const bool valid = r < n && r >= row0 && r < row1;
    const bool lng = (smask[s] >> lane) & 1u;
    const int64_t base = sptr[s];
    const int width = (int)((sptr[s + 1] - base) >> 5);
    double pi = 0.0, po = 0.0;
    if (valid) {
      if (PCG) { po = pold[r]; pi = z[r] + beta * po; }
      else pi = z[r];
    }
    double acc = 0.0;
#pragma unroll 4
    for (int k = 0; k < width; ++k) {
      const int64_t idx = base + k * 32 + lane;
      const int32_t j = scol[idx];
      const double pj = PCG ? z[j] + beta * pold[j] : z[j];
      acc += sw[idx] * (pi - pj);
    }
    if (valid && !lng) {
      q[r] = acc;
      if (PCG) {
        pnew[r] = pi;
        x[r] += alpha * po;
        d += pi * acc;
      }
    }
  }
  for (int64_t i = warp; i < nlong; i += nwarps) {  // warp per long row
    const int64_t r = long_rows[i];
    if (r < row0 || r >= row1) continue;
    const double po = PCG ? pold[r] : 0.0;
    const double pi = PCG ? z[r] + beta * po : z[r];
    double acc = row_dot<32>(col, w, rowptr[r], rowptr[r + 1], lane, pi,
                             [&](int32_t j) { return PCG ? z[j] + beta * pold[j] : z[j]; });
    acc = warp_sum(acc);
    if (lane == 0) {
      q[r] = acc;
      if (PCG) {
        pnew[r] = pi;
        x[r] += alpha * po;
        d += pi * acc;
      }
    }
  }
  for (int64_t s = blockIdx.x; s < hd.nseg; s += gridDim.x) {  // CTA per huge-row segment
    const int4 sg = hd.seg[s];
    const int64_t r = long_rows[nlong + sg.x];
    if (r < row0 || r >= row1) continue;  // block-uniform
    const double po = PCG ? pold[r] : 0.0;
    const double pi = PCG ? z[r] + beta * po : z[r];
    double acc = row_dot<TPB>(col, w, sg.y, sg.z, threadIdx.x, pi,
                              [&](int32_t j) { return PCG ? z[j] + beta * pold[j] : z[j]; });
    acc = block_sum<TPB>(acc);
    double tot;
    if (threadIdx.x == 0 && huge_last(hd, sg.x, s, acc, &tot)) {
      q[r] = tot;
      if (PCG) {
        pnew[r] = pi;
        x[r] += alpha * po;
        hd.dot[sg.x] = pi * tot;  // summed in row order at the end
      }
    }
  }
  if (!PCG) return;
  pdl_trigger();
  const double bs = block_sum<TPB>(d);
  if (threadIdx.x < 32) {  // only warp 0 waits on the ticket
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (warp_last_block(&cnt[C_SPMV])) {
      const double pq = warp_sum_partials(part, gridDim.x) + huge_dot_sum(hd, long_rows, nlong, row0, row1);
      if (threadIdx.x == 0) {
        scal[S_PQ] = pq;
        scal[S_ALPHA] = scal[S_RHO] / pq;
        cnt[C_SPMV] = 0;
      }
    }
  }
}


// Software-pipelined SELL SpMV for slices no wider than MW (fused PCG form):
// while slice s is gathered and reduced, the slice pointers of s+2 and the
// column / weight / row vectors of s+1 are already in flight.
#undef TRACE_KID
#define TRACE_KID 6
// hot-vertex cache fill (power-law graphs, setup.cu build_hot_cache): the
// (z, p_old) pairs of the nhot highest-degree rows, copied into one compact
// L2-resident array before the SpMV gathers them
__global__ void k_hot_gather(int64_t nhot, const int32_t* __restrict__ rows, const double2* __restrict__ zp,
                             double2* __restrict__ hot, const unsigned* __restrict__ cnt) {
  pdl_wait();
  if (cnt[C_DONE]) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nhot; k += (int64_t)gridDim.x * blockDim.x)
    hot[k] = zp[rows[k]];
}

template <int MW, bool UNIF, bool SEP = false, bool HOT = false>
__global__ void __launch_bounds__(TPB, MSP_SPMV_LB) k_spmv_pipe(int64_t n, int64_t nslices, const int64_t* __restrict__ sptr,
                                                      const int32_t* __restrict__ scol, const double* __restrict__ sw,
                                                      const uint32_t* __restrict__ smask, int64_t nlong, const HugeDesc hd,
                                                      const int32_t* __restrict__ long_rows,
                                                      const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                      const double* __restrict__ w, const double2* __restrict__ zp,
                                                      double* __restrict__ zpout,
                                                      double* __restrict__ q, double* __restrict__ x,
                                                      double* __restrict__ part, double* __restrict__ scal,
                                                      unsigned int* __restrict__ cnt, int64_t row0, int64_t row1,
                                                      const double* __restrict__ zs, const double* __restrict__ ps,
                                                      double* __restrict__ pn, int64_t nmed,
                                                      const double2* __restrict__ hot) {
  // pairs (!SEP): zp[i] = (z_i, p_old_i), the new p_i goes to zpout[2 i + 1];
  // SEP: z, p_old and the new p in three plain vectors zs, ps, pn (every
  // store a full sector: no L2 fill of a half-written pair line).  Rows
  // [row0, row1) only (a rank's own rows; all of them on one GPU)
  auto zpj = [&](int64_t j) -> double2 {
    if (SEP) return make_double2(zs[j], ps[j]);
    return zp[j];
  };
  // a gathered neighbour: HOT columns with HOT_BIT read the cache
  uint64_t keep_pol = 0;
  if (HOT) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep_pol));
  auto zpg = [&](int32_t j) -> double2 {
    if (HOT && (j & HOT_BIT)) {  // the hot-vertex cache, kept resident in L2 (evict-last)
      double2 v;
      asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                   : "=d"(v.x), "=d"(v.y)
                   : "l"(hot + (j & (HOT_BIT - 1))), "l"(keep_pol));
      return v;
    }
    return zpj(j);
  };
  auto put_p = [&](int64_t r, double v) {
    if (SEP) pn[r] = v;
    else zpout[2 * r + 1] = v;
  };
  if ((MSP_EARLY & 16) != 0) pdl_trigger();
  TRACE(0);
#ifdef MSP_SPMV_PF_PRE  // off since the SpMV launches without PDL (configs[1] 61.7 -> 61.4 us/iteration)
  if (UNIF && (threadIdx.x & 31) == 0) {  // constant streams of the first slices, before the dependency
    const int64_t w0 = (blockIdx.x * (int64_t)TPB + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * TPB) >> 5;
    for (int64_t sp = w0; sp < nslices && sp <= w0 + nw; sp += nw) {
      l2_prefetch(scol + sp * 32 * MW, 32 * MW * 4);
      l2_prefetch(sw + sp * 32 * MW, 32 * MW * 8);
    }
  }
#endif
  pdl_wait();
  TRACE(1);
  if (cnt[C_DONE]) return;
  const double beta = scal[S_BETA];
  const double alpha = scal[S_ALPHA];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)TPB + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * TPB) >> 5;
  double d = 0.0;
  // stage A (slice s): pointers; stage B (slice s): columns, weights, own row
  const int64_t s_end = (row1 + 31) >> 5;
  int64_t s = (row0 >> 5) + warp;
  int64_t b0 = 0, b1 = 0;
  if (UNIF) { b0 = s * 32 * MW; b1 = b0 + 32 * MW; }
  else if (s < s_end) { b0 = sptr[s]; b1 = sptr[s + 1]; }
  int32_t jc[MW];
  double wc[MW];
  double po = 0.0, zr = 0.0;
  uint32_t mk = 0;
  auto load_B = [&](int64_t ss, int64_t bb0, int64_t bb1) {
    const int wd = UNIF ? MW : (int)((bb1 - bb0) >> 5);
    const int64_t r = ss * 32 + lane;
#pragma unroll
    for (int k = 0; k < MW; ++k) {
      if (k < wd) {
#ifndef MSP_NO_SPMV_CS  // streamed once per iteration: evict-first, so the
                        // vectors the next kernels re-read stay in L2
        jc[k] = __ldcs(scol + bb0 + k * 32 + lane);
        wc[k] = __ldcs(sw + bb0 + k * 32 + lane);
#else
        jc[k] = scol[bb0 + k * 32 + lane];
        wc[k] = sw[bb0 + k * 32 + lane];
#endif
      }
    }
    mk = smask[ss];
    if (r < n) { const double2 v = zpj(r); zr = v.x; po = v.y; }
  };
  if (s < s_end) load_B(s, b0, b1);
  while (s < s_end) {
    const int64_t s1 = s + nwarps;
#if MSP_PF_DIST > 0
    if (UNIF && lane == 0) {  // the streams of slice s + PF * nwarps into L2
      const int64_t sp = s + MSP_PF_DIST * nwarps;
      if ((sp + 1) * 32 <= n) {
        l2_prefetch(scol + sp * 32 * MW, 32 * MW * 4);
        l2_prefetch(sw + sp * 32 * MW, 32 * MW * 8);
        if (SEP) {
          l2_prefetch(zs + sp * 32, 32 * 8);
          l2_prefetch(ps + sp * 32, 32 * 8);
        } else {
          l2_prefetch(zp + sp * 32, 32 * 16);
        }
        l2_prefetch(x + sp * 32, 32 * 8);
      }
    }
#endif
    int64_t n0 = 0, n1 = 0;
    if (UNIF) { n0 = s1 * 32 * MW; n1 = n0 + 32 * MW; }
    else if (s1 < s_end) { n0 = sptr[s1]; n1 = sptr[s1 + 1]; }  // next pointers, in flight
    // current slice: gathers and reduction
    const int wd = UNIF ? MW : (int)((b1 - b0) >> 5);
    const int64_t r = s * 32 + lane;
    const double pi = zr + beta * po;
    double g[MW];
#pragma unroll
    for (int k = 0; k < MW; ++k)
      if (k < wd) {
        const double2 v = zpg(jc[k]);
        g[k] = v.x + beta * v.y;
      }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < MW; ++k)
      if (k < wd) acc += wc[k] * (pi - g[k]);
    if (r < row1 && r >= row0 && !((mk >> lane) & 1u)) {
      q[r] = acc;
      put_p(r, pi);
#ifndef MSP_NO_X_CS
      __stcs(x + r, __ldcs(x + r) + alpha * po);
#else
      x[r] += alpha * po;
#endif
      d += pi * acc;
    }
    // next slice's columns / weights / row vectors
    s = s1;
    b0 = n0;
    b1 = n1;
    if (s < s_end) load_B(s, b0, b1);
  }
  {  // medium rows: 8 lanes per row, four rows per warp (warp-uniform trip count)
    constexpr int MG = 8;
    const int sub = lane & (MG - 1);
    for (int64_t base = warp * (32 / MG); base < nmed; base += nwarps * (32 / MG)) {
      const int64_t i = base + lane / MG;
      const bool ok = i < nmed;
      const int64_t r = ok ? long_rows[i] : 0;
      const bool mine = ok && r >= row0 && r < row1;
      double pi = 0.0, pr = 0.0, xr = 0.0, acc = 0.0;
      if (mine) {
        const double2 vr = zpj(r);
        pr = vr.y;
        pi = vr.x + beta * pr;
        if (sub == 0) xr = x[r];
        acc = row_dot<MG>(col, w, rowptr[r], rowptr[r + 1], sub, pi, [&](int32_t j) {
          const double2 v = zpg(j);
          return v.x + beta * v.y;
        });
      }
#pragma unroll
      for (int o = MG / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (mine && sub == 0) {
        q[r] = acc;
        put_p(r, pi);
        x[r] = xr + alpha * pr;
        d += pi * acc;
      }
    }
  }
  for (int64_t i = nmed + warp; i < nlong; i += nwarps) {  // warp per long row
    const int64_t r = long_rows[i];
    if (r < row0 || r >= row1) continue;
    const double2 vr = zpj(r);
    const double pr = vr.y;
    const double pi = vr.x + beta * pr;
    const double xr = (lane == 0) ? x[r] : 0.0;  // in flight with the row
    double acc = row_dot<32>(col, w, rowptr[r], rowptr[r + 1], lane, pi, [&](int32_t j) {
      const double2 v = zpg(j);
      return v.x + beta * v.y;
    });
    acc = warp_sum(acc);
    if (lane == 0) {
      q[r] = acc;
      put_p(r, pi);
      x[r] = xr + alpha * pr;
      d += pi * acc;
    }
  }
  for (int64_t s = blockIdx.x; s < hd.nseg; s += gridDim.x) {  // CTA per huge-row segment
    const int4 sg = hd.seg[s];
    const int64_t row = long_rows[nlong + sg.x];
    if (row < row0 || row >= row1) continue;  // block-uniform
    const double2 vr = zpj(row);
    const double pr = vr.y;
    const double pi = vr.x + beta * pr;
    double acc = row_dot<TPB>(col, w, sg.y, sg.z, threadIdx.x, pi, [&](int32_t j) {
      const double2 v = zpg(j);
      return v.x + beta * v.y;
    });
    acc = block_sum<TPB>(acc);
    double tot;
    if (threadIdx.x == 0 && huge_last(hd, sg.x, s, acc, &tot)) {
      q[row] = tot;
      put_p(row, pi);
      x[row] += alpha * pr;
      hd.dot[sg.x] = pi * tot;  // summed in row order at the end
    }
  }
  TRACE(2);
  pdl_trigger();
  const double bs = block_sum<TPB>(d);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (warp_last_block(&cnt[C_SPMV])) {
      const double pq = warp_sum_partials(part, gridDim.x) + huge_dot_sum(hd, long_rows, nlong, row0, row1);
      if (threadIdx.x == 0) {
        scal[S_PQ] = pq;
        scal[S_ALPHA] = scal[S_RHO] / pq;
        cnt[C_SPMV] = 0;
      }
    }
  }
  TRACE_END();
}

// x += alpha p for the last direction (the in-loop updates are deferred into
// the next L p); p is the buffer the C_IT-th product wrote
__global__ void k_x_final(int64_t n, double* __restrict__ x, const double* __restrict__ vp,
                          const double* __restrict__ vp2, const double* __restrict__ scal,
                          const unsigned* __restrict__ cnt) {
  pdl_wait();
  const unsigned it = cnt[C_IT];
  if (it == 0) return;
  const double* p = (it & 1u) ? vp2 : vp;
  const double alpha = scal[S_ALPHA];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += alpha * p[i];
}

// per-level shared-memory pointers of a tile / of the coarse levels
// (byte offsets from the dynamic shared-memory base, so the compiler keeps
// shared-space loads; -1 = absent)
struct LvlPtr {
  int cp;            // child pointers of this level's nodes (as parents)
  int ki;            // K'^{-1} triples of this level's aggregates
  int lo;            // leftover triples of this level's nodes (as children)
  int y, nn, z, w;
  int a, cnt;        // first node, node count
  double ck;         // c(k)
};
#define SMP(T, off) reinterpret_cast<T*>(sm + (off))

// ------------------------------------------------------------ tile staging
// Stage [lo, hi) of a global array (absolute element indices, element size
// es = 4 or 8) into shared memory at dst with one TMA bulk copy; the window
// starts at the 16-byte-aligned element at or below lo.  Returns the skew
// lo - window start (elements).  Called by one thread per segment; the
// barrier's single arrival comes after every segment's expect_tx.
template <bool KEEP = false>
__device__ __forceinline__ int stage_window(uint64_t* bar, char* dst, const void* src, int es, int64_t lo,
                                            int64_t hi) {
  const int64_t m = (es == 4) ? 3 : 1;
  const int64_t a0 = lo & ~m;
  if (hi > lo) {
    const int64_t e0 = (hi + m) & ~m;
    const uint32_t bytes = (uint32_t)((e0 - a0) * es);
    mbar_expect_tx(bar, bytes);
    if (KEEP) tma_1d_keep(dst, (const char*)src + a0 * es, bytes, bar);
    else tma_1d(dst, (const char*)src + a0 * es, bytes, bar);
  }
  return (int)(lo - a0);
}

// same for the interleaved (z, p) pairs: iteration k writes p into the
// buffer of parity k & 1
__global__ void k_x_final_pairs(int64_t n, double* __restrict__ x, const double* __restrict__ zp1,
                                const double* __restrict__ zp2, const double* __restrict__ scal,
                                const unsigned* __restrict__ cnt) {
  pdl_wait();
  const unsigned it = cnt[C_IT];
  if (it == 0) return;
  const double* zp = (it & 1u) ? zp2 : zp1;
  const double alpha = scal[S_ALPHA];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += alpha * zp[2 * i + 1];
}

// ------------------------------------------------------------ tile up-sweep
// Tier k0..k1, one CTA per tile.  FIRST (k0 == 1): level 1 is the PCG update
// r -= alpha q (mode ITER) with (r, r) and gdot = (r, H); otherwise y_k0 is
// staged from Y.  y_k1 = (P^T)^{k1-k0} y_k0 is formed directly, each level-k1
// node summing its contiguous range of level-k0 descendants (one warp per
// node), and written to global Y.
#undef TRACE_KID
#define TRACE_KID (FIRST ? 4 : 5)
template <bool FIRST>
__global__ void __launch_bounds__(UT) k_tile_up(const __grid_constant__ Lv lv, const __grid_constant__ TierDesc td,
                                                const int32_t* __restrict__ tstart, const int32_t* __restrict__ firstk0,
                                                const double* __restrict__ q, double* __restrict__ r,
                                                const double* __restrict__ H, double* __restrict__ Yg,
                                                double* __restrict__ part_rr, double* __restrict__ part_gd,
                                                double* __restrict__ scal, unsigned int* __restrict__ cnt, int mode_in,
                                                int tile0) {
  const int mode = mode_in & 15;
  const bool dist = (mode_in & M_DIST) != 0;
  extern __shared__ __align__(16) char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int sa0, sn0, sa1, sn1, skf, sky0, sdone, skr, skq, skh;
  __shared__ double salpha;
  // this CTA's tiles [tA, tB): `group` consecutive tiles (1 when distributed)
  const int grp = td.up_group;
  const int tA = tile0 + blockIdx.x * grp, tB = min(tA + grp, td.ntiles);
  const int tile = blockIdx.x;  // partial-sum slot
  const int nl = td.nl, k0 = td.k0, nt1 = td.ntiles + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // early trigger (MSP_EARLY bit 1: tier >= 2 up, bit 2: first-tier up): the
  // next kernel's CTAs may launch and stage their constants now; its
  // griddepcontrol.wait still waits for this whole grid
  if ((FIRST ? (MSP_EARLY & 2) : (MSP_EARLY & 1)) != 0) pdl_trigger();
  TRACE(0);
  PHASE_START();
  if (tid == 0) {
    mbar_init(&bar, 1);
    sa0 = tstart[tA];
    sn0 = tstart[tB] - sa0;
    if (nl > 1) {
      sa1 = tstart[(nl - 1) * nt1 + tA];
      sn1 = tstart[(nl - 1) * nt1 + tB] - sa1;
      skf = stage_window<true>(&bar, sm + td.o_uf, firstk0, 4, sa1, (int64_t)sa1 + sn1 + 1);
    }
    // FIRST: the level-1 H (constant) and, in PCG iterations, r (last written
    // by the previous iteration's up kernel) are staged before the grid
    // dependency resolves; q after it
    if (FIRST && sn0 > 0) {
      skh = stage_window<true>(&bar, sm + td.o_uh, H, 8, sa0, (int64_t)sa0 + sn0);
      if (mode == M_ITER) skr = stage_window(&bar, sm + td.o_uy0, r, 8, sa0, (int64_t)sa0 + sn0);
    }
  }
  TRACE(1);
  PHASE(0);
  pdl_wait();
  TRACE(2);
  PHASE(1);
  if (tid == 0) {
    sdone = (mode == M_ITER) ? (int)cnt[C_DONE] : 0;
    salpha = (mode == M_ITER) ? scal[S_ALPHA] : 0.0;
    if (!FIRST && !sdone) {
      const int64_t base = lv.off[k0 - 1];
      sky0 = stage_window(&bar, sm + td.o_uy0, Yg, 8, base + sa0, base + sa0 + sn0);
    }
    if (FIRST && sn0 > 0) {
      if (mode == M_ITER) skq = stage_window(&bar, sm + td.o_uq, q, 8, sa0, (int64_t)sa0 + sn0);
      else skr = stage_window(&bar, sm + td.o_uy0, r, 8, sa0, (int64_t)sa0 + sn0);
    }
    mbar_arrive(&bar);
  }
  __syncthreads();
  const int done = sdone;
  double rr = 0.0, gd = 0.0;
  double* y0 = reinterpret_cast<double*>(sm + td.o_uy0);
  TRACE(3);
  mbar_wait(&bar, 0);
  TRACE(4);
  PHASE(2);
  if (done) return;
  constexpr int FG = MSP_FLAT_G;
  const int sub = tid & (FG - 1);
  if (FIRST && nl > 1) {
    // one pass: FG lanes per level-k1 node update its level-1 descendants
    // (r -= alpha q), accumulate (r, r), (H, r) and the node's sum y_k1
    const double alpha = salpha;
    const int a1 = sa0, np = sn1;
    double* rs = y0 + skr;
    const double* qs = reinterpret_cast<const double*>(sm + td.o_uq) + skq;
    const double* hs = reinterpret_cast<const double*>(sm + td.o_uh) + skh;
    const int* f = reinterpret_cast<const int*>(sm + td.o_uf) + skf;
    double* yp = Yg + lv.off[k0 + nl - 2] + sa1;
    #pragma unroll 1
    for (int base = 0; base < np; base += UT / FG) {  // block-uniform trip count
      const int i = base + tid / FG;
      double y = 0.0;
      if (i < np) {
        const int c1 = f[i + 1] - a1;
        #pragma unroll 1
        for (int c = f[i] - a1 + sub; c < c1; c += FG) {
          double ri = rs[c];
          if (mode == M_ITER) {
            ri -= alpha * qs[c];
            r[a1 + c] = ri;
          }
          rr += ri * ri;
          gd += hs[c] * ri;
          y += ri;
        }
      }
#pragma unroll
      for (int o = FG / 2; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (sub == 0 && i < np) yp[i] = y;
    }
    PHASE(3);
  } else if (FIRST) {  // a level-1-only tier: the update alone
    const double alpha = salpha;
    const int a1 = sa0, n1 = sn0;
    double* rs = y0 + skr;
    const double* qs = reinterpret_cast<const double*>(sm + td.o_uq) + skq;
    const double* hs = reinterpret_cast<const double*>(sm + td.o_uh) + skh;
    for (int i = tid; i < n1; i += UT) {
      double ri = rs[i];
      if (mode == M_ITER) {
        ri -= alpha * qs[i];
        r[a1 + i] = ri;
      }
      rr += ri * ri;
      gd += hs[i] * ri;
    }
    PHASE(3);
  } else if (nl > 1) {
    const int* f = reinterpret_cast<const int*>(sm + td.o_uf) + skf;
    const double* yc = y0 + sky0;
    const int a0 = sa0, np = sn1;
    double* yp = Yg + lv.off[k0 + nl - 2] + sa1;
    // FG lanes per level-k1 node, two partial sums per lane, then a
    // butterfly over the group (fixed order)
    for (int base = 0; base < np; base += UT / FG) {  // block-uniform trip count
      const int i = base + tid / FG;
      double ya = 0.0, yb = 0.0;
      if (i < np) {
        const int c0 = f[i] - a0, c1 = f[i + 1] - a0;
        int c = c0 + sub;
        for (; c + FG < c1; c += 2 * FG) { ya += yc[c]; yb += yc[c + FG]; }
        if (c < c1) ya += yc[c];
      }
      double y = ya + yb;
#pragma unroll
      for (int o = FG / 2; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (sub == 0 && i < np) yp[i] = y;
    }
  }
  TRACE(5);
  PHASE(4);
  pdl_trigger();
  if (FIRST) {
    const double2 v = block_sum2<UT>(make_double2(rr, gd));
    TRACE(6);
    PHASE(5);
    if (tid < 32) {  // only warp 0 waits on the ticket
      if (tid == 0) { part_rr[tile] = v.x; part_gd[tile] = v.y; }
      if (mode != M_APPLY && warp_last_block(&cnt[C_UPD])) {
        const double2 t2 = warp_sum_partials2(part_rr + tile0, part_gd + tile0, gridDim.x);
        const double tot = t2.x, tgd = t2.y;  // (r, r); (H, r) for the coarse levels
        if (dist) {  // local totals; k_dist_finish runs after the all-reduce
          if (tid == 0) { scal[S_RR] = tot; scal[S_GD] = tgd; cnt[C_UPD] = 0; }
        } else if (tid == 0) {
          scal[S_GD] = tgd;
          finish_rr(tot, scal, cnt, mode);
          cnt[C_UPD] = 0;
        }
      }
    }
    TRACE(7);
    PHASE(6);
  }
#ifdef MSP_TRACE
  if (threadIdx.x == 0) atomicAdd(&g_phase[TRACE_KID][15], 1ull);
#endif
  TRACE_END();
}

// ------------------------------------------------- first-tier up, streamed
// The first tier's up sweep as a plain stream (no staging): FG lanes per
// level-k1 node, each lane loading r, q, H of four of the node's level-1
// descendants at a time straight from global memory, so every lane keeps 12
// independent loads in flight and the grid (a few CTAs per SM, striding over
// the nodes) stays balanced.  Per node: r -= alpha q (mode ITER), the node's
// sum y_k1; per CTA: (r, r) and gdot = (H, r) partials, last-CTA ticket.
// FLAT: a level-1-only tier (no y), one element per lane and step.
template <bool FLAT>
__global__ void __launch_bounds__(UT) k_up_stream(int64_t nnodes, const int32_t* __restrict__ f, int64_t n1,
                                                  const double* __restrict__ q, double* __restrict__ r,
                                                  const double* __restrict__ H, double* __restrict__ yk1,
                                                  double* __restrict__ part_rr, double* __restrict__ part_gd,
                                                  double* __restrict__ scal, unsigned int* __restrict__ cnt, int mode) {
  constexpr int FG = MSP_FLAT_G;
  constexpr int U = 4;  // elements per lane in flight
  mode &= 15;
  const int sub = threadIdx.x & (FG - 1);
  const int64_t base0 = (int64_t)blockIdx.x * (UT / FG);
  pdl_wait();
  if (mode == M_ITER && cnt[C_DONE]) return;  // uniform
  const double alpha = (mode == M_ITER) ? scal[S_ALPHA] : 0.0;
  const bool upd = (mode == M_ITER);
  double rr = 0.0, gd = 0.0;
  auto elem = [&](int64_t c, double rv, double qv, double hv, double& y) {
    double ri = rv;
    if (upd) {
      ri -= alpha * qv;
      r[c] = ri;
    }
    rr += ri * ri;
    gd += hv * ri;
    y += ri;
  };
  if (FLAT) {
    const int64_t T = (int64_t)gridDim.x * UT;
    double y = 0.0;
    for (int64_t c0 = (int64_t)blockIdx.x * UT + threadIdx.x; c0 < n1; c0 += U * T) {
      double rv[U], qv[U], hv[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t c = c0 + k * T;
        if (c < n1) { rv[k] = r[c]; qv[k] = upd ? __ldcs(q + c) : 0.0; hv[k] = H[c]; }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t c = c0 + k * T;
        if (c < n1) elem(c, rv[k], qv[k], hv[k], y);
      }
    }
  } else {
    const int64_t ngrp = (int64_t)gridDim.x * UT / FG;
    // block-uniform trip count (the groups of a warp shuffle together)
    for (int64_t b = base0; b < nnodes; b += ngrp) {
      const int64_t i = b + (threadIdx.x / FG);
      double y = 0.0;
      if (i < nnodes) {
        const int64_t e0 = f[i], e1 = f[i + 1];
        for (int64_t c0 = e0 + sub; c0 < e1; c0 += U * FG) {
          double rv[U], qv[U], hv[U];
#pragma unroll
          for (int k = 0; k < U; ++k) {
            const int64_t c = c0 + k * FG;
            if (c < e1) { rv[k] = r[c]; qv[k] = upd ? __ldcs(q + c) : 0.0; hv[k] = H[c]; }
          }
#pragma unroll
          for (int k = 0; k < U; ++k) {
            const int64_t c = c0 + k * FG;
            if (c < e1) elem(c, rv[k], qv[k], hv[k], y);
          }
        }
      }
#pragma unroll
      for (int o = FG / 2; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
      if (sub == 0 && i < nnodes) yk1[i] = y;
    }
  }
  pdl_trigger();
  const double2 v = block_sum2<UT>(make_double2(rr, gd));
  if (threadIdx.x < 32) {  // only warp 0 waits on the ticket
    if (threadIdx.x == 0) { part_rr[blockIdx.x] = v.x; part_gd[blockIdx.x] = v.y; }
    if (mode != M_APPLY && warp_last_block(&cnt[C_UPD])) {
      const double2 t2 = warp_sum_partials2(part_rr, part_gd, gridDim.x);
      if (threadIdx.x == 0) {
        scal[S_GD] = t2.y;
        finish_rr(t2.x, scal, cnt, mode);
        cnt[C_UPD] = 0;
      }
    }
  }
}

// --------------------------------------------------------- coarse kernel
// Levels Kc..L of the coarse kernel when the top has <= 32 nodes.  Level t
// (n_{Kc+t} nodes, one per thread) runs on its first W(t) = ceil(n/32) warps
// only; the barrier before a level spans exactly the warps of the larger of
// the two levels it separates (a named barrier, __syncwarp for one warp), so
// the small upper levels cost a warp-level sync instead of a 32-warp one.  The
// top solve runs on warp 0.  Level Kc goes straight to global memory.
// Barrier ids: 1 for the up sweep (its warp sets only shrink, so every warp
// of an instance has left the previous one); one id per down level (2 + t),
// because a warp that joins the down sweep late arrives at its first barrier
// while the others are still levels above.
__device__ __forceinline__ void named_sync(int id, int nw) {
  if (nw == 1) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nw * 32) : "memory");
}

#undef TRACE_KID
#define TRACE_KID 1
__device__ __forceinline__ void coarse_levels(const Lv& lv, const LvlPtr* tb, char* sm, const double* __restrict__ pinv,
                                           double* __restrict__ Zg, double* __restrict__ Wg,
                                           double* __restrict__ zout, double* __restrict__ scal, double gd,
                                           int mode_in, int o_tt, bool kc_to_smem = false,
                                           const double* __restrict__ mtop = nullptr, int tj = 0, int nj = 0,
                                           int nwl = CT / 32) {
  // nwl: the warps [0, nwl) that run the coarse levels (the others are busy)
  // mtop (shared memory): levels Kc+tj .. L by the dense top map instead of
  // sweeps and the top solve (build_top_map)
  // kc_to_smem: level Kc stays in shared memory (the merged tier-2 down kernel)
  const int NW = nwl;
  const int mode = mode_in & 15;
  const int L = lv.L, Kc = lv.Kc, nl = L - Kc + 1, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ double srho;
  auto W = [&](int t) {  // tb[t].cnt = n_{Kc+t} (shared memory)
    const int c = (tb[t].cnt + 31) >> 5;
    return c < 1 ? 1 : (c > NW ? NW : c);
  };
  if (NW == CT / 32) __syncthreads();  // pointer table and staged segments
  else named_sync(1, NW);
  // ---- up: level t on warps [0, W(t)) (up to level Kc+tj with the top map)
  const int tup = mtop ? tj : nl - 1;
  __shared__ double sgd;
  if (mtop && tid == 0) sgd = gd;
  for (int t = 1; t <= tup; ++t) {
    if (t >= 2) {
      const int wp = W(t - 1);
      if (warp >= wp) break;
      named_sync(1, wp);
    }
    if (t <= 7) TRACE(6 + t);
    const int wt = W(t);
    if (warp < wt) {
      const int* cp = SMP(const int, tb[t].cp);
      const double* yc = SMP(const double, tb[t - 1].y);
      double* yp = SMP(double, tb[t].y);
      const int np = tb[t].cnt;
      #pragma unroll 1
      for (int i = tid; i < np; i += 32 * wt) {
        double y = 0.0;
        const int c1 = cp[i + 1];
        #pragma unroll 1
        for (int c = cp[i]; c < c1; ++c) y += yc[c];
        yp[i] = y;
      }
    }
  }
  // ---- top solve (warp 0), or the top map (warps [0, W(tj)))
  double rz = 0.0;
  const int ntop = tb[nl - 1].cnt;
  if (mtop) {
    const int wj = W(tj);
    if (warp < wj) {
      named_sync(1, wj);  // y at level Kc+tj complete, sgd visible
      const double* yj = SMP(const double, tb[tj].y);
      double* zj = SMP(double, tb[tj].z);
      double* wjs = SMP(double, tb[tj].w);
      const double g0 = sgd;
      #pragma unroll 1
      for (int row = tid; row < 2 * nj; row += 32 * wj) {
        const double* m = mtop + (int64_t)row * (nj + 1);
        double a0 = 0.0, a1 = 0.0;
        int c = 0;
        #pragma unroll 1
        for (; c + 1 < nj; c += 2) { a0 += m[c] * yj[c]; a1 += m[c + 1] * yj[c + 1]; }
        if (c < nj) a0 += m[c] * yj[c];
        const double v = (a0 + a1) + m[nj] * g0;
        if (row < nj) zj[row] = v;
        else wjs[row - nj] = v;
      }
      if (warp == 0) {  // rho from the same y (sums are preserved up the tree)
        double ysum = 0.0;
        #pragma unroll 1
        for (int i = lane; i < nj; i += 32) ysum += yj[i];
        ysum = warp_sum(ysum);
        if (lane == 0) {
          srho = lv.c_sum * ysum / lv.n_tilde;
          if (mode != M_COLUMN) scal[S_SHIFT] = srho;
        }
      }
    }
  } else if (warp == 0) {
    __syncwarp();
    const double* yt = SMP(const double, tb[nl - 1].y);
    const double* Nt = SMP(const double, tb[nl - 1].nn);
    double ysum = 0.0;
    #pragma unroll 1
    for (int i = lane; i < ntop; i += 32) ysum += yt[i];
    ysum = warp_sum(ysum);
    gd = warp_sum(gd);
    const double rho = lv.c_sum * ysum / lv.n_tilde;
    double* tt = reinterpret_cast<double*>(sm + o_tt);
    #pragma unroll 1
    for (int i = lane; i < ntop; i += 32) tt[i] = lv.ck[L] * yt[i] - rho * Nt[i];
    __syncwarp();
    double* zt = SMP(double, tb[nl - 1].z);
    double* wt = SMP(double, tb[nl - 1].w);
    double nz = 0.0;
    #pragma unroll 1
    for (int i = lane; i < ntop; i += 32) {
      double zi = 0.0;
      #pragma unroll 1
      for (int j = 0; j < ntop; ++j) zi += pinv[i * ntop + j] * tt[j];
      zt[i] = zi;
      nz += Nt[i] * zi;
    }
    nz = warp_sum(nz);
    const double m = (nz + gd - rho * lv.GN) / lv.n_tilde;
    #pragma unroll 1
    for (int i = lane; i < ntop; i += 32) {
      const double z = zt[i] - m;
      zt[i] = z;
      wt[i] = z;
      if (L == 1) {
        rz += yt[i] * z;
        zout[((mode_in & M_ZS2) ? 2 : 1) * i] = z;
      } else if (nl == 1) {  // the top is level Kc: to global
        if (mode == M_COLUMN) {
          Zg[(int64_t)blockIdx.x * 2 * ntop + i] = z;
          Zg[(int64_t)blockIdx.x * 2 * ntop + ntop + i] = z;
        } else {
          Zg[lv.off[Kc - 1] + i] = z;
          Wg[lv.off[Kc - 1] + i] = z;
        }
      }
    }
    if (lane == 0) {
      srho = rho;
      if (mode != M_COLUMN) scal[S_SHIFT] = rho;
    }
    __syncwarp();
  }
  TRACE(5);
  // ---- down: level t on warps [0, W(t)) (W grows as t falls)
  const double negmu = lv.negmu;
  for (int t = mtop ? tj - 1 : nl - 2; t >= 0; --t) {
    const int wt = W(t);
    if (warp >= wt) continue;
    named_sync(2 + t, wt);
    const double rho = srho;
    const int* cp = SMP(const int, tb[t + 1].cp);
    const double* ki = SMP(const double, tb[t + 1].ki);
    const double* zp = SMP(const double, tb[t + 1].z);
    const double* wp = SMP(const double, tb[t + 1].w);
    const double* lo = SMP(const double, tb[t].lo);
    const double* yc = SMP(const double, tb[t].y);
    const double* nc = SMP(const double, tb[t].nn);
    double* zc = SMP(double, tb[t].z);
    double* wc = SMP(double, tb[t].w);
    const double ckk = tb[t].ck;
    const int np = tb[t + 1].cnt;
    const int nk = tb[t].cnt;
    if (t > 0 || kc_to_smem) {
      #pragma unroll 1
      for (int i = tid; i < np; i += 32 * wt) {
        const int lb = -3 * (2 * i + 2);
        block_solve(
            cp[i], cp[i + 1], [&](int j) { return ki[3 * i + j]; }, [&](int p, int j) { return lo[lb + 3 * p + j]; },
            zp[i], negmu * wp[i], [&](int p) { return ckk * yc[p] - rho * nc[p]; },
            [&](int p, double z, double w) { zc[p] = z; wc[p] = w; });
      }
    } else if (Kc == 1) {  // level-1 output and (r, R r)
      const int zs = (mode_in & M_ZS2) ? 2 : 1;
      #pragma unroll 1
      for (int i = tid; i < np; i += 32 * wt) {
        const int lb = -3 * (2 * i + 2);
        block_solve(
            cp[i], cp[i + 1], [&](int j) { return ki[3 * i + j]; }, [&](int p, int j) { return lo[lb + 3 * p + j]; },
            zp[i], negmu * wp[i], [&](int p) { return yc[p] - rho; },
            [&](int p, double z, double w) { rz += yc[p] * w; zout[zs * p] = w; });
      }
    } else {  // level Kc to global: Z, W (or column blockIdx.x of the GEMV map)
      double* zg = (mode == M_COLUMN) ? Zg + (int64_t)blockIdx.x * 2 * nk : Zg + lv.off[Kc - 1];
      double* wg = (mode == M_COLUMN) ? zg + nk : Wg + lv.off[Kc - 1];
      #pragma unroll 1
      for (int i = tid; i < np; i += 32 * wt) {
        const int lb = -3 * (2 * i + 2);
        block_solve(
            cp[i], cp[i + 1], [&](int j) { return ki[3 * i + j]; }, [&](int p, int j) { return lo[lb + 3 * p + j]; },
            zp[i], negmu * wp[i], [&](int p) { return ckk * yc[p] - rho * nc[p]; },
            [&](int p, double z, double w) { zg[p] = z; wg[p] = w; });
      }
    }
  }
  TRACE(6);
  if (!kc_to_smem || (MSP_EARLY & 32) == 0) pdl_trigger();
  if (Kc == 1) {
    rz = block_sum<CT>(rz);
    if (tid == 0 && mode != M_APPLY) finish_rz(rz, scal, mode);
  }
}

// Single CTA: levels Kc..L up-sweep, the top solve, levels L..Kc down-sweep,
// everything staged in / computed into shared memory (layout: CoarseDesc).
// When Kc == 1 it also produces the level-1 output and (r, R r).
#undef TRACE_KID
#define TRACE_KID 1
// Shared state of the coarse levels (k_coarse, and the merged tier-2 down
// kernel that runs them first).
struct CoarseState {
  uint64_t bar;
  int skc[MAXT + 8], skk[MAXT + 8], skl[MAXT + 8], skn[MAXT + 8];
  int sky0, skp, skm;
  LvlPtr tb[MAXT + 8];
};

// static segments of levels Kc..L (before the grid dependency), one per
// thread spread over the warps: [0, nl-1) child pointers, [nl-1, 2nl-2)
// factors, [2nl-2, 3nl-3) leftover coefficients, [3nl-3, 4nl-3) subtree
// sizes, 4nl-3 the top pseudo-inverse.  C.bar must be initialised and visible.
template <int NT>
__device__ __forceinline__ void coarse_stage_static(CoarseState& C, char* smc, const Lv& lv, const CoarseDesc& cd,
                                                    const int32_t* __restrict__ cptr,
                                                    const double* __restrict__ kinv,
                                                    const double* __restrict__ lof,
                                                    const double* __restrict__ Nsub,
                                                    const double* __restrict__ pinv_g,
                                                    const double* __restrict__ mtop_g) {
  const int tid = threadIdx.x, L = lv.L, Kc = lv.Kc, nl = cd.nl;
  const int64_t n1 = lv.n[0];
  const int g = (tid & 31) * (NT / 32) + (tid >> 5);
  const int m1 = nl - 1;
  if (g < m1) {
    const int t = g + 1;
    const int64_t base = lv.cpo[Kc + t - 2];
    C.skc[t] = stage_window<true>(&C.bar, smc + cd.o_cp[t], cptr, 4, base, base + lv.n[Kc + t - 1] + 1);
  } else if (g < 2 * m1) {
    const int t = g - m1 + 1;
    const int64_t base = 3 * (lv.off[Kc + t - 1] - n1);
    C.skk[t] = stage_window<true>(&C.bar, smc + cd.o_ki[t], kinv, 8, base, base + 3 * lv.n[Kc + t - 1]);
  } else if (g < 3 * m1) {
    const int t = g - 2 * m1;
    const int64_t base = 3 * lv.lo[Kc + t - 1];
    C.skl[t] = stage_window<true>(&C.bar, smc + cd.o_lo[t], lof, 8, base,
                                  base + 3 * (lv.n[Kc + t - 1] - 2 * lv.n[Kc + t]));
  } else if (g < 3 * m1 + nl) {
    const int t = g - 3 * m1;
    const int64_t base = lv.off[Kc + t - 1];
    C.skn[t] = stage_window<true>(&C.bar, smc + cd.o_n[t], Nsub, 8, base, base + lv.n[Kc + t - 1]);
  } else if (g == 3 * m1 + nl && cd.stage_pinv) {
    const int64_t nt = lv.n[L - 1];
    C.skp = stage_window<true>(&C.bar, smc + cd.o_pinv, pinv_g, 8, 0, nt * nt);
  } else if (g == 3 * m1 + nl + 1 && cd.topmap_t > 0 && mtop_g) {
    const int64_t nj = cd.mtop_n;
    C.skm = stage_window<true>(&C.bar, smc + cd.o_mtop, mtop_g, 8, 0, 2 * nj * (nj + 1));
  }
}

// per-level pointer table of the coarse levels (threads t < nl)
__device__ __forceinline__ void coarse_table(CoarseState& C, const Lv& lv, const CoarseDesc& cd, int coff) {
  const int t = threadIdx.x, nl = cd.nl, Kc = lv.Kc;
  if (t < nl) {
    LvlPtr e;
    e.cp = (t >= 1) ? coff + cd.o_cp[t] + 4 * C.skc[t] : -1;
    e.ki = (t >= 1) ? coff + cd.o_ki[t] + 8 * C.skk[t] : -1;
    e.lo = (t + 1 < nl) ? coff + cd.o_lo[t] + 8 * C.skl[t] : -1;
    e.y = coff + cd.o_y[t] + (t == 0 ? 8 * C.sky0 : 0);
    e.nn = coff + cd.o_n[t] + 8 * C.skn[t];
    e.z = coff + cd.o_z[t];
    e.w = coff + cd.o_w[t];
    e.a = 0;
    e.cnt = (int)lv.n[Kc + t - 1];
    e.ck = lv.ck[Kc + t];
    C.tb[t] = e;
  }
}

// ---------------------------------------------------------- tile down-sweep
// Tier k0..k1: recompute y (and subtree sizes N) of levels k0+1..k1-1 from
// y_k0, read z, w at level k1, solve / prolong down to level k0.  FIRST: the
// output R r and the partial (r, R r); otherwise z, w at level k0 to global.
#undef TRACE_KID
#define TRACE_KID (FIRST ? 2 : 3)
// COARSE (tier 2 = the last tier, one CTA of CT threads per tile): the CTA
// first runs the coarse levels Kc..L itself (every CTA the same, into its own
// shared memory at byte offset coff) and takes its tile's level-Kc z, w from
// there -- no coarse kernel, no round trip of z_Kc, w_Kc through global memory.
template <bool FIRST, bool COARSE = false>
__global__ void __launch_bounds__(COARSE ? CT : TT) k_tile_down(const __grid_constant__ Lv lv, const __grid_constant__ TierDesc td,
                                                  const int32_t* __restrict__ tstart, const int32_t* __restrict__ cptr,
                                                  const double* __restrict__ kinv, const double* __restrict__ lof,
                                                  const double* __restrict__ Nsub, const double* __restrict__ y0src,
                                                  double* __restrict__ Zg, double* __restrict__ Wg,
                                                  double* __restrict__ zout, double* __restrict__ part,
                                                  double* __restrict__ scal, unsigned int* __restrict__ cnt, int mode_in,
                                                  const double* __restrict__ Mco, const double* __restrict__ part_gd,
                                                  int npart_gd, const double* __restrict__ Ygl, int tile0,
                                                  const int4* __restrict__ segs,
                                                  const __grid_constant__ CoarseDesc cd, int coff,
                                                  const double* __restrict__ pinv_g,
                                                  const double* __restrict__ mtop_g) {
  constexpr int NT = COARSE ? CT : TT;
  const int mode = mode_in & 15;
  const bool dist = (mode_in & M_DIST) != 0;
  extern __shared__ __align__(16) char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int sa[MAXT], sn[MAXT], skc[MAXT], skk[MAXT], skl[MAXT];
  __shared__ int sky0, skn0, skz, skw, sdone;
  __shared__ double srho, srho_g;
  __shared__ LvlPtr tb[MAXT];
  __shared__ CoarseState C;
  __shared__ double sgd;
  const int nl = td.nl, k0 = td.k0, nt1 = td.ntiles + 1;
  // first tier (not distributed): tpc consecutive tiles per CTA, one after
  // another (the block reduction and ticket once per CTA)
  const int tpc = (FIRST && !COARSE && td.tpc > 1) ? td.tpc : 1;
  const int tid = threadIdx.x;
  const int64_t n1 = lv.n[0];
  if ((COARSE ? (MSP_EARLY & 4) : FIRST ? (MSP_EARLY & 8) : (MSP_EARLY & 4)) != 0) pdl_trigger();
  TRACE(0);
  PHASE_START();
  if (tid == 0) {
    mbar_init(&bar, 1);
    if (COARSE) mbar_init(&C.bar, 1);
  }
  double rz = 0.0;
  // the next tile's ranges and segment descriptors are loaded into registers
  // while the current one computes
  int pa = 0, pb = 0;
  int4 psd = make_int4(0, 0, 0, 0);
  auto load_idx = [&](int tl) {
    if (tid < nl) { pa = tstart[tid * nt1 + tl]; pb = tstart[tid * nt1 + tl + 1]; }
    if (tid < td.nseg) psd = __ldg(segs + (int64_t)tl * td.nseg + tid);
  };
  load_idx((int)blockIdx.x * tpc + tile0);
  #pragma unroll 1
  for (int tt = 0; tt < tpc; ++tt) {
  const int tile = (int)blockIdx.x * tpc + tt + tile0;
  if (tile >= td.ntiles) break;  // uniform
  if (tid < nl) {
    sa[tid] = pa;
    sn[tid] = pb - pa;
  }
  // static segments (child pointers, factors, leftover coefficients, N_k0),
  // one per thread from the tile's precomputed descriptors; after the grid
  // dependency: y_k0, z, w
  const int4 sd = psd;
  __syncthreads();
  if (tid < td.nseg) {
    const int kind = sd.x & 3, t = (sd.x >> 2) & 63, dst = sd.x >> 8;
    if (sd.y > 0) {
      mbar_expect_tx(&bar, (uint32_t)sd.y);
      const char* src = (kind == SEG_CP)   ? (const char*)cptr + (int64_t)sd.z * 4
                        : (kind == SEG_KI) ? (const char*)kinv + (int64_t)sd.z * 8
                        : (kind == SEG_LO) ? (const char*)lof + (int64_t)sd.z * 8
                                           : (const char*)Nsub + (int64_t)sd.z * 8;
      tma_1d_keep(sm + dst, src, (uint32_t)sd.y, &bar);
    }
    if (kind == SEG_CP) skc[t] = sd.w;
    else if (kind == SEG_KI) skk[t] = sd.w;
    else if (kind == SEG_LO) skl[t] = sd.w;
    else skn0 = sd.w;
  }
  const int g = (tid & 31) * (NT / 32) + (tid >> 5);  // dynamic segments below
  const int m1 = nl - 1;
  if (COARSE) coarse_stage_static<NT>(C, sm + coff, lv, cd, cptr, kinv, lof, Nsub, pinv_g, mtop_g);
  TRACE(1);
  PHASE(0);
  pdl_wait();
  TRACE(2);
  PHASE(1);
  // dynamic segments (y_k0, z and w at level k1) go out at once; the done
  // flag and rho are read alongside (a finished solve only wastes the copies)
  if (tid == 0) {
    sdone = (mode != M_APPLY) ? (int)cnt[C_DONE] : 0;
    if (!COARSE) srho = scal[S_SHIFT];
    if (COARSE) {  // y_Kc for the coarse levels, and gdot
      const int Kc = lv.Kc;
      C.sky0 = stage_window(&C.bar, sm + coff + cd.o_y[0], Ygl, 8, lv.off[Kc - 1], lv.off[Kc - 1] + lv.n[Kc - 1]);
      if (mode != M_APPLY) sgd = scal[S_GD];
    }
  }
  const bool gemv = td.gemv_n > 0;
  if (g == 3 * m1 + 1) {
    const int64_t base = FIRST ? 0 : lv.off[k0 - 1];
    sky0 = stage_window(&bar, sm + td.o_y[0], y0src, 8, base + sa[0], base + sa[0] + sn[0]);
  } else if (!COARSE && !gemv && (g == 3 * m1 + 2 || g == 3 * m1 + 3)) {
    const bool isz = (g == 3 * m1 + 2);
    const int64_t base = lv.off[k0 + nl - 2] + sa[nl - 1];
    const int v = stage_window(&bar, sm + (isz ? td.o_z[nl - 1] : td.o_w[nl - 1]), isz ? Zg : Wg, 8, base,
                               base + sn[nl - 1]);
    if (isz) skz = v; else skw = v;
  }
  if (gemv) {
    // Coarse GEMV (levels Kc..L folded into a dense map at setup): z, w of
    // this tile's level-Kc nodes = Mco [y_Kc; gdot]; rho from the same y_Kc
    const int nk = td.gemv_n;
    double* v = reinterpret_cast<double*>(sm + td.o_v);
    const int64_t okc = lv.off[k0 + nl - 2];
    double ys = 0.0, gd = 0.0;
    for (int j = tid; j < nk; j += NT) {
      const double yv = __ldcg(Ygl + okc + j);
      v[j] = yv;
      ys += yv;
    }
    for (int j = tid; j < npart_gd; j += NT) gd += __ldcg(part_gd + j);
    const double2 sums = block_sum2<NT>(make_double2(ys, gd));
    if (tid == 0) {
      v[nk] = sums.y;
      srho_g = lv.c_sum * sums.x / lv.n_tilde;
      skz = 0;
      skw = 0;
    }
    __syncthreads();
    // warp per output row: rows [a, a+cnt) of z then of w
    const int a = sa[nl - 1], cnt = sn[nl - 1], lane = tid & 31, warp = tid >> 5;
    double* zt = reinterpret_cast<double*>(sm + td.o_z[nl - 1]);
    double* wt = reinterpret_cast<double*>(sm + td.o_w[nl - 1]);
    for (int rr = warp; rr < 2 * cnt; rr += NT / 32) {
      const int row = (rr < cnt) ? a + rr : nk + a + (rr - cnt);
      const double* Mr = Mco + (int64_t)row * (nk + 1);
      double acc = 0.0;
      for (int j = lane; j <= nk; j += 32) acc += Mr[j] * v[j];
      acc = warp_sum(acc);
      if (lane == 0) {
        if (rr < cnt) zt[rr] = acc;
        else wt[rr - cnt] = acc;
      }
    }
    if (tid == 0 && blockIdx.x == 0 && mode != M_COLUMN) scal[S_SHIFT] = srho_g;
  }
  __syncthreads();
  const int done = sdone;
  if (gemv && tid == 0) srho = srho_g;
  if (tid == 0) {  // every expect_tx of both barriers precedes (the barrier above)
    mbar_arrive(&bar);
    if (COARSE) mbar_arrive(&C.bar);
  }
  mbar_wait(&bar, (uint32_t)(tt & 1));
  if (tt + 1 < tpc && tile + 1 < td.ntiles) load_idx(tile + 1);
  TRACE(3);
  PHASE(2);
  // per-level pointer table (one thread per level), so every phase starts
  // with a handful of independent shared-memory loads
  auto build_table = [&](int t) {
    LvlPtr e;
    e.cp = (t >= 1) ? td.o_cp[t] + 4 * skc[t] : -1;
    e.ki = (t >= 1) ? td.o_ki[t] + 8 * skk[t] : -1;
    e.lo = (t + 1 < nl) ? td.o_lo[t] + 8 * skl[t] : -1;
    e.y = (t == 0) ? td.o_y[0] + 8 * sky0 : (t + 1 < nl ? td.o_y[t] : -1);
    e.nn = (t == 0) ? (FIRST ? -1 : td.o_n[0] + 8 * skn0) : (t + 1 < nl ? td.o_n[t] : -1);
    e.z = (t == nl - 1) ? (COARSE ? coff + cd.o_z[0] + 8 * sa[t] : td.o_z[t] + 8 * skz) : (t >= 1 ? td.o_z[t] : -1);
    e.w = (t == nl - 1) ? (COARSE ? coff + cd.o_w[0] + 8 * sa[t] : td.o_w[t] + 8 * skw) : (t >= 1 ? td.o_w[t] : -1);
    e.a = sa[t];
    e.cnt = sn[t];
    e.ck = lv.ck[k0 + t];
    tb[t] = e;
  };
  // ---- recompute y and N of levels k0+1 .. k1-1 (threads base, base +
  // stride, ...; sync() before every level)
  auto recompute = [&](int base, int stride, auto sync) {
#ifndef MSP_NO_RECOMP2
    // two levels per step where both need recomputing: a thread takes a
    // level-(t+1) parent, forms y, N of each child c (level t) from c's
    // children and sums them -- the same additions in the same order, one
    // barrier fewer
    int t = 1;
    for (; t + 2 < nl; t += 2) {
      sync();
      const int* cp1 = SMP(const int, tb[t].cp);
      const int* cp2 = SMP(const int, tb[t + 1].cp);
      const double* yg = SMP(const double, tb[t - 1].y);
      const double* ng = tb[t - 1].nn >= 0 ? SMP(const double, tb[t - 1].nn) : nullptr;
      double* yc = SMP(double, tb[t].y);
      double* nc = SMP(double, tb[t].nn);
      double* yp = SMP(double, tb[t + 1].y);
      double* np = SMP(double, tb[t + 1].nn);
      const int ag = tb[t - 1].a, ac = tb[t].a, npar = tb[t + 1].cnt;
      #pragma unroll 1
      for (int i = base; i < npar; i += stride) {
        const int c0 = cp2[i] - ac, c1 = cp2[i + 1] - ac;
        double y2 = 0.0, N2 = 1.0;
        #pragma unroll 1
        for (int c = c0; c < c1; ++c) {
          const int g0 = cp1[c] - ag, g1 = cp1[c + 1] - ag;
          double y = 0.0, N = 1.0;
          if (ng) {
            #pragma unroll 1
            for (int gg = g0; gg < g1; ++gg) { y += yg[gg]; N += ng[gg]; }
          } else {
            #pragma unroll 1
            for (int gg = g0; gg < g1; ++gg) y += yg[gg];
            N = (double)(1 + g1 - g0);
          }
          yc[c] = y;
          nc[c] = N;
          y2 += y;
          N2 += N;
        }
        yp[i] = y2;
        np[i] = N2;
      }
    }
    for (; t + 1 < nl; ++t) {
#else
    for (int t = 1; t + 1 < nl; ++t) {
#endif
      sync();
      const int* cp = SMP(const int, tb[t].cp);
      const double* yc = SMP(const double, tb[t - 1].y);
      const double* nc = tb[t - 1].nn >= 0 ? SMP(const double, tb[t - 1].nn) : nullptr;
      double* yp = SMP(double, tb[t].y);
      double* np = SMP(double, tb[t].nn);
      const int ac = tb[t - 1].a, npar = tb[t].cnt;
      if (nc) {
        #pragma unroll 1
        for (int i = base; i < npar; i += stride) {
          const int c0 = cp[i] - ac, c1 = cp[i + 1] - ac;
          double y = 0.0, N = 1.0;
          #pragma unroll 1
          for (int c = c0; c < c1; ++c) {
            y += yc[c];
            N += nc[c];
          }
          yp[i] = y;
          np[i] = N;
        }
      } else {  // level-1 children: N = 1 each
        #pragma unroll 1
        for (int i = base; i < npar; i += stride) {
          const int c0 = cp[i] - ac, c1 = cp[i + 1] - ac;
          double y = yc[c0] + yc[c0 + 1];  // every aggregate has its matched pair
          #pragma unroll 1
          for (int c = c0 + 2; c < c1; ++c) y += yc[c];
          yp[i] = y;
          np[i] = (double)(1 + c1 - c0);
        }
      }
    }
  };
  bool recomputed = false;
  if (COARSE) {
    mbar_wait(&C.bar, 0);
    if (done) return;
    double gd = 0.0;
    if (mode != M_APPLY) gd = (tid == 0) ? sgd : 0.0;
    else if (tid < 32) {  // apply_R: the partials are summed here
      const double t = warp_sum_partials(part_gd, npart_gd);
      gd = (tid == 0) ? t : 0.0;
    }
    // overlap: warps 16..31 recompute the tile's levels (barrier id 15)
    // while warps 0..15 run the coarse levels (ids 1 .. nl_c < 15)
    const bool ovl = cd.overlap != 0;
    const int warp_ = tid >> 5;
    if (ovl && warp_ >= 16) {
      const int u = tid - 512;
      if (u < nl) build_table(u);
      recompute(u, NT - 512, [&] { named_sync(15, 16); });
    } else {
      coarse_table(C, lv, cd, coff);
      const double* pinv =
          cd.stage_pinv ? reinterpret_cast<const double*>(sm + coff + cd.o_pinv) + C.skp : pinv_g;
      const double* mtop = (cd.topmap_t > 0 && mtop_g)
                               ? reinterpret_cast<const double*>(sm + coff + cd.o_mtop) + C.skm : nullptr;
      coarse_levels(lv, C.tb, sm, pinv, Zg, Wg, zout, scal, gd, mode_in, coff + cd.o_tt, true, mtop, cd.topmap_t,
                    cd.mtop_n, ovl ? 16 : NT / 32);
    }
    __syncthreads();
    if (tid == 0) srho = scal[S_SHIFT];  // written by warp 0 above
    recomputed = ovl;
    __syncthreads();
  }
  if (done) return;
  if (!recomputed) {
    if (tid < nl) build_table(tid);
    recompute(tid, NT, [] { __syncthreads(); });
  }
  TRACE(4);
  PHASE(3);
  // ---- down: levels k1-1 .. k0+1 in shared memory, then level k0 out
  const double rho = srho;
  const double negmu = lv.negmu;
  for (int t = nl - 2; t >= 1; --t) {  // child level k = k0+t, parent level k+1
    __syncthreads();
    TRACE(6 + t);
    const int* cp = SMP(const int, tb[t + 1].cp);
    const double* ki = SMP(const double, tb[t + 1].ki);
    const double* zp = SMP(const double, tb[t + 1].z);
    const double* wp = SMP(const double, tb[t + 1].w);
    const double* lo = SMP(const double, tb[t].lo);
    const double* yc = SMP(const double, tb[t].y);
    const double* nc = SMP(const double, tb[t].nn);
    double* zc = SMP(double, tb[t].z);
    double* wc = SMP(double, tb[t].w);
    const int ac = tb[t].a, npar = tb[t + 1].cnt;
    const double ckk = tb[t].ck;
    #pragma unroll 1
    for (int i = tid; i < npar; i += NT) {
      const int lb = -3 * (2 * i + 2);
      block_solve(
          cp[i] - ac, cp[i + 1] - ac, [&](int j) { return ki[3 * i + j]; },
          [&](int p, int j) { return lo[lb + 3 * p + j]; }, zp[i], negmu * wp[i],
          [&](int p) { return ckk * yc[p] - rho * nc[p]; },
          [&](int p, double z, double w) { zc[p] = z; wc[p] = w; });
    }
  }
  {
    __syncthreads();
    PHASE(4);
    const int* cp = SMP(const int, tb[1].cp);
    const double* ki = SMP(const double, tb[1].ki);
    const double* zp = SMP(const double, tb[1].z);
    const double* wp = SMP(const double, tb[1].w);
    const double* lo = SMP(const double, tb[0].lo);
    const double* yc = SMP(const double, tb[0].y);
    const double* nc = SMP(const double, tb[0].nn >= 0 ? tb[0].nn : 0);
    const int ac = tb[0].a, npar = tb[1].cnt;
    const double ckk = tb[0].ck;
    const int zs = (mode_in & M_ZS2) ? 2 : 1;
    double* zg = FIRST ? zout + zs * ac : Zg + lv.off[k0 - 1] + ac;
    double* wg = Wg + lv.off[k0 - 1] + ac;
    #pragma unroll 1
    for (int i = tid; i < npar; i += NT) {
      const int lb = -3 * (2 * i + 2);
      if (FIRST)
        block_solve(
            cp[i] - ac, cp[i + 1] - ac, [&](int j) { return ki[3 * i + j]; },
            [&](int p, int j) { return lo[lb + 3 * p + j]; }, zp[i], negmu * wp[i],
            [&](int p) { return yc[p] - rho; },
            [&](int p, double z, double w) { rz += yc[p] * w; zg[zs * p] = w; });
      else
        block_solve(
            cp[i] - ac, cp[i + 1] - ac, [&](int j) { return ki[3 * i + j]; },
            [&](int p, int j) { return lo[lb + 3 * p + j]; }, zp[i], negmu * wp[i],
            [&](int p) { return ckk * yc[p] - rho * nc[p]; },
            [&](int p, double z, double w) { zg[p] = z; wg[p] = w; });
    }
  }
  if (tt + 1 < tpc) __syncthreads();  // the next tile's copies overwrite shared memory
  }  // tiles of this CTA
  TRACE(5);
  PHASE(5);
  pdl_trigger();
  if (FIRST) {
    rz = block_sum<NT>(rz);
    if (tid < 32) {  // only warp 0 waits on the ticket
      if (tid == 0) part[blockIdx.x + tile0] = rz;
      if (mode != M_APPLY && warp_last_block(&cnt[C_DOWN])) {
        const double tot = warp_sum_partials(part + tile0, gridDim.x);
        if (tid == 0) {
          if (dist) scal[S_RZ] = tot;
          else finish_rz(tot, scal, mode);
          cnt[C_DOWN] = 0;
        }
      }
    }
  }
  PHASE(6);
#ifdef MSP_TRACE
  if (threadIdx.x == 0) atomicAdd(&g_phase[TRACE_KID][15], 1ull);
#endif
  TRACE_END();
}

// ------------------------------------------------- first-tier down, per warp
// The first tier's down sweep with one warp per tile (tiles of ~MSP_WTILE
// level-1 nodes): every warp stages its own tile with TMA bulk copies onto
// its own mbarrier and runs the tile's levels with __syncwarp between them,
// so the warps of an SM are independent chains (no CTA barrier per level)
// and the next tile's copies of one warp overlap the other warps' compute.
// Same arithmetic, in the same order, as k_tile_down<true> (its header and
// DESIGN.md "MSP apply"): recompute y, N of levels 2 .. k1-1, then the block
// solves down to level 1, whose output w_1 = R r goes to zout (stride zs)
// with (r, R r) accumulated.
#ifndef MSP_WD
#define MSP_WD 4
#endif
constexpr int WD = MSP_WD;  // warps per CTA
__global__ void __launch_bounds__(WD * 32) k_wtile_down(const __grid_constant__ Lv lv, const __grid_constant__ TierDesc td,
                                                       const int32_t* __restrict__ tstart,
                                                       const int32_t* __restrict__ cptr, const double* __restrict__ kinv,
                                                       const double* __restrict__ lof, const double* __restrict__ rin,
                                                       const double* __restrict__ Zg, const double* __restrict__ Wg,
                                                       double* __restrict__ zout, double* __restrict__ part,
                                                       double* __restrict__ scal, unsigned int* __restrict__ cnt,
                                                       int mode_in, const int4* __restrict__ segs, int region) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[WD];
  __shared__ LvlPtr tbs[WD][MAXT];
  __shared__ int ssa[WD][MAXT], ssn[WD][MAXT], skc_[WD][MAXT], skk_[WD][MAXT], skl_[WD][MAXT], skd[WD][4];
  const int mode = mode_in & 15;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  char* sm = smem + (size_t)wid * region;
  uint64_t* bar = &bars[wid];
  LvlPtr* tb = tbs[wid];
  int* sa = ssa[wid];
  int* sn = ssn[wid];
  const int nl = td.nl, nt1 = td.ntiles + 1, m1 = nl - 1;
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  const int zs = (mode_in & M_ZS2) ? 2 : 1;
  const double negmu = lv.negmu;
  const int64_t okz = lv.off[nl - 1];  // level k1 = nl (k0 = 1)
  double rz = 0.0;
  double rho = 0.0;
  int done = 0;
  bool waited = false;
  uint32_t phase = 0;
  const int gw = blockIdx.x * WD + wid, nw = gridDim.x * WD;
  #pragma unroll 1
  for (int tile = gw; tile < td.ntiles; tile += nw) {
    // ranges of the tile at every level (lane t), static segments (lane < nseg)
    int a = 0, b = 0;
    if (lane < nl) { a = tstart[lane * nt1 + tile]; b = tstart[lane * nt1 + tile + 1]; sa[lane] = a; sn[lane] = b - a; }
    const int4 sd = (lane < td.nseg) ? __ldg(segs + (int64_t)tile * td.nseg + lane) : make_int4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the last tile before the copies
    if (lane < td.nseg) {
      const int kind = sd.x & 3, t = (sd.x >> 2) & 63, dst = sd.x >> 8;
      if (sd.y > 0) {
        mbar_expect_tx(bar, (uint32_t)sd.y);
        const char* src = (kind == SEG_CP)   ? (const char*)cptr + (int64_t)sd.z * 4
                          : (kind == SEG_KI) ? (const char*)kinv + (int64_t)sd.z * 8
                                             : (const char*)lof + (int64_t)sd.z * 8;
        tma_1d_keep(sm + dst, src, (uint32_t)sd.y, bar);
      }
      if (kind == SEG_CP) skc_[wid][t] = sd.w;
      else if (kind == SEG_KI) skk_[wid][t] = sd.w;
      else skl_[wid][t] = sd.w;
    }
    if (!waited) {
      pdl_wait();
      waited = true;
      done = (mode != M_APPLY) ? (int)cnt[C_DONE] : 0;
      rho = scal[S_SHIFT];
    }
    const int a0 = __shfl_sync(0xffffffffu, a, 0), n0 = __shfl_sync(0xffffffffu, b - a, 0);
    const int ak = __shfl_sync(0xffffffffu, a, m1), nk = __shfl_sync(0xffffffffu, b - a, m1);
    if (!done) {  // dynamic segments: y_1 = r, z and w at level k1
      if (lane == 29) skd[wid][0] = stage_window(bar, sm + td.o_y[0], rin, 8, a0, (int64_t)a0 + n0);
      else if (lane == 30) skd[wid][1] = stage_window(bar, sm + td.o_z[m1], Zg, 8, okz + ak, okz + ak + nk);
      else if (lane == 31) skd[wid][2] = stage_window(bar, sm + td.o_w[m1], Wg, 8, okz + ak, okz + ak + nk);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
    mbar_wait(bar, phase);
    phase ^= 1u;
    if (done) break;  // warp-uniform; the copies have landed
    if (lane < nl) {
      const int t = lane;
      LvlPtr e;
      e.cp = (t >= 1) ? td.o_cp[t] + 4 * skc_[wid][t] : -1;
      e.ki = (t >= 1) ? td.o_ki[t] + 8 * skk_[wid][t] : -1;
      e.lo = (t + 1 < nl) ? td.o_lo[t] + 8 * skl_[wid][t] : -1;
      e.y = (t == 0) ? td.o_y[0] + 8 * skd[wid][0] : (t + 1 < nl ? td.o_y[t] : -1);
      e.nn = (t == 0) ? -1 : (t + 1 < nl ? td.o_n[t] : -1);
      e.z = (t == m1) ? td.o_z[t] + 8 * skd[wid][1] : (t >= 1 ? td.o_z[t] : -1);
      e.w = (t == m1) ? td.o_w[t] + 8 * skd[wid][2] : (t >= 1 ? td.o_w[t] : -1);
      e.a = sa[t];
      e.cnt = sn[t];
      e.ck = lv.ck[1 + t];
      tb[t] = e;
    }
    __syncwarp();
    // ---- recompute y, N of levels 2 .. k1-1 (two levels per step where both
    // need it: the same additions in the same order as one level at a time)
    {
      int t = 1;
      #pragma unroll 1
      for (; t + 2 < nl; t += 2) {
        const int* cp1 = SMP(const int, tb[t].cp);
        const int* cp2 = SMP(const int, tb[t + 1].cp);
        const double* yg = SMP(const double, tb[t - 1].y);
        const double* ng = tb[t - 1].nn >= 0 ? SMP(const double, tb[t - 1].nn) : nullptr;
        double* yc = SMP(double, tb[t].y);
        double* nc = SMP(double, tb[t].nn);
        double* yp = SMP(double, tb[t + 1].y);
        double* np = SMP(double, tb[t + 1].nn);
        const int ag = tb[t - 1].a, ac = tb[t].a, npar = tb[t + 1].cnt;
        #pragma unroll 1
        for (int i = lane; i < npar; i += 32) {
          const int c0 = cp2[i] - ac, c1 = cp2[i + 1] - ac;
          double y2 = 0.0, N2 = 1.0;
          #pragma unroll 1
          for (int c = c0; c < c1; ++c) {
            const int g0 = cp1[c] - ag, g1 = cp1[c + 1] - ag;
            double y = 0.0, N = 1.0;
            if (ng) {
              #pragma unroll 1
              for (int gg = g0; gg < g1; ++gg) { y += yg[gg]; N += ng[gg]; }
            } else {
              #pragma unroll 1
              for (int gg = g0; gg < g1; ++gg) y += yg[gg];
              N = (double)(1 + g1 - g0);
            }
            yc[c] = y;
            nc[c] = N;
            y2 += y;
            N2 += N;
          }
          yp[i] = y2;
          np[i] = N2;
        }
        __syncwarp();
      }
      #pragma unroll 1
      for (; t + 1 < nl; ++t) {
        const int* cp = SMP(const int, tb[t].cp);
        const double* yc = SMP(const double, tb[t - 1].y);
        const double* nc = tb[t - 1].nn >= 0 ? SMP(const double, tb[t - 1].nn) : nullptr;
        double* yp = SMP(double, tb[t].y);
        double* np = SMP(double, tb[t].nn);
        const int ac = tb[t - 1].a, npar = tb[t].cnt;
        #pragma unroll 1
        for (int i = lane; i < npar; i += 32) {
          const int c0 = cp[i] - ac, c1 = cp[i + 1] - ac;
          double y = 0.0, N = 1.0;
          if (nc) {
            #pragma unroll 1
            for (int c = c0; c < c1; ++c) { y += yc[c]; N += nc[c]; }
          } else {
            y = yc[c0] + yc[c0 + 1];
            #pragma unroll 1
            for (int c = c0 + 2; c < c1; ++c) y += yc[c];
            N = (double)(1 + c1 - c0);
          }
          yp[i] = y;
          np[i] = N;
        }
        __syncwarp();
      }
    }
    // ---- down: levels k1-1 .. 2 in shared memory, then level 1 out
    #pragma unroll 1
    for (int t = nl - 2; t >= 1; --t) {
      const int* cp = SMP(const int, tb[t + 1].cp);
      const double* ki = SMP(const double, tb[t + 1].ki);
      const double* zp = SMP(const double, tb[t + 1].z);
      const double* wp = SMP(const double, tb[t + 1].w);
      const double* lo = SMP(const double, tb[t].lo);
      const double* yc = SMP(const double, tb[t].y);
      const double* nc = SMP(const double, tb[t].nn);
      double* zc = SMP(double, tb[t].z);
      double* wc = SMP(double, tb[t].w);
      const int ac = tb[t].a, npar = tb[t + 1].cnt;
      const double ckk = tb[t].ck;
      #pragma unroll 1
      for (int i = lane; i < npar; i += 32) {
        const int lb = -3 * (2 * i + 2);
        block_solve(
            cp[i] - ac, cp[i + 1] - ac, [&](int j) { return ki[3 * i + j]; },
            [&](int p, int j) { return lo[lb + 3 * p + j]; }, zp[i], negmu * wp[i],
            [&](int p) { return ckk * yc[p] - rho * nc[p]; },
            [&](int p, double z, double w) { zc[p] = z; wc[p] = w; });
      }
      __syncwarp();
    }
    {
      const int* cp = SMP(const int, tb[1].cp);
      const double* ki = SMP(const double, tb[1].ki);
      const double* zp = SMP(const double, tb[1].z);
      const double* wp = SMP(const double, tb[1].w);
      const double* lo = SMP(const double, tb[0].lo);
      const double* yc = SMP(const double, tb[0].y);
      const int ac = tb[0].a, npar = tb[1].cnt;
      double* zg = zout + (int64_t)zs * ac;
      #pragma unroll 1
      for (int i = lane; i < npar; i += 32) {
        const int lb = -3 * (2 * i + 2);
        block_solve(
            cp[i] - ac, cp[i + 1] - ac, [&](int j) { return ki[3 * i + j]; },
            [&](int p, int j) { return lo[lb + 3 * p + j]; }, zp[i], negmu * wp[i],
            [&](int p) { return yc[p] - rho; },
            [&](int p, double z, double w) { rz += yc[p] * w; zg[zs * p] = w; });
      }
    }
    __syncwarp();  // every lane is done with this tile's shared memory
  }
  if (!waited) {  // a warp without tiles
    pdl_wait();
    done = (mode != M_APPLY) ? (int)cnt[C_DONE] : 0;
  }
  if (done) return;  // the whole grid (the flag is constant during this kernel)
  pdl_trigger();
  rz = block_sum<WD * 32>(rz);
  if (threadIdx.x < 32) {  // only warp 0 waits on the ticket
    if (threadIdx.x == 0) part[blockIdx.x] = rz;
    if (mode != M_APPLY && warp_last_block(&cnt[C_DOWN])) {
      const double tot = warp_sum_partials(part, gridDim.x);
      if (threadIdx.x == 0) {
        finish_rz(tot, scal, mode);
        cnt[C_DOWN] = 0;
      }
    }
  }
}

#undef TRACE_KID
#define TRACE_KID 0
// ------------------------------------------------------ per-level kernels
// (a tier whose aggregates are too large to tile: one level, one thread per
// aggregate)  y_{k+1} = P^T y_k
__global__ void __launch_bounds__(TPB) k_up_lvl(const __grid_constant__ Lv lv, int k, const int32_t* __restrict__ cptr,
                                                const double* __restrict__ yin, double* __restrict__ yout,
                                                const unsigned int* __restrict__ cnt, int mode_in,
                                                const int32_t* __restrict__ heavy, int nheavy, int64_t B0, int64_t nB,
                                                const HeavyChunks hc, const double* __restrict__ lof) {
  // parents B0 .. B0+nB-1 of level k+1 (a rank's own range; all of them on one GPU)
  // blocks [0, G - nheavy - nch): a thread per aggregate (heavy ones skipped);
  // then a CTA per heavy aggregate (nheavy) or per heavy chunk (hc.nch)
  const int mode = mode_in & 15;
  pdl_wait();
  if (mode == M_ITER && cnt[C_DONE]) return;
  const int32_t* cp = cptr + lv.cpo[k - 1];
  if ((int)blockIdx.x >= (int)gridDim.x - hc.nch) {  // a chunk of a heavy aggregate
    const int c = (int)blockIdx.x - ((int)gridDim.x - hc.nch);
    const int4 sg = hc.seg[c];
    const int64_t B = sg.x, s0 = cp[B];
    const int64_t lb = 3 * (lv.lo[k - 1] - 2 * B - 2);
    double y = 0.0, a = 0.0, b = 0.0;
    for (int64_t p = sg.y + threadIdx.x; p < sg.z; p += TPB) {
      const double v = yin[p];
      y += v;
      if (p >= s0 + 2) {
        a += lof[lb + 3 * p + 0] * v;
        b += lof[lb + 3 * p + 1] * v;
      }
    }
    const double2 yb = block_sum2<TPB>(make_double2(y, a));
    const double bb = block_sum<TPB>(b);
    if (threadIdx.x == 0) {
      const int g = hc.c0 + c;
      hc.part[3 * g] = yb.x;
      hc.part[3 * g + 1] = yb.y;
      hc.part[3 * g + 2] = bb;
      __threadfence();
      const int f0 = hc.first[sg.w], f1 = hc.first[sg.w + 1];
      if (atomicAdd(&hc.cnt[sg.w], 1u) == (unsigned)(f1 - f0 - 1)) {  // the aggregate's last chunk
        __threadfence();
        double ty = 0.0, ta = 0.0, tb = 0.0;
        for (int j = f0; j < f1; ++j) {
          ty += __ldcg(hc.part + 3 * j);
          ta += __ldcg(hc.part + 3 * j + 1);
          tb += __ldcg(hc.part + 3 * j + 2);
        }
        yout[B] = ty;
        hc.sum[2 * sg.w] = ta;
        hc.sum[2 * sg.w + 1] = tb;
        hc.cnt[sg.w] = 0;
      }
    }
    return;
  }
  const int nnorm = (int)gridDim.x - nheavy - hc.nch;
  if ((int)blockIdx.x < nnorm) {
    const int64_t B = B0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (B < B0 + nB) {
      const int32_t c0 = cp[B], c1 = cp[B + 1];
      if (c1 - c0 <= HEAVY_AGG) {
        double y = 0.0;
#pragma unroll 1
        for (int32_t c = c0; c < c1; ++c) y += yin[c];
        yout[B] = y;
      }
    }
  } else {
    const int64_t B = heavy[blockIdx.x - nnorm];
    double y = 0.0;
    for (int32_t c = cp[B] + threadIdx.x; c < cp[B + 1]; c += TPB) y += yin[c];
    y = block_sum<TPB>(y);
    if (threadIdx.x == 0) yout[B] = y;
  }
}

// z_k, w_k from z_{k+1}, w_{k+1}; at level 1 the output R r and (r, R r)
template <bool LEVEL1>
__global__ void __launch_bounds__(TPB) k_down_lvl(const __grid_constant__ Lv lv, int k, const int32_t* __restrict__ cptr,
                                                  const double* __restrict__ kinv, const double* __restrict__ lof,
                                                  const double* __restrict__ yk, const double* __restrict__ Nsub,
                                                  const double* __restrict__ zB, const double* __restrict__ wB,
                                                  double* __restrict__ zk, double* __restrict__ wk,
                                                  double* __restrict__ part, double* __restrict__ scal,
                                                  unsigned int* __restrict__ cnt, int mode_in,
                                                  const int32_t* __restrict__ heavy, int nheavy, int64_t B0,
                                                  int64_t nB, const HeavyChunks hc) {
  const int mode = mode_in & 15;
  const bool dist = (mode_in & M_DIST) != 0;
  const int zs = (mode_in & M_ZS2) ? 2 : 1;
  pdl_wait();
  if (mode != M_APPLY && cnt[C_DONE]) return;
  const double rho = scal[S_SHIFT];
  const double ckk = lv.ck[k];
  const int32_t* cp = cptr + lv.cpo[k - 1];
  const double* Nk = Nsub + lv.off[k - 1];
  auto tf = [&](int64_t p) { return LEVEL1 ? yk[p] - rho : ckk * yk[p] - rho * Nk[p]; };
  double rz = 0.0;
  auto ef = [&](int64_t p, double z, double w) {
    if (LEVEL1) { rz += yk[p] * w; wk[zs * p] = w; }
    else { zk[p] = z; wk[p] = w; }
  };
  const int nnorm = (int)gridDim.x - nheavy - hc.nch;
  if ((int)blockIdx.x >= nnorm + nheavy) {  // a chunk of a heavy aggregate: no reduction needed
    const int4 sg = hc.seg[(int)blockIdx.x - nnorm - nheavy];
    const int64_t B = sg.x, s0 = cp[B];
    const double* ki = kinv + 3 * (lv.off[k] - lv.n[0] + B);
    const int64_t lb = 3 * (lv.lo[k - 1] - 2 * B - 2);
    const double kuu = ki[0], kuv = ki[1], kvv = ki[2];
    const double zb = zB[B], wbm = lv.negmu * wB[B];
    // sum_x C(x, j) t_x = c(k) S_j - rho K_j (t_x = c(k) y_x - rho N_x)
    const double au = tf(s0) + (ckk * hc.sum[2 * sg.w] - rho * hc.cst[2 * sg.w]);
    const double av = tf(s0 + 1) + (ckk * hc.sum[2 * sg.w + 1] - rho * hc.cst[2 * sg.w + 1]);
    const double zu = kuu * au + kuv * av, zv = kuv * au + kvv * av;
    if (threadIdx.x == 0 && sg.y == s0) {
      { const double z = zb + zu; ef(s0, z, z + wbm); }
      { const double z = zb + zv; ef(s0 + 1, z, z + wbm); }
    }
    for (int64_t p = max((int64_t)sg.y, s0 + 2) + threadIdx.x; p < sg.z; p += TPB) {
      const double zx = lof[lb + 3 * p + 2] * tf(p) + lof[lb + 3 * p + 0] * zu + lof[lb + 3 * p + 1] * zv;
      const double z = zb + zx;
      ef(p, z, z + wbm);
    }
  } else if ((int)blockIdx.x < nnorm) {
    const int64_t B = B0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (B < B0 + nB && cp[B + 1] - cp[B] <= HEAVY_AGG) {
      const double* ki = kinv + 3 * (lv.off[k] - lv.n[0] + B);
      const int64_t lb = 3 * (lv.lo[k - 1] - 2 * B - 2);
      block_solve(  // (an unrolled leftover loop measured slower on configs[4]: 1.26 -> 1.32 ms)
          cp[B], cp[B + 1], [&](int j) { return ki[j]; }, [&](int64_t p, int j) { return lof[lb + 3 * p + j]; },
          zB[B], lv.negmu * wB[B], tf, ef);
    }
  } else {  // a CTA per heavy aggregate: the leftover sums by a block reduction
    const int64_t B = heavy[blockIdx.x - nnorm];
    const int64_t s0 = cp[B], s1 = cp[B + 1];
    const double* ki = kinv + 3 * (lv.off[k] - lv.n[0] + B);
    const int64_t lb = 3 * (lv.lo[k - 1] - 2 * B - 2);
    const double kuu = ki[0], kuv = ki[1], kvv = ki[2];
    const double zb = zB[B], wbm = lv.negmu * wB[B];
    double su = 0.0, sv = 0.0;
    for (int64_t p = s0 + 2 + threadIdx.x; p < s1; p += TPB) {
      const double tx = tf(p);
      su += lof[lb + 3 * p + 0] * tx;
      sv += lof[lb + 3 * p + 1] * tx;
    }
    const double2 s2 = block_sum2<TPB>(make_double2(su, sv));
    const double au = tf(s0) + s2.x, av = tf(s0 + 1) + s2.y;
    const double zu = kuu * au + kuv * av, zv = kuv * au + kvv * av;
    if (threadIdx.x == 0) {
      { const double z = zb + zu; ef(s0, z, z + wbm); }
      { const double z = zb + zv; ef(s0 + 1, z, z + wbm); }
    }
    for (int64_t p = s0 + 2 + threadIdx.x; p < s1; p += TPB) {
      const double zx = lof[lb + 3 * p + 2] * tf(p) + lof[lb + 3 * p + 0] * zu + lof[lb + 3 * p + 1] * zv;
      const double z = zb + zx;
      ef(p, z, z + wbm);
    }
  }
  if (LEVEL1) {
    rz = block_sum<TPB>(rz);
    if (threadIdx.x == 0) part[blockIdx.x] = rz;
    if (mode != M_APPLY && last_block(&cnt[C_DOWN])) {
      const double tot = block_sum_partials<TPB>(part, gridDim.x);
      if (threadIdx.x == 0) {
        if (dist) scal[S_RZ] = tot;  // local total: the caller all-reduces
        else finish_rz(tot, scal, mode);
        cnt[C_DOWN] = 0;
      }
    }
  }
}

__global__ void __launch_bounds__(CT) k_coarse(const __grid_constant__ Lv lv_p, const __grid_constant__ CoarseDesc cd,
                                               const int32_t* __restrict__ cptr, const double* __restrict__ kinv,
                                               const double* __restrict__ lof, const double* __restrict__ Nsub,
                                               const double* __restrict__ pinv_g, const double* __restrict__ y0src,
                                               double* __restrict__ Zg, double* __restrict__ Wg,
                                               double* __restrict__ zout, const double* __restrict__ part_gd,
                                               int npart, double* __restrict__ scal, unsigned int* __restrict__ cnt,
                                               int mode_in, const double* __restrict__ mtop_g) {
  const int mode = mode_in & 15;
  const bool dist = (mode_in & M_DIST) != 0;
  extern __shared__ __align__(16) char sm[];
  __shared__ CoarseState C;
  __shared__ int sdone;
  // the level table is read level by level; a single CTA would take a cold
  // constant-cache miss at nearly every level, so it is copied to shared
  // memory once, all words in parallel
  __shared__ __align__(16) Lv slv;
  static_assert(sizeof(Lv) % 8 == 0, "Lv copied as 8-byte words");
  for (int i = threadIdx.x; i < (int)(sizeof(Lv) / 8); i += CT)
    reinterpret_cast<uint64_t*>(&slv)[i] = reinterpret_cast<const uint64_t*>(&lv_p)[i];
  const Lv& lv = slv;
  const int tid = threadIdx.x;
  TRACE(0);
  if (tid == 0) mbar_init(&C.bar, 1);
  __syncthreads();
  const int L = lv.L, Kc = lv.Kc, nl = cd.nl;
  coarse_stage_static<CT>(C, sm, lv, cd, cptr, kinv, lof, Nsub, pinv_g, mode == M_COLUMN ? nullptr : mtop_g);
  TRACE(1);
  pdl_wait();
  TRACE(2);
  if (tid == 0) sdone = (mode == M_INIT || mode == M_ITER) ? (int)cnt[C_DONE] : 0;
  __syncthreads();
  const int done = sdone;
  if (tid == 0 && !done) {
    // M_COLUMN (setup of the coarse GEMV matrix): CTA j solves for the j-th
    // unit input, whose y_Kc is row j of y0src (n_Kc x n_Kc identity, then 0)
    const int64_t base = (mode == M_COLUMN) ? (int64_t)blockIdx.x * lv.n[Kc - 1] : ((Kc == 1) ? 0 : lv.off[Kc - 1]);
    C.sky0 = stage_window(&C.bar, sm + cd.o_y[0], y0src, 8, base, base + lv.n[Kc - 1]);
  }
  __syncthreads();
  if (tid == 0) mbar_arrive(&C.bar);
  // small top (<= 32 nodes): the levels run on as many warps as they have
  // nodes for, the top solve on warp 0 (so gdot is summed there)
#ifndef MSP_NO_SMALLTOP
  const bool small_top = lv.n[L - 1] <= 32 && nl <= 14;
#else
  const bool small_top = false;
#endif
  double gd = 0.0;
  if (mode == M_COLUMN) {
    if (tid == 0) gd = ((int64_t)blockIdx.x == lv.n[Kc - 1]) ? 1.0 : 0.0;
  } else if (dist || mode != M_APPLY) {
    // summed by the up kernel's last CTA (all-reduced by the caller if dist)
    if (tid == 0 && !done) gd = scal[S_GD];
  } else if (small_top) {  // apply_R: the partials are summed here (warp 0 holds gdot)
    if (tid < 32) {
      const double t = warp_sum_partials(part_gd, npart);
      gd = (tid == 0) ? t : 0.0;
    }
  } else {
    for (int i = tid; i < npart; i += CT) gd += __ldcg(part_gd + i);
  }
  mbar_wait(&C.bar, 0);
  TRACE(3);
  if (done) return;
  coarse_table(C, lv, cd, 0);
  LvlPtr* tb = C.tb;
  const int skp = C.skp;
  if (small_top) {
    const double* pinv = cd.stage_pinv ? reinterpret_cast<const double*>(sm + cd.o_pinv) + skp : pinv_g;
    const bool map = cd.topmap_t > 0 && mode != M_COLUMN && mtop_g;
    const double* mtop = map ? reinterpret_cast<const double*>(sm + cd.o_mtop) + C.skm : nullptr;
    coarse_levels(lv, tb, sm, pinv, Zg, Wg, zout, scal, gd, mode_in, cd.o_tt, false, mtop, cd.topmap_t, cd.mtop_n);
    return;
  }
  // ---- up
  for (int t = 1; t < nl; ++t) {  // child level Kc+t-1, parent Kc+t
    __syncthreads();
    const int* cp = SMP(const int, tb[t].cp);
    const double* yc = SMP(const double, tb[t - 1].y);
    double* yp = SMP(double, tb[t].y);
    const int np = tb[t].cnt;
    #pragma unroll 1
    for (int i = tid; i < np; i += CT) {
      double y = 0.0;
      const int c1 = cp[i + 1];
      #pragma unroll 1
      for (int c = cp[i]; c < c1; ++c) y += yc[c];
      yp[i] = y;
    }
  }
  // ---- top solve
  __syncthreads();
  TRACE(7);
  const int ntop = tb[nl - 1].cnt;
  const double* yt = SMP(const double, tb[nl - 1].y);
  const double* Nt = SMP(const double, tb[nl - 1].nn);
  double ysum = 0.0;
  #pragma unroll 1
  for (int i = tid; i < ntop; i += CT) ysum += yt[i];
  {
    const double2 v = block_sum2<CT>(make_double2(ysum, gd));
    ysum = v.x;
    gd = v.y;
  }
  TRACE(8);
  const double rho = lv.c_sum * ysum / lv.n_tilde;
  double* tt = reinterpret_cast<double*>(sm + cd.o_tt);
  #pragma unroll 1
  for (int i = tid; i < ntop; i += CT) tt[i] = lv.ck[L] * yt[i] - rho * Nt[i];
  __syncthreads();
  const double* pinv = cd.stage_pinv ? reinterpret_cast<const double*>(sm + cd.o_pinv) + skp : pinv_g;
  double* zt = SMP(double, tb[nl - 1].z);
  double* wt = SMP(double, tb[nl - 1].w);
  double nz = 0.0;
  #pragma unroll 1
  for (int i = tid; i < ntop; i += CT) {
    double zi = 0.0;
    #pragma unroll 1
    for (int j = 0; j < ntop; ++j) zi += pinv[i * ntop + j] * tt[j];
    zt[i] = zi;
    nz += Nt[i] * zi;
  }
  TRACE(9);
  nz = block_sum<CT>(nz);
  TRACE(10);
  if (tid == 0 && mode != M_COLUMN) scal[S_SHIFT] = rho;
  const double m = (nz + gd - rho * lv.GN) / lv.n_tilde;
  double rz = 0.0;
  #pragma unroll 1
  for (int i = tid; i < ntop; i += CT) {
    const double z = zt[i] - m;
    zt[i] = z;
    wt[i] = z;
    if (L == 1) { rz += yt[i] * z; zout[((mode_in & M_ZS2) ? 2 : 1) * i] = z; }
  }
  TRACE(5);
  // ---- down
  const double negmu = lv.negmu;
  for (int t = nl - 2; t >= 0; --t) {  // child level k = Kc+t, parent k+1
    __syncthreads();
    const int* cp = SMP(const int, tb[t + 1].cp);
    const double* ki = SMP(const double, tb[t + 1].ki);
    const double* zp = SMP(const double, tb[t + 1].z);
    const double* wp = SMP(const double, tb[t + 1].w);
    const double* lo = SMP(const double, tb[t].lo);
    const double* yc = SMP(const double, tb[t].y);
    const double* nc = SMP(const double, tb[t].nn);
    double* zc = SMP(double, tb[t].z);
    double* wc = SMP(double, tb[t].w);
    const double ckk = tb[t].ck;
    const bool out1 = (Kc + t == 1);
    const int np = tb[t + 1].cnt;
    #pragma unroll 1
    for (int i = tid; i < np; i += CT) {
      const int lb = -3 * (2 * i + 2);
      block_solve(
          cp[i], cp[i + 1], [&](int j) { return ki[3 * i + j]; }, [&](int p, int j) { return lo[lb + 3 * p + j]; },
          zp[i], negmu * wp[i], [&](int p) { return out1 ? yc[p] - rho : ckk * yc[p] - rho * nc[p]; },
          [&](int p, double z, double w) {
            if (out1) { rz += yc[p] * w; zout[((mode_in & M_ZS2) ? 2 : 1) * p] = w; }
            else { zc[p] = z; wc[p] = w; }
          });
    }
  }
  __syncthreads();
  TRACE(6);
  pdl_trigger();
  if (mode == M_COLUMN) {  // column j of the GEMV matrix: [z_Kc; w_Kc]
    const int nk = tb[0].cnt;
    double* col = Zg + (int64_t)blockIdx.x * 2 * nk;
    const double* zc = SMP(const double, tb[0].z);
    const double* wc = SMP(const double, tb[0].w);
    for (int i = tid; i < nk; i += CT) { col[i] = zc[i]; col[nk + i] = wc[i]; }
  } else if (Kc > 1) {
    const int nk = tb[0].cnt;
    const int64_t base = lv.off[Kc - 1];
    const double* zc = SMP(const double, tb[0].z);
    const double* wc = SMP(const double, tb[0].w);
    for (int i = tid; i < nk; i += CT) { Zg[base + i] = zc[i]; Wg[base + i] = wc[i]; }
  } else {
    rz = block_sum<CT>(rz);
    if (tid == 0 && mode != M_APPLY) finish_rz(rz, scal, mode);
  }
}

// ------------------------------------------------------- unpreconditioned
// R = I: r -= alpha q, rr; z = r so rz = rr -> beta  (x deferred into L p)
__global__ void __launch_bounds__(TPB) k_update_cg(int64_t n, double* __restrict__ r, const double* __restrict__ q,
                                                   double* __restrict__ part, double* __restrict__ scal,
                                                   unsigned int* __restrict__ cnt, int mode, int set_rz) {
  pdl_wait();
  if (mode == M_ITER && cnt[C_DONE]) return;
  const double alpha = (mode == M_ITER) ? scal[S_ALPHA] : 0.0;
  double d = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double ri = r[i];
    if (mode == M_ITER) {
      ri -= alpha * q[i];
      r[i] = ri;
    }
    d += ri * ri;
  }
  pdl_trigger();
  d = block_sum<TPB>(d);
  if (threadIdx.x == 0) part[blockIdx.x] = d;
  if (last_block(&cnt[C_UPD])) {
    const double rr = block_sum_partials<TPB>(part, gridDim.x);
    if (threadIdx.x == 0) {
      finish_rr(rr, scal, cnt, mode);
      if (set_rz && !cnt[C_DONE]) finish_rz(rr, scal, mode);
      cnt[C_UPD] = 0;
    }
  }
}

// rz = (r, z) after an externally applied preconditioner -> beta, rho
__global__ void __launch_bounds__(TPB) k_rz(int64_t n, const double* __restrict__ r, const double* __restrict__ z,
                                            double* __restrict__ part, double* __restrict__ scal,
                                            unsigned int* __restrict__ cnt, int mode) {
  pdl_wait();
  double d = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d += r[i] * z[i];
  d = block_sum<TPB>(d);
  if (threadIdx.x == 0) part[blockIdx.x] = d;
  if (last_block(&cnt[C_DOWN])) {
    const double rz = block_sum_partials<TPB>(part, gridDim.x);
    if (threadIdx.x == 0) { finish_rz(rz, scal, mode); cnt[C_DOWN] = 0; }
  }
}

__global__ void k_init_state(double* scal, unsigned int* cnt, double rtol2) {
  pdl_wait();
  for (int i = 0; i < S_NSCAL; ++i) scal[i] = 0.0;
  for (int i = 0; i < C_NCNT; ++i) cnt[i] = 0;
  scal[S_RTOL2] = rtol2;
}

// ------------------------------------------------------------- host side
bool use_pdl() {
  static const bool on = std::getenv("MSP_NO_PDL") == nullptr;
  return on;
}

// launches of kernel category `cat` (1 plain SpMV, 2 pipelined SpMV, 4 tile
// up, 8 tile down, 16 per-level kernels) without the PDL attribute when its
// bit is set in MSP_NOPDL_MASK.  Default 3, the SpMVs: their grid-stride
// CTAs, launched early, land unevenly on the SMs the previous kernel is still
// leaving (without PDL there: configs[1] 64.0 -> 61.7, configs[2] 1362 -> 942,
// configs[3] 472 -> 426 us/iteration)
bool pdl_for(int cat) {
  static const int mask = std::getenv("MSP_NOPDL_MASK") ? std::atoi(std::getenv("MSP_NOPDL_MASK")) : 3;
  return use_pdl() && !(mask & cat);
}

template <typename... KArgs, typename... Args>
void launch_c(int cat, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_for(cat) ? 1 : 0;
  MSP_CUDA(cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...));
}

template <typename... KArgs, typename... Args>
void launch(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  MSP_CUDA(cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...));
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

// the scalars of one PCG step after a collective (the steps of a finished
// solve leave everything, the iteration count included, untouched)
__global__ void k_dist_finish(int stage, double* scal, unsigned int* cnt, int mode) {
  if (mode == M_ITER && cnt[C_DONE]) return;
  if (stage == 0) {
    scal[S_ALPHA] = scal[S_RHO] / scal[S_PQ];
  } else if (stage == 1) {
    finish_rr(scal[S_RR], scal, cnt, mode);
  } else if (!cnt[C_DONE] || mode == M_INIT) {
    finish_rz(scal[S_RZ], scal, mode);
  }
}

// One tier of the sweep schedule as one GPU (or one rank) runs it: the
// tier's layout and either its tiles (all of them, or a rank's clipped list)
// or, for a generic tier, the range of parent nodes [B0, B0 + nB) at level
// k0 + 1 with the heavy aggregates among them.
struct TierRun {
  bool generic = false;
  int k0 = 1, k1 = 1;
  const TierDesc* desc = nullptr;
  const int32_t* tstart = nullptr;
  const int32_t* firstk0 = nullptr;
  const int4* segs = nullptr;
  int64_t ntiles = 0;
  int up_group = 1, tpc = 1;
  int64_t B0 = 0, nB = 0;
  const int32_t* heavy = nullptr;
  int nheavy = 0;
  size_t smem_up = 0, smem_down = 0;
};

std::vector<TierRun> tier_runs(Handle& h) {
  std::vector<TierRun> v;
  for (auto& T : h.tiers) {
    TierRun t;
    t.generic = T.generic;
    t.k0 = T.k0;
    t.k1 = T.k1;
    if (T.generic) {
      const int k = T.k0;
      t.B0 = 0;
      t.nB = h.lv[k].n;
      t.heavy = h.heavy.p + h.heavy_off[k - 1];
      t.nheavy = (int)(h.heavy_off[k] - h.heavy_off[k - 1]);
    } else {
      t.desc = &T.desc;
      t.tstart = T.tstart.p;
      t.firstk0 = T.firstk0.p;
      t.segs = T.segs.p;
      t.ntiles = T.ntiles;
      t.up_group = T.up_group;
      t.tpc = T.desc.tpc;
      t.smem_up = T.smem_up;
      t.smem_down = T.smem_down;
    }
    v.push_back(t);
  }
  return v;
}

enum { PH_UP_LOW = 1, PH_UPPER = 2, PH_DOWN_LOW = 4, PH_ALL = 7 };

// The first tier's up sweep streamed (k_up_stream) instead of tile-staged
// (k_tile_up<true>): measured per iteration (us) staged -> streamed, configs[2]
// 839 -> 803, configs[3] 401 -> 392, configs[4] at scale 0.1 (a level-1-only
// tier) 292 -> 286, but configs[1] 60.5 -> 64.2 (its 1M-row problem is small
// enough that the staged kernel's prologue, TMA of r and H before the grid
// dependency, overlaps a large part of the SpMV's tail).  Streamed for
// level-1-only tiers and from 2^21 rows on; MSP_UP_STREAM=1 / 0 forces it.
bool use_up_stream(const Handle& h, const TierRun& T) {
  static const int v = std::getenv("MSP_UP_STREAM") ? std::atoi(std::getenv("MSP_UP_STREAM")) : -1;
  if (v >= 0) return v != 0;
  return T.k1 == T.k0 || h.n >= (int64_t(1) << 21);
}

// grid of k_up_stream: a few CTAs per SM (MSP_UPS_PER_SM), no more than the
// nodes (or elements) need
unsigned up_stream_grid(const Handle& h, const TierRun& T) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    MSP_CUDA(cudaGetDevice(&dev));
    MSP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  int per_sm = 4;
  if (const char* e = std::getenv("MSP_UPS_PER_SM")) per_sm = std::max(1, std::atoi(e));
  const int64_t need = (T.k1 == T.k0) ? (h.n + UT * 4 - 1) / (UT * 4)
                                      : (h.lv[T.k1 - 1].n + UT / MSP_FLAT_G - 1) / (UT / MSP_FLAT_G);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * per_sm));
}

// R r (MSP) on nested vectors.  mode APPLY: r -> z;  INIT / ITER: the PCG
// step (ITER first updates r) with the scalars of reading R10.  Tiers
// 0..tp are the "low" ones (a rank's own part when distributed: M_DIST makes
// their reductions rank-local totals, and the levels above run replicated);
// `phases` selects the up sweep of the low tiers, everything above them
// (upper tiers, coarse levels), and the down sweep of the low tiers.
void msp_sweeps_runs(Handle& h, const Lv& lv, const std::vector<TierRun>& runs, int tp, const double* q, double* r,
                     double* z, cudaStream_t st, int mode, Prof& P, int phases) {
  double* part_rr = h.red.p;                  // [cap/4]
  double* part_rz = h.red.p + h.red_cap / 4;
  double* part_gd = h.red.p + h.red_cap / 2;
  unsigned* cnt = h.counters.p;
  double* scal = h.scal.p;
  const int nt = (int)runs.size();
  const bool dist = (mode & M_DIST) != 0;
  // the first tier's up sweep streamed (k_up_stream) on one GPU
  const bool stream = !dist && !runs.empty() && !runs[0].generic && runs[0].k0 == 1 && use_up_stream(h, runs[0]);
  const unsigned sgrid = stream ? up_stream_grid(h, runs[0]) : 0u;
  const int npart_up = runs.empty() || runs[0].generic
                           ? 0
                           : stream ? (int)sgrid : (int)((runs[0].ntiles + runs[0].up_group - 1) / runs[0].up_group);
  auto up = [&](int i) {
    const TierRun& T = runs[i];
    const int md = (i <= tp) ? mode : (mode & ~M_DIST);
    P.begin();
    if (i == 0 && stream) {
      if (T.k1 == T.k0)
        launch_c(4, k_up_stream<true>, sgrid, UT, 0, st, (int64_t)0, (const int32_t*)nullptr, h.n, q, r,
                 (const double*)h.Hvec.p, (double*)nullptr, part_rr, part_gd, scal, cnt, md);
      else
        launch_c(4, k_up_stream<false>, sgrid, UT, 0, st, h.lv[T.k1 - 1].n, T.firstk0, h.n, q, r,
                 (const double*)h.Hvec.p, h.Y.p + h.lv[T.k1 - 1].off, part_rr, part_gd, scal, cnt, md);
      P.end(PC_TILE_UP);
    } else if (T.generic) {
      const int k = T.k0;
      const double* yin = (k == 1) ? r : h.Y.p + h.lv[k - 1].off;
      const HeavyChunks hc = dist ? HeavyChunks{} : h.heavy_chunks(k);
      const int nhv = hc.nch > 0 ? 0 : T.nheavy;
      launch_c(16, k_up_lvl, grid_for(std::max<int64_t>(T.nB, 1)) + nhv + hc.nch, TPB, 0, st, lv, k,
               (const int32_t*)h.cptr.p, yin, h.Y.p + h.lv[k].off, (const unsigned*)cnt, md, T.heavy, nhv, T.B0,
               T.nB, hc, (const double*)h.lof.p);
      P.end(PC_MID_UP);
    } else {
      const unsigned grid = (unsigned)std::max<int64_t>(1, (T.ntiles + T.up_group - 1) / T.up_group);
      if (T.k0 == 1)
        launch_c(4, k_tile_up<true>, grid, UT, T.smem_up, st, lv, *T.desc, T.tstart, T.firstk0, q, r,
                 (const double*)h.Hvec.p, h.Y.p, part_rr, part_gd, scal, cnt, md, 0);
      else
        launch_c(4, k_tile_up<false>, grid, UT, T.smem_up, st, lv, *T.desc, T.tstart, T.firstk0, q, r,
                 (const double*)h.Hvec.p, h.Y.p, part_rr, part_gd, scal, cnt, md & ~M_DIST, 0);
      P.end(T.k0 == 1 ? PC_TILE_UP : PC_MID_UP);
    }
    ++h.launches;
  };
  const bool merged = h.merged_coff > 0 && (!dist || tp < nt - 1);
  auto down = [&](int i) {
    const TierRun& T = runs[i];
    if (!T.generic && T.k1 == T.k0) return;  // the (1,1) update-only tier
    const int md = (i <= tp) ? mode : (mode & ~M_DIST);
    P.begin();
    if (T.generic) {
      const int k = T.k0;
      const int64_t ok = h.lv[k - 1].off, op = h.lv[k].off;
      const HeavyChunks hc = dist ? HeavyChunks{} : h.heavy_chunks(k);
      const int nhv = hc.nch > 0 ? 0 : T.nheavy;
      const unsigned grid = grid_for(std::max<int64_t>(T.nB, 1)) + nhv + hc.nch;
      if (k == 1)
        launch_c(16, k_down_lvl<true>, grid, TPB, 0, st, lv, k, (const int32_t*)h.cptr.p, (const double*)h.kinv.p,
                 (const double*)h.lof.p, (const double*)r, (const double*)h.Nsub.p, (const double*)(h.Z.p + op),
                 (const double*)(h.W.p + op), (double*)nullptr, z, part_rz, scal, cnt, md, T.heavy, nhv, T.B0,
                 T.nB, hc);
      else
        launch_c(16, k_down_lvl<false>, grid, TPB, 0, st, lv, k, (const int32_t*)h.cptr.p, (const double*)h.kinv.p,
                 (const double*)h.lof.p, (const double*)(h.Y.p + ok), (const double*)h.Nsub.p,
                 (const double*)(h.Z.p + op), (const double*)(h.W.p + op), h.Z.p + ok, h.W.p + ok, part_rz, scal,
                 cnt, md & ~M_DIST, T.heavy, nhv, T.B0, T.nB, hc);
      P.end(k == 1 ? PC_TILE_DOWN : PC_MID_DOWN);
    } else {
      if (T.k0 == 1 && !dist && h.wdown_grid > 0)
        launch_c(8, k_wtile_down, h.wdown_grid, WD * 32, (size_t)WD * h.wdown_region, st, lv, *T.desc, T.tstart,
                 (const int32_t*)h.cptr.p, (const double*)h.kinv.p, (const double*)h.lof.p, (const double*)r,
                 (const double*)h.Z.p, (const double*)h.W.p, z, part_rz, scal, cnt, md, T.segs, h.wdown_region);
      else if (T.k0 == 1)
        launch_c(8, k_tile_down<true>, (unsigned)std::max<int64_t>(1, (T.ntiles + T.tpc - 1) / T.tpc), TT,
                 T.smem_down, st, lv, *T.desc, T.tstart, (const int32_t*)h.cptr.p, (const double*)h.kinv.p,
                 (const double*)h.lof.p, (const double*)h.Nsub.p, (const double*)r, h.Z.p, h.W.p, z, part_rz, scal,
                 cnt, md, (const double*)h.Mco.p, (const double*)part_gd, npart_up, (const double*)h.Y.p, 0, T.segs,
                 h.cdesc, 0, (const double*)nullptr, (const double*)nullptr);
      else if (merged && i == nt - 1)  // the coarse levels run inside this kernel
        launch_c(8, k_tile_down<false, true>, (unsigned)T.ntiles, CT, h.merged_smem, st, lv, *T.desc, T.tstart,
                 (const int32_t*)h.cptr.p, (const double*)h.kinv.p, (const double*)h.lof.p, (const double*)h.Nsub.p,
                 (const double*)h.Y.p, h.Z.p, h.W.p, z, part_rz, scal, cnt, md & ~M_DIST, (const double*)h.Mco.p,
                 (const double*)part_gd, npart_up, (const double*)h.Y.p, 0, T.segs, h.cdesc, (int)h.merged_coff,
                 (const double*)h.top_pinv.p, (const double*)h.Mtop.p);
      else
        launch_c(8, k_tile_down<false>, (unsigned)std::max<int64_t>(1, T.ntiles), TT, T.smem_down, st, lv, *T.desc,
                 T.tstart, (const int32_t*)h.cptr.p, (const double*)h.kinv.p, (const double*)h.lof.p,
                 (const double*)h.Nsub.p, (const double*)h.Y.p, h.Z.p, h.W.p, z, part_rz, scal, cnt, md & ~M_DIST,
                 (const double*)h.Mco.p, (const double*)part_gd, npart_up, (const double*)h.Y.p, 0, T.segs, h.cdesc,
                 0, (const double*)nullptr, (const double*)nullptr);
      P.end(T.k0 == 1 ? PC_TILE_DOWN : PC_MID_DOWN);
    }
    ++h.launches;
  };
  if (phases & PH_UP_LOW)
    for (int i = 0; i <= tp && i < nt; ++i) up(i);
  if (phases & PH_UPPER) {
    for (int i = tp + 1; i < nt; ++i) up(i);
    // coarse (folded into the top tier's down kernel in GEMV mode, and into
    // the last tier's down kernel when merged)
    if (!h.gemv && !merged) {
      P.begin();
      const double* y0 = (h.Kc == 1) ? r : h.Y.p;
      launch(k_coarse, 1u, CT, h.coarse_smem, st, lv, h.cdesc, (const int32_t*)h.cptr.p, (const double*)h.kinv.p,
             (const double*)h.lof.p, (const double*)h.Nsub.p, (const double*)h.top_pinv.p, y0, h.Z.p, h.W.p, z,
             (const double*)part_gd, npart_up, scal, cnt, mode, (const double*)h.Mtop.p);
      P.end(PC_COARSE);
      ++h.launches;
    }
    for (int i = nt - 1; i > tp; --i) down(i);
  }
  if (phases & PH_DOWN_LOW)
    for (int i = std::min(tp, nt - 1); i >= 0; --i) down(i);
}

void msp_sweeps(Handle& h, const Lv& lv, const double* q, double* r, double* z, cudaStream_t st, int mode, Prof& P) {
  const std::vector<TierRun> runs = tier_runs(h);
  msp_sweeps_runs(h, lv, runs, (int)runs.size() - 1, q, r, z, st, mode, P, PH_ALL);
}

template <bool PCG>
void launch_spmv(Handle& h, const double* z, const double* pold, double* pnew, double* q, double* x,
                 cudaStream_t st, int64_t row0 = 0, int64_t row1 = -1) {
  if (row1 < 0) row1 = h.n;
  launch_c(1, k_spmv<PCG>, h.spmv_grid, TPB, 0, st, h.n, h.nslices, (const int64_t*)h.sell_ptr.p,
         (const int32_t*)h.sell_col.p, (const double*)h.sell_w.p, (const uint32_t*)h.sell_mask.p, h.nlong, h.huge_desc(),
         (const int32_t*)h.long_rows.p, (const int32_t*)h.rowptr1.p, (const int32_t*)h.col1.p,
         (const double*)h.w1.p, z, pold, pnew, q, x, h.red.p, h.scal.p, h.counters.p, row0, row1);
  ++h.launches;
}

// SpMV of the MSP iteration on interleaved (z, p) pairs (M_ZS2)
void launch_spmv_pairs(Handle& h, const double* zp_in, double* zp_out, double* q, double* x, cudaStream_t st,
                       int64_t row0 = 0, int64_t row1 = -1, bool hot_ok = true) {
  if (row1 < 0) row1 = h.n;
  const bool hot = hot_ok && h.nhot > 0;
  if (hot) {
    launch_c(16, k_hot_gather, (unsigned)std::min<int64_t>(grid_for(h.nhot), 148 * 8), TPB, 0, st, h.nhot,
             (const int32_t*)h.hot_rows.p, reinterpret_cast<const double2*>(zp_in),
             reinterpret_cast<double2*>(h.hot_pairs.p), (const unsigned*)h.counters.p);
    ++h.launches;
  }
  const int32_t* sc = hot ? h.sell_colh.p : h.sell_col.p;
  const int32_t* cc = hot ? h.col1h.p : h.col1.p;
  auto go = [&](auto kern) {
    launch_c(2, kern, h.spmv_grid, TPB, 0, st, h.n, h.nslices, (const int64_t*)h.sell_ptr.p, sc,
           (const double*)h.sell_w.p, (const uint32_t*)h.sell_mask.p, h.nlong, h.huge_desc(), (const int32_t*)h.long_rows.p,
           (const int32_t*)h.rowptr1.p, cc, (const double*)h.w1.p,
           reinterpret_cast<const double2*>(zp_in), zp_out, q, x, h.red.p, h.scal.p, h.counters.p, row0, row1,
           (const double*)nullptr, (const double*)nullptr, (double*)nullptr, h.nmed,
           reinterpret_cast<const double2*>(h.hot_pairs.p));
  };
  if (hot) {
    if (h.sell_uniform && h.sell_maxw == 4) go(k_spmv_pipe<4, true, false, true>);
    else if (h.sell_uniform && h.sell_maxw == 8) go(k_spmv_pipe<8, true, false, true>);
    else if (h.sell_maxw <= 4) go(k_spmv_pipe<4, false, false, true>);
    else if (h.sell_maxw <= 8) go(k_spmv_pipe<8, false, false, true>);
    else go(k_spmv_pipe<16, false, false, true>);
  } else if (h.sell_uniform && h.sell_maxw == 4) go(k_spmv_pipe<4, true>);
  else if (h.sell_uniform && h.sell_maxw == 6) go(k_spmv_pipe<6, true>);
  else if (h.sell_uniform && h.sell_maxw == 8) go(k_spmv_pipe<8, true>);
  else if (h.sell_maxw <= 4) go(k_spmv_pipe<4, false>);
  else if (h.sell_maxw <= 8) go(k_spmv_pipe<8, false>);
  else go(k_spmv_pipe<16, false>);
  ++h.launches;
}

// SpMV of the MSP iteration on separate z, p_old, p vectors (the pipelined
// kernel, full-sector stores)
void launch_spmv_sep(Handle& h, const double* z, const double* pold, double* pnew, double* q, double* x,
                     cudaStream_t st, int64_t row0 = 0, int64_t row1 = -1) {
  if (row1 < 0) row1 = h.n;
  auto go = [&](auto kern) {
    launch_c(2, kern, h.spmv_grid, TPB, 0, st, h.n, h.nslices, (const int64_t*)h.sell_ptr.p, (const int32_t*)h.sell_col.p,
             (const double*)h.sell_w.p, (const uint32_t*)h.sell_mask.p, h.nlong, h.huge_desc(),
             (const int32_t*)h.long_rows.p, (const int32_t*)h.rowptr1.p, (const int32_t*)h.col1.p, (const double*)h.w1.p,
             (const double2*)nullptr, (double*)nullptr, q, x, h.red.p, h.scal.p, h.counters.p, row0, row1, z, pold,
             pnew, h.nmed, (const double2*)nullptr);
  };
  if (h.sell_uniform && h.sell_maxw == 4) go(k_spmv_pipe<4, true, true>);
  else if (h.sell_uniform && h.sell_maxw == 6) go(k_spmv_pipe<6, true, true>);
  else if (h.sell_uniform && h.sell_maxw == 8) go(k_spmv_pipe<8, true, true>);
  else if (h.sell_maxw <= 4) go(k_spmv_pipe<4, false, true>);
  else if (h.sell_maxw <= 8) go(k_spmv_pipe<8, false, true>);
  else go(k_spmv_pipe<16, false, true>);
  ++h.launches;
}

// Separate vectors unless the graph has long (power-law hub) rows: a gather
// of (z_j, p_j) is then one sector instead of two, which wins on scattered
// neighbours (configs[4] at scale 0.1: 292 vs 304 us per iteration), while
// on meshes the pair layout's half-sector stores cost an L2 fill each
// (configs[2]: 941 -> 840, configs[1]: 61.4 -> 60.5 us per iteration with
// separate vectors).  MSP_SPMV_SEP=1 / 0 forces either.
bool use_sep(const Handle& h) {
  static const int mode = std::getenv("MSP_SPMV_SEP") ? std::atoi(std::getenv("MSP_SPMV_SEP")) : -1;
  static const bool off = std::getenv("MSP_NO_SPMV_PIPE") != nullptr;
  if (off || h.sell_maxw > 16) return false;
  if (mode >= 0) return mode == 1;
  return h.nlong == 0 && h.nhuge == 0;
}

bool use_pairs(const Handle& h) {
  static const bool off = std::getenv("MSP_NO_SPMV_PIPE") != nullptr;
  return !off && h.sell_maxw <= 16 && !use_sep(h);
}

// one PCG iteration (reading R10): p = z + beta p, q = L p (x += alpha p
// deferred), r -= alpha q, z = R r
void pcg_iteration(Handle& h, const Lv& lv, int precond, double* x, cudaStream_t st, Prof& P) {
  if (precond == MSP_PRECOND_MSP && use_pairs(h)) {
    double* zin = h.pparity ? h.zp2.p : h.zp1.p;
    double* zout = h.pparity ? h.zp1.p : h.zp2.p;
    h.pparity ^= 1;
    P.begin();
    launch_spmv_pairs(h, zin, zout, h.vq.p, x, st);
    P.end(PC_SPMV);
    msp_sweeps(h, lv, h.vq.p, h.vr.p, zout, st, M_ITER | M_ZS2, P);
    return;
  }
  double* pold = h.pparity ? h.vp2.p : h.vp.p;
  double* pnew = h.pparity ? h.vp.p : h.vp2.p;
  h.pparity ^= 1;
  const double* z = (precond == MSP_PRECOND_MSP) ? h.vz.p : h.vr.p;
  P.begin();
  if (precond == MSP_PRECOND_MSP && use_sep(h)) launch_spmv_sep(h, z, pold, pnew, h.vq.p, x, st);
  else launch_spmv<true>(h, z, pold, pnew, h.vq.p, x, st);
  P.end(PC_SPMV);
  if (precond == MSP_PRECOND_MSP) {
    msp_sweeps(h, lv, h.vq.p, h.vr.p, h.vz.p, st, M_ITER, P);
  } else {
    P.begin();
    launch(k_update_cg, std::min<unsigned>(grid_for(h.n), 148u * 8u), TPB, 0, st, h.n, h.vr.p,
           (const double*)h.vq.p, h.red.p, h.scal.p, h.counters.p, (int)M_ITER, 1);
    P.end(PC_TILE_UP);
    ++h.launches;
  }
}

}  // namespace

// The coarse levels Kc..L map (y_Kc, gdot) linearly to (z_Kc, w_Kc): run the
// coarse kernel once per unit input (n_Kc + 1 CTAs) and keep the map as a
// dense row-major matrix for the GEMV in the top tier's down kernel.
__global__ void k_unit_rows(int64_t nk, double* __restrict__ E) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < (nk + 1) * nk) E[i] = ((i / nk) == (i % nk)) ? 1.0 : 0.0;
}

__global__ void k_transpose(int64_t rows, int64_t cols, const double* __restrict__ C, double* __restrict__ M) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // i = r * cols + c of M
  if (i < rows * cols) M[i] = C[(i % cols) * rows + (i / cols)];
}

void build_coarse_matrix(Handle& h, cudaStream_t st) {
  if (!h.gemv) return;
  const int64_t nk = h.lv[h.Kc - 1].n;
  DBuf<double> E, C;
  E.alloc((nk + 1) * nk + 8);
  C.alloc(2 * nk * (nk + 1) + 8);
  h.Mco.alloc(2 * nk * (nk + 1) + 8);
  k_unit_rows<<<grid_for((nk + 1) * nk), TPB, 0, st>>>(nk, E.p);
  const Lv lv = make_level_table(h);
  launch(k_coarse, (unsigned)(nk + 1), CT, h.coarse_smem, st, lv, h.cdesc, (const int32_t*)h.cptr.p,
         (const double*)h.kinv.p, (const double*)h.lof.p, (const double*)h.Nsub.p, (const double*)h.top_pinv.p,
         (const double*)E.p, C.p, C.p, (double*)nullptr, (const double*)nullptr, 0, h.scal.p, h.counters.p,
         (int)M_COLUMN, (const double*)nullptr);
  k_transpose<<<grid_for(2 * nk * (nk + 1)), TPB, 0, st>>>(2 * nk, nk + 1, C.p, h.Mco.p);
  MSP_LAUNCH_CHECK();
  MSP_CUDA(cudaStreamSynchronize(st));
}

// Top map: when a coarse level j (Kc < j <= L-2) has at most 48 nodes, the
// levels j..L -- up-sweep, top solve, down-sweep -- are one linear map
// (y_j, gdot) -> (z_j, w_j) (the coarse GEMV idea of DESIGN.md, restricted to
// the few top levels, where each output is a sum of at most 49 products, not
// ~300): built here column by column by the coarse kernel itself (one CTA per
// unit input) and applied in coarse_levels by a small GEMV from shared memory.
void build_top_map(Handle& h, cudaStream_t st) {
  h.cdesc.topmap_t = 0;
  if (std::getenv("MSP_NO_TOPMAP") || h.gemv) return;
  const int L = h.levels, Kc = h.Kc, nl = L - Kc + 1;
  if (!(h.lv[L - 1].n <= 32 && nl <= 14)) return;  // the small-top coarse path only
  int j = 0;
  for (int k = Kc + 1; k <= L - 2; ++k)
    if (h.lv[k - 1].n <= 48) { j = k; break; }
  if (j == 0) return;
  const int64_t nj = h.lv[j - 1].n;
  const bool stage_pinv = h.lv[L - 1].n <= 32;
  const CoarseDesc cdj = coarse_desc(h, j, stage_pinv);
  Lv lvj = make_level_table(h);
  lvj.Kc = j;
  DBuf<double> E, C;
  E.alloc((nj + 1) * nj + 8);
  C.alloc(2 * nj * (nj + 1) + 8);
  h.Mtop.alloc(2 * nj * (nj + 1) + 8);
  k_unit_rows<<<grid_for((nj + 1) * nj), TPB, 0, st>>>(nj, E.p);
  raise_smem_limit((const void*)k_coarse, std::max<size_t>(h.coarse_smem, cdj.smem));
  launch(k_coarse, (unsigned)(nj + 1), CT, (size_t)cdj.smem, st, lvj, cdj, (const int32_t*)h.cptr.p,
         (const double*)h.kinv.p, (const double*)h.lof.p, (const double*)h.Nsub.p, (const double*)h.top_pinv.p,
         (const double*)E.p, C.p, C.p, (double*)nullptr, (const double*)nullptr, 0, h.scal.p, h.counters.p,
         (int)M_COLUMN, (const double*)nullptr);
  k_transpose<<<grid_for(2 * nj * (nj + 1)), TPB, 0, st>>>(2 * nj, nj + 1, C.p, h.Mtop.p);
  MSP_LAUNCH_CHECK();
  MSP_CUDA(cudaStreamSynchronize(st));
  h.cdesc.topmap_t = j - Kc;
  h.cdesc.mtop_n = (int)nj;
  h.cdesc.o_mtop = (int)((h.cdesc.smem + 15) & ~15);
  h.cdesc.smem = (int)((h.cdesc.o_mtop + (2 * nj * (nj + 1) + 2) * 8 + 15) & ~(int64_t)15);
  h.coarse_smem = h.cdesc.smem;
}

void raise_smem_limit(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;  // per device and kernel
  int dev = 0;
  MSP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cur[{dev, func}];
  if (bytes <= c) return;
  MSP_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  c = bytes;
}

void release_graph(Handle& h) {
  if (h.graph) cudaGraphExecDestroy(h.graph);
  h.graph = nullptr;
  h.graph_batch = 0;
}

void alloc_solve_workspace(Handle& h) {
  const int64_t nt = h.n_tilde;
  h.Y.alloc(nt + 8); h.Z.alloc(nt + 8); h.W.alloc(nt + 8);
  MSP_CUDA(cudaMemset(h.Y.p, 0, (nt + 8) * sizeof(double)));
  {
    int dev = 0, sms = 148;
    MSP_CUDA(cudaGetDevice(&dev));
    MSP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // pipelined SpMV: 4 CTAs/SM (its register budget); the plain one: 8
    // (configs[3]: 426 -> 397 us/iteration)
    int per_sm = (use_pairs(h) || use_sep(h)) ? 4 : 8;
    if (const char* e = std::getenv("MSP_SPMV_BLOCKS_PER_SM")) per_sm = std::max(1, std::atoi(e));
    const int64_t want = grid_for(std::max<int64_t>(h.nslices, 1) * 32);
    h.spmv_grid = (unsigned)std::min<int64_t>(want, (int64_t)sms * per_sm);
  }
  // partials: [0, cap/4) SpMV / rr, [cap/4, cap/2) rz, [cap/2, cap) gdot
  int64_t need = std::max<int64_t>({(int64_t)h.spmv_grid, (int64_t)grid_for(h.n), 1});
  for (auto& T : h.tiers) need = std::max<int64_t>(need, T.ntiles);
  if (h.lv.size() > 1) need = std::max<int64_t>(need, grid_for(h.lv[1].n));
  // generic level-1 down kernel: a block per 256 parents plus a CTA per heavy
  // aggregate or per heavy chunk, each with an (r, R r) partial
  need += (h.hch_off.empty() ? 0 : h.hch_off.back()) + (h.heavy_off.empty() ? 0 : h.heavy_off.back());
  h.red_cap = 4 * need + 64;
  h.red.alloc(h.red_cap);
  MSP_CUDA(cudaMemset(h.red.p, 0, h.red_cap * sizeof(double)));
  for (auto* v : {&h.vx, &h.vr, &h.vp, &h.vp2, &h.vq, &h.vz, &h.vb}) {
    v->alloc(h.n + 8);
    MSP_CUDA(cudaMemset(v->p, 0, (h.n + 8) * sizeof(double)));
  }
  for (auto* v : {&h.zp1, &h.zp2}) {
    v->alloc(2 * h.n + 8);
    MSP_CUDA(cudaMemset(v->p, 0, (2 * h.n + 8) * sizeof(double)));
  }
  h.counters.alloc(C_NCNT);
  h.scal.alloc(S_NSCAL);
  MSP_CUDA(cudaMemset(h.counters.p, 0, C_NCNT * sizeof(unsigned)));
  MSP_CUDA(cudaMemset(h.scal.p, 0, S_NSCAL * sizeof(double)));
  build_top_map(h, 0);  // may extend the coarse layout: before the attributes below
  size_t up = 0, down = 0;
  for (auto& T : h.tiers) { up = std::max(up, T.smem_up); down = std::max(down, T.smem_down); }
  for (auto f : {(const void*)k_tile_up<true>, (const void*)k_tile_up<false>})
    raise_smem_limit(f, up);
  for (auto f : {(const void*)k_tile_down<true>, (const void*)k_tile_down<false>})
    raise_smem_limit(f, down);
  // first tier down: tiles per CTA -- about one wave of resident CTAs, at most
  // 8 tiles each (configs[1..3]: 2 / 8 / 8 measured best or within 0.5 %)
  for (auto& T : h.tiers) {
    if (T.generic || T.k0 != 1 || T.k1 == T.k0) continue;
    int per_sm = 0, dev = 0, nsm = 0;
    MSP_CUDA(cudaFuncSetAttribute((const void*)k_tile_down<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    MSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_tile_down<true>, TT,
                                                           T.smem_down));
    MSP_CUDA(cudaGetDevice(&dev));
    MSP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t slots = std::max<int64_t>(1, (int64_t)per_sm * nsm);
    int tpc = (int)std::min<int64_t>(8, (T.ntiles + slots - 1) / slots);
    if (const char* e = std::getenv("MSP_DOWN_TPC")) tpc = std::max(1, std::atoi(e));
    T.desc.tpc = std::max(1, tpc);
  }
  for (auto f : {(const void*)k_tile_up<true>, (const void*)k_tile_up<false>, (const void*)k_tile_down<true>,
                 (const void*)k_tile_down<false>})
    MSP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  // warp-per-tile first-tier down kernel: WD regions per CTA, about one
  // wave of resident CTAs (each warp then strides over the tiles)
  h.wdown_grid = 0;
  if (h.wdown && !h.tiers.empty() && !h.tiers[0].generic && h.tiers[0].k0 == 1 && h.tiers[0].k1 > 1) {
    auto& T = h.tiers[0];
    h.wdown_region = (int)((T.smem_down + 127) & ~(size_t)127);
    const size_t smem = (size_t)WD * h.wdown_region;
    if (smem <= 220 * 1024) {
      raise_smem_limit((const void*)k_wtile_down, smem);
      MSP_CUDA(cudaFuncSetAttribute((const void*)k_wtile_down, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      int per_sm = 0, dev = 0, nsm = 0;
      MSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_wtile_down, WD * 32, smem));
      MSP_CUDA(cudaGetDevice(&dev));
      MSP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      const int64_t want = (T.ntiles + WD - 1) / WD;
      h.wdown_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)std::max(per_sm, 1) * nsm));
    }
  }
  raise_smem_limit((const void*)k_coarse, h.coarse_smem);
  // merged last-tier down + coarse kernel (tier k1 == Kc, small top)
  h.merged_coff = 0;
  h.merged_smem = 0;
  {
    const int L = h.levels, nlc = L - h.Kc + 1;
    const bool small_top = h.lv[L - 1].n <= 32 && nlc <= 14;
    if (!std::getenv("MSP_NO_MERGE") && !h.gemv && h.tiers.size() >= 2 && small_top && h.Kc > 1) {
      auto& T = h.tiers.back();
      if (!T.generic && T.k1 == h.Kc && T.k0 > 1) {
        const size_t coff = (T.smem_down + 15) & ~(size_t)15;
        const size_t tot = coff + h.coarse_smem;
        if (tot <= 220 * 1024) {
          raise_smem_limit((const void*)k_tile_down<false, true>, tot);
          h.merged_coff = std::max<size_t>(coff, 16);
          h.merged_smem = h.merged_coff + h.coarse_smem;
          // coarse levels on 16 warps beside the tile recompute when every
          // coarse level fits them (n_Kc <= 512)
          h.cdesc.overlap = (!std::getenv("MSP_NO_OVERLAP") && h.lv[h.Kc - 1].n <= 512) ? 1 : 0;
        }
      }
    }
  }

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
  launch_spmv<false>(h, x, nullptr, nullptr, y, nullptr, st);
}

void apply_R_msp_nested(Handle& h, const double* r, double* z, cudaStream_t st) {
  // r is read-only in APPLY mode (the tile kernels read it as y_1)
  Prof P(h, st);
  const Lv lv = make_level_table(h);
  msp_sweeps(h, lv, nullptr, const_cast<double*>(r), z, st, M_APPLY, P);
}

// PCG (reading R10) on nested-numbered vectors b -> x.
void pcg_nested(Handle& h, int precond, const double* b, double* x, double rtol, int maxit, cudaStream_t st,
                msp_report* rep) {
  const int64_t n = h.n;
  const Lv lv = make_level_table(h);
  cudaEvent_t e0, e1;
  MSP_CUDA(cudaEventCreate(&e0));
  MSP_CUDA(cudaEventCreate(&e1));
  const int64_t launches0 = h.launches;
  MSP_CUDA(cudaEventRecord(e0, st));
  // x = 0, r = b, p_old = 0, scalars; z = R r, rho = (r, z), beta = 0
  MSP_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  MSP_CUDA(cudaMemcpyAsync(h.vr.p, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  h.pparity = 0;
  MSP_CUDA(cudaMemsetAsync(h.vp.p, 0, n * sizeof(double), st));
  launch(k_init_state, 1u, 1u, 0, st, h.scal.p, h.counters.p, rtol * rtol);
  ++h.launches;
  {
    Prof P(h, st);
    if (precond == MSP_PRECOND_MSP && use_pairs(h)) {
      MSP_CUDA(cudaMemsetAsync(h.zp1.p, 0, 2 * n * sizeof(double), st));
      msp_sweeps(h, lv, nullptr, h.vr.p, h.zp1.p, st, M_INIT | M_ZS2, P);
    } else if (precond == MSP_PRECOND_MSP) {
      msp_sweeps(h, lv, nullptr, h.vr.p, h.vz.p, st, M_INIT, P);
    } else if (precond == MSP_PRECOND_NONE) {
      launch(k_update_cg, std::min<unsigned>(grid_for(n), 148u * 8u), TPB, 0, st, n, h.vr.p, (const double*)nullptr,
             h.red.p, h.scal.p, h.counters.p, (int)M_INIT, 1);
      ++h.launches;
    }
  }
  unsigned host_cnt[C_NCNT];
  if (precond == MSP_PRECOND_PEGP) {
    // PEGP: the inner solve is host-driven, so iterations run one by one
    unsigned hc[C_NCNT];
    auto flag = [&]() {
      MSP_CUDA(cudaMemcpyAsync(hc, h.counters.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
      return hc[C_DONE] != 0;
    };
    const unsigned gv = std::min<unsigned>(grid_for(n), 148u * 8u);
    launch(k_update_cg, gv, TPB, 0, st, n, h.vr.p, (const double*)nullptr, h.red.p, h.scal.p, h.counters.p,
           (int)M_INIT, 0);
    h.pegp_solve_inner = 0;
    if (!flag()) {
      apply_R_pegp_nested(h, h.vr.p, h.vz.p, st);
      h.pegp_solve_inner += h.pegp_last_inner;
      launch(k_rz, gv, TPB, 0, st, n, (const double*)h.vr.p, (const double*)h.vz.p, h.red.p, h.scal.p, h.counters.p,
             (int)M_INIT);
      for (int it = 0; it < maxit; ++it) {
        double* pold = h.pparity ? h.vp2.p : h.vp.p;
        double* pnew = h.pparity ? h.vp.p : h.vp2.p;
        h.pparity ^= 1;
        launch_spmv<true>(h, h.vz.p, pold, pnew, h.vq.p, x, st);
        launch(k_update_cg, gv, TPB, 0, st, n, h.vr.p, (const double*)h.vq.p, h.red.p, h.scal.p, h.counters.p,
               (int)M_ITER, 0);
        h.launches += 2;
        if (flag()) break;
        apply_R_pegp_nested(h, h.vr.p, h.vz.p, st);
        h.pegp_solve_inner += h.pegp_last_inner;
        launch(k_rz, gv, TPB, 0, st, n, (const double*)h.vr.p, (const double*)h.vz.p, h.red.p, h.scal.p,
               h.counters.p, (int)M_ITER);
        ++h.launches;
      }
    }
  } else {
  // iterations in batches; a batch is a captured CUDA graph (even length so
  // the p / p_old ping-pong is periodic), the done flag read once per batch
  int batch = 64;  // 16 / 32 / 64 / 128 measured: 75.6 / 75.2 / 74.9 / 74.9 us per iteration
  if (const char* e = std::getenv("MSP_PCG_BATCH")) batch = std::max(2, std::atoi(e) & ~1);
  const bool use_graph = !h.profile && std::getenv("MSP_NO_GRAPH") == nullptr;
  int it = 0;
  Prof P(h, st);
  while (it < maxit) {
    const int nb = std::min(batch, maxit - it);
    if (use_graph && nb == batch) {
      if (!h.own_stream) {
        MSP_CUDA(cudaStreamCreateWithFlags(&h.own_stream, cudaStreamNonBlocking));
        MSP_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
        MSP_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
      }
      cudaStream_t gs = h.own_stream;
      const int key = batch * 4 + precond;
      if (h.graph && h.graph_batch != key) release_graph(h);
      MSP_CUDA(cudaEventRecord(h.ev_fork, st));
      MSP_CUDA(cudaStreamWaitEvent(gs, h.ev_fork, 0));
      if (!h.graph) {
        const int64_t l0 = h.launches;
        cudaGraph_t g;
        MSP_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        for (int b2 = 0; b2 < nb; ++b2) pcg_iteration(h, lv, precond, x, gs, P);
        MSP_CUDA(cudaStreamEndCapture(gs, &g));
        MSP_CUDA(cudaGraphInstantiate(&h.graph, g, 0));
        cudaGraphDestroy(g);
        h.graph_batch = key;
        h.graph_launches = h.launches - l0;
      } else {
        h.launches += h.graph_launches;
      }
      MSP_CUDA(cudaGraphLaunch(h.graph, gs));
      MSP_CUDA(cudaEventRecord(h.ev_join, gs));
      MSP_CUDA(cudaStreamWaitEvent(st, h.ev_join, 0));
    } else {
      for (int b2 = 0; b2 < nb; ++b2) pcg_iteration(h, lv, precond, x, st, P);
    }
    it += nb;
    P.flush();
    MSP_CUDA(cudaMemcpyAsync(host_cnt, h.counters.p, sizeof(host_cnt), cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    if (host_cnt[C_DONE]) break;
  }
  }
  if (precond == MSP_PRECOND_MSP && use_pairs(h))
    launch(k_x_final_pairs, std::min<unsigned>(grid_for(n), 148u * 8u), TPB, 0, st, n, x, (const double*)h.zp1.p,
           (const double*)h.zp2.p, (const double*)h.scal.p, (const unsigned*)h.counters.p);
  else
    launch(k_x_final, std::min<unsigned>(grid_for(n), 148u * 8u), TPB, 0, st, n, x, (const double*)h.vp.p,
           (const double*)h.vp2.p, (const double*)h.scal.p, (const unsigned*)h.counters.p);
  ++h.launches;
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
    rep->solve_ms = ms;
    rep->kernel_launches = h.launches - launches0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace msp

#ifdef MSP_TRACE
extern "C" int msp_debug_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, msp::g_trace, sizeof(msp::g_trace)) == cudaSuccess ? 0 : -2;
}
extern "C" int msp_debug_phase(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, msp::g_phase, sizeof(msp::g_phase)) != cudaSuccess) return -2;
  if (reset) {
    static unsigned long long z[8][16] = {};
    if (cudaMemcpyToSymbol(msp::g_phase, z, sizeof(z)) != cudaSuccess) return -2;
  }
  return 0;
}
#endif

namespace msp {

// One rank of the partitioned PCG-MSP solve (msp_dist_solve), nested vectors.
#include "dist_solve.cuh"

}  // namespace msp

