// internal.cuh -- private types and helpers of libmsp_b200.so (sm_100a).
// Not part of the C ABI (include/msp_b200.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/msp_b200.h"

namespace msp {

enum { PC_SPMV = 0, PC_UPDATE, PC_UP1, PC_UPC, PC_TOP, PC_DOWNC, PC_DOWN1, PC_PUPD };

// ---------------------------------------------------------------- errors
struct Error {
  int code;
  std::string msg;
};
void set_error(const std::string& m);

#define MSP_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::msp::Error{MSP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                           " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
  } while (0)

#define MSP_LAUNCH_CHECK() MSP_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- device buffer
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) MSP_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  T* get() const { return p; }
};

// One level of the aggregation hierarchy.
//   Canonical numbering (reading R3) is what the MWM produces and what the
//   oracle uses; nested numbering is the GPU layout (every aggregate of every
//   level is a contiguous range of the level below).
struct LevelHost {
  int64_t n = 0;          // n_k
  int64_t nnz = 0;        // entries of the level-k adjacency CSR
  int64_t off = 0;        // offset of level k in the expanded (n~) vector
};

// Device-resident state of a handle.
struct Handle {
  // ---- problem
  int64_t n = 0, nnz_adj = 0;  // vertices, adjacency entries (2m)
  double mu = 0.8;
  uint64_t seed = 0;
  int32_t levels = 0, mwm_rounds = 0, top_max = 256, levels_req = 0;
  double setup_ms = 0.0;
  std::vector<LevelHost> lv;   // k = 1..l  (index k-1)
  int64_t n_tilde = 0;

  // ---- canonical hierarchy (kept for parity queries)
  std::vector<DBuf<int32_t>> agg_canon;   // [l-1]: level-k canonical -> level-(k+1) canonical
  std::vector<DBuf<int64_t>> canon_rowptr;  // [l]: canonical CSR of each level
  std::vector<DBuf<int32_t>> canon_col;
  std::vector<DBuf<double>> canon_w;
  std::vector<DBuf<int32_t>> nested_of_canon;  // [l]: canonical id -> nested position
  std::vector<DBuf<int32_t>> order_nested;     // [l]: nested position -> canonical id
  std::vector<DBuf<int32_t>> mates_canon;      // [l-1]: matched partner or <0 (leftover)
  std::vector<DBuf<double>> apar_canon;        // [l-1]: MSP parent-edge weight per node

  // ---- solve-phase layout (nested numbering)
  DBuf<int32_t> perm;         // nested position -> original vertex (level 1)
  DBuf<int32_t> rowptr1;      // level-1 adjacency in nested numbering (int32 offsets)
  DBuf<int32_t> col1;
  DBuf<double> w1;
  DBuf<int32_t> cptr;         // concatenated child pointers: level k block at cptr_off[k-1]
  std::vector<int64_t> cptr_off;
  DBuf<double> c0, c1, c2;    // per expanded node (nested): block-tree factor data
  DBuf<double> Nsub;          // subtree sizes N_i (double)
  DBuf<double> gvec;          // g = K_S^{-1} N_S per node
  DBuf<double> top_pinv;      // dense (sigma_l L_l)^+ of the top level, nested order
  double c_sum = 0.0;         // sum_{k=1}^{l} (-mu)^{k-1}
  double GN = 0.0;            // sum over non-top nodes g_i N_i
  std::vector<double> neg_mu_pow;  // (-mu)^j, j = 0..l

  // ---- solve workspaces
  DBuf<double> Y, S, Z, W;    // n~-layout sweep vectors
  DBuf<double> red;           // reduction partials
  DBuf<double> vx, vr, vp, vq, vz, vb;  // PCG vectors (nested numbering)
  DBuf<unsigned int> counters;
  DBuf<double> scal;          // device scalars of PCG
  DBuf<double> stage_in, stage_out;   // host-mode staging
  int64_t red_cap = 0;
  int64_t launches = 0;       // kernels launched (counted on the host)
  int profile = 0;            // bracket solve launches with events (msp_set_profiling)
  double prof_ms[MSP_PROF_NCAT] = {0};
  int64_t prof_cnt[MSP_PROF_NCAT] = {0};
};

// setup.cu
void validate_csr(Handle& h, const int64_t* rowptr, const int32_t* col, const double* w,
                  cudaStream_t st);
void build_setup(Handle& h, const int64_t* rowptr, const int32_t* col, const double* w,
                 cudaStream_t st);
// solve.cu
void apply_L_nested(Handle& h, const double* x, double* y, cudaStream_t st);
void apply_R_msp_nested(Handle& h, const double* r, double* z, cudaStream_t st);
void gather_to_nested(Handle& h, const double* src_orig, double* dst_nested, cudaStream_t st);
void scatter_from_nested(Handle& h, const double* src_nested, double* dst_orig, cudaStream_t st);
void pcg_nested(Handle& h, int precond, const double* b, double* x, double rtol, int maxit,
                cudaStream_t st, msp_report* rep);
void alloc_solve_workspace(Handle& h);

}  // namespace msp
