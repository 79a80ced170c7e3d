// internal.cuh -- private types and helpers of libmsp_b200.so (sm_100a).
// Not part of the C ABI (include/msp_b200.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/msp_b200.h"
#include "sched.cuh"

namespace msp {

constexpr int HEAVY_AGG = 64;

enum { PC_SPMV = 0, PC_TILE_UP, PC_MID_UP, PC_COARSE, PC_MID_DOWN, PC_TILE_DOWN, PC_PEGP_SPMV, PC_PEGP_SWEEPS };

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

// cudaFuncAttributeMaxDynamicSharedMemorySize is per kernel and process-wide:
// raise it to the largest request any handle has made, never lower it (a
// second, smaller handle must not break launches of a larger one).  The
// occupancy of a launch depends on the bytes it passes, not on this cap.
void raise_smem_limit(const void* func, size_t bytes);

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

struct DistRank;                 // dist_solve.cuh: one rank's partition, plan and communicator
void dist_free(DistRank* d);

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
  // heavy aggregates (more than HEAVY_AGG children), per parent level k+1:
  // nested ids heavy[heavy_off[k-1] .. heavy_off[k]) -- a CTA each in the
  // per-level sweep kernels
  DBuf<int32_t> heavy;
  std::vector<int64_t> heavy_off;
  // their chunks (sched.cuh HeavyChunks), per parent level k+1: chunks
  // hch_off[k-1] .. hch_off[k)
  DBuf<int4> hch_seg;
  std::vector<int64_t> hch_off;
  DBuf<int32_t> hch_first;
  DBuf<unsigned> hch_cnt;
  DBuf<double> hch_part, hch_sum, hch_cst;
  HeavyChunks heavy_chunks(int k) const {  // parent level k+1
    if (hch_off.empty() || hch_off[k] == hch_off[k - 1]) return HeavyChunks{nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    return HeavyChunks{hch_seg.p + hch_off[k - 1], (int)(hch_off[k] - hch_off[k - 1]), hch_first.p, hch_cnt.p,
                       hch_part.p, hch_sum.p, hch_cst.p, (int)hch_off[k - 1]};
  }
  // MSP block-tree factors, packed:
  //   kinv[3 (off_{k+1} - n + B) + {0,1,2}] = K'^{-1} (uu, uv, vv) of aggregate B at level k+1
  //   lof[3 (lo_off[k-1] + p - 2B - 2) + {0,1,2}] = (s w_xu / d, s w_xv / d, 1 / d) of leftover p
  DBuf<double> kinv, lof;
  std::vector<int64_t> lo_off;  // [l]: first leftover slot of the level-k children
  DBuf<double> Nsub;          // subtree sizes N_i (double)
  DBuf<double> gvec;          // g = K_S^{-1} N_S per node
  DBuf<double> Hvec;          // [n]: gdot weights, gdot = (r, H)
  DBuf<double> top_pinv;      // dense (sigma_l L_l)^+ of the top level, nested order
  double c_sum = 0.0;         // sum_{k=1}^{l} (-mu)^{k-1}
  double GN = 0.0;            // sum over non-top nodes g_i N_i
  std::vector<double> neg_mu_pow;  // (-mu)^j, j = 0..l

  // ---- level-1 Laplacian in SELL-32 (slices of 32 rows, column-major,
  // padded with (self, 0)); rows of degree > LCAP are "long": empty in SELL,
  // flagged in sell_mask and handled warp-per-row from the nested CSR
  int64_t nslices = 0, nlong = 0, nhuge = 0, nmed = 0;  // long_rows: [0, nmed) medium, [nmed, nlong) long, then huge  // long rows: warp per row; huge: CTA per row (after them)
  int sell_maxw = 0;          // widest slice (padded row length)
  bool sell_uniform = false;  // every slice padded to sell_maxw (no slice pointers needed)
  DBuf<int64_t> sell_ptr;
  DBuf<int32_t> sell_col;
  DBuf<double> sell_w;
  DBuf<uint32_t> sell_mask;
  DBuf<int32_t> long_rows;
  // hot-vertex gather cache (power-law graphs): the nhot highest-degree rows
  // (hot_rows, by decreasing degree), their (z, p) pairs copied each
  // iteration into hot_pairs (L2-resident), and column copies in which a hot
  // column j reads HOT_BIT | rank(j)
  int64_t nhot = 0;
  DBuf<int32_t> hot_rows, sell_colh, col1h;
  DBuf<double> hot_pairs;
  // huge rows cut into segments (sched.cuh HugeDesc)
  DBuf<int4> hseg;
  DBuf<int32_t> hfirst;
  DBuf<unsigned> hcnt;
  DBuf<double> hpart;
  int64_t nhseg = 0;
  DBuf<double> hdot;
  HugeDesc huge_desc() const { return HugeDesc{hseg.p, nhseg, hfirst.p, hcnt.p, hpart.p, hdot.p, nhuge}; }

  // ---- solve schedule: tiers of tile
  // kernels over levels 1..Kc, then one single-CTA kernel for Kc..L
  struct Tier {
    int32_t k0 = 1, k1 = 1;
    int64_t ntiles = 0;
    DBuf<int32_t> tstart;     // [k1-k0+1][ntiles+1]: first level-(k0+t) node of tile j
    size_t smem_up = 0, smem_down = 0;
    bool generic = false;     // one level by per-node kernels (an aggregate too large to tile)
    TierDesc desc{};
    DBuf<int32_t> firstk0;    // [n_k1 + 1]: first level-k0 descendant of each level-k1 node
    DBuf<int4> segs;          // [ntiles][desc.nseg] static segments of the down kernel (sched.cuh)
    int up_group = 1;         // tiles per CTA of the up kernel
  };
  std::vector<Tier> tiers;
  // first tier's down sweep by k_wtile_down (a warp per tile): grid and
  // per-warp shared-memory region
  bool wdown = false;
  unsigned wdown_grid = 0;
  int wdown_region = 0;
  int32_t Kc = 1;
  size_t coarse_smem = 0;
  CoarseDesc cdesc{};
  // coarse levels Kc..L as a dense map:
  // [z_Kc; w_Kc] = Mco [y_Kc; gdot], row-major (2 n_Kc) x (n_Kc + 1)
  bool gemv = false;
  DBuf<double> Mco;
  DBuf<double> Mtop;          // top map (CoarseDesc::topmap_t), row-major (2 n_j) x (n_j + 1)
  std::vector<double> ck;     // c(k) = sum_{j<k} (-mu)^j, k = 0..L (ck[0] unused)
  unsigned spmv_grid = 1;
  size_t merged_coff = 0, merged_smem = 0;  // merged last-tier down + coarse kernel (0: off)

  // ---- PEGP (built lazily on first use, pegp.cu)
  bool pegp_ready = false;
  DBuf<int32_t> parent;       // [n~]: expanded index of the parent aggregate, -1 on top
  DBuf<int64_t> hrow;         // explicit CSR of the H~ edge weights over n~ (nested; no diagonal)
  DBuf<int32_t> hcol;
  DBuf<double> hw;
  int64_t hnnz = 0;
  DBuf<int32_t> hrows;        // H~ rows by degree class (short / warp / CTA rows), nested order within
  int64_t hclass[3] = {0, 0, 0};
  DBuf<int4> hseg2;           // long-row segments (pegp.cu HMat)
  DBuf<int32_t> hlnseg;
  DBuf<double> hsegpart, hlpq;
  DBuf<unsigned> hltick;
  int64_t hnseg = 0;
  DBuf<double> ex, er, eq, es, ey, eres, ecor;  // expanded-space CG vectors
  DBuf<double> ezp[2];        // (z, p) pairs of the inner CG, ping-pong
  DBuf<double> edots, epart, eup, ezs, espmv_part;  // device scalars, block partials
  DBuf<unsigned> etick;       // ticket counters of the inner CG
  int pegp_Kc = 1;            // levels above pegp_Kc run in the single coarse CTA
  double pegp_rtol = 1e-13;
  int pegp_maxit = 5000;
  int pegp_refine = 0;        // refinement steps after the inner CG (reading R13)
  double pegp_build_ms = 0.0; // H~ assembly time (device)
  int64_t pegp_solve_inner = 0;  // inner iterations of the last PCG-PEGP solve
  int pegp_last_inner = 0;
  DistRank* dist = nullptr;   // msp_dist_init / the loopback group

  // ---- solve workspaces
  DBuf<double> Y, Z, W;       // n~-layout sweep vectors (y = P^T sums, z, w)
  DBuf<double> red;           // reduction partials
  DBuf<double> vx, vr, vp, vq, vz, vb;  // PCG vectors (nested numbering)
  DBuf<double> vp2;           // ping-pong partner of vp (p = z + beta p fused into L p)
  DBuf<double> zp1, zp2;      // MSP path: interleaved (z_i, p_i) pairs, ping-pong
  int pparity = 0;            // which of vp / vp2 holds the current p
  cudaGraphExec_t graph = nullptr;  // captured batch of PCG iterations
  cudaGraphExec_t pegp_graph = nullptr;  // captured batch of PEGP inner CG iterations
  int64_t pegp_graph_launches = 0;
  const double* pegp_graph_z = nullptr;  // the output vector the PEGP graph was captured with
  int graph_batch = 0;
  int64_t graph_launches = 0;
  cudaStream_t own_stream = nullptr;  // capture / replay stream of the graph
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DBuf<unsigned int> counters;
  DBuf<double> scal;          // device scalars of PCG
  DBuf<double> stage_in, stage_out;   // host-mode staging
  int64_t red_cap = 0;
  int64_t launches = 0;       // kernels launched (counted on the host)
  int profile = 0;            // bracket solve launches with events (msp_set_profiling)
  double prof_ms[MSP_PROF_NCAT] = {0};
  int64_t prof_cnt[MSP_PROF_NCAT] = {0};
  Handle() = default;
  Handle(const Handle&) = delete;
  ~Handle() {
    if (dist) dist_free(dist);
    if (graph) cudaGraphExecDestroy(graph);
    if (pegp_graph) cudaGraphExecDestroy(pegp_graph);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
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
DistRank* dist_build(Handle& h, int world, int rank, const void* id128, cudaStream_t st);
void pcg_dist_group(std::vector<Handle*>& hs, bool loop, double rtol, int maxit, cudaStream_t st, msp_report* rep);
void dist_unique_id(void* id128);
void dist_range(const Handle& h, int64_t* out8);
void add_into(Handle& h, const double* a, double* y, cudaStream_t st);
void alloc_solve_workspace(Handle& h);
void build_schedule(Handle& h, cudaStream_t st);   // setup.cu: tiers, tiles, Kc
void build_heavy_chunks(Handle& h, cudaStream_t st);  // setup.cu: chunks of the heavy aggregates
void build_hot_cache(Handle& h, cudaStream_t st);     // setup.cu: hot-vertex gather cache
// pegp.cu
void pegp_build(Handle& h, cudaStream_t st);
void apply_LH_nested(Handle& h, const double* x, double* y, cudaStream_t st);
void apply_LT_pinv_nested(Handle& h, const double* rt, double* z, cudaStream_t st);
int solve_LH_nested(Handle& h, const double* rt, double* z, cudaStream_t st);
void apply_R_pegp_nested(Handle& h, const double* r, double* z, cudaStream_t st);
void expanded_to_nested(Handle& h, const double* src, double* dst, cudaStream_t st);
void nested_to_expanded(Handle& h, const double* src, double* dst, cudaStream_t st);
Lv make_level_table(const Handle& h);              // setup.cu
void release_graph(Handle& h);
void build_coarse_matrix(Handle& h, cudaStream_t st);  // solve.cu
void build_top_map(Handle& h, cudaStream_t st);        // solve.cu
CoarseDesc coarse_desc(const Handle& h, int Kc, bool stage_pinv);  // setup.cu
std::vector<int4> make_tile_segs(const Handle& h, int k0, int nl, const TierDesc& d, const std::vector<int32_t>& ts,
                                 int64_t ntiles);                   // setup.cu

}  // namespace msp
