// sched.cuh -- solve-schedule data shared by setup.cu (host: layout) and
// solve.cu (device: kernels).  Private to libmsp_b200.so.
//
// A tier covers levels k0..k1 of the nested hierarchy.  Its tiles are
// contiguous ranges of level-k1 nodes; by the nested numbering a tile's
// descendants form one contiguous range at every level k0..k1, so a tile is
// processed by one CTA with every intermediate level in shared memory.  The
// shared-memory layout of a tier is fixed on the host (one slot per level and
// array, sized for the largest tile), so a CTA only computes its TMA windows:
// thread i stages segment i with a 1-D TMA bulk copy (cp.async.bulk).
#pragma once

#include <stdint.h>

namespace msp {

constexpr int MAXL = 40;   // levels

// Rows of degree > hcap ("huge", power-law hubs: up to millions of entries)
// are cut into segments of at most HUGE_SEG entries, a CTA each in the SpMV;
// the CTA that finishes a row's last segment (ticket cnt[row]) sums the
// row's partials in segment order (deterministic) and writes the row.
constexpr int HUGE_SEG = 16384;
constexpr int32_t HOT_BIT = 1 << 30;  // column flag: read the hot-vertex cache (rank in the low bits)
constexpr int MED_ROW = 64;  // medium rows (lcap < degree <= MED_ROW): 8 lanes per row in the SpMV
struct HugeDesc {
  const int4* seg;       // [nseg]: x = huge-row index (into long_rows[nlong + x]), y = e0, z = e1
  int64_t nseg;
  const int32_t* first;  // [nhuge + 1]: first segment of each huge row
  unsigned* cnt;         // [nhuge]: arrival tickets (zero between launches)
  double* part;          // [nseg]: segment partial sums
  double* dot;           // [nhuge]: the row's p_i (L p)_i, added to (p, q) in row order by the
                         // SpMV's last block (which CTA finishes a row varies run to run)
  int64_t nhuge;
};
constexpr int MAXT = 16;   // levels per tier

// Heavy aggregates (more than HEAVY_AGG children; power-law hubs hold up to
// millions) of one parent level, cut into chunks of at most HEAVY_CHUNK
// children, a CTA each in the generic per-level sweeps.  The up kernel sums
// y and the leftover-weighted sums S_j = sum_x C(x, j) y_x (j = 0, 1) per
// chunk; the CTA that finishes an aggregate's last chunk (ticket cnt[h])
// adds the chunk partials in chunk order (deterministic).  The down kernel's
// chunks then need no reduction: sum_x C(x, j) t_x = c(k) S_j - rho K_j with
// K_j = sum_x C(x, j) N_x fixed at setup.
constexpr int HEAVY_CHUNK = 4096;
struct HeavyChunks {
  const int4* seg;      // [nch]: x = aggregate B (nested, parent level), y = first child, z = end, w = heavy index h
  int nch;              // chunks of this level (0: CTA-per-aggregate path)
  const int32_t* first; // [nheavy_total + 1]: first chunk (global) of heavy aggregate h
  unsigned* cnt;        // [nheavy_total]: tickets (zero between launches)
  double* part;         // [3 * chunks_total]: per-chunk (sum y, S_0, S_1)
  double* sum;          // [2 * nheavy_total]: (S_0, S_1) of the last up sweep
  const double* cst;    // [2 * nheavy_total]: (K_0, K_1)
  int c0;               // global index of this level's first chunk
};

struct Lv {
  int L, Kc;
  int64_t n[MAXL];     // n_k                           (index k-1)
  int64_t off[MAXL];   // offset of level k in n~ vectors
  int64_t cpo[MAXL];   // children of level-(k+1) nodes start at cptr + cpo[k-1]
  int64_t lo[MAXL];    // first leftover slot of the level-k children
  double ck[MAXL + 1]; // c(k) = sum_{j<k} (-mu)^j, k = 1..L
  double negmu, c_sum, n_tilde, GN;
};

// Shared-memory layout of one tier (byte offsets, 16-byte aligned), t = level
// k0+t.  Staged windows start at the 16-byte-aligned element at or below the
// tile's first element; the skew (0..3 elements) is kept per CTA.
struct TierDesc {
  int k0, nl, ntiles;
  int o_cp[MAXT];  // child pointers of level-(k0+t) parents, t >= 1 (int32)
  int o_ki[MAXT];  // K'^{-1} triples of level-(k0+t) aggregates, t >= 1
  int o_lo[MAXT];  // leftover triples of level-(k0+t) children, t <= nl-2
  int o_y[MAXT];   // y of level k0+t: t = 0 staged (or computed in FIRST up), 1..nl-2 computed
  int o_n[MAXT];   // N of level k0+t: t = 0 staged (k0 > 1), 1..nl-2 computed
  int o_z[MAXT];   // z, w of level k0+t: t = nl-1 staged, 1..nl-2 computed
  int o_w[MAXT];
  int o_v;         // GEMV input [y_Kc; gdot] (top tier in GEMV mode), -1 otherwise
  int gemv_n;      // n_Kc when this tier's down kernel forms z, w at Kc by the GEMV
  int smem_down;
  // up kernel (its own layout): first level-k0 descendant of each level-k1
  // node of the tile (int32, [a, b]) and y at level k0
  int o_uf, o_uy0, o_uq, o_uh, smem_up;
  int up_group;    // tiles per CTA of the up kernel (1 when distributed)
  int nseg;        // static (constant-data) segments per tile of the down kernel
  int tpc;         // tiles per CTA of the down kernel (first tier; one after another)
};

// One static TMA segment of a tile of the down kernel, precomputed at setup
// (the window stage_window would compute): x = kind | t << 2 | dst << 8
// (kind 0 child pointers, 1 factors, 2 leftover coefficients, 3 N_k0; t the
// tier level; dst the shared-memory byte offset), y = bytes (0: nothing to
// copy), z = first element of the 16-byte aligned window, w = skew.
enum { SEG_CP = 0, SEG_KI = 1, SEG_LO = 2, SEG_N0 = 3 };

// coarse kernel (levels Kc..L, one CTA), t = level Kc+t; same conventions,
// every range is a whole level
struct CoarseDesc {
  int nl, stage_pinv;
  int o_cp[MAXT + 8], o_ki[MAXT + 8], o_lo[MAXT + 8], o_n[MAXT + 8];
  int o_y[MAXT + 8], o_z[MAXT + 8], o_w[MAXT + 8];
  int o_pinv, o_tt;
  // top map: levels j..L replaced by the dense linear map (y_j, gdot) ->
  // (z_j, w_j), j = Kc + topmap_t (0: off), n_j = mtop_n, staged at o_mtop
  int topmap_t, mtop_n, o_mtop;
  int overlap;  // merged kernel: coarse levels on warps 0..15 while warps 16..31 recompute the tile
  int smem;
};

}  // namespace msp
