// sched.cuh -- solve-schedule data shared by setup.cu (host: sizing) and
// solve.cu (device: kernels).  Private to libmsp_b200.so.
//
// A tier covers levels k0..k1 of the nested hierarchy.  Its tiles are
// contiguous ranges of level-k1 nodes; by the nested numbering a tile's
// descendants form one contiguous range at every level k0..k1, so a tile is
// processed by one CTA with every intermediate level in shared memory.  The
// constant data a tile needs (child pointers, factors) and its inputs are
// staged into shared memory with 1-D TMA bulk copies (cp.async.bulk); the
// layout below is computed identically on the host (to size the dynamic
// shared memory) and on the device.
#pragma once

#include <stdint.h>

namespace msp {

constexpr int MAXL = 40;   // levels
constexpr int MAXT = 24;   // levels per tier

struct Lv {
  int L, Kc;
  int64_t n[MAXL];     // n_k                           (index k-1)
  int64_t off[MAXL];   // offset of level k in n~ vectors
  int64_t cpo[MAXL];   // children of level-(k+1) nodes start at cptr + cpo[k-1]
  int64_t lo[MAXL];    // first leftover slot of the level-k children
  double ck[MAXL + 1]; // c(k) = sum_{j<k} (-mu)^j, k = 1..L
  double negmu, c_sum, n_tilde, GN;
};

// One staged (or computed) shared-memory segment.  Element e of the level's
// index space lives at smem byte soff + (e - org) * elem.  nbytes > 0: bytes
// to bulk-copy from the source array starting at absolute element gstart.
struct Seg {
  int32_t soff;
  int32_t nbytes;
  int64_t gstart;
  int64_t org;
};

struct TileLayout {
  // tile_down segments, t = level k0 + t
  Seg cp[MAXT];   // child pointers of level-(k0+t) parents, t >= 1
  Seg ki[MAXT];   // K_S^{-1} of level-(k0+t) aggregates, t >= 1
  Seg lo[MAXT];   // leftover coefficients of level-(k0+t) children, t <= nl-2
  Seg y0, n0;     // y and N at level k0 (n0 only when k0 > 1)
  Seg zt, wt;     // z and w at level k1
  Seg y[MAXT], nn[MAXT], z[MAXT], w[MAXT];  // computed, 1 <= t <= nl-2
  int32_t total;  // bytes
};

struct TileLayoutUp {
  Seg cp[MAXT];   // child pointers of level-(k0+t) parents, t >= 1
  Seg y0;         // level-k0 input (staged when k0 > 1; computed from r when k0 == 1)
  Seg y[MAXT];    // computed, 1 <= t <= nl-2
  int32_t total;
};

__host__ __device__ inline int32_t align16(int64_t b) { return (int32_t)((b + 15) & ~(int64_t)15); }

// staged window of elements [lo, hi) (absolute in the source array, element
// size es): 16-byte aligned start and length.  org = origin in level indices.
__host__ __device__ inline int32_t stage(Seg& s, int32_t cur, int64_t lo, int64_t hi, int es, int64_t base) {
  const int64_t per = 16 / es;
  const int64_t a0 = (lo / per) * per;
  int64_t e0 = ((hi + per - 1) / per) * per;
  if (hi <= lo) e0 = a0;
  s.soff = align16(cur);
  s.nbytes = (int32_t)((e0 - a0) * es);
  s.gstart = a0;
  s.org = a0 - base;
  return s.soff + s.nbytes;
}

__host__ __device__ inline int32_t computed(Seg& s, int32_t cur, int64_t count, int es, int64_t org) {
  s.soff = align16(cur);
  s.nbytes = 0;
  s.gstart = 0;
  s.org = org;
  return s.soff + (int32_t)(count * es);
}

// a[t], b[t]: the tile's level-(k0+t) range, t = 0..nl-1 (nl = k1-k0+1 >= 2)
__host__ __device__ inline int32_t tile_layout_down(const Lv& lv, int k0, int nl, const int64_t* a,
                                                    const int64_t* b, TileLayout& T) {
  const int64_t n1 = lv.n[0];
  int32_t cur = 0;
  for (int t = 1; t < nl; ++t) {
    const int k = k0 + t;  // parent level
    cur = stage(T.cp[t], cur, lv.cpo[k - 2] + a[t], lv.cpo[k - 2] + b[t] + 1, 4, lv.cpo[k - 2]);
  }
  for (int t = 1; t < nl; ++t) {
    const int k = k0 + t;
    const int64_t base = 3 * (lv.off[k - 1] - n1);
    cur = stage(T.ki[t], cur, base + 3 * a[t], base + 3 * b[t], 8, base);
  }
  for (int t = 0; t + 1 < nl; ++t) {
    const int k = k0 + t;  // child level
    const int64_t base = 3 * lv.lo[k - 1];
    cur = stage(T.lo[t], cur, base + 3 * (a[t] - 2 * a[t + 1]), base + 3 * (b[t] - 2 * b[t + 1]), 8, base);
  }
  const int64_t b0 = (k0 == 1) ? 0 : lv.off[k0 - 1];
  cur = stage(T.y0, cur, b0 + a[0], b0 + b[0], 8, b0);
  if (k0 > 1) cur = stage(T.n0, cur, b0 + a[0], b0 + b[0], 8, b0);
  else T.n0 = Seg{0, 0, 0, 0};
  const int64_t bt = lv.off[k0 + nl - 2];
  cur = stage(T.zt, cur, bt + a[nl - 1], bt + b[nl - 1], 8, bt);
  cur = stage(T.wt, cur, bt + a[nl - 1], bt + b[nl - 1], 8, bt);
  for (int t = 1; t + 1 < nl; ++t) {
    const int64_t s = b[t] - a[t];
    cur = computed(T.y[t], cur, s, 8, a[t]);
    cur = computed(T.nn[t], cur, s, 8, a[t]);
    cur = computed(T.z[t], cur, s, 8, a[t]);
    cur = computed(T.w[t], cur, s, 8, a[t]);
  }
  T.total = align16(cur);
  return T.total;
}

__host__ __device__ inline int32_t tile_layout_up(const Lv& lv, int k0, int nl, const int64_t* a, const int64_t* b,
                                                  TileLayoutUp& T) {
  int32_t cur = 0;
  for (int t = 1; t < nl; ++t) {
    const int k = k0 + t;
    cur = stage(T.cp[t], cur, lv.cpo[k - 2] + a[t], lv.cpo[k - 2] + b[t] + 1, 4, lv.cpo[k - 2]);
  }
  if (k0 == 1) {
    cur = computed(T.y0, cur, b[0] - a[0], 8, a[0]);
  } else {
    const int64_t b0 = lv.off[k0 - 1];
    cur = stage(T.y0, cur, b0 + a[0], b0 + b[0], 8, b0);
  }
  for (int t = 1; t + 1 < nl; ++t) cur = computed(T.y[t], cur, b[t] - a[t], 8, a[t]);
  T.total = align16(cur);
  return T.total;
}

// coarse kernel (levels Kc..L, one CTA): everything staged / computed
struct CoarseLayout {
  Seg cp[MAXT];   // child pointers of level-(Kc+t) parents, t >= 1
  Seg ki[MAXT];   // K_S^{-1} of level-(Kc+t) aggregates, t >= 1
  Seg lo[MAXT];   // leftover coefficients of level-(Kc+t) children
  Seg nn[MAXT];   // N of level Kc+t
  Seg y0;         // y at level Kc
  Seg pinv;       // dense top pseudo-inverse (when staged)
  Seg y[MAXT], z[MAXT], w[MAXT], tt;
  int32_t total;
};

__host__ __device__ inline int32_t coarse_layout(const Lv& lv, bool stage_pinv, CoarseLayout& C) {
  const int Kc = lv.Kc, L = lv.L, nl = L - Kc + 1;
  const int64_t n1 = lv.n[0];
  int32_t cur = 0;
  for (int t = 1; t < nl; ++t) {
    const int k = Kc + t;
    cur = stage(C.cp[t], cur, lv.cpo[k - 2], lv.cpo[k - 2] + lv.n[k - 1] + 1, 4, lv.cpo[k - 2]);
    const int64_t base = 3 * (lv.off[k - 1] - n1);
    cur = stage(C.ki[t], cur, base, base + 3 * lv.n[k - 1], 8, base);
  }
  for (int t = 0; t + 1 < nl; ++t) {
    const int k = Kc + t;
    const int64_t base = 3 * lv.lo[k - 1];
    cur = stage(C.lo[t], cur, base, base + 3 * (lv.n[k - 1] - 2 * lv.n[k]), 8, base);
  }
  for (int t = 0; t < nl; ++t) {
    const int k = Kc + t;
    cur = stage(C.nn[t], cur, lv.off[k - 1], lv.off[k - 1] + lv.n[k - 1], 8, lv.off[k - 1]);
  }
  const int64_t b0 = (Kc == 1) ? 0 : lv.off[Kc - 1];
  cur = stage(C.y0, cur, b0, b0 + lv.n[Kc - 1], 8, b0);
  const int64_t ntop = lv.n[L - 1];
  if (stage_pinv) cur = stage(C.pinv, cur, 0, ntop * ntop, 8, 0);
  else C.pinv = Seg{0, 0, 0, 0};
  for (int t = 1; t < nl; ++t) cur = computed(C.y[t], cur, lv.n[Kc + t - 1], 8, 0);
  for (int t = 0; t < nl; ++t) {
    cur = computed(C.z[t], cur, lv.n[Kc + t - 1], 8, 0);
    cur = computed(C.w[t], cur, lv.n[Kc + t - 1], 8, 0);
  }
  cur = computed(C.tt, cur, ntop, 8, 0);
  C.total = align16(cur);
  return C.total;
}

}  // namespace msp
