// dist.cu -- host-side partition and halo plan of the multi-GPU solve (no
// CUDA calls: runs and is tested without a GPU).
//
// Partition: the ranks split the nodes of one
// "partition level" kp of the nested hierarchy into contiguous ranges,
// balanced by a prefix cost (the solve's per-row work: adjacency entries plus
// a per-row constant); by the nested numbering a rank then owns a contiguous
// range of every level k <= kp -- the subtrees of its level-kp nodes, down to
// its level-1 rows.  Levels above kp are replicated.  The data-path
// exchanges are the SpMV halo (p of the neighbour rows the own rows
// reference), the all-gather of y at level kp, and three all-reduces.
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/msp_b200.h"

extern "C" {

int msp_dist_boundaries(int64_t m, const int64_t* cost, int32_t world, int64_t* bnd) {
  if (m < 1 || !cost || world < 1 || !bnd) return MSP_ERR_ARG;
  for (int64_t i = 0; i < m; ++i)
    if (cost[i + 1] < cost[i]) return MSP_ERR_ARG;
  const long double tot = (long double)(cost[m] - cost[0]);
  bnd[0] = 0;
  bnd[world] = m;
  for (int r = 1; r < world; ++r) {
    const long double target = (long double)cost[0] + tot * r / world;
    // first node whose prefix cost reaches the target
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((long double)cost[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    bnd[r] = lo;
  }
  // every rank must own at least one node: the check depends only on the
  // shared inputs, so all ranks fail together, before any collective
  for (int r = 0; r < world; ++r)
    if (bnd[r + 1] <= bnd[r]) return MSP_ERR_UNSUPPORTED;
  return MSP_OK;
}

int msp_halo_plan(int64_t n, const int32_t* rowptr, const int32_t* col, int32_t world, const int64_t* row_bnd,
                  int32_t rank, int64_t* recv_counts, int64_t* send_counts, int64_t* recv_rows, int64_t recv_cap,
                  int64_t* send_rows, int64_t send_cap) {
  if (n < 1 || !rowptr || !col || world < 1 || rank < 0 || rank >= world || !row_bnd || !recv_counts ||
      !send_counts)
    return MSP_ERR_ARG;
  if (row_bnd[0] != 0 || row_bnd[world] != n) return MSP_ERR_ARG;
  for (int r = 0; r < world; ++r)
    if (row_bnd[r + 1] <= row_bnd[r]) return MSP_ERR_UNSUPPORTED;
  const int64_t r0 = row_bnd[rank], r1 = row_bnd[rank + 1];
  auto owner = [&](int64_t j) {
    return (int)(std::upper_bound(row_bnd, row_bnd + world + 1, j) - row_bnd) - 1;
  };
  // recv: neighbour columns outside [r0, r1), unique, sorted (hence grouped by
  // owner); send: own rows with a neighbour in peer q's range, per q, sorted.
  // The graph is symmetric, so what r sends to q is what q receives from r,
  // in the same (increasing row) order.
  std::vector<int64_t> halo;
  std::vector<std::vector<int64_t>> snd(world);
  std::vector<int> qs;
  for (int64_t i = r0; i < r1; ++i) {
    qs.clear();
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t j = col[e];
      if (j >= r0 && j < r1) continue;
      halo.push_back(j);
      qs.push_back(owner(j));
    }
    std::sort(qs.begin(), qs.end());
    qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
    for (int q : qs) snd[q].push_back(i);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  for (int q = 0; q < world; ++q) {
    recv_counts[q] = 0;
    send_counts[q] = (int64_t)snd[q].size();
  }
  for (int64_t j : halo) recv_counts[owner(j)] += 1;
  if (recv_rows) {
    if ((int64_t)halo.size() > recv_cap) return MSP_ERR_ARG;
    std::copy(halo.begin(), halo.end(), recv_rows);
  }
  if (send_rows) {
    int64_t tot = 0;
    for (auto& v : snd) tot += (int64_t)v.size();
    if (tot > send_cap) return MSP_ERR_ARG;
    int64_t k = 0;
    for (auto& v : snd)
      for (int64_t i : v) send_rows[k++] = i;
  }
  return MSP_OK;
}

}  // extern "C"
