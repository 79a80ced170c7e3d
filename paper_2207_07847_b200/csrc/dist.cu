// dist.cu -- row partition and halo plan of the multi-GPU solve (host code;
// no CUDA calls, so it runs and is tested without a GPU).
//
// The graph is partitioned at the first tier's tiles:
// rank r owns a contiguous range of tier-1 tiles, hence a contiguous range of
// level-1 rows and, by the nested numbering, every level of their subtrees up
// to the first tier's top level k1.  Levels above k1 are replicated.  The
// only data-path exchanges are the SpMV halo (p values of the neighbour rows a
// rank's rows reference) and the all-gather of y at level k1.
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/msp_b200.h"

namespace {

// first tile whose first row is >= target
int64_t lower_tile(const int32_t* tile_rows, int64_t ntiles, int64_t target) {
  return std::lower_bound(tile_rows, tile_rows + ntiles + 1, (int32_t)std::min<int64_t>(target, INT32_MAX)) -
         tile_rows;
}

}  // namespace

extern "C" {

int msp_partition_plan(int64_t n, const int32_t* rowptr, const int32_t* col, int64_t ntiles,
                       const int32_t* tile_rows, int32_t world, int32_t rank, int64_t* range,
                       int64_t* recv_counts, int64_t* send_counts, int64_t* recv_rows, int64_t recv_cap,
                       int64_t* send_rows, int64_t send_cap) {
  if (n < 1 || !rowptr || !col || ntiles < 1 || !tile_rows || world < 1 || rank < 0 || rank >= world || !range ||
      !recv_counts || !send_counts)
    return MSP_ERR_ARG;
  if (tile_rows[0] != 0 || tile_rows[ntiles] != n) return MSP_ERR_ARG;
  // tile boundaries of every rank, balanced by rows
  std::vector<int64_t> tb(world + 1), rb(world + 1);
  tb[0] = 0;
  tb[world] = ntiles;
  for (int r = 1; r < world; ++r) tb[r] = std::max(tb[r - 1], lower_tile(tile_rows, ntiles, (n * r) / world));
  for (int r = 0; r <= world; ++r) rb[r] = tile_rows[tb[r]];
  // every rank must own at least one tile: the check depends only on the
  // shared inputs, so all ranks fail together, before any collective
  for (int r = 0; r < world; ++r)
    if (tb[r + 1] <= tb[r]) return MSP_ERR_UNSUPPORTED;
  const int64_t r0 = rb[rank], r1 = rb[rank + 1];
  range[0] = r0;
  range[1] = r1;
  range[2] = tb[rank];
  range[3] = tb[rank + 1];
  auto owner = [&](int64_t j) {
    return (int)(std::upper_bound(rb.begin(), rb.end(), j) - rb.begin()) - 1;
  };
  // recv: neighbour columns outside [r0, r1), unique, grouped by owner (sorted)
  std::vector<int64_t> halo;
  // send: own rows with a neighbour in peer q's range, per q (sorted)
  std::vector<std::vector<int64_t>> snd(world);
  for (int64_t i = r0; i < r1; ++i) {
    int last_q = -1;
    std::vector<int> qs;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t j = col[e];
      if (j >= r0 && j < r1) continue;
      halo.push_back(j);
      const int q = owner(j);
      if (q != last_q) qs.push_back(q);
      last_q = q;
    }
    std::sort(qs.begin(), qs.end());
    qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
    for (int q : qs) snd[q].push_back(i);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  for (int q = 0; q < world; ++q) { recv_counts[q] = 0; send_counts[q] = (int64_t)snd[q].size(); }
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
