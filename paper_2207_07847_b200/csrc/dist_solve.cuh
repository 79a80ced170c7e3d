// dist_solve.cuh -- the partitioned (multi-GPU) PCG-MSP solve; included by
// solve.cu inside namespace msp (it uses solve.cu's kernels and sweeps).
//
// Partition (dist.cu): rank r owns the nodes
// [lo_k(r), hi_k(r)) of every level k <= kp (the subtrees of its range at
// the partition level kp, which is the top level of tier tp).  Tiers 0..tp
// run on the owned part only -- a tier's tiles clipped at the rank's range
// (a tile is a set of whole subtrees, so a clipped tile still is one), a
// generic tier on the owned parent range -- with rank-local reductions
// (M_DIST); the tiers above tp and the coarse levels run replicated, on y_kp
// all-gathered from every rank.  One PCG iteration:
//
//   pack p = z + beta p_old of the rows peers reference -> halo exchange ->
//   rows received go into the pair buffer as (p, 0) -> SpMV on own rows
//   (p, q) local -> all-reduce -> alpha -> up sweep of tiers 0..tp (r -= alpha
//   q, (r, r), gdot and y up to kp, local) -> all-gather [y_kp own, (r, r),
//   gdot] -> convergence test -> tiers above tp, coarse, down sweep of tiers
//   0..tp ((r, R r) local) -> all-reduce -> beta.
//
// Every step is stream-ordered on the device: NCCL calls (one process per
// GPU), or -- to run and test the same decomposition on one GPU -- a
// "loopback group" of W ranks' handles in one process on one stream, whose
// collectives are device copies and fixed-order sums.  Nothing waits on the
// host inside an iteration; batches of iterations are captured as one CUDA
// graph and the host reads the (replicated) done flag once per batch.
// (nccl.h, <cstring> and <memory> are included at the top of solve.cu)

#define MSP_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      throw ::msp::Error{MSP_ERR_CUDA, std::string(#call) + ": " + ncclGetErrorString(r_)};    \
  } while (0)

struct DistRank {
  int world = 1, rank = 0;
  int tp = 0, kp = 1;
  std::vector<int64_t> bnd_kp;                 // [world+1] boundaries at level kp
  std::vector<std::vector<int64_t>> lvl_bnd;   // [kp][world+1]: boundaries at level k (index k-1)
  int64_t row0 = 0, row1 = 0, kp_max = 1;
  std::vector<TierRun> runs;                   // every tier (0..tp: this rank's part)
  std::vector<TierDesc> descs;
  std::vector<DBuf<int32_t>> tstarts, heavies;
  std::vector<DBuf<int4>> segs;
  std::vector<int64_t> send_cnt, recv_cnt, send_off, recv_off;
  int64_t nsend = 0, nrecv = 0;
  DBuf<int32_t> send_idx, recv_idx;
  DBuf<double> sendbuf, recvbuf, gsend, grecv;
  ncclComm_t comm = nullptr;
  ~DistRank() {
    if (comm) ncclCommDestroy(comm);
  }
};

void dist_free(DistRank* d) { delete d; }

__global__ void k_zero_outside(int64_t n, int64_t r0, int64_t r1, double* __restrict__ x);

namespace {

// p of the rows peers need: sendbuf[k] = z + beta p_old at send row k (z at
// z[s i], p_old at po[s i]: the pair buffer (s = 2, po = z + 1) or two arrays)
__global__ void k_halo_pack(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ z,
                            const double* __restrict__ po, int s, double* __restrict__ out,
                            const double* __restrict__ scal, const unsigned* __restrict__ cnt) {
  if (cnt[C_DONE]) return;
  const double beta = scal[S_BETA];
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) {
    const int64_t i = idx[k];
    out[k] = z[s * i] + beta * po[s * i];
  }
}

// received p as (z, p_old) = (p, 0): the SpMV's z + beta p_old is then p
__global__ void k_halo_unpack(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ in,
                              double* __restrict__ z, double* __restrict__ po, int s,
                              const unsigned* __restrict__ cnt) {
  if (cnt[C_DONE]) return;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) {
    const int64_t j = idx[k];
    z[s * j] = in[k];
    po[s * j] = 0.0;
  }
}

// all-gather payload of one rank: [y_kp on its range, padded to M - 2, (r, r), gdot]
__global__ void k_pack_y(int64_t cnt, const double* __restrict__ y, const double* __restrict__ scal,
                         double* __restrict__ out, int64_t M) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < M - 2) out[i] = (i < cnt) ? y[i] : 0.0;
  if (i == M - 2) out[i] = scal[S_RR];
  if (i == M - 1) out[i] = scal[S_GD];
}

struct Bnd16 {
  int64_t b[17];
};

// every rank's y_kp range into Y; (r, r) and gdot summed in rank order
__global__ void k_unpack_y(int world, Bnd16 bnd, const double* __restrict__ g, int64_t M, double* __restrict__ ykp,
                           double* __restrict__ scal) {
  for (int q = 0; q < world; ++q) {
    const int64_t c = bnd.b[q + 1] - bnd.b[q];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x)
      ykp[bnd.b[q] + i] = g[q * M + i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double rr = 0.0, gd = 0.0;
    for (int q = 0; q < world; ++q) { rr += g[q * M + M - 2]; gd += g[q * M + M - 1]; }
    scal[S_RR] = rr;
    scal[S_GD] = gd;
  }
}

struct Ptr16 {
  double* p[16];
};

// loopback all-reduce: the sum over ranks (rank order) of scal[slot..slot+c)
__global__ void k_loop_allreduce(int world, Ptr16 scal, int slot, int c) {
  const int j = threadIdx.x;
  if (j >= c) return;
  double s = 0.0;
  for (int q = 0; q < world; ++q) s += scal.p[q][slot + j];
  for (int q = 0; q < world; ++q) scal.p[q][slot + j] = s;
}

// the boundaries of every level k <= kp: b_k = children pointers of b_{k+1}
__global__ void k_descend(int64_t m, const int32_t* __restrict__ cptr, const int64_t* __restrict__ above,
                          int64_t* __restrict__ below) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < m) below[j] = cptr[above[j]];
}

__global__ void k_gather_i32_at(int64_t m, const int32_t* __restrict__ src, const int64_t* __restrict__ at,
                                int64_t* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < m) out[j] = src[at[j]];
}

template <typename T>
std::vector<T> d2h(const T* d, int64_t m, cudaStream_t st) {
  std::vector<T> v(std::max<int64_t>(m, 1));
  if (m > 0) MSP_CUDA(cudaMemcpyAsync(v.data(), d, m * sizeof(T), cudaMemcpyDeviceToHost, st));
  MSP_CUDA(cudaStreamSynchronize(st));
  v.resize(m);
  return v;
}

int tier_top(const Handle::Tier& T) { return T.generic ? T.k0 + 1 : T.k1; }

}  // namespace

// The partition of rank `rank` of `world` (every rank computes the same plan
// from the same hierarchy) and, with a unique id, its NCCL communicator.
DistRank* dist_build(Handle& h, int world, int rank, const void* id128, cudaStream_t st) {
  if (world < 1 || world > 16 || rank < 0 || rank >= world) throw Error{MSP_ERR_ARG, "bad world / rank (1..16)"};
  if (h.tiers.empty()) throw Error{MSP_ERR_UNSUPPORTED, "no tiers (graph too small to partition)"};
  auto d = std::make_unique<DistRank>();
  d->world = world;
  d->rank = rank;
  const int nt = (int)h.tiers.size();
  // partition level: the top of the highest tier with >= 32 nodes per rank
  // there (the levels above are replicated: cheap when small)
  int tp = -1;
  for (int t = 0; t < nt; ++t)
    if (h.lv[tier_top(h.tiers[t]) - 1].n >= 32 * (int64_t)world) tp = t;
  if (tp < 0) throw Error{MSP_ERR_UNSUPPORTED, "graph too small for this many ranks"};
  // keep the merged top-tier + coarse kernel replicated
  if (tp == nt - 1 && h.merged_coff > 0 && nt >= 2) tp = nt - 2;
  d->tp = tp;
  d->kp = tier_top(h.tiers[tp]);
  const int kp = d->kp;
  const int64_t nkp = h.lv[kp - 1].n;
  // prefix cost over level-kp nodes: adjacency entries + 8 per row of their
  // level-1 descendants (first descendants by descending the child pointers)
  DBuf<int64_t> f, g;
  f.alloc(nkp + 1);
  g.alloc(nkp + 1);
  {
    std::vector<int64_t> io(nkp + 1);
    for (int64_t i = 0; i <= nkp; ++i) io[i] = i;
    MSP_CUDA(cudaMemcpyAsync(f.p, io.data(), (nkp + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    for (int k = kp - 1; k >= 1; --k) {
      k_descend<<<grid_for(nkp + 1), TPB, 0, st>>>(nkp + 1, h.cptr.p + h.cptr_off[k - 1], f.p, g.p);
      std::swap(f, g);
    }
    k_gather_i32_at<<<grid_for(nkp + 1), TPB, 0, st>>>(nkp + 1, h.rowptr1.p, f.p, g.p);
    MSP_LAUNCH_CHECK();
  }
  std::vector<int64_t> f1 = d2h(f.p, nkp + 1, st), e1 = d2h(g.p, nkp + 1, st);
  std::vector<int64_t> cost(nkp + 1);
  for (int64_t i = 0; i <= nkp; ++i) cost[i] = e1[i] + 8 * f1[i];
  d->bnd_kp.assign(world + 1, 0);
  int rc = msp_dist_boundaries(nkp, cost.data(), world, d->bnd_kp.data());
  if (rc) throw Error{rc, "partition: too few nodes at the partition level for this many ranks"};
  // boundaries at every level k <= kp
  d->lvl_bnd.assign(kp, std::vector<int64_t>(world + 1));
  d->lvl_bnd[kp - 1] = d->bnd_kp;
  {
    DBuf<int64_t> a, b;
    a.alloc(world + 1);
    b.alloc(world + 1);
    MSP_CUDA(cudaMemcpyAsync(a.p, d->bnd_kp.data(), (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    for (int k = kp - 1; k >= 1; --k) {
      k_descend<<<1, 32, 0, st>>>(world + 1, h.cptr.p + h.cptr_off[k - 1], a.p, b.p);
      MSP_LAUNCH_CHECK();
      d->lvl_bnd[k - 1] = d2h(b.p, world + 1, st);
      std::swap(a, b);
    }
  }
  d->row0 = d->lvl_bnd[0][rank];
  d->row1 = d->lvl_bnd[0][rank + 1];
  // this rank's runs of tiers 0..tp; tiers above: as on one GPU
  d->runs = tier_runs(h);
  d->descs.resize(nt);
  d->tstarts.resize(nt);
  d->segs.resize(nt);
  d->heavies.resize(nt);
  for (int t = 0; t <= tp; ++t) {
    auto& T = h.tiers[t];
    TierRun& R = d->runs[t];
    if (T.generic) {
      const int k = T.k0;  // parents at level k + 1
      const int64_t B0 = d->lvl_bnd[k][rank], B1 = d->lvl_bnd[k][rank + 1];
      R.B0 = B0;
      R.nB = B1 - B0;
      const int64_t nh = h.heavy_off[k] - h.heavy_off[k - 1];
      std::vector<int32_t> hv = d2h(h.heavy.p + h.heavy_off[k - 1], nh, st), mine;
      for (int32_t x : hv)
        if (x >= B0 && x < B1) mine.push_back(x);
      d->heavies[t].alloc(std::max<size_t>(mine.size(), 1));
      if (!mine.empty())
        MSP_CUDA(cudaMemcpyAsync(d->heavies[t].p, mine.data(), mine.size() * 4, cudaMemcpyHostToDevice, st));
      R.heavy = d->heavies[t].p;
      R.nheavy = (int)mine.size();
      continue;
    }
    const int nl = T.k1 - T.k0 + 1;
    const int64_t nt1 = T.ntiles + 1;
    std::vector<int32_t> ts = d2h(T.tstart.p, (int64_t)nl * nt1, st);
    const int64_t a = d->lvl_bnd[T.k1 - 1][rank], b = d->lvl_bnd[T.k1 - 1][rank + 1];
    std::vector<int64_t> top{a};
    for (int64_t j = 0; j <= T.ntiles; ++j) {
      const int64_t v = ts[(size_t)(nl - 1) * nt1 + j];
      if (v > a && v < b) top.push_back(v);
    }
    top.push_back(b);
    const int64_t ntr = (int64_t)top.size() - 1;
    // starts per level by descending the clipped top starts
    std::vector<int32_t> rts((size_t)nl * (ntr + 1));
    {
      DBuf<int64_t> x, y;
      x.alloc(ntr + 1);
      y.alloc(ntr + 1);
      MSP_CUDA(cudaMemcpyAsync(x.p, top.data(), (ntr + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      for (int64_t j = 0; j <= ntr; ++j) rts[(size_t)(nl - 1) * (ntr + 1) + j] = (int32_t)top[j];
      for (int u = nl - 2; u >= 0; --u) {
        const int kc = T.k0 + u;  // child level
        k_descend<<<grid_for(ntr + 1), TPB, 0, st>>>(ntr + 1, h.cptr.p + h.cptr_off[kc - 1], x.p, y.p);
        MSP_LAUNCH_CHECK();
        std::vector<int64_t> lvl = d2h(y.p, ntr + 1, st);
        for (int64_t j = 0; j <= ntr; ++j) rts[(size_t)u * (ntr + 1) + j] = (int32_t)lvl[j];
        std::swap(x, y);
      }
    }
    TierDesc ds = T.desc;
    ds.ntiles = (int)ntr;
    // the up kernel's grouping of consecutive tiles, its layout re-sized for
    // the clipped tiles; the down kernel's tiles per CTA as on one GPU
    const int G = T.up_group;
    {
      auto a16 = [](int64_t b) { return (int)((b + 15) & ~(int64_t)15); };
      int64_t c0 = 0, c1 = 0;
      for (int64_t j = 0; j < ntr; j += G) {
        const int64_t je = std::min<int64_t>(j + G, ntr);
        c0 = std::max<int64_t>(c0, (int64_t)rts[je] - rts[j]);
        c1 = std::max<int64_t>(c1, (int64_t)rts[(size_t)(nl - 1) * (ntr + 1) + je] - rts[(size_t)(nl - 1) * (ntr + 1) + j]);
      }
      ds.o_uf = 0;
      ds.o_uy0 = a16((c1 + 1 + 8) * 4);
      ds.o_uq = a16(ds.o_uy0 + (c0 + 2) * 8);
      ds.o_uh = a16(ds.o_uq + (c0 + 2) * 8);
      ds.smem_up = (T.k0 == 1) ? a16(ds.o_uh + (c0 + 2) * 8) : a16(ds.o_uy0 + (c0 + 2) * 8);
      ds.up_group = G;
      raise_smem_limit(T.k0 == 1 ? (const void*)k_tile_up<true> : (const void*)k_tile_up<false>, ds.smem_up);
    }
    d->descs[t] = ds;
    d->tstarts[t].alloc(rts.size());
    MSP_CUDA(cudaMemcpyAsync(d->tstarts[t].p, rts.data(), rts.size() * 4, cudaMemcpyHostToDevice, st));
    if (nl > 1) {
      const std::vector<int4> sg = make_tile_segs(h, T.k0, nl, ds, rts, ntr);
      d->segs[t].alloc(std::max<size_t>(sg.size(), 1));
      if (!sg.empty())
        MSP_CUDA(cudaMemcpyAsync(d->segs[t].p, sg.data(), sg.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    }
    R.desc = &d->descs[t];
    R.tstart = d->tstarts[t].p;
    R.segs = nl > 1 ? d->segs[t].p : nullptr;
    R.ntiles = ntr;
    R.up_group = G;
    R.tpc = ds.tpc;
    R.smem_up = ds.smem_up;
  }
  MSP_CUDA(cudaStreamSynchronize(st));
  // halo plan (host, from the level-1 nested CSR)
  {
    std::vector<int32_t> rp = d2h(h.rowptr1.p, h.n + 1, st), cl = d2h(h.col1.p, h.nnz_adj, st);
    d->send_cnt.assign(world, 0);
    d->recv_cnt.assign(world, 0);
    const std::vector<int64_t>& rb = d->lvl_bnd[0];
    rc = msp_halo_plan(h.n, rp.data(), cl.data(), world, rb.data(), rank, d->recv_cnt.data(), d->send_cnt.data(),
                       nullptr, 0, nullptr, 0);
    if (rc) throw Error{rc, "halo plan"};
    for (int q = 0; q < world; ++q) { d->nsend += d->send_cnt[q]; d->nrecv += d->recv_cnt[q]; }
    std::vector<int64_t> rr(std::max<int64_t>(d->nrecv, 1)), sr(std::max<int64_t>(d->nsend, 1));
    rc = msp_halo_plan(h.n, rp.data(), cl.data(), world, rb.data(), rank, d->recv_cnt.data(), d->send_cnt.data(),
                       rr.data(), d->nrecv, sr.data(), d->nsend);
    if (rc) throw Error{rc, "halo plan"};
    d->send_off.assign(world + 1, 0);
    d->recv_off.assign(world + 1, 0);
    for (int q = 0; q < world; ++q) {
      d->send_off[q + 1] = d->send_off[q] + d->send_cnt[q];
      d->recv_off[q + 1] = d->recv_off[q] + d->recv_cnt[q];
    }
    std::vector<int32_t> si(sr.begin(), sr.end()), ri(rr.begin(), rr.end());
    d->send_idx.alloc(si.size());
    d->recv_idx.alloc(ri.size());
    MSP_CUDA(cudaMemcpyAsync(d->send_idx.p, si.data(), si.size() * 4, cudaMemcpyHostToDevice, st));
    MSP_CUDA(cudaMemcpyAsync(d->recv_idx.p, ri.data(), ri.size() * 4, cudaMemcpyHostToDevice, st));
    d->sendbuf.alloc(std::max<int64_t>(d->nsend, 1));
    d->recvbuf.alloc(std::max<int64_t>(d->nrecv, 1));
    MSP_CUDA(cudaStreamSynchronize(st));
  }
  d->kp_max = 1;
  for (int q = 0; q < world; ++q) d->kp_max = std::max<int64_t>(d->kp_max, d->bnd_kp[q + 1] - d->bnd_kp[q]);
  d->gsend.alloc(d->kp_max + 2);
  d->grecv.alloc((d->kp_max + 2) * world);
  if (id128) {
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&id, id128, sizeof(id));
    MSP_NCCL(ncclCommInitRank(&d->comm, world, id, rank));
  }
  return d.release();
}

namespace {

// The ranks this process drives: one (NCCL), or all of them (loopback).
struct DistGroup {
  std::vector<Handle*> hs;
  bool loop = false;
  int world = 1;
  cudaStream_t st = nullptr;
};

void coll_allreduce(DistGroup& g, int slot, int c) {
  if (g.loop) {
    Ptr16 p{};
    for (int q = 0; q < g.world; ++q) p.p[q] = g.hs[q]->scal.p;
    k_loop_allreduce<<<1, 32, 0, g.st>>>(g.world, p, slot, c);
    MSP_LAUNCH_CHECK();
  } else {
    Handle& h = *g.hs[0];
    MSP_NCCL(ncclAllReduce(h.scal.p + slot, h.scal.p + slot, c, ncclDouble, ncclSum, h.dist->comm, g.st));
  }
}

void coll_halo(DistGroup& g) {
  if (g.loop) {
    for (int r = 0; r < g.world; ++r) {
      DistRank& dr = *g.hs[r]->dist;
      for (int q = 0; q < g.world; ++q) {
        if (q == r || dr.recv_cnt[q] == 0) continue;
        DistRank& dq = *g.hs[q]->dist;
        MSP_CUDA(cudaMemcpyAsync(dr.recvbuf.p + dr.recv_off[q], dq.sendbuf.p + dq.send_off[r],
                                 dr.recv_cnt[q] * sizeof(double), cudaMemcpyDeviceToDevice, g.st));
      }
    }
  } else {
    DistRank& d = *g.hs[0]->dist;
    MSP_NCCL(ncclGroupStart());
    for (int q = 0; q < g.world; ++q) {
      if (q == d.rank) continue;
      if (d.send_cnt[q]) MSP_NCCL(ncclSend(d.sendbuf.p + d.send_off[q], d.send_cnt[q], ncclDouble, q, d.comm, g.st));
      if (d.recv_cnt[q]) MSP_NCCL(ncclRecv(d.recvbuf.p + d.recv_off[q], d.recv_cnt[q], ncclDouble, q, d.comm, g.st));
    }
    MSP_NCCL(ncclGroupEnd());
  }
}

void coll_allgather_y(DistGroup& g) {
  const DistRank& d0 = *g.hs[0]->dist;
  const int64_t M = d0.kp_max + 2;
  for (Handle* h : g.hs) {
    DistRank& d = *h->dist;
    const int64_t lo = d.bnd_kp[d.rank], cnt = d.bnd_kp[d.rank + 1] - lo;
    k_pack_y<<<grid_for(M), TPB, 0, g.st>>>(cnt, h->Y.p + h->lv[d.kp - 1].off + lo, h->scal.p, d.gsend.p, M);
  }
  MSP_LAUNCH_CHECK();
  if (g.loop) {
    for (int r = 0; r < g.world; ++r)
      for (int q = 0; q < g.world; ++q)
        MSP_CUDA(cudaMemcpyAsync(g.hs[r]->dist->grecv.p + q * M, g.hs[q]->dist->gsend.p, M * sizeof(double),
                                 cudaMemcpyDeviceToDevice, g.st));
  } else {
    DistRank& d = *g.hs[0]->dist;
    MSP_NCCL(ncclAllGather(d.gsend.p, d.grecv.p, M, ncclDouble, d.comm, g.st));
  }
  for (Handle* h : g.hs) {
    DistRank& d = *h->dist;
    Bnd16 b{};
    for (int q = 0; q <= d.world; ++q) b.b[q] = d.bnd_kp[q];
    const int64_t m = std::max<int64_t>(d.kp_max, 1);
    k_unpack_y<<<std::min<unsigned>(grid_for(m), 512u), TPB, 0, g.st>>>(d.world, b, d.grecv.p, M,
                                                                        h->Y.p + h->lv[d.kp - 1].off, h->scal.p);
  }
  MSP_LAUNCH_CHECK();
}

void dist_finish(DistGroup& g, int stage, int mode) {
  for (Handle* h : g.hs) k_dist_finish<<<1, 1, 0, g.st>>>(stage, h->scal.p, h->counters.p, mode);
  MSP_LAUNCH_CHECK();
}

// the sweeps of one PCG step (mode INIT or ITER), both halves around the all-gather
void dist_sweeps(DistGroup& g, int mode, double* const* zout, Prof* const* P) {
  for (size_t i = 0; i < g.hs.size(); ++i) {
    Handle& h = *g.hs[i];
    const Lv lv = make_level_table(h);
    const int zs = use_pairs(h) ? M_ZS2 : 0;
    msp_sweeps_runs(h, lv, h.dist->runs, h.dist->tp, mode == M_ITER ? h.vq.p : nullptr, h.vr.p, zout[i], g.st,
                    mode | zs | M_DIST, *P[i], PH_UP_LOW);
  }
  coll_allgather_y(g);
  dist_finish(g, 1, mode);
  for (size_t i = 0; i < g.hs.size(); ++i) {
    Handle& h = *g.hs[i];
    const Lv lv = make_level_table(h);
    const int zs = use_pairs(h) ? M_ZS2 : 0;
    msp_sweeps_runs(h, lv, h.dist->runs, h.dist->tp, mode == M_ITER ? h.vq.p : nullptr, h.vr.p, zout[i], g.st,
                    mode | zs | M_DIST, *P[i], PH_UPPER | PH_DOWN_LOW);
  }
  coll_allreduce(g, S_RZ, 1);
  dist_finish(g, 2, mode);
}

void dist_iteration(DistGroup& g, Prof* const* P) {
  const size_t m = g.hs.size();
  std::vector<double*> zin(m), zout(m), pold(m), pnew(m);
  const bool pairs = use_pairs(*g.hs[0]);
  for (size_t i = 0; i < m; ++i) {
    Handle& h = *g.hs[i];
    if (pairs) {
      zin[i] = h.pparity ? h.zp2.p : h.zp1.p;
      zout[i] = h.pparity ? h.zp1.p : h.zp2.p;
    } else {
      zin[i] = zout[i] = h.vz.p;
      pold[i] = h.pparity ? h.vp2.p : h.vp.p;
      pnew[i] = h.pparity ? h.vp.p : h.vp2.p;
    }
    h.pparity ^= 1;
    DistRank& d = *h.dist;
    if (d.nsend)
      k_halo_pack<<<grid_for(d.nsend), TPB, 0, g.st>>>(d.nsend, d.send_idx.p, zin[i], pairs ? zin[i] + 1 : pold[i],
                                                         pairs ? 2 : 1, d.sendbuf.p, h.scal.p, h.counters.p);
  }
  MSP_LAUNCH_CHECK();
  coll_halo(g);
  for (size_t i = 0; i < m; ++i) {
    Handle& h = *g.hs[i];
    DistRank& d = *h.dist;
    if (d.nrecv)
      k_halo_unpack<<<grid_for(d.nrecv), TPB, 0, g.st>>>(d.nrecv, d.recv_idx.p, d.recvbuf.p, zin[i],
                                                           pairs ? zin[i] + 1 : pold[i], pairs ? 2 : 1,
                                                           h.counters.p);
    MSP_LAUNCH_CHECK();
    P[i]->begin();
    if (pairs) launch_spmv_pairs(h, zin[i], zout[i], h.vq.p, h.vx.p, g.st, d.row0, d.row1, false);
    else if (use_sep(h)) launch_spmv_sep(h, zin[i], pold[i], pnew[i], h.vq.p, h.vx.p, g.st, d.row0, d.row1);
    else launch_spmv<true>(h, zin[i], pold[i], pnew[i], h.vq.p, h.vx.p, g.st, d.row0, d.row1);
    P[i]->end(PC_SPMV);
  }
  coll_allreduce(g, S_PQ, 1);
  dist_finish(g, 0, M_ITER);
  dist_sweeps(g, M_ITER, zout.data(), P);
}

}  // namespace

// PCG-MSP (reading R10) on the partitioned system: every handle of the group
// holds b (nested) in vb; x (nested, own rows; zero elsewhere) in vx.
void pcg_dist_group(std::vector<Handle*>& hs, bool loop, double rtol, int maxit, cudaStream_t st, msp_report* rep) {
  DistGroup g;
  g.hs = hs;
  g.loop = loop;
  g.world = hs[0]->dist->world;
  g.st = st;
  std::vector<std::unique_ptr<Prof>> profs;
  std::vector<Prof*> P;
  for (Handle* h : hs) {
    profs.emplace_back(new Prof(*h, st));
    P.push_back(profs.back().get());
  }
  cudaEvent_t e0, e1;
  MSP_CUDA(cudaEventCreate(&e0));
  MSP_CUDA(cudaEventCreate(&e1));
  const int64_t l0 = hs[0]->launches;
  MSP_CUDA(cudaEventRecord(e0, st));
  std::vector<double*> z1;
  for (Handle* h : hs) {
    const int64_t n = h->n;
    MSP_CUDA(cudaMemsetAsync(h->vx.p, 0, n * sizeof(double), st));
    MSP_CUDA(cudaMemcpyAsync(h->vr.p, h->vb.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    MSP_CUDA(cudaMemsetAsync(h->zp1.p, 0, 2 * n * sizeof(double), st));
    MSP_CUDA(cudaMemsetAsync(h->vp.p, 0, n * sizeof(double), st));
    MSP_CUDA(cudaMemsetAsync(h->vz.p, 0, n * sizeof(double), st));
    h->pparity = 0;
    k_init_state<<<1, 1, 0, st>>>(h->scal.p, h->counters.p, rtol * rtol);
    z1.push_back(use_pairs(*h) ? h->zp1.p : h->vz.p);
  }
  MSP_LAUNCH_CHECK();
  dist_sweeps(g, M_INIT, z1.data(), P.data());
  int batch = 64;
  if (const char* e = std::getenv("MSP_PCG_BATCH")) batch = std::max(2, std::atoi(e) & ~1);
  const bool use_graph = std::getenv("MSP_NO_GRAPH") == nullptr && !hs[0]->profile;
  cudaGraphExec_t gx = nullptr;
  int64_t graph_launches = 0;  // kernels of one captured batch (counted on rank 0's handle)
  unsigned hc[C_NCNT];
  auto done = [&]() {
    MSP_CUDA(cudaMemcpyAsync(hc, hs[0]->counters.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    MSP_CUDA(cudaStreamSynchronize(st));
    return hc[C_DONE] != 0;
  };
  int it = 0;
  if (!done()) {
    while (it < maxit) {
      const int nb = std::min(batch, maxit - it);
      if (use_graph && nb == batch) {
        if (!gx) {
          cudaStream_t cs;
          MSP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
          cudaGraph_t gr;
          DistGroup gc = g;
          gc.st = cs;
          const int64_t lc0 = hs[0]->launches;
          MSP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
          for (int b2 = 0; b2 < nb; ++b2) dist_iteration(gc, P.data());
          MSP_CUDA(cudaStreamEndCapture(cs, &gr));
          MSP_CUDA(cudaGraphInstantiate(&gx, gr, 0));
          cudaGraphDestroy(gr);
          cudaStreamDestroy(cs);
          graph_launches = hs[0]->launches - lc0;  // the capture pass counted the first replay
        } else {
          hs[0]->launches += graph_launches;
        }
        MSP_CUDA(cudaGraphLaunch(gx, st));
      } else {
        for (int b2 = 0; b2 < nb; ++b2) dist_iteration(g, P.data());
      }
      it += nb;
      if (done()) break;
    }
  }
  if (gx) cudaGraphExecDestroy(gx);
  for (Handle* h : hs) {
    if (use_pairs(*h))
      launch(k_x_final_pairs, std::min<unsigned>(grid_for(h->n), 148u * 8u), TPB, 0, st, h->n, h->vx.p,
             (const double*)h->zp1.p, (const double*)h->zp2.p, (const double*)h->scal.p,
             (const unsigned*)h->counters.p);
    else
      launch(k_x_final, std::min<unsigned>(grid_for(h->n), 148u * 8u), TPB, 0, st, h->n, h->vx.p,
             (const double*)h->vp.p, (const double*)h->vp2.p, (const double*)h->scal.p,
             (const unsigned*)h->counters.p);
    k_zero_outside<<<grid_for(h->n), TPB, 0, st>>>(h->n, h->dist->row0, h->dist->row1, h->vx.p);
  }
  MSP_LAUNCH_CHECK();
  MSP_CUDA(cudaEventRecord(e1, st));
  MSP_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  MSP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  double hsc[S_NSCAL];
  MSP_CUDA(cudaMemcpy(hsc, hs[0]->scal.p, sizeof(hsc), cudaMemcpyDeviceToHost));
  MSP_CUDA(cudaMemcpy(hc, hs[0]->counters.p, sizeof(hc), cudaMemcpyDeviceToHost));
  if (rep) {
    rep->iterations = (int32_t)hc[C_IT];
    rep->converged = hc[C_DONE] ? 1 : 0;
    rep->relres = hsc[S_BB] > 0 ? std::sqrt(hsc[S_RR] / hsc[S_BB]) : 0.0;
    rep->solve_ms = ms;
    rep->kernel_launches = hs[0]->launches - l0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

__global__ void k_zero_outside(int64_t n, int64_t r0, int64_t r1, double* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && (i < r0 || i >= r1)) x[i] = 0.0;
}

void dist_unique_id(void* id128) {
  ncclUniqueId id;
  MSP_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
}

namespace {
__global__ void k_add_into(int64_t n, const double* __restrict__ a, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] += a[i];
}
}  // namespace

void add_into(Handle& h, const double* a, double* y, cudaStream_t st) {
  k_add_into<<<grid_for(h.n), TPB, 0, st>>>(h.n, a, y);
  MSP_LAUNCH_CHECK();
}

// (row0, row1, kp, tp, nsend, nrecv, world, rank) of the handle's rank
void dist_range(const Handle& h, int64_t* o) {
  const DistRank& d = *h.dist;
  o[0] = d.row0; o[1] = d.row1; o[2] = d.kp; o[3] = d.tp;
  o[4] = d.nsend; o[5] = d.nrecv; o[6] = d.world; o[7] = d.rank;
}
