// capi.cu -- extern "C" boundary of libmsp_b200.so (declared in
// include/msp_b200.h).  Argument checking and host<->device marshalling only;
// every step of the method runs in the kernels of setup.cu / solve.cu.
#include <algorithm>
#include <cstring>
#include <exception>
#include <vector>

#include "internal.cuh"

namespace msp {
namespace {
thread_local std::string g_last_error = "no error";
}
void set_error(const std::string& m) { g_last_error = m; }
}  // namespace msp

using msp::DBuf;
using msp::Error;
using msp::Handle;

struct msp_handle {
  Handle h;
};

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MSP_OK;
  } catch (const Error& e) {
    msp::set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    msp::set_error(e.what());
    return MSP_ERR_CUDA;
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void need(bool ok, const char* what) {
  if (!ok) throw Error{MSP_ERR_ARG, what};
}

// stage a vector of n doubles in device memory when mem == MSP_MEM_HOST
const double* stage_in(Handle& h, const double* p, int mem, DBuf<double>& buf, cudaStream_t st) {
  if (mem == MSP_MEM_DEVICE) return p;
  if (buf.n < (size_t)h.n) buf.alloc(h.n);
  MSP_CUDA(cudaMemcpyAsync(buf.p, p, h.n * sizeof(double), cudaMemcpyHostToDevice, st));
  return buf.p;
}

}  // namespace

extern "C" {

const char* msp_last_error(void) { return msp::g_last_error.c_str(); }

int msp_setup(int64_t n, const int64_t* rowptr, const int32_t* col, const double* w, int mem,
              const msp_params* params, void* stream, msp_handle** out) {
  return guarded([&] {
    need(out != nullptr, "out is NULL");
    *out = nullptr;
    need(n >= 2, "n must be >= 2");
    need(rowptr && col && w, "null CSR pointer");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    cudaStream_t st = S(stream);
    auto* H = new msp_handle();
    try {
      Handle& h = H->h;
      h.n = n;
      h.mu = (params && params->mu > 0) ? params->mu : 0.8;
      h.levels_req = params ? params->max_levels : 0;
      h.seed = params ? params->seed : 0;
      h.top_max = (params && params->top_max > 0) ? params->top_max : 256;
      if (h.top_max > 256) throw Error{MSP_ERR_ARG, "top_max must be <= 256"};
      // row offsets: host copy to validate and learn nnz
      std::vector<int64_t> rp(n + 1);
      if (mem == MSP_MEM_HOST) std::memcpy(rp.data(), rowptr, (n + 1) * sizeof(int64_t));
      else MSP_CUDA(cudaMemcpy(rp.data(), rowptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
      if (rp[0] != 0) throw Error{MSP_ERR_GRAPH, "rowptr[0] != 0"};
      for (int64_t i = 0; i < n; ++i)
        if (rp[i + 1] < rp[i]) throw Error{MSP_ERR_GRAPH, "rowptr not monotone"};
      h.nnz_adj = rp[n];
      if (h.nnz_adj <= 0) throw Error{MSP_ERR_GRAPH, "graph has no edges"};
      const int64_t* drp = rowptr;
      const int32_t* dcol = col;
      const double* dw = w;
      DBuf<int64_t> brp;
      DBuf<int32_t> bcol;
      DBuf<double> bw;
      if (mem == MSP_MEM_HOST) {
        brp.alloc(n + 1); bcol.alloc(h.nnz_adj); bw.alloc(h.nnz_adj);
        MSP_CUDA(cudaMemcpyAsync(brp.p, rowptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        MSP_CUDA(cudaMemcpyAsync(bcol.p, col, h.nnz_adj * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        MSP_CUDA(cudaMemcpyAsync(bw.p, w, h.nnz_adj * sizeof(double), cudaMemcpyHostToDevice, st));
        drp = brp.p; dcol = bcol.p; dw = bw.p;
      }
      msp::validate_csr(h, drp, dcol, dw, st);
      msp::build_setup(h, drp, dcol, dw, st);
      msp::alloc_solve_workspace(h);
      msp::build_coarse_matrix(h, st);
      MSP_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      delete H;
      throw;
    }
    *out = H;
  });
}

int msp_destroy(msp_handle* H) {
  return guarded([&] { delete H; });
}

int msp_info(const msp_handle* H, msp_info_t* out) {
  return guarded([&] {
    need(H && out, "null argument");
    const Handle& h = H->h;
    out->n = h.n;
    out->nnz = h.nnz_adj + h.n;
    out->n_tilde = h.n_tilde;
    out->levels = h.levels;
    out->mwm_rounds = h.mwm_rounds;
    out->mu = h.mu;
    out->setup_ms = h.setup_ms;
    int32_t tl = 1;
    int64_t nt = 0;
    for (const auto& T : h.tiers) {
      if (!T.generic && T.k0 == 1) { tl = T.k1; nt = T.ntiles; }
    }
    out->tile_level = tl;
    out->coarse_level = h.Kc;
    out->ntiles = nt;
    out->ntiers = (int32_t)h.tiers.size();
    out->spmv_grid = (int32_t)h.spmv_grid;
    out->merged_coarse = h.merged_coff > 0 ? 1 : 0;
  });
}

int msp_level_sizes(const msp_handle* H, int64_t* sizes) {
  return guarded([&] {
    need(H && sizes, "null argument");
    for (int k = 0; k < H->h.levels; ++k) sizes[k] = H->h.lv[k].n;
  });
}

int msp_get_aggregates(const msp_handle* H, int32_t level, int32_t* agg) {
  return guarded([&] {
    need(H && agg, "null argument");
    need(level >= 1 && level < H->h.levels, "level out of range (1..levels-1)");
    const Handle& h = H->h;
    MSP_CUDA(cudaMemcpy(agg, h.agg_canon[level - 1].p, h.lv[level - 1].n * sizeof(int32_t),
                        cudaMemcpyDeviceToHost));
  });
}

int msp_get_msp_edges(const msp_handle* H, int64_t* count, int64_t* I, int64_t* J, double* Wt) {
  return guarded([&] {
    need(H && count, "null argument");
    const Handle& h = H->h;
    const int L = h.levels;
    std::vector<int64_t> ei, ej;
    std::vector<double> ew;
    double sigma = 1.0;  // mu^{2(k-1)}
    for (int k = 1; k <= L; ++k) {
      const int64_t nk = h.lv[k - 1].n, nnz = h.lv[k - 1].nnz, off = h.lv[k - 1].off;
      std::vector<int64_t> rp(nk + 1);
      std::vector<int32_t> cl(nnz);
      std::vector<double> ww(nnz);
      MSP_CUDA(cudaMemcpy(rp.data(), h.canon_rowptr[k - 1].p, (nk + 1) * 8, cudaMemcpyDeviceToHost));
      MSP_CUDA(cudaMemcpy(cl.data(), h.canon_col[k - 1].p, nnz * 4, cudaMemcpyDeviceToHost));
      MSP_CUDA(cudaMemcpy(ww.data(), h.canon_w[k - 1].p, nnz * 8, cudaMemcpyDeviceToHost));
      std::vector<int32_t> agg;
      std::vector<double> apar;
      if (k < L) {
        agg.resize(nk);
        apar.resize(nk);
        MSP_CUDA(cudaMemcpy(agg.data(), h.agg_canon[k - 1].p, nk * 4, cudaMemcpyDeviceToHost));
        MSP_CUDA(cudaMemcpy(apar.data(), h.apar_canon[k - 1].p, nk * 8, cudaMemcpyDeviceToHost));
      }
      for (int64_t i = 0; i < nk; ++i) {
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
          const int64_t j = cl[e];
          if (j <= i) continue;
          if (k == L || agg[i] == agg[j]) {  // top level, or inside an aggregate (R8)
            ei.push_back(off + i); ej.push_back(off + j); ew.push_back(sigma * ww[e]);
          }
        }
        if (k < L && apar[i] > 0) {  // node -> own aggregate (R8)
          ei.push_back(off + i); ej.push_back(h.lv[k].off + agg[i]); ew.push_back(apar[i]);
        }
      }
      sigma *= h.mu * h.mu;
    }
    if (I && J && Wt) {
      need((int64_t)ei.size() <= *count, "arrays too small");
      std::memcpy(I, ei.data(), ei.size() * 8);
      std::memcpy(J, ej.data(), ej.size() * 8);
      std::memcpy(Wt, ew.data(), ew.size() * 8);
    }
    *count = (int64_t)ei.size();
  });
}

int msp_apply_L(msp_handle* H, const double* x, double* y, int mem, void* stream) {
  return guarded([&] {
    need(H && x && y, "null argument");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    Handle& h = H->h;
    cudaStream_t st = S(stream);
    const double* xd = stage_in(h, x, mem, h.stage_in, st);
    msp::gather_to_nested(h, xd, h.vp.p, st);
    msp::apply_L_nested(h, h.vp.p, h.vq.p, st);
    if (mem == MSP_MEM_DEVICE) {
      msp::scatter_from_nested(h, h.vq.p, y, st);
    } else {
      if (h.stage_out.n < (size_t)h.n) h.stage_out.alloc(h.n);
      msp::scatter_from_nested(h, h.vq.p, h.stage_out.p, st);
      MSP_CUDA(cudaMemcpyAsync(y, h.stage_out.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
    }
  });
}

int msp_apply_R(msp_handle* H, int precond, const double* r, double* z, int mem, void* stream) {
  return guarded([&] {
    need(H && r && z, "null argument");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    need(precond == MSP_PRECOND_MSP || precond == MSP_PRECOND_NONE || precond == MSP_PRECOND_PEGP, "bad precond");
    Handle& h = H->h;
    cudaStream_t st = S(stream);
    const double* rd = stage_in(h, r, mem, h.stage_in, st);
    msp::gather_to_nested(h, rd, h.vr.p, st);
    if (precond == MSP_PRECOND_MSP) msp::apply_R_msp_nested(h, h.vr.p, h.vz.p, st);
    else if (precond == MSP_PRECOND_PEGP) msp::apply_R_pegp_nested(h, h.vr.p, h.vz.p, st);
    else MSP_CUDA(cudaMemcpyAsync(h.vz.p, h.vr.p, h.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (mem == MSP_MEM_DEVICE) {
      msp::scatter_from_nested(h, h.vz.p, z, st);
    } else {
      if (h.stage_out.n < (size_t)h.n) h.stage_out.alloc(h.n);
      msp::scatter_from_nested(h, h.vz.p, h.stage_out.p, st);
      MSP_CUDA(cudaMemcpyAsync(z, h.stage_out.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
    }
  });
}

int msp_pcg_solve(msp_handle* H, int precond, const double* b, double* x, double rtol, int32_t maxit,
                  int mem, void* stream, msp_report* rep) {
  return guarded([&] {
    need(H && b && x, "null argument");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    need(rtol >= 0 && maxit >= 0, "bad rtol / maxit");
    need(precond == MSP_PRECOND_MSP || precond == MSP_PRECOND_NONE || precond == MSP_PRECOND_PEGP, "bad precond");
    Handle& h = H->h;
    cudaStream_t st = S(stream);
    const double* bd = stage_in(h, b, mem, h.stage_in, st);
    msp::gather_to_nested(h, bd, h.vb.p, st);
    msp::pcg_nested(h, precond, h.vb.p, h.vx.p, rtol, maxit, st, rep);
    if (mem == MSP_MEM_DEVICE) {
      msp::scatter_from_nested(h, h.vx.p, x, st);
      MSP_CUDA(cudaStreamSynchronize(st));
    } else {
      if (h.stage_out.n < (size_t)h.n) h.stage_out.alloc(h.n);
      msp::scatter_from_nested(h, h.vx.p, h.stage_out.p, st);
      MSP_CUDA(cudaMemcpyAsync(x, h.stage_out.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, st));
      MSP_CUDA(cudaStreamSynchronize(st));
    }
  });
}

int msp_pegp_params(msp_handle* H, double inner_rtol, int32_t inner_maxit, int32_t refine_steps) {
  return guarded([&] {
    need(H != nullptr, "null handle");
    need(inner_rtol > 0 && inner_rtol < 1 && inner_maxit > 0 && refine_steps >= 0 && refine_steps <= 16,
         "bad PEGP parameters");
    H->h.pegp_rtol = inner_rtol;
    H->h.pegp_maxit = inner_maxit;
    H->h.pegp_refine = refine_steps;
  });
}

}  // extern "C"

namespace {
// run f(x_nested, y_nested) on expanded vectors given in the canonical
// expanded numbering (n~ entries in `mem`)
template <typename F>
void expanded_call(Handle& h, const double* x, double* y, int mem, cudaStream_t st, F&& f) {
  const int64_t nt = h.n_tilde;
  msp::pegp_build(h, st);
  DBuf<double> xin, xn, yn, yout;
  xn.alloc(nt + 8);
  yn.alloc(nt + 8);
  const double* xd = x;
  if (mem == MSP_MEM_HOST) {
    xin.alloc(nt);
    MSP_CUDA(cudaMemcpyAsync(xin.p, x, nt * sizeof(double), cudaMemcpyHostToDevice, st));
    xd = xin.p;
  }
  msp::expanded_to_nested(h, xd, xn.p, st);
  f(xn.p, yn.p);
  if (mem == MSP_MEM_DEVICE) {
    msp::nested_to_expanded(h, yn.p, y, st);
  } else {
    yout.alloc(nt);
    msp::nested_to_expanded(h, yn.p, yout.p, st);
    MSP_CUDA(cudaMemcpyAsync(y, yout.p, nt * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  MSP_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

extern "C" {

int msp_apply_LH(msp_handle* H, const double* x, double* y, int mem, void* stream) {
  return guarded([&] {
    need(H && x && y, "null argument");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    Handle& h = H->h;
    expanded_call(h, x, y, mem, S(stream), [&](const double* xn, double* yn) {
      msp::apply_LH_nested(h, xn, yn, S(stream));
    });
  });
}

int msp_solve_LH(msp_handle* H, const double* r, double* z, int mem, void* stream, int32_t* inner_iterations) {
  return guarded([&] {
    need(H && r && z, "null argument");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    Handle& h = H->h;
    int it = 0;
    expanded_call(h, r, z, mem, S(stream), [&](const double* rn, double* zn) {
      it = msp::solve_LH_nested(h, rn, zn, S(stream));
    });
    if (inner_iterations) *inner_iterations = it;
  });
}

int msp_pegp_info(msp_handle* H, void* stream, int64_t* out5) {
  return guarded([&] {
    need(H && out5, "null argument");
    Handle& h = H->h;
    msp::pegp_build(h, S(stream));
    out5[0] = h.hnnz;
    out5[1] = h.pegp_last_inner;
    out5[2] = h.pegp_Kc;
    out5[3] = (int64_t)(h.pegp_build_ms * 1000.0);
    out5[4] = h.pegp_solve_inner;
  });
}

int msp_dist_unique_id(void* id128) {
  return guarded([&] {
    need(id128 != nullptr, "null argument");
    msp::dist_unique_id(id128);
  });
}

int msp_dist_init(msp_handle* H, int32_t world, int32_t rank, const void* id128, void* stream) {
  return guarded([&] {
    need(H != nullptr, "null handle");
    need(world >= 1 && world <= 16 && rank >= 0 && rank < world, "bad world / rank");
    Handle& h = H->h;
    if (h.dist) { msp::dist_free(h.dist); h.dist = nullptr; }
    h.dist = msp::dist_build(h, world, rank, id128, S(stream));
  });
}

int msp_dist_range(msp_handle* H, int64_t* out) {
  return guarded([&] {
    need(H && out, "null argument");
    need(H->h.dist != nullptr, "msp_dist_init was not called");
    msp::dist_range(H->h, out);
  });
}

namespace {
// b (caller numbering, host or device) into every handle's vb; x out as the
// sum of the handles' own rows
void dist_io_in(std::vector<Handle*>& hs, const double* b, int mem, cudaStream_t st) {
  for (Handle* hp : hs) {
    const double* bd = stage_in(*hp, b, mem, hp->stage_in, st);
    msp::gather_to_nested(*hp, bd, hp->vb.p, st);
  }
}
}  // namespace

int msp_dist_solve(msp_handle* H, const double* b, double* x, double rtol, int32_t maxit, int mem, void* stream,
                   msp_report* rep) {
  return guarded([&] {
    need(H && b && x, "null argument");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    need(rtol >= 0 && maxit >= 0, "bad rtol / maxit");
    Handle& h = H->h;
    need(h.dist != nullptr, "msp_dist_init was not called");
    cudaStream_t st = S(stream);
    std::vector<Handle*> hs{&h};
    dist_io_in(hs, b, mem, st);
    msp::pcg_dist_group(hs, false, rtol, maxit, st, rep);
    if (mem == MSP_MEM_DEVICE) {
      msp::scatter_from_nested(h, h.vx.p, x, st);
    } else {
      if (h.stage_out.n < (size_t)h.n) h.stage_out.alloc(h.n);
      msp::scatter_from_nested(h, h.vx.p, h.stage_out.p, st);
      MSP_CUDA(cudaMemcpyAsync(x, h.stage_out.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    MSP_CUDA(cudaStreamSynchronize(st));
  });
}

int msp_dist_group_solve(msp_handle** Hs, int32_t world, const double* b, double* x, double rtol, int32_t maxit,
                         int mem, void* stream, msp_report* rep) {
  return guarded([&] {
    need(Hs && b && x, "null argument");
    need(world >= 1 && world <= 16, "world must be 1..16");
    need(mem == MSP_MEM_DEVICE || mem == MSP_MEM_HOST, "bad mem");
    need(rtol >= 0 && maxit >= 0, "bad rtol / maxit");
    cudaStream_t st = S(stream);
    std::vector<Handle*> hs;
    for (int r = 0; r < world; ++r) {
      need(Hs[r] != nullptr, "null handle");
      Handle& h = Hs[r]->h;
      need(h.n == Hs[0]->h.n && h.n_tilde == Hs[0]->h.n_tilde, "handles of different graphs");
      if (h.dist) { msp::dist_free(h.dist); h.dist = nullptr; }
      h.dist = msp::dist_build(h, world, r, nullptr, st);
      hs.push_back(&h);
    }
    dist_io_in(hs, b, mem, st);
    msp::pcg_dist_group(hs, true, rtol, maxit, st, rep);
    // assemble: the sum of the ranks' own rows (each zero outside its rows)
    Handle& h0 = *hs[0];
    for (int r = 1; r < world; ++r) msp::add_into(h0, hs[r]->vx.p, h0.vx.p, st);
    if (mem == MSP_MEM_DEVICE) {
      msp::scatter_from_nested(h0, h0.vx.p, x, st);
    } else {
      if (h0.stage_out.n < (size_t)h0.n) h0.stage_out.alloc(h0.n);
      msp::scatter_from_nested(h0, h0.vx.p, h0.stage_out.p, st);
      MSP_CUDA(cudaMemcpyAsync(x, h0.stage_out.p, h0.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    MSP_CUDA(cudaStreamSynchronize(st));
    for (Handle* hp : hs) { msp::dist_free(hp->dist); hp->dist = nullptr; }
  });
}

// debugging aid (not in the header): the device scalars of the last solve
int msp_debug_scalars(msp_handle* H, double* out, int64_t n) {
  return guarded([&] {
    need(H && out && n > 0, "null argument");
    MSP_CUDA(cudaMemcpy(out, H->h.scal.p, std::min<int64_t>(n, (int64_t)H->h.scal.n) * sizeof(double),
                        cudaMemcpyDeviceToHost));
  });
}

int msp_set_profiling(msp_handle* H, int on) {
  return guarded([&] {
    need(H != nullptr, "null handle");
    H->h.profile = on ? 1 : 0;
  });
}

int msp_get_profile(msp_handle* H, double* ms, int64_t* counts) {
  return guarded([&] {
    need(H && ms && counts, "null argument");
    for (int i = 0; i < MSP_PROF_NCAT; ++i) {
      ms[i] = H->h.prof_ms[i];
      counts[i] = H->h.prof_cnt[i];
      H->h.prof_ms[i] = 0.0;
      H->h.prof_cnt[i] = 0;
    }
  });
}

}  // extern "C"
