// C ABI of include/phiks.h: handles, planning, apply, building blocks.
#include "host.h"

namespace phiks {
namespace host {
thread_local std::string g_err;
}  // namespace host
}  // namespace phiks

extern "C" {

const char* phiks_last_error(void) { return g_err.c_str(); }
const char* phiks_version(void) { return "phiks-b200 0.1.0 (sm_100a, fp64 DMMA)"; }

}  // extern "C"

namespace {

// Real form of a complex n×n column-major matrix given as interleaved (re, im)
// doubles: the 2n×2n matrix acting on interleaved vectors,
// R[(c+2j) + (c'+2k)·2n] = [[Ar, −Ai], [Ai, Ar]]_{cc'}(j, k).
std::vector<double> realify(int n, const double* Az) {
  const size_t m = 2 * static_cast<size_t>(n);
  std::vector<double> R(m * m);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      const double ar = Az[2 * (j + static_cast<size_t>(k) * n)], ai = Az[2 * (j + static_cast<size_t>(k) * n) + 1];
      R[(2 * j) + (2 * k) * m] = ar;
      R[(2 * j + 1) + (2 * k) * m] = ai;
      R[(2 * j) + (2 * k + 1) * m] = -ai;
      R[(2 * j + 1) + (2 * k + 1) * m] = ar;
    }
  return R;
}

phiks_status create_impl(int d, const int* n, const double* const* A_host, bool cplx, phiks_handle* out,
                         int nblocks = 1) {
  if (!out || !n || !A_host) return fail(PHIKS_ERR_ARG, "null argument");
  *out = nullptr;
  if (d < 1 || d > PHIKS_MAX_D) return fail(PHIKS_ERR_ARG, "d out of range");
  if (nblocks < 1 || nblocks > kMaxBlocks) return fail(PHIKS_ERR_ARG, "nblocks out of range");
  for (int k = 0; k < nblocks * d; ++k)
    if (!A_host[k]) return fail(PHIKS_ERR_ARG, "null A");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PHIKS_ERR_CUDA, "no CUDA device");
  auto* h = new phiks_ctx();
  h->d = d;
  h->cplx = cplx;
  h->nblocks = nblocks;
  h->Nc = 1;
  for (int mu = 0; mu < d; ++mu) {
    if (n[mu] < 1 || n[mu] > PHIKS_MAX_N || !A_host[mu]) {
      delete h;
      return fail(PHIKS_ERR_ARG, "n[mu] out of range or null A");
    }
    h->n[mu] = n[mu];
    h->gn[mu] = n[mu];
    h->Nc *= n[mu];
  }
  h->N = cplx ? 2 * h->Nc : h->Nc;
  const int per = cplx ? 2 : 1;  // doubles per matrix entry
  // dedupe bitwise-identical factors (across modes and blocks)
  std::vector<int> rep;  // A_host index of each distinct factor
  for (int bm = 0; bm < nblocks * d; ++bm) {
    const int mu = bm % d;
    const double* Ah = A_host[bm];
    int found = -1;
    for (size_t f = 0; f < rep.size(); ++f) {
      const int m2 = rep[f];
      if (n[m2 % d] == n[mu] &&
          std::memcmp(A_host[m2], Ah, sizeof(double) * per * static_cast<size_t>(n[mu]) * n[mu]) == 0) {
        found = static_cast<int>(f);
        break;
      }
    }
    if (found < 0) {
      Factor F;
      // complex factors are stored (and exponentiated) in their 2n×2n real form:
      // exp of the real form is the real form of exp (an algebra homomorphism)
      std::vector<double> Rz;
      const double* A = Ah;
      if (cplx) {
        Rz = realify(n[mu], Ah);
        A = Rz.data();
      }
      F.n = per * n[mu];
      const size_t bytes = sizeof(double) * static_cast<size_t>(F.n) * F.n;
      if (cudaMalloc(&F.dA, bytes) != cudaSuccess) {
        phiks_destroy(h);
        return fail(PHIKS_ERR_NOMEM, "cudaMalloc A");
      }
      if (cudaMemcpy(F.dA, A, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(F.dA);
        phiks_destroy(h);
        return fail(PHIKS_ERR_CUDA, "copy A");
      }
      double nrm = 0.0;
      for (int j = 0; j < F.n; ++j) {
        double c = 0.0;
        for (int i = 0; i < F.n; ++i) c += std::fabs(A[i + static_cast<size_t>(j) * F.n]);
        nrm = std::max(nrm, c);
      }
      F.norm1 = nrm;
      F.metzler = !cplx;
      for (int j = 0; j < F.n && F.metzler; ++j)
        for (int i = 0; i < F.n; ++i)
          if (i != j && !(A[i + static_cast<size_t>(j) * F.n] >= 0.0)) {
            F.metzler = false;
            break;
          }
      F.fr = cplx ? plan::factor_range_complex(n[mu], Ah) : plan::factor_range(F.n, A);
      h->factors.push_back(F);
      rep.push_back(bm);
      found = static_cast<int>(h->factors.size()) - 1;
    }
    h->fac_of_block[bm / d][mu] = found;
  }
  if (cudaMallocHost(reinterpret_cast<void**>(&h->h_pinned), 64 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&h->h_barrier_err), sizeof(int)) != cudaSuccess) {
    phiks_destroy(h);
    return fail(PHIKS_ERR_NOMEM, "pinned host scratch");
  }
  *h->h_barrier_err = 0;
  *out = h;
  return PHIKS_OK;
}

}  // namespace

extern "C" {

phiks_status phiks_create(int d, const int* n, const double* const* A_host, phiks_handle* out) {
  return create_impl(d, n, A_host, false, out);
}

phiks_status phiks_create_complex(int d, const int* n, const double* const* A_host, phiks_handle* out) {
  return create_impl(d, n, A_host, true, out);
}

phiks_status phiks_create_blocks(int nblocks, int d, const int* n, const double* const* A_host, phiks_handle* out) {
  return create_impl(d, n, A_host, false, out, nblocks);
}

phiks_status phiks_create_blocks_complex(int nblocks, int d, const int* n, const double* const* A_host,
                                         phiks_handle* out) {
  return create_impl(d, n, A_host, true, out, nblocks);
}

phiks_status phiks_destroy(phiks_handle h) {
  if (!h) return PHIKS_OK;
  for (auto& F : h->factors)
    if (F.dA) cudaFree(F.dA);
  if (h->ws_own) cudaFree(h->ws_own);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  if (h->h_barrier_err) cudaFreeHost(h->h_barrier_err);
  if (h->d_kcount) cudaFree(h->d_kcount);
  for (int k = 0; k < kMaxRanks; ++k)
    if (h->peer_ipc[k] && h->peer[k]) cudaIpcCloseMemHandle(h->peer[k]);
  for (cudaEvent_t e : {h->ev_h2d, h->ev_d2h[0], h->ev_d2h[1], h->ev_cdone[0], h->ev_cdone[1], h->ev_ready})
    if (e) cudaEventDestroy(e);
  for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
  if (h->s_cap) cudaStreamDestroy(h->s_cap);
  if (h->s_pre) cudaStreamDestroy(h->s_pre);
  if (h->ev_pre) cudaEventDestroy(h->ev_pre);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  if (h->sym) cudaFree(h->sym);
  for (auto& e : h->ev) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  delete h;
  return PHIKS_OK;
}

}  // extern "C"

namespace phiks {
namespace host {


phiks_status validate(phiks_handle h, const phiks_request* req, int& p) {
  if (!h || !req) return fail(PHIKS_ERR_ARG, "null argument");
  if (req->mode != PHIKS_MODE_SAME_VECTOR && req->mode != PHIKS_MODE_LINCOMB) return fail(PHIKS_ERR_ARG, "mode");
  if (req->n_ells < 1 || req->n_ells > PHIKS_MAX_P + 1 || !req->ells) return fail(PHIKS_ERR_ARG, "n_ells");
  if (req->n_scales < 1 || req->n_scales > PHIKS_MAX_SCALES) return fail(PHIKS_ERR_LIMIT, "n_scales");
  if (!(req->tau > 0.0) || !std::isfinite(req->tau)) return fail(PHIKS_ERR_ARG, "tau must be > 0");
  if (req->mem_kind != PHIKS_MEM_DEVICE && req->mem_kind != PHIKS_MEM_HOST && req->mem_kind != PHIKS_MEM_HOST_ASYNC)
    return fail(PHIKS_ERR_ARG, "mem_kind");
  p = -1;
  for (int i = 0; i < req->n_ells; ++i) {
    const int e = req->ells[i];
    if (e < 0 || e > PHIKS_MAX_P) return fail(PHIKS_ERR_LIMIT, "order out of range");
    if (i > 0 && e <= req->ells[i - 1]) return fail(PHIKS_ERR_ARG, "ells must be strictly increasing");
    p = std::max(p, e);
  }
  if (req->force_s >= 0 && p >= 1 && req->force_q < 2) return fail(PHIKS_ERR_ARG, "force_q < 2");
  if (req->force_s >= 0 && req->force_s < req->n_scales - 1) return fail(PHIKS_ERR_ARG, "force_s < n_scales-1");
  return PHIKS_OK;
}

// Tucker operators run_jobs executes (reading R9): θ_q = 1 costs none; at the
// last squaring step (or at s = 0) only the output combinations are formed —
// Ψ_p for a linear combination, the requested φ_ℓ for the same vector
// (PAPER.md l.953-956); a linear combination's quadrature at s ≥ 1 runs one
// operator per node and given vector v_ℓ (ℓ ≥ 1).  Lincomb with v_1..v_p, without
// v_0, ŝ = 1: (q−2)p + sp + 1 (Table 1).
int tucker_executed(const phiks_request* req, int p, const plan::Plan& pl) {
  const bool same = req->mode == PHIKS_MODE_SAME_VECTOR;
  const bool has0 = req->ells[0] == 0;
  const int n0 = has0 ? req->n_scales : 0;
  if (p == 0) return n0;
  int given = 0;  // requested orders ℓ ≥ 1 (lincomb: the given vectors v_ℓ)
  for (int i = 0; i < req->n_ells; ++i) given += req->ells[i] >= 1;
  const int last = same ? given : 1;
  const int sq = pl.s >= 1 ? (pl.s - 1) * p + last : 0;
  const int quad = same ? pl.q - 1 : (pl.q - 1) * (pl.s >= 1 ? given : 1);
  return quad + sq + n0;
}

phiks_status make_plan(phiks_handle h, const phiks_request* req, int p, const std::vector<double>& norms,
                       plan::Plan& out, int block) {
  const int s_min = req->n_scales - 1;
  if (req->force_s >= 0) {
    out.s = req->force_s;
    out.q = (p >= 1) ? req->force_q : 0;
    out.T = plan::tucker_count(req->mode, out.s, req->n_scales, out.q, p);
    out.ok = true;
    return PHIKS_OK;
  }
  const double tol = req->tol > 0 ? req->tol : std::ldexp(1.0, -53);
  PlanKey key{req->mode, p, req->n_scales, req->tau, tol, norms, block};
  auto it = h->plan_cache.find(key);
  if (it != h->plan_cache.end()) {
    out = it->second;
    return PHIKS_OK;
  }
  plan::Rect rect{};
  double cr = 0.0, ci = 0.0, hr = 0.0, hi = 0.0;
  for (int mu = 0; mu < h->d; ++mu) {
    const auto& fr = h->factors[h->fac_of_block[block][mu]].fr;
    cr += req->tau * fr.sigma;
    ci += req->tau * fr.sigma_im;
    hr += req->tau * fr.hnorm;
    hi += req->tau * fr.snorm;
  }
  rect.center = std::complex<double>(cr, ci);
  rect.hr = hr;
  rect.hi = hi;
  if (p == 0) {
    out = plan::select_plan(req->mode, rect, 0, norms, 0.0, req->n_scales, s_min);
  } else if (req->mode == PHIKS_MODE_SAME_VECTOR) {
    // reading R2: δ = tol·||v||, and ||v|| cancels in ||R||·||v|| ≤ δ 2^{ℓs}
    out = plan::select_plan(req->mode, rect, p, std::vector<double>{1.0}, tol, req->n_scales, s_min);
  } else {
    double mx = 0.0;
    for (double v : norms) mx = std::max(mx, v);
    if (mx == 0.0) {
      out.s = s_min;
      out.q = 2;
      out.T = plan::tucker_count(req->mode, s_min, req->n_scales, 2, p);
      out.ok = true;
    } else {
      out = plan::select_plan(req->mode, rect, p, norms, tol * mx, req->n_scales, s_min);
    }
  }
  if (!out.ok) return fail(PHIKS_ERR_PLAN, "no admissible (s, q) in the §3.3 search");
  h->plan_cache[key] = out;
  return PHIKS_OK;
}


// error flag of the cross-rank barrier (sticky; read with a synchronous copy)
phiks_status check_barrier_flag(phiks_handle h) {
  if (!h->sharded() || !h->sym) return PHIKS_OK;
  int err = 0;
  CUDA_TRY(cudaMemcpy(&err, h->sym + kCtrlErr, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) return fail(PHIKS_ERR_CUDA, "cross-rank barrier timed out (a peer rank did not arrive)");
  return PHIKS_OK;
}


}  // namespace host
}  // namespace phiks


extern "C" {

phiks_status phiks_plan(phiks_handle h, const phiks_request* req, const double* vec_norms, phiks_plan_info* out) {
  int p = 0;
  phiks_status st = validate(h, req, p);
  if (st != PHIKS_OK) return st;
  if (!out) return fail(PHIKS_ERR_ARG, "null out");
  std::vector<double> norms;
  if (req->mode == PHIKS_MODE_LINCOMB && p >= 1) {
    if (!vec_norms) return fail(PHIKS_ERR_ARG, "lincomb plan needs vec_norms");
    norms.assign(vec_norms, vec_norms + p);
  }
  plan::Plan pl;
  st = make_plan(h, req, p, norms, pl);
  if (st != PHIKS_OK) return st;
  out->s = pl.s;
  out->q = pl.q;
  out->T_formula = pl.T;
  out->T_executed = tucker_executed(req, p, pl);
  return PHIKS_OK;
}

}  // extern "C"

extern "C" {

static phiks_status apply_impl(phiks_handle h, const phiks_request* req, int n_vecs, const double* const* vecs,
                               double* const* outs, void* workspace, size_t ws_bytes, void* stream,
                               bool size_only, const phiks_plan_info* forced, size_t* size_out) {
  // sharded handles: the barrier's sticky error flag of earlier applies, copied to pinned
  // memory at the end of each apply (stream-ordered, no synchronisation): a device-memory
  // apply reports a timed-out peer at the latest on the next call
  if (!size_only && h && h->sharded() && h->h_barrier_err && *static_cast<volatile int*>(h->h_barrier_err))
    return fail(PHIKS_ERR_CUDA, "cross-rank barrier timed out in an earlier apply (a peer rank did not arrive)");
  ApplyRun run;
  phiks_status st = run.init(h, req, n_vecs, vecs, outs, stream, size_only);
  if (st != PHIKS_OK) return st;
  if (!forced && run.need_norms) {
    st = run.norms_enqueue(true);
    if (st != PHIKS_OK) return st;
    st = run.norms_finish(h->sym);
  } else {
    st = run.plan_direct(forced);
  }
  if (st != PHIKS_OK) return st;
  size_t need = 0;
  st = run.measure(&need);
  if (st != PHIKS_OK) return st;
  if (size_out) *size_out = need;
  if (size_only) return PHIKS_OK;
  char* base = nullptr;
  st = run.workspace(workspace, ws_bytes, need, &base);
  if (st != PHIKS_OK) return st;
  const bool graphs_on = h->opt_graphs != 0;
  // graphs pay off where launch overhead matters (small tensors); large applies
  // keep direct launches so their exponential stage overlaps on the side stream
  const bool small_apply = h->N <= (int64_t(1) << 22);
  if (graphs_on && small_apply && !run.host_mem && !h->profiling) {
    const cudaStream_t cs = run.cs;
    // key: everything the recorded launches depend on
    std::vector<uint64_t> key;
    auto bits = [](double x) {
      uint64_t u;
      std::memcpy(&u, &x, sizeof(u));
      return u;
    };
    key.insert(key.end(), {static_cast<uint64_t>(req->mode), static_cast<uint64_t>(req->n_scales), bits(req->tau),
                           bits(req->tol), static_cast<uint64_t>(run.split), reinterpret_cast<uint64_t>(base), need});
    for (const auto& pl : run.pls) key.insert(key.end(), {static_cast<uint64_t>(pl.s), static_cast<uint64_t>(pl.q)});
    for (int i = 0; i < req->n_ells; ++i) key.push_back(static_cast<uint64_t>(req->ells[i]));
    for (int i = 0; i < n_vecs; ++i) key.push_back(reinterpret_cast<uint64_t>(vecs[i]));
    for (int i = 0; i < run.nouts; ++i) key.push_back(reinterpret_cast<uint64_t>(outs[i]));
    cudaGraphExec_t exec = nullptr;
    for (auto& g : h->graphs)
      if (g.key == key) exec = g.exec;
    if (!exec) {
      if (!h->s_cap) CUDA_TRY(cudaStreamCreateWithFlags(&h->s_cap, cudaStreamNonBlocking));
      if (h->graphs.size() >= 32) {
        CUDA_TRY(cudaStreamSynchronize(cs));
        for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
        h->graphs.clear();
      }
      run.cs = h->s_cap;
      CUDA_TRY(cudaStreamBeginCapture(h->s_cap, cudaStreamCaptureModeThreadLocal));
      st = run.execute(base, need, nullptr);
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(h->s_cap, &graph);
      run.cs = cs;
      if (st != PHIKS_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (ce != cudaSuccess) return fail(PHIKS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) return fail(PHIKS_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
      h->graphs.push_back({key, exec});
    } else {
      ++h->graph_replays;
    }
    CUDA_TRY(cudaGraphLaunch(exec, cs));
    for (int k = 0; k < 2; ++k)
      if (!h->ev_cdone[k]) CUDA_TRY(cudaEventCreateWithFlags(&h->ev_cdone[k], cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(h->ev_cdone[run.half], cs));  // orders later side-stream work after this replay
    if (h->sharded())
      CUDA_TRY(cudaMemcpyAsync(h->h_barrier_err, h->sym + kCtrlErr, sizeof(int), cudaMemcpyDeviceToHost, cs));
    run.finish_stats(need);
    return PHIKS_OK;
  }
  st = run.execute(base, need, nullptr);
  if (st != PHIKS_OK) return st;
  if (h->sharded())
    CUDA_TRY(cudaMemcpyAsync(h->h_barrier_err, h->sym + kCtrlErr, sizeof(int), cudaMemcpyDeviceToHost, run.cs));
  if (run.host_mem && !run.host_async) {
    CUDA_TRY(cudaEventSynchronize(h->ev_d2h[run.half]));
    CUDA_TRY(cudaStreamSynchronize(run.cs));
    st = check_barrier_flag(h);
    if (st != PHIKS_OK) return st;
  }
  run.finish_stats(need);
  return PHIKS_OK;
}

phiks_status phiks_apply(phiks_handle h, const phiks_request* req, int n_vecs, const double* const* vecs,
                         double* const* outs, void* workspace, size_t ws_bytes, void* stream) {
  return apply_impl(h, req, n_vecs, vecs, outs, workspace, ws_bytes, stream, false, nullptr, nullptr);
}

phiks_status phiks_workspace_size(phiks_handle h, const phiks_request* req, const phiks_plan_info* plan,
                                  size_t* bytes) {
  if (!bytes) return fail(PHIKS_ERR_ARG, "null bytes");
  return apply_impl(h, req, 0, nullptr, nullptr, nullptr, 0, nullptr, true, plan, bytes);
}

phiks_status phiks_get_stats(phiks_handle h, phiks_stats* out) {
  if (!h || !out) return fail(PHIKS_ERR_ARG, "null argument");
  {
    phiks_status st = check_barrier_flag(h);
    if (st != PHIKS_OK) return st;
  }
  *out = h->stats;
  out->mode_product_launches = 0;
  out->mode_product_ms = 0.0;
  out->mode_product_flops = 0.0;
  out->expm_launches = 0;
  out->expm_ms = 0.0;
  out->i8_launches = 0;
  out->i8_ms = 0.0;
  out->i8_flops = 0.0;
  out->i8_gemm_launches = 0;
  out->i8_gemm_ms = 0.0;
  out->i8_kblocks = out->i8_kblocks_run = 0;
  if (h->profiling) {
    if (h->d_kcount) {
      unsigned long long kc[2] = {0, 0};
      CUDA_TRY(cudaMemcpy(kc, h->d_kcount, sizeof(kc), cudaMemcpyDeviceToHost));
      out->i8_kblocks = static_cast<int64_t>(kc[0]);
      out->i8_kblocks_run = static_cast<int64_t>(kc[1]);
    }
    for (int i = 0; i < h->ev_used; ++i) {
      CUDA_TRY(cudaEventSynchronize(h->ev[i].second));
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, h->ev[i].first, h->ev[i].second));
      if (h->ev_expm[i] == 1) {
        out->expm_ms += ms;
        ++out->expm_launches;
      } else {
        out->mode_product_ms += ms;
        out->mode_product_flops += h->ev_flops[i];
        ++out->mode_product_launches;
        if (h->ev_expm[i] >= 2) {
          out->i8_ms += ms;
          out->i8_flops += h->ev_flops[i];
          ++out->i8_launches;
        }
        if (h->ev_expm[i] == 2) {
          out->i8_gemm_ms += ms;
          ++out->i8_gemm_launches;
        }
      }
    }
  }
  return PHIKS_OK;
}

phiks_status phiks_set_gemm_path(phiks_handle h, int path) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  if (path != PHIKS_GEMM_AUTO && path != PHIKS_GEMM_DMMA && path != PHIKS_GEMM_I8)
    return fail(PHIKS_ERR_ARG, "unknown gemm path");
  if (h->gemm_path != path) {
    for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);  // captured with the other path
    h->graphs.clear();
    h->gemm_path = path;
  }
  return PHIKS_OK;
}

phiks_status phiks_set_option(phiks_handle h, int option, int value) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  int* slot = nullptr;
  int lo = 0, hi = 0;
  switch (option) {
    case PHIKS_OPT_SPLIT: slot = &h->opt_split; hi = 2; break;
    case PHIKS_OPT_CHAIN: slot = &h->opt_chain; hi = 2; break;
    case PHIKS_OPT_GRAPHS: slot = &h->opt_graphs; hi = 1; break;
    case PHIKS_OPT_PRESPLIT: slot = &h->opt_presplit; hi = 1; break;
    case PHIKS_OPT_KSKIP: slot = &h->opt_kskip; hi = 1; break;
    default: return fail(PHIKS_ERR_ARG, "unknown option");
  }
  if (value < lo || value > hi) return fail(PHIKS_ERR_ARG, "option value out of range");
  if (*slot != value) {
    for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);  // captured under the other setting
    h->graphs.clear();
    *slot = value;
  }
  return PHIKS_OK;
}

phiks_status phiks_get_option(phiks_handle h, int option, int* value) {
  if (!h || !value) return fail(PHIKS_ERR_ARG, "null argument");
  switch (option) {
    case PHIKS_OPT_SPLIT: *value = h->opt_split; break;
    case PHIKS_OPT_CHAIN: *value = h->opt_chain; break;
    case PHIKS_OPT_GRAPHS: *value = h->opt_graphs; break;
    case PHIKS_OPT_PRESPLIT: *value = h->opt_presplit; break;
    case PHIKS_OPT_KSKIP: *value = h->opt_kskip; break;
    default: return fail(PHIKS_ERR_ARG, "unknown option");
  }
  return PHIKS_OK;
}

phiks_status phiks_set_profiling(phiks_handle h, int on) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  h->profiling = on != 0;
  h->ev_used = 0;
  if (h->profiling) {  // k-block counters since profiling was switched on
    if (!h->d_kcount) CUDA_TRY(cudaMalloc(&h->d_kcount, 2 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemset(h->d_kcount, 0, 2 * sizeof(unsigned long long)));
  }
  return PHIKS_OK;
}

phiks_status phiks_mode_product(int d, const int* n, int mu, int batch, const double* const* in,
                                const double* const* M, double* const* out, void* stream) {
  if (d < 1 || d > PHIKS_MAX_D || !n || mu < 0 || mu >= d || batch < 0 || (batch > 0 && (!in || !M || !out)))
    return fail(PHIKS_ERR_ARG, "bad argument");
  int64_t L = 1, R = 1;
  for (int k = 0; k < mu; ++k) L *= n[k];
  for (int k = mu + 1; k < d; ++k) R *= n[k];
  size_t i = 0;
  while (i < static_cast<size_t>(batch)) {
    ModeParams* pp = new ModeParams();
    pp->L = L;
    pp->R = R;
    pp->n = n[mu];
    int g = 0;
    for (; g < kMaxGroups && i < static_cast<size_t>(batch); ++g, ++i) {
      pp->groups[g] = GroupSpec{g, g + 1};
      pp->terms[g] = TermSpec{in[i], M[i], g, 1};
      pp->outs[g] = OutSpec{out[i], 1.0, 0, 0};
    }
    pp->ngroups = g;
    cudaError_t e = launch_mode_product(*pp, static_cast<cudaStream_t>(stream));
    delete pp;
    if (e != cudaSuccess) return fail(PHIKS_ERR_CUDA, std::string("mode_product: ") + cudaGetErrorString(e));
  }
  return PHIKS_OK;
}

phiks_status phiks_mode_product_i8_workspace(int d, const int* n, int mu, int slices, int batch, size_t* bytes) {
  if (d < 1 || d > PHIKS_MAX_D || !n || mu < 0 || mu >= d || batch < 0 || !bytes) return fail(PHIKS_ERR_ARG, "bad argument");
  int64_t L = 1, R = 1;
  for (int k = 0; k < mu; ++k) L *= n[k];
  for (int k = mu + 1; k < d; ++k) R *= n[k];
  if (!ozaki_supported(L, n[mu], R, slices)) return fail(PHIKS_ERR_ARG, "int8 mode product: unsupported size or slices");
  const int cap = std::min(std::max(batch, 1), kMaxTerms);
  *bytes = ozaki_workspace_bytes(L, n[mu], R, slices, cap, cap);
  return PHIKS_OK;
}

phiks_status phiks_mode_product_i8(int d, const int* n, int mu, int slices, int batch, const double* const* in,
                                   const double* const* M, double* const* out, void* workspace, size_t ws_bytes,
                                   void* stream) {
  size_t need = 0;
  phiks_status st = phiks_mode_product_i8_workspace(d, n, mu, slices, batch, &need);
  if (st != PHIKS_OK) return st;
  if (batch > 0 && (!in || !M || !out)) return fail(PHIKS_ERR_ARG, "bad argument");
  if (!workspace || ws_bytes < need) return fail(PHIKS_ERR_ARG, "workspace too small");
  int64_t L = 1, R = 1;
  for (int k = 0; k < mu; ++k) L *= n[k];
  for (int k = mu + 1; k < d; ++k) R *= n[k];
  for (int i0 = 0; i0 < batch; i0 += kMaxTerms) {
    OzakiParams* pp = new OzakiParams();
    OzakiParams& p = *pp;
    p.L = L;
    p.R = R;
    p.n = n[mu];
    p.S = slices;
    p.kskip = 1;
    p.nx = p.ne = p.nterms = 0;
    for (int i = i0; i < std::min(batch, i0 + kMaxTerms); ++i) {
      int xs = -1, es = -1;
      for (int k = 0; k < p.nx; ++k)
        if (p.x[k] == in[i]) xs = k;
      for (int k = 0; k < p.ne; ++k)
        if (p.e[k] == M[i]) es = k;
      if (xs < 0) {
        xs = p.nx;
        p.x[p.nx++] = in[i];
      }
      if (es < 0) {
        es = p.ne;
        p.e[p.ne++] = M[i];
      }
      p.terms[p.nterms++] = OzakiTerm{xs, es, out[i], 1.0};
    }
    ozaki_bind_workspace(p, workspace);
    cudaError_t e = launch_ozaki_mode(p, static_cast<cudaStream_t>(stream));
    delete pp;
    if (e != cudaSuccess) return fail(PHIKS_ERR_CUDA, std::string("int8 mode product: ") + cudaGetErrorString(e));
  }
  return PHIKS_OK;
}

phiks_status phiks_tucker(int d, const int* n, const double* in, const double* const* M, double* out,
                          double* scratch, void* stream) {
  if (d < 1 || d > PHIKS_MAX_D || !n || !in || !M || !out || (d > 1 && !scratch))
    return fail(PHIKS_ERR_ARG, "bad argument");
  int64_t N = 1;
  for (int k = 0; k < d; ++k) N *= n[k];
  const double* cur = in;
  for (int mu = 0; mu < d; ++mu) {
    double* dst = (mu == d - 1) ? out : scratch + (mu % 2) * N;
    phiks_status st = phiks_mode_product(d, n, mu, 1, &cur, &M[mu], &dst, stream);
    if (st != PHIKS_OK) return st;
    cur = dst;
  }
  return PHIKS_OK;
}

phiks_status phiks_expm(int n, const double* A, double c, double* E, double* scratch, void* stream) {
  if (n < 1 || n > PHIKS_MAX_N || !A || !E || !scratch) return fail(PHIKS_ERR_ARG, "bad argument");
  // temporary single-factor context on caller memory
  phiks_ctx h;
  h.d = 1;
  h.n[0] = n;
  h.N = n;
  h.Nc = n;
  Factor F;
  F.n = n;
  F.dA = const_cast<double*>(A);
  // ||A||_1 needs host data: read back (small, test/bench API only)
  std::vector<double> hA(static_cast<size_t>(n) * n);
  CUDA_TRY(cudaMemcpy(hA.data(), A, sizeof(double) * hA.size(), cudaMemcpyDeviceToHost));
  double nrm = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::fabs(hA[i + static_cast<size_t>(j) * n]);
    nrm = std::max(nrm, s);
  }
  F.norm1 = nrm;
  h.factors.push_back(F);
  Arena ar;
  ar.measure = true;
  {
    Exec exm{&h, static_cast<cudaStream_t>(stream), true, &ar};
    std::vector<ExpReq> r0{{0, c}};
    expm_batch(exm, 1.0, r0);
  }
  if (ar.off > sizeof(double) * (8 * static_cast<size_t>(n) * n + 256)) {
    h.factors.clear();
    return fail(PHIKS_ERR_WORKSPACE, "expm scratch too small");
  }
  ar.off = 0;
  ar.base = reinterpret_cast<char*>(scratch);
  ar.cap = sizeof(double) * (8 * static_cast<size_t>(n) * n + 256);
  ar.measure = false;
  Exec ex{&h, static_cast<cudaStream_t>(stream), false, &ar};
  std::vector<ExpReq> reqs{{0, c}};
  expm_batch(ex, 1.0, reqs);
  h.factors.clear();
  if (!ex.ok()) return ex.status;
  CUDA_TRY(cudaMemcpyAsync(E, reqs[0].result, sizeof(double) * static_cast<size_t>(n) * n, cudaMemcpyDeviceToDevice,
                           static_cast<cudaStream_t>(stream)));
  return PHIKS_OK;
}

static phiks_status plan_host_impl(int d, const int* n, const double* const* A_host, bool cplx,
                                   const phiks_request* req, const double* vec_norms, phiks_plan_info* out) {
  if (!n || !A_host || !req || !out || d < 1 || d > PHIKS_MAX_D) return fail(PHIKS_ERR_ARG, "bad argument");
  phiks_ctx h;  // host-only context: factor ranges, no device buffers
  h.d = d;
  h.N = 1;
  for (int mu = 0; mu < d; ++mu) {
    if (n[mu] < 1 || n[mu] > PHIKS_MAX_N || !A_host[mu]) return fail(PHIKS_ERR_ARG, "bad factor");
    h.n[mu] = n[mu];
    h.gn[mu] = n[mu];
    h.N *= n[mu];
    h.Nc = h.N;
    Factor F;
    F.n = n[mu];
    F.fr = cplx ? plan::factor_range_complex(F.n, A_host[mu]) : plan::factor_range(F.n, A_host[mu]);
    h.factors.push_back(F);
    h.fac_of_block[0][mu] = mu;
  }
  return phiks_plan(&h, req, vec_norms, out);
}

phiks_status phiks_plan_host(int d, const int* n, const double* const* A_host, const phiks_request* req,
                             const double* vec_norms, phiks_plan_info* out) {
  return plan_host_impl(d, n, A_host, false, req, vec_norms, out);
}

phiks_status phiks_plan_host_complex(int d, const int* n, const double* const* A_host, const phiks_request* req,
                                     const double* vec_norms, phiks_plan_info* out) {
  return plan_host_impl(d, n, A_host, true, req, vec_norms, out);
}

phiks_status phiks_select_plan(int mode, double center_re, double center_im, double hr, double hi, int p,
                               const double* norms, double delta, int s_hat, int s_min, int s_fixed,
                               phiks_plan_info* out) {
  if (!out || p < 0 || p > PHIKS_MAX_P || (p > 0 && !norms)) return fail(PHIKS_ERR_ARG, "bad argument");
  plan::Rect rect{std::complex<double>(center_re, center_im), hr, hi};
  const int nn = (mode == PHIKS_MODE_SAME_VECTOR) ? 1 : p;
  std::vector<double> nv(norms, norms + (p > 0 ? nn : 0));
  if (s_fixed >= 0) {
    out->s = s_fixed;
    out->q = p > 0 ? plan::q_for_s(mode, rect, p, nv, delta, s_fixed) : 0;
    out->T_formula = plan::tucker_count(mode, s_fixed, s_hat, out->q, p);
    out->T_executed = -1;
    return PHIKS_OK;
  }
  plan::Plan pl = plan::select_plan(mode, rect, p, nv, delta, s_hat, s_min);
  if (!pl.ok) return fail(PHIKS_ERR_PLAN, "no admissible (s, q)");
  out->s = pl.s;
  out->q = pl.q;
  out->T_formula = pl.T;
  out->T_executed = -1;
  return PHIKS_OK;
}

phiks_status phiks_fp64_peak_launch(int kind, int blocks, int64_t iters, double* sink, void* stream, double* flops) {
  if (!sink || !flops || blocks < 1 || iters < 1 || (kind != 0 && kind != 1)) return fail(PHIKS_ERR_ARG, "bad argument");
  cudaError_t e = launch_fp64_peak(kind, blocks, iters, sink, static_cast<cudaStream_t>(stream), flops);
  if (e != cudaSuccess) return fail(PHIKS_ERR_CUDA, cudaGetErrorString(e));
  return PHIKS_OK;
}

}  // extern "C"
