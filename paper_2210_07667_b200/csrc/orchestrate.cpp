// The job of one apply as kernel launches: the exponential stage and the
// quadrature / squaring / exp-action Tucker batches (see host.h).
#include "host.h"

namespace phiks {
namespace host {

void expm_batch(Exec& ex, double tau, std::vector<ExpReq>& reqs) {
  phiks_ctx* h = ex.h;
  const int nf = static_cast<int>(h->factors.size());
  std::vector<char> used(nf, 0);
  for (auto& r : reqs) used[r.f] = 1;
  // per-factor powers
  std::vector<double*> X1(nf, nullptr), X2(nf), X3(nf), X4(nf);
  std::map<int, double*> Ident;
  for (int f = 0; f < nf; ++f) {
    if (!used[f]) continue;
    const int n = h->factors[f].n;
    const int64_t nn = static_cast<int64_t>(n) * n;
    X1[f] = ex.ar->alloc_doubles(nn);
    X2[f] = ex.ar->alloc_doubles(nn);
    X3[f] = ex.ar->alloc_doubles(nn);
    X4[f] = ex.ar->alloc_doubles(nn);
    if (!Ident.count(n)) {
      Ident[n] = ex.ar->alloc_doubles(nn);
      double* I = Ident[n];
      ex.emit("set_identity", [I, n](cudaStream_t s) { return launch_set_identity(I, n, 1.0, s); });
    }
  }
  // distinct n values
  std::vector<int> ns;
  for (int f = 0; f < nf; ++f)
    if (used[f] && std::find(ns.begin(), ns.end(), h->factors[f].n) == ns.end()) ns.push_back(h->factors[f].n);
  for (int n : ns) {
    const int64_t nn = static_cast<int64_t>(n) * n;
    std::vector<Out> sc;
    for (int f = 0; f < nf; ++f)
      if (used[f] && h->factors[f].n == n) sc.push_back(Out{X1[f], 0.0, {Src{h->factors[f].dA, tau}}});
    ex.combine(nn, sc);
    std::vector<Exec::LaunchTerm> t2, t3, t4;
    for (int f = 0; f < nf; ++f)
      if (used[f] && h->factors[f].n == n) t2.push_back({X1[f], X1[f], f, {Out{X2[f], 1.0, {}}}});
    ex.gemm_batch(n, t2);
    for (int f = 0; f < nf; ++f)
      if (used[f] && h->factors[f].n == n) {
        t3.push_back({X1[f], X2[f], f, {Out{X3[f], 1.0, {}}}});   // X2·X1
        t4.push_back({X2[f], X2[f], f, {Out{X4[f], 1.0, {}}}});   // X2·X2
      }
    for (auto& t : t4) t3.push_back(t);
    for (size_t i = 0; i < t3.size(); ++i) t3[i].group = static_cast<int>(i);
    ex.gemm_batch(n, t3);
  }
  // per request: scaling, Horner in X4, squarings
  struct St {
    double a;
    int sigma;
    double* buf[2];
    int cur;
  };
  std::vector<St> sts(reqs.size());
  int max_sigma = 0;
  for (size_t i = 0; i < reqs.size(); ++i) {
    const Factor& F = h->factors[reqs[i].f];
    const double nrm = std::fabs(reqs[i].c) * tau * F.norm1;
    int sigma = 0;
    if (nrm > 0.5) sigma = static_cast<int>(std::ceil(std::log2(nrm / 0.5)));
    sts[i].sigma = sigma;
    sts[i].a = reqs[i].c / std::ldexp(1.0, sigma);
    const int64_t nn = static_cast<int64_t>(F.n) * F.n;
    sts[i].buf[0] = ex.ar->alloc_doubles(nn);
    sts[i].buf[1] = ex.ar->alloc_doubles(nn);
    sts[i].cur = 0;
    max_sigma = std::max(max_sigma, sigma);
  }
  auto coefs = [](double a, int base) {  // B_m coefficients a^r/(base+r)!, r = 0..3 (base = 4m)
    std::vector<double> c(4);
    for (int r = 0; r < 4; ++r) c[r] = std::pow(a, r) / factorial(base + r);
    return c;
  };
  for (int n : ns) {
    const int64_t nn = static_cast<int64_t>(n) * n;
    // H = Y4/16! + B3 = a^4/16! X4 + B3
    std::vector<Out> h0;
    for (size_t i = 0; i < reqs.size(); ++i) {
      const int f = reqs[i].f;
      if (h->factors[f].n != n) continue;
      const double a = sts[i].a;
      auto c = coefs(a, 12);
      h0.push_back(Out{sts[i].buf[0], 0.0,
                       {Src{X4[f], std::pow(a, 4) / factorial(16)}, Src{Ident[n], c[0]}, Src{X1[f], c[1]},
                        Src{X2[f], c[2]}, Src{X3[f], c[3]}}});
    }
    ex.combine(nn, h0);
    // three Horner GEMMs: H <- a^4 X4 H + B_m, m = 2, 1, 0
    for (int m = 2; m >= 0; --m) {
      std::vector<Exec::LaunchTerm> tl;
      for (size_t i = 0; i < reqs.size(); ++i) {
        const int f = reqs[i].f;
        if (h->factors[f].n != n) continue;
        const double a = sts[i].a;
        auto c = coefs(a, 4 * m);
        St& s = sts[i];
        tl.push_back({s.buf[s.cur], X4[f], static_cast<int>(tl.size()),
                      {Out{s.buf[s.cur ^ 1], std::pow(a, 4),
                           {Src{Ident[n], c[0]}, Src{X1[f], c[1]}, Src{X2[f], c[2]}, Src{X3[f], c[3]}}}}});
        s.cur ^= 1;
      }
      ex.gemm_batch(n, tl);
    }
    // σ squarings
    for (int k = 0; k < max_sigma; ++k) {
      std::vector<Exec::LaunchTerm> tl;
      for (size_t i = 0; i < reqs.size(); ++i) {
        const int f = reqs[i].f;
        St& s = sts[i];
        if (h->factors[f].n != n || s.sigma <= k) continue;
        tl.push_back({s.buf[s.cur], s.buf[s.cur], static_cast<int>(tl.size()), {Out{s.buf[s.cur ^ 1], 1.0, {}}}});
        s.cur ^= 1;
      }
      if (!tl.empty()) ex.gemm_batch(n, tl);
    }
  }
  for (size_t i = 0; i < reqs.size(); ++i) reqs[i].result = sts[i].buf[sts[i].cur];
}

// Stage A of one apply.  Slab-sharded handles split it over the ranks:
// request i is computed by rank i mod P, which stores the n×n result into slot i of every
// rank's exponential pool (symmetric region, the apply's half) by NVLink peer stores; a
// channel-1 barrier, then every rank reads all results from its own pool.  The request list
// and the slot offsets are identical on every rank (same plans).
void expm_stage(Exec& ex, double tau, std::vector<ExpReq>& reqs) {
  phiks_ctx* h = ex.h;
  const int P = h->world;
  std::vector<size_t> off(reqs.size());
  size_t need = 0;
  for (size_t i = 0; i < reqs.size(); ++i) {
    off[i] = need;
    const size_t n = static_cast<size_t>(h->factors[reqs[i].f].n);
    need += (n * n * sizeof(double) + 255) & ~size_t(255);
  }
  if (!h->sharded() || !h->xpool_off || need > h->xpool_half || reqs.size() < 2) {
    expm_batch(ex, tau, reqs);
    return;
  }
  std::vector<ExpReq> mine;
  std::vector<size_t> mine_idx;
  for (size_t i = h->rank; i < reqs.size(); i += P) {
    mine.push_back(reqs[i]);
    mine_idx.push_back(i);
  }
  if (!mine.empty()) expm_batch(ex, tau, mine);
  if (!ex.ok()) return;
  const size_t pool = h->xpool_off + static_cast<size_t>(ex.half) * h->xpool_half;
  for (size_t c0 = 0; c0 < mine.size(); c0 += kMaxPeerCopy) {
    auto pc = std::make_shared<PeerCopyParams>();
    std::memset(pc.get(), 0, sizeof(PeerCopyParams));
    pc->world = P;
    for (int k = 0; k < P; ++k) pc->base[k] = h->peer[k];
    for (size_t i = c0; i < std::min(mine.size(), c0 + kMaxPeerCopy); ++i) {
      const int64_t n = h->factors[mine[i].f].n;
      pc->src[pc->nitems] = mine[i].result;
      pc->off[pc->nitems] = pool + off[mine_idx[i]];
      pc->count[pc->nitems] = n * n;
      ++pc->nitems;
    }
    ex.emit("peer_copy_expm", [pc](cudaStream_t s) { return launch_peer_copy(*pc, s); });
  }
  ex.barrier(1);
  for (size_t i = 0; i < reqs.size(); ++i) reqs[i].result = reinterpret_cast<double*>(h->sym + pool + off[i]);
}

// ---------------------------------------------------------------------------
// The whole φ-action (stages A-D) on device pointers.
// vin[ℓ] (ℓ = 0..p) device input tensors or nullptr; out_same[ℓ][j] / out_lin[j]
// device output tensors or nullptr (not requested).
// ---------------------------------------------------------------------------
// All blocks' jobs of one apply (one job per diagonal block of K̂, PAPER.md
// §4.4; a single job for an ordinary handle).  Each job follows PAPER.md §3
// with its own plan (s_b, q_b); their exponential requests form one stage A
// and their Tucker operators are merged phase by phase into the same batches
// (quadrature, then squaring level j for every job with s_b ≥ j, then the
// exp-action terms), so the blocks share launches.
void run_jobs(Exec& ex, const std::vector<Job>& jobs) {
  phiks_ctx* h = ex.h;
  const int d = h->d;
  const int64_t N = h->N;
  const int nj = static_cast<int>(jobs.size());
  if (nj == 0) return;
  const int p = jobs[0].p;
  const bool same = jobs[0].mode == PHIKS_MODE_SAME_VECTOR;
  const double tau = jobs[0].tau;

  struct JS {
    const Job* jb;
    int s, q, jmin, n_nodes, gbase;
    std::vector<double> theta, w;
    std::vector<int> facs;  // distinct factor indices of the block
    size_t req0;            // first stage-A request of this job
    std::vector<std::vector<const double*>> nodeE;  // [i][f]
    std::vector<std::vector<double*>> Es;           // [j][f]
    std::vector<std::vector<double*>> state;        // [j][ℓ]
    std::vector<double*> pool[2];
  };
  const int nf = static_cast<int>(h->factors.size());
  std::vector<JS> js(nj);
  std::vector<ExpReq> reqs;
  for (int b = 0; b < nj; ++b) {
    JS& J = js[b];
    const Job& jb = jobs[b];
    J.jb = &jb;
    J.s = jb.s;
    J.q = jb.q;
    J.gbase = 10000 * b;  // epilogue groups of different jobs never merge
    // ---- which level matrices exp(τA/2^j) are needed ----
    bool want_phi0 = false;
    if (same) {
      for (int j = 0; j < jb.n_scales; ++j) want_phi0 |= jb.out_same[0][j] != nullptr;
    } else {
      want_phi0 = jb.vin[0] != nullptr;
    }
    J.jmin = J.s;
    if (p >= 1) J.jmin = std::min(J.jmin, 1);
    if (want_phi0) J.jmin = 0;
    if (p >= 1 && J.s == 0) J.jmin = 0;
    if (p >= 1) plan::gll_rule(J.q, J.theta, J.w);
    J.n_nodes = (p >= 1) ? J.q - 1 : 0;
    for (int mu = 0; mu < d; ++mu) {
      const int f = h->fac_of_block[jb.block][mu];
      if (std::find(J.facs.begin(), J.facs.end(), f) == J.facs.end()) J.facs.push_back(f);
    }
    // ---- Stage A requests: node exponentials (θ_i ≠ 1): c_i = (1 − θ_i)/2^s;
    // node 0 (θ = 0) gives exp(τA/2^s) ----
    J.req0 = reqs.size();
    for (int i = 0; i < J.n_nodes; ++i)
      for (int f : J.facs) reqs.push_back({f, (1.0 - J.theta[i]) / std::ldexp(1.0, J.s)});
    if (p == 0)
      for (int f : J.facs) reqs.push_back({f, 1.0 / std::ldexp(1.0, J.s)});
  }
  expm_stage(ex, tau, reqs);
  if (!ex.ok()) return;
  int max_lev = 0;
  for (JS& J : js) {
    const size_t nfb = J.facs.size();
    J.nodeE.assign(J.n_nodes, std::vector<const double*>(nf, nullptr));
    for (int i = 0; i < J.n_nodes; ++i)
      for (size_t k = 0; k < nfb; ++k) J.nodeE[i][J.facs[k]] = reqs[J.req0 + i * nfb + k].result;
    J.Es.assign(J.s + 1, std::vector<double*>(nf, nullptr));
    for (size_t k = 0; k < nfb; ++k)
      J.Es[J.s][J.facs[k]] = (p >= 1) ? const_cast<double*>(J.nodeE[0][J.facs[k]]) : reqs[J.req0 + k].result;
    max_lev = std::max(max_lev, J.s - J.jmin);
  }
  // level matrices Es[j] = Es[j+1]², j = s_b−1..jmin_b: the k-th squaring of every job in one batch
  for (int k = 0; k < max_lev; ++k) {
    std::map<int, std::vector<Exec::LaunchTerm>> byn;
    for (JS& J : js) {
      const int j = J.s - k;
      if (j <= J.jmin) continue;
      for (int f : J.facs) {
        const int n = h->factors[f].n;
        J.Es[j - 1][f] = ex.ar->alloc_doubles(static_cast<int64_t>(n) * n);
        auto& v = byn[n];
        v.push_back({J.Es[j][f], J.Es[j][f], static_cast<int>(v.size()), {Out{J.Es[j - 1][f], 1.0, {}}}});
      }
    }
    for (auto& kv : byn) ex.gemm_batch(kv.first, kv.second);
  }
  auto mats_for = [&](const JS& J, const std::vector<double*>& perf, const double** mats) {
    for (int mu = 0; mu < d; ++mu) mats[mu] = perf[h->fac_of_block[J.jb->block][mu]];
  };
  auto node_mats = [&](const JS& J, int i, const double** mats) {
    for (int mu = 0; mu < d; ++mu) mats[mu] = J.nodeE[i][h->fac_of_block[J.jb->block][mu]];
  };

  // inputs staged from host memory are needed from here on (stage A overlaps their copy)
  ex.stage_a = false;
  if (ex.on_inputs) ex.on_inputs();

  // ---- Stage D (same vector): exp(τK/2^j)v needs only the level matrices and
  // reads the same v as the quadrature, so with p ≥ 1 it joins the quadrature
  // batch (one launch per mode for both); a host-memory apply copies it out
  // while the squaring runs ----
  std::vector<TuckerItem> d_items;
  std::vector<double*> d_ready;
  if (same) {
    for (JS& J : js) {
      const Job& jb = *J.jb;
      for (int j = 0; j < jb.n_scales; ++j) {
        if (!jb.out_same[0][j]) continue;
        TuckerItem it;
        it.in = jb.vin[0];
        mats_for(J, J.Es[j], it.mats);
        it.group = J.gbase + 1000 + j;
        it.outs.push_back(Out{jb.out_same[0][j], 1.0, {}});
        d_items.push_back(it);
        d_ready.push_back(jb.out_same[0][j]);
      }
    }
    if (p == 0) {
      ex.batch(d_items, false);
      if (!ex.ok()) return;
      if (ex.on_outputs && !d_ready.empty()) ex.on_outputs(d_ready);
      d_items.clear();
      d_ready.clear();
    }
  }

  // ---- state buffers: state[j][ℓ] for the scale j (ℓ = 1..p) ----
  for (JS& J : js) {
    const Job& jb = *J.jb;
    J.state.assign(J.s + 1, std::vector<double*>(p + 1, nullptr));
    for (int j = 0; j <= J.s; ++j)
      for (int ell = 1; ell <= p; ++ell) {
        double* u = (same && j < jb.n_scales) ? jb.out_same[ell][j] : nullptr;
        if (!u) {
          auto& pl = J.pool[j % 2];
          while (static_cast<int>(pl.size()) <= ell) pl.push_back(nullptr);
          if (!pl[ell]) pl[ell] = ex.ar->alloc_doubles(N);
          u = pl[ell];
        }
        J.state[j][ell] = u;
      }
  }

  if (p >= 1) {
    // ---- Stage B: quadrature at scale s_b, every job in one batch ----
    std::vector<TuckerItem> items;
    std::vector<Out> prep;
    for (JS& J : js) {
      const Job& jb = *J.jb;
      const int s = J.s, q = J.q;
      const std::vector<double>& theta = J.theta;
      const std::vector<double>& w = J.w;
      const double wq = w[q - 1];  // θ_q = 1 term: exp(0) = I, no Tucker operator (l.948-952)
      auto& state = J.state;
      if (same) {
        for (int i = 0; i < J.n_nodes; ++i) {
          TuckerItem it;
          it.in = jb.vin[0];
          node_mats(J, i, it.mats);
          it.group = J.gbase;
          for (int ell = 1; ell <= p; ++ell) {
            Out o;
            o.dst = state[s][ell];
            o.beta = w[i] * std::pow(theta[i], ell - 1) / factorial(ell - 1);
            if (i == 0)
              o.srcs.push_back(Src{jb.vin[0], wq / factorial(ell - 1)});
            else
              o.srcs.push_back(Src{o.dst, 1.0});
            it.outs.push_back(o);
          }
          items.push_back(it);
        }
      } else {
        // Ψ_ℓ^{(s)} = Σ_i w_i E_i x_iℓ,  x_iℓ = Σ_{k=1}^ℓ θ_i^{ℓ−k}/(ℓ−k)! v_{p+1−k}/2^{(ℓ−k+1)s}
        auto xcoef = [&](double th, int ell, int k) {
          return std::pow(th, ell - k) / factorial(ell - k) / std::ldexp(1.0, (ell - k + 1) * s);
        };
        std::vector<std::vector<TuckerItem>> per_ell(p + 1);
        std::vector<TuckerItem> jitems;
        // s ≥ 1 (every Ψ_ℓ^{(s)} feeds the squaring): by the linearity of the Tucker operator,
        // E_i x_iℓ = Σ_k c_iℓk E_i v_{p+1−k}, so one operator per node and GIVEN vector feeds every
        // Ψ_ℓ that uses that vector — each v split once, no pre-combined inputs, and with only some
        // v_ℓ given fewer operators than one per (node, ℓ) (reading R9).  s = 0: only Ψ_p is an
        // output, from the pre-combined x_ip (one operator per node).
        if (s >= 1) {
          std::vector<char> started(p + 1, 0);
          auto initial = [&](int ell, Out& o) {  // the θ_q = 1 term w_q x_qℓ
            for (int k = 1; k <= ell; ++k) {
              const double* v = jb.vin[p + 1 - k];
              if (v) o.srcs.push_back(Src{v, wq * xcoef(1.0, ell, k)});
            }
          };
          for (int i = 0; i < J.n_nodes; ++i)
            for (int m = 1; m <= p; ++m) {
              const double* v = jb.vin[m];
              if (!v) continue;
              const int k = p + 1 - m;
              TuckerItem it;
              it.in = v;
              node_mats(J, i, it.mats);
              it.group = J.gbase;
              for (int ell = k; ell <= p; ++ell) {
                const double c = xcoef(theta[i], ell, k);
                if (c == 0.0) continue;
                Out o;
                o.dst = state[s][ell];
                o.beta = w[i] * c;
                if (!started[ell]) {
                  initial(ell, o);
                  started[ell] = 1;
                } else {
                  o.srcs.push_back(Src{o.dst, 1.0});
                }
                it.outs.push_back(o);
              }
              if (!it.outs.empty()) jitems.push_back(it);
            }
          for (int ell = 1; ell <= p; ++ell)
            if (!started[ell]) {  // no node contributed: Ψ_ℓ = w_q x_qℓ
              Out o{state[s][ell], 0.0, {}};
              initial(ell, o);
              prep.push_back(o);
              if (ell == p && s < jb.n_scales && jb.out_lin[s]) {
                o.dst = jb.out_lin[s];
                prep.push_back(o);
              }
            }
        }
        for (int ell = 1; ell <= p && s == 0; ++ell) {
          // s = 0: level 0 is the output level and only Ψ_p^{(0)} is an output
          // (Table 1's lincomb T = (q−2)p + sp + 1, reading R9)
          if (s == 0 && ell != p) continue;
          bool first = true;
          for (int i = 0; i < J.n_nodes; ++i) {
            std::vector<Src> comb;
            for (int k = 1; k <= ell; ++k) {
              const double* v = jb.vin[p + 1 - k];
              const double c = xcoef(theta[i], ell, k);
              if (v && c != 0.0) comb.push_back(Src{v, c});
            }
            if (comb.empty()) continue;
            TuckerItem it;
            node_mats(J, i, it.mats);
            it.group = J.gbase + ell;
            if (comb.size() == 1) {
              it.in = comb[0].ptr;
              it.in_scale = comb[0].coef;
            } else {
              double* x = ex.ar->alloc_doubles(N);
              prep.push_back(Out{x, 0.0, comb});
              it.in = x;
            }
            Out o;
            o.dst = state[s][ell];
            o.beta = w[i];
            if (first) {
              for (int k = 1; k <= ell; ++k) {
                const double* v = jb.vin[p + 1 - k];
                if (v) o.srcs.push_back(Src{v, wq * xcoef(1.0, ell, k)});
              }
            } else {
              o.srcs.push_back(Src{o.dst, 1.0});
            }
            it.outs.push_back(o);
            first = false;
            per_ell[ell].push_back(it);
          }
          if (first) {  // no node contributed: Ψ_ℓ = w_q x_qℓ
            Out o{state[s][ell], 0.0, {}};
            for (int k = 1; k <= ell; ++k) {
              const double* v = jb.vin[p + 1 - k];
              if (v) o.srcs.push_back(Src{v, wq * xcoef(1.0, ell, k)});
            }
            prep.push_back(o);
            if (ell == p && s < jb.n_scales && jb.out_lin[s]) {
              o.dst = jb.out_lin[s];
              prep.push_back(o);
            }
          }
        }
        for (int ell = 1; ell <= p; ++ell)
          for (auto& it : per_ell[ell]) jitems.push_back(it);
        if (s < jb.n_scales && jb.out_lin[s]) {
          // scale s output = Ψ_p^{(s)} (+ exp term later): mirror the Ψ_p accumulation
          for (auto& it : jitems) {
            const size_t no = it.outs.size();
            for (size_t oi = 0; oi < no; ++oi)
              if (it.outs[oi].dst == state[s][p]) {
                Out o = it.outs[oi];
                o.dst = jb.out_lin[s];
                for (auto& sr : o.srcs)
                  if (sr.ptr == state[s][p]) sr.ptr = jb.out_lin[s];
                it.outs.push_back(o);
              }
          }
        }
        for (auto& it : jitems) items.push_back(it);
      }
    }
    // ---- Stage C: squaring, level j for every job with s_b ≥ j ----
    int max_s = 0;
    for (const JS& J : js) max_s = std::max(max_s, J.s);
    auto squaring_items = [&](int j) {
      std::vector<TuckerItem> sq;
      for (JS& J : js) {
        if (J.s < j) continue;
        const Job& jb = *J.jb;
        auto& state = J.state;
        for (int ell = p; ell >= 1; --ell) {
          // level j−1 = 0 is output only: Ψ_p alone (linear combination), the
          // requested φ_ℓ (same vector) — PAPER.md l.953-956, reading R9
          if (j == 1 && (same ? !(jb.n_scales > 0 && jb.out_same[ell][0]) : ell != p)) continue;
          TuckerItem it;
          it.in = state[j][ell];
          mats_for(J, J.Es[j], it.mats);
          it.group = J.gbase + ell;
          Out o;
          o.dst = state[j - 1][ell];
          if (same) {
            const double sc = std::ldexp(1.0, -ell);
            o.beta = sc;
            for (int k = 1; k <= ell; ++k) o.srcs.push_back(Src{state[j][k], sc / factorial(ell - k)});
          } else {
            o.beta = 1.0;
            for (int k = 1; k <= ell; ++k)
              o.srcs.push_back(Src{state[j][k], 1.0 / (factorial(ell - k) * std::ldexp(1.0, (ell - k) * j))});
          }
          it.outs.push_back(o);
          if (!same && ell == p && (j - 1) < jb.n_scales && jb.out_lin[j - 1]) {
            Out o2 = o;
            o2.dst = jb.out_lin[j - 1];
            it.outs.push_back(o2);
          }
          sq.push_back(it);
        }
      }
      return sq;
    };
    // the inputs of the next squaring level come out of this batch's combination, which then
    // also writes their mode-1 digits (Exec::pre_want)
    auto want_next = [&](int j, bool producer_split) {
      if (j < 1 || !producer_split) return;
      for (const TuckerItem& it : squaring_items(j)) ex.pre_want.push_back(it.in);
    };

    ex.combine(N, prep);
    for (auto& it : d_items) items.push_back(it);
    want_next(max_s, ex.split >= 1);
    ex.batch(items, ex.split >= 1);
    if (!ex.ok()) return;
    if (ex.on_outputs && !d_ready.empty()) ex.on_outputs(d_ready);
    if (!ex.ok()) return;

    for (int j = max_s; j >= 1; --j) {
      std::vector<TuckerItem> sq = squaring_items(j);
      want_next(j - 1, ex.split >= 2);
      ex.batch(sq, ex.split >= 2);
      if (!ex.ok()) return;
    }
  }

  // ---- Stage D (linear combination): exp(τK/2^j)v_0 added to the result ----
  std::vector<TuckerItem> ex_items;
  if (!same) {
    for (JS& J : js) {
      const Job& jb = *J.jb;
      for (int j = 0; j < jb.n_scales; ++j) {
        if (!jb.out_lin[j]) continue;
        if (jb.vin[0]) {
          TuckerItem it;
          it.in = jb.vin[0];
          mats_for(J, J.Es[j], it.mats);
          it.group = J.gbase + j;
          Out o{jb.out_lin[j], 1.0, {}};
          if (p >= 1) o.srcs.push_back(Src{jb.out_lin[j], 1.0});
          it.outs.push_back(o);
          ex_items.push_back(it);
        }
      }
    }
  }
  ex.batch(ex_items, false);
}

}  // namespace host
}  // namespace phiks
