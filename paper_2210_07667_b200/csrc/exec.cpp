// Out-of-line members of Exec (host.h): the launch builders of the Tucker batches
// (per-mode, chained int8, split with a streaming combination, slab-sharded).
#include "host.h"

namespace phiks {
namespace host {

void Exec::oz_emit(const std::shared_ptr<OzakiParams>& pp, bool split_x, const std::function<void()>& mid) {
  const OzakiParams& p = *pp;
  ++i8_launches;
  for (int phase = 0; phase < 2; ++phase) {
    if (phase == 1 && mid) mid();
    const bool prof = !measure && h->profiling && !rec;
    if (prof) {
      if (h->ev_used == static_cast<int>(h->ev.size())) {
        cudaEvent_t a, b;
        check(cudaEventCreate(&a), "cudaEventCreate");
        check(cudaEventCreate(&b), "cudaEventCreate");
        h->ev.emplace_back(a, b);
        h->ev_flops.push_back(0.0);
        h->ev_expm.push_back(0);
      }
      h->ev_flops[h->ev_used] =
          phase == 0 ? 0.0 : 2.0 * static_cast<double>(p.L * p.R) * p.n * static_cast<double>(p.n) * p.nterms;
      h->ev_expm[h->ev_used] = phase == 0 ? 3 : 2;
      check(cudaEventRecord(h->ev[h->ev_used].first, st), "cudaEventRecord");
    }
    if (phase == 0) {
      emit("digits_i8", [pp, split_x](cudaStream_t s2) { return launch_ozaki_mode(*pp, s2, split_x, true, false); });
      if (split_x) ++launches;  // split_x + split_e (+ chain)
      if (p.n_next > 0 && !p.shard_stage0) ++launches;
    } else {
      emit("mode_product_i8", [pp](cudaStream_t s2) { return launch_ozaki_mode(*pp, s2, false, false, true); });
    }
    if (prof) check(cudaEventRecord(h->ev[h->ev_used++].second, st), "cudaEventRecord");
  }
}

bool Exec::ozaki_chain_route(const std::vector<TuckerItem>& items, size_t c0, size_t c1, int mlast) const {
  if (in_expm || h->cplx || h->gemm_path == PHIKS_GEMM_DMMA || h->opt_chain == 0) return false;
  // guard (R15): the exponent bound ‖e_j‖₁·max|x| is attained when every exponential is
  // entrywise nonnegative; rows with cancellation would lose bits against it
  if (h->opt_chain == 1 && !h->chain_safe()) return false;
  const int d = h->d;
  if (mlast < 0) mlast = d - 1;
  if (d < 2 || mlast < 1) return false;
  const int64_t N = h->N;
  int64_t L = 1;
  for (int mu = 0; mu <= mlast; ++mu) {
    const int n = h->n[mu];
    const int64_t R = N / (L * n);
    if (!ozaki_supported(L, n, R, kOzDigits) || n % 16 != 0) return false;
    if (mu > 0 && (L % 128 != 0 || L >= (int64_t(1) << 31) || R >= (int64_t(1) << 31))) return false;
    if (h->gemm_path == PHIKS_GEMM_AUTO && (n < 128 || N < (int64_t(1) << 20))) return false;
    L *= n;
  }
  std::set<int> groups;  // last mode: one plain output per operator, distinct groups
  for (size_t b = c0; b < c1; ++b) {
    const TuckerItem& it = items[b];
    if (it.outs.size() != 1 || !it.outs[0].srcs.empty()) return false;
    if (!groups.insert(it.group).second) return false;
  }
  return true;
}

void Exec::tucker_chain_i8(const std::vector<TuckerItem>& items, size_t c0, size_t c1, int mlast,
                     const Remap* rm, const Remap* rm1) {
  const int d = h->d, S = kOzDigits;
  if (mlast < 0) mlast = d - 1;
  const int64_t N = h->N;
  const int nt = static_cast<int>(c1 - c0);
  const int st0 = rm1 ? d - 2 : -1;  // the stage-0 mode of the sharded digit path
  int nmin = h->n[0];
  for (int mu = 1; mu < d; ++mu) nmin = std::min(nmin, h->n[mu]);
  if (oz_chain_cap < static_cast<size_t>(nt)) {
    const size_t cap = chain_cap();
    for (int k = 0; k < 2; ++k) {
      oz_dig[k] = reinterpret_cast<int8_t*>(ar->alloc_doubles(static_cast<int64_t>((cap * S * N + 7) / 8)));
      oz_ex[k] = ar->alloc_doubles(static_cast<int64_t>(cap) * (N / nmin));
    }
    oz_mx = ar->alloc_doubles(static_cast<int64_t>(cap) * (N / (static_cast<int64_t>(nmin) * nmin)));
    oz_chain_cap = cap;
  }
  int64_t L = 1;
  std::vector<const double*> prev_e;  // the previous mode's matrices, split in oz_ws (bind: E region first)
  int prev_n = -1;
  double* prev_ws = nullptr;
  for (int mu = 0; mu <= mlast && ok(); ++mu) {
    int n = h->n[mu];
    int64_t R = N / (L * n);
    if (rm1 && mu == d - 1) {  // stage 1: layout S_{d-1}, dims (L0·cb, n_d, 1)
      n = h->gn[d - 1];
      L = N / n;
      R = 1;
    }
    auto pp = std::make_shared<OzakiParams>();
    OzakiParams& p = *pp;
    std::memset(&p, 0, sizeof(p));
    p.L = L;
    p.R = R;
    p.n = n;
    p.S = S;
    p.kskip = h->opt_kskip;
    p.kcount = h->profiling ? h->d_kcount : nullptr;
    p.n_next = mu < mlast ? (mu == st0 ? h->gn[d - 1] : h->n[mu + 1]) : 0;
    if (mu == mlast && rm) p.remap = rm1 ? *rm1 : *rm;
    if (mu == st0) {
      p.remap = *rm;
      p.shard_stage0 = 1;
    }
    const int64_t Cn = mu < mlast ? N / h->n[mu + 1] : 0;
    for (int b = 0; b < nt; ++b) {
      const TuckerItem& it = items[c0 + b];
      int xs = b, es = -1;
      if (mu == 0) {
        xs = -1;
        for (int k = 0; k < p.nx; ++k)
          if (p.x[k] == it.in) xs = k;
        if (xs < 0) {
          xs = p.nx;
          p.x[p.nx++] = it.in;
        }
      }
      for (int k = 0; k < p.ne; ++k)
        if (p.e[k] == it.mats[mu]) es = k;
      if (es < 0) {
        es = p.ne;
        p.e[p.ne++] = it.mats[mu];
      }
      OzakiTerm t{xs, es, nullptr, 1.0, nullptr, nullptr, nullptr};
      if (mu == st0) {  // the owners' T pools as digit pools: term b's plane s at (b·S + s)·N bytes
        t.dig = reinterpret_cast<int8_t*>(kCtrlBytes + static_cast<size_t>(b) * S * N);
        t.nmx = oz_mx + static_cast<int64_t>(b) * L;
      } else if (mu < mlast) {
        t.dig = oz_dig[mu % 2] + static_cast<int64_t>(b) * S * N;
        t.nex = oz_ex[mu % 2] + static_cast<int64_t>(b) * Cn;
        t.nmx = oz_mx + static_cast<int64_t>(b) * (N / (static_cast<int64_t>(n) * h->n[mu + 1]));
      } else if (rm1) {
        t.out = reinterpret_cast<double*>(kCtrlBytes + static_cast<size_t>(kShardChunk + c0 + b) * h->sym_slot);
      } else if (rm) {
        t.out = reinterpret_cast<double*>(kCtrlBytes + static_cast<size_t>(c0 + b) * h->sym_slot);
      } else {
        t.out = it.outs[0].dst;
        t.beta = it.outs[0].beta * it.in_scale;
      }
      p.terms[p.nterms++] = t;
    }
    // mode 1 of a batch whose inputs the previous batch's combination already split (pre_ready;
    // mode 1 is local on slab-sharded handles too)
    bool pre = mu == 0 && !pre_ready.empty();
    for (int k = 0; pre && k < p.nx; ++k) pre = pre_ready.count(p.x[k]) != 0;
    const int nx_split = mu == 0 && !pre ? p.nx : 0;
    oz_ws_reserve(ozaki_workspace_bytes(L, n, R, S, nx_split, p.ne));
    const int nx_keep = p.nx;
    p.nx = nx_split;
    ozaki_bind_workspace(p, oz_ws);
    // the same factor in every mode (configs[2]-[4]): each distinct matrix is split once per batch
    p.e_ready = (prev_ws == oz_ws && prev_n == n && prev_e.size() == static_cast<size_t>(p.ne) &&
                 std::equal(prev_e.begin(), prev_e.end(), p.e)) ? 1 : 0;
    prev_e.assign(p.e, p.e + p.ne);
    prev_n = n;
    prev_ws = oz_ws;
    if (mu > 0) {  // A: the previous product's digit planes and exponent bounds
      p.nx = nt;
      p.xs = (rm1 && mu == d - 1) ? reinterpret_cast<int8_t*>(h->sym + kCtrlBytes) : oz_dig[(mu - 1) % 2];
      p.xsc = oz_ex[(mu - 1) % 2];
      p.a_mn = 1;
    } else if (pre) {  // A: the pre-split slots (same Kp: n rounded up to 128)
      for (int b = 0; b < p.nterms; ++b) p.terms[b].xslot = pre_ready.at(p.x[p.terms[b].xslot]);
      p.nx = pre_slots;
      p.xs = pre_xs;
      p.xsc = pre_xsc;
      pre_hits += nx_keep;
    } else {
      p.nx = nx_keep;
    }
    if (mu == st0) {
      // next-mode exponents across the ranks: partial maxima to every peer, barrier, tables
      OzShardExch ex{};
      ex.rank = h->rank;
      ex.world = h->world;
      ex.nterms = nt;
      ex.L0 = L;
      ex.R = R;
      ex.kstart = static_cast<int>(blk_start(h->gn[d - 2], h->world, h->rank));
      ex.cb = static_cast<int>(blk_cnt(h->gn[d - 2], h->world, h->rank));
      ex.exch = reinterpret_cast<const double*>(h->sym + h->exch_off);
      for (int k = 0; k < h->world; ++k) ex.dst[k] = reinterpret_cast<double*>(h->peer[k] + h->exch_off);
      for (int b = 0; b < nt; ++b) {
        ex.xsc[b] = p.xsc + static_cast<int64_t>(p.terms[b].xslot) * (L * R);
        ex.eb[b] = p.eb + static_cast<int64_t>(p.terms[b].eslot) * n;
        ex.nmx[b] = p.terms[b].nmx;
        ex.xsc1[b] = oz_ex[mu % 2] + static_cast<int64_t>(b) * (L * ex.cb);
      }
      auto exs = std::make_shared<OzShardExch>(ex);
      oz_emit(pp, mu == 0, [this, exs] {
        emit("oz_shard_pmax", [exs](cudaStream_t s2) { return launch_oz_shard_pmax(*exs, s2); });
        barrier();
        emit("oz_shard_tables", [exs](cudaStream_t s2) { return launch_oz_shard_tables(*exs, s2); });
      });
      barrier();  // every rank's digit planes are in place before stage 1 reads them
    } else {
      oz_emit(pp, mu == 0 && !pre);
    }
    L *= n;
  }
  i8_chained += nt;
  if (mlast < d - 1 || rm1) return;  // the sharded caller completes and counts the operators
  int64_t nsum = 0;
  for (int mu = 0; mu < d; ++mu) nsum += h->n[mu];
  tucker_ops += nt;
  mu_flops += static_cast<double>(nt) * 2.0 * static_cast<double>(N) * static_cast<double>(nsum);
}

void Exec::mode_launch(int64_t L, int n, int64_t R, const std::vector<LaunchTerm>& terms, const Remap* rm) {
  if (!ok() || terms.empty()) return;
  if (ozaki_route(L, n, R, terms, rm)) {
    ozaki_launch(L, n, R, terms, rm);
    return;
  }
  // chunk so every launch fits ModeParams; a group's terms stay in order
  size_t i = 0;
  while (i < terms.size() && ok()) {
    ModeParams* pp = new ModeParams();
    ModeParams& p = *pp;
    p.L = L;
    p.R = R;
    p.n = n;
    p.ngroups = 0;
    if (rm) p.remap = *rm;
    int nt = 0, no = 0, ns = 0;
    std::map<int, int> gslot;  // group key -> slot in this launch
    std::vector<std::vector<int>> gterms;
    size_t j = i;
    for (; j < terms.size(); ++j) {
      const LaunchTerm& t = terms[j];
      int need_s = 0;
      for (const Out& o : t.outs) need_s += static_cast<int>(o.srcs.size());
      const bool new_group = gslot.find(t.group) == gslot.end();
      if (nt + 1 > kMaxTerms || no + static_cast<int>(t.outs.size()) > kMaxOuts || ns + need_s > kMaxSrcs ||
          (new_group && static_cast<int>(gterms.size()) + 1 > kMaxGroups))
        break;
      if (new_group) {
        gslot[t.group] = static_cast<int>(gterms.size());
        gterms.emplace_back();
      }
      gterms[gslot[t.group]].push_back(static_cast<int>(j));
      ++nt;
      no += static_cast<int>(t.outs.size());
      ns += need_s;
    }
    if (j == i) {
      status = PHIKS_ERR_LIMIT;
      g_err = "term exceeds launch descriptor limits";
      delete pp;
      return;
    }
    // lay out groups contiguously
    int tt = 0, oo = 0, ss = 0;
    for (size_t g = 0; g < gterms.size(); ++g) {
      p.groups[g].t0 = tt;
      for (int ti : gterms[g]) {
        const LaunchTerm& t = terms[ti];
        TermSpec& ts = p.terms[tt++];
        ts.in = t.in;
        ts.M = t.M;
        ts.cswap = t.cswap;
        ts.out0 = oo;
        ts.nout = static_cast<int>(t.outs.size());
        for (const Out& o : t.outs) {
          OutSpec& os = p.outs[oo++];
          os.dst = o.dst;
          os.beta = o.beta;
          os.src0 = ss;
          os.nsrc = static_cast<int>(o.srcs.size());
          for (const Src& s : o.srcs) p.srcs[ss++] = SrcRef{s.ptr, s.coef};
        }
      }
      p.groups[g].t1 = tt;
    }
    p.ngroups = static_cast<int>(gterms.size());
    if (rec) {
      ++launches;
      if (!measure) {
        std::shared_ptr<ModeParams> sp(pp);
        rec->push_back(Op{false, [sp](cudaStream_t s) { return launch_mode_product(*sp, s); }, "mode_product", stage_a});
      } else {
        delete pp;
      }
      i = j;
      continue;
    }
    if (!measure && h->profiling) {
      if (h->ev_used == static_cast<int>(h->ev.size())) {
        cudaEvent_t a, b;
        check(cudaEventCreate(&a), "cudaEventCreate");
        check(cudaEventCreate(&b), "cudaEventCreate");
        h->ev.emplace_back(a, b);
        h->ev_flops.push_back(0.0);
        h->ev_expm.push_back(0);
      }
      h->ev_flops[h->ev_used] = 2.0 * static_cast<double>(L * R) * n * static_cast<double>(n) * nt;
      h->ev_expm[h->ev_used] = in_expm ? 1 : 0;
      check(cudaEventRecord(h->ev[h->ev_used].first, st), "cudaEventRecord");
    }
    if (!measure) check(launch_mode_product(p, st), "mode_product");
    if (!measure && h->profiling) check(cudaEventRecord(h->ev[h->ev_used++].second, st), "cudaEventRecord");
    ++launches;
    delete pp;
    i = j;
  }
}

void Exec::combine(int64_t count, const std::vector<Out>& outs) {
  if (!ok() || outs.empty()) return;
  size_t i = 0;
  while (i < outs.size() && ok()) {
    CombineParams* pp = new CombineParams();
    CombineParams& p = *pp;
    p.count = count;
    p.nout = 0;
    int ns = 0;
    size_t j = i;
    for (; j < outs.size(); ++j) {
      const int need = static_cast<int>(outs[j].srcs.size());
      if (p.nout + 1 > kMaxCombOuts || ns + need > kMaxCombSrcs) break;
      OutSpec& os = p.outs[p.nout++];
      os.dst = outs[j].dst;
      os.beta = 0.0;
      os.src0 = ns;
      os.nsrc = need;
      for (const Src& s : outs[j].srcs) p.srcs[ns++] = SrcRef{s.ptr, s.coef};
    }
    std::shared_ptr<CombineParams> sp(pp);
    emit("combine", [sp](cudaStream_t s) { return launch_combine(*sp, s); });
    i = j;
  }
}

bool Exec::pre_ok() const {
  // the conditions of ozaki_chain_route on mode 1, for the pre-split's fibre layout
  if (!h->opt_presplit || h->cplx || h->gemm_path == PHIKS_GEMM_DMMA || h->opt_chain == 0 || h->d < 2) return false;
  if (h->opt_chain == 1 && !h->chain_safe()) return false;
  const int n = h->n[0];
  // mode 2's A operand is MN-major over L = n_1 fibres: the chain needs n_1 % 128 == 0
  if (n % 128 != 0 || n > kOzMaxN || !ozaki_supported(1, n, h->N / n, kOzDigits)) return false;
  if (h->gemm_path == PHIKS_GEMM_AUTO && (n < 128 || h->N < (int64_t(1) << 20))) return false;
  return true;
}

void Exec::mcombine(int64_t count, const std::vector<const double*>& srcs, const std::vector<double*>& dsts,
              const std::vector<std::vector<double>>& coef, const std::vector<int>* dslot) {
  if (!ok() || dsts.empty()) return;
  bool any = false;
  for (size_t o = 0; dslot && o < dsts.size(); ++o) any |= (*dslot)[o] >= 0;
  if (any && static_cast<int>(srcs.size()) <= kMcMaxSrc && count == h->N) {
    // the combination fused with the next batch's mode-1 split (up to 8 outputs per launch for
    // n_1 ≤ 256, 4 above)
    const int n = h->n[0];
    const int64_t C = count / n;
    const int Kp = (n + 127) / 128 * 128;
    const size_t mo = static_cast<size_t>(oz_multi_combine_split_max_out(n));
    for (size_t o0 = 0; o0 < dsts.size(); o0 += mo) {
      MultiCombineParams* pp = new MultiCombineParams();
      std::memset(pp, 0, sizeof(MultiCombineParams));
      pp->count = count;
      pp->fn = n;
      pp->Kp = Kp;
      pp->nsrc = static_cast<int>(srcs.size());
      for (size_t k = 0; k < srcs.size(); ++k) pp->src[k] = srcs[k];
      pp->nout = static_cast<int>(std::min(dsts.size() - o0, mo));
      for (int o = 0; o < pp->nout; ++o) {
        pp->dst[o] = dsts[o0 + o];
        for (size_t k = 0; k < srcs.size(); ++k) pp->coef[o][k] = coef[o0 + o][k];
        const int sl = (*dslot)[o0 + o];
        if (sl >= 0) {
          pp->dig[o] = pre_xs + static_cast<int64_t>(sl) * kOzDigits * C * Kp;
          pp->dsc[o] = pre_xsc + static_cast<int64_t>(sl) * C;
          pre_next[dsts[o0 + o]] = sl;
        }
      }
      std::shared_ptr<MultiCombineParams> sp(pp);
      emit("multi_combine_split", [sp](cudaStream_t s) { return launch_multi_combine_split(*sp, s); });
    }
    return;
  }
  if (static_cast<int>(srcs.size()) <= kMcMaxSrc) {
    for (size_t o0 = 0; o0 < dsts.size(); o0 += kMcMaxOut) {
      MultiCombineParams* pp = new MultiCombineParams();
      std::memset(pp, 0, sizeof(MultiCombineParams));
      pp->count = count;
      pp->nsrc = static_cast<int>(srcs.size());
      for (size_t k = 0; k < srcs.size(); ++k) pp->src[k] = srcs[k];
      pp->nout = static_cast<int>(std::min(dsts.size() - o0, static_cast<size_t>(kMcMaxOut)));
      for (int o = 0; o < pp->nout; ++o) {
        pp->dst[o] = dsts[o0 + o];
        for (size_t k = 0; k < srcs.size(); ++k) pp->coef[o][k] = coef[o0 + o][k];
      }
      std::shared_ptr<MultiCombineParams> sp(pp);
      emit("multi_combine", [sp](cudaStream_t s) { return launch_multi_combine(*sp, s); });
    }
    return;
  }
  // many sources: per output, chunks of 63 sources accumulating into the output
  for (size_t o = 0; o < dsts.size(); ++o) {
    std::vector<Out> one;
    for (size_t k0 = 0; k0 < srcs.size(); k0 += 63) {
      Out ou{dsts[o], 0.0, {}};
      if (k0 > 0) ou.srcs.push_back(Src{dsts[o], 1.0});
      for (size_t k = k0; k < std::min(srcs.size(), k0 + 63); ++k)
        if (coef[o][k] != 0.0) ou.srcs.push_back(Src{srcs[k], coef[o][k]});
      combine(count, {ou});
    }
  }
}

void Exec::tucker_batch_split(const std::vector<TuckerItem>& items) {
  if (!ok() || items.empty()) return;
  const int64_t N = h->N;
  const bool shard = h->sharded();
  const size_t chunk = shard ? static_cast<size_t>(kShardChunk) : items.size();
  if (!shard)
    while (y_pool.size() < items.size()) y_pool.push_back(ar->alloc_doubles(N));
  // symbolic keys of the Y_b: the real buffers (local) or tags (sharded, pooled per chunk)
  auto ykey = [&](size_t b) -> const double* {
    return shard ? reinterpret_cast<const double*>(static_cast<uintptr_t>(16 + 16 * b)) : y_pool[b];
  };
  auto yitem = [&](const double* key) -> int64_t {  // item index of a Y key, -1 for externals
    if (shard) {
      const uintptr_t v = reinterpret_cast<uintptr_t>(key);
      return (v >= 16 && v < 16 + 16 * items.size() && v % 16 == 0) ? static_cast<int64_t>(v / 16 - 1) : -1;
    }
    for (size_t b = 0; b < items.size(); ++b)
      if (y_pool[b] == key) return static_cast<int64_t>(b);
    return -1;
  };
  typedef std::vector<std::pair<const double*, double>> Lin;
  std::map<const double*, Lin> val;
  std::vector<double*> order;
  auto add = [](Lin& acc, const double* ptr, double c) {
    for (auto& t : acc)
      if (t.first == ptr) {
        t.second += c;
        return;
      }
    acc.emplace_back(ptr, c);
  };
  // items with one output, no sources, whose destination nothing else in the
  // batch reads or writes, write it directly (no Y buffer, no combination)
  std::vector<char> direct(items.size(), 0);
  if (!shard) {
    std::map<const double*, int> refs;
    for (const TuckerItem& it : items)
      for (const Out& o : it.outs) {
        ++refs[o.dst];
        for (const Src& sr : o.srcs) ++refs[sr.ptr];
      }
    for (size_t b = 0; b < items.size(); ++b)
      direct[b] = items[b].outs.size() == 1 && items[b].outs[0].srcs.empty() && refs[items[b].outs[0].dst] == 1;
  }
  for (size_t b = 0; b < items.size(); ++b) {
    if (direct[b]) continue;
    for (const Out& o : items[b].outs) {
      Lin lin;
      add(lin, ykey(b), o.beta * items[b].in_scale);
      for (const Src& sr : o.srcs) {
        auto it = val.find(sr.ptr);
        if (it != val.end())
          for (auto& t : it->second) add(lin, t.first, sr.coef * t.second);
        else
          add(lin, sr.ptr, sr.coef);
      }
      if (!val.count(o.dst)) order.push_back(o.dst);
      val[o.dst] = lin;
    }
  }
  for (size_t c0 = 0; c0 < items.size() && ok(); c0 += chunk) {
    const size_t c1 = std::min(items.size(), c0 + chunk);
    std::vector<TuckerItem> raw(items.begin() + c0, items.begin() + c1);
    for (size_t b = 0; b < raw.size(); ++b) {
      const double beta = direct[c0 + b] ? raw[b].outs[0].beta * raw[b].in_scale : 1.0;
      double* dst = direct[c0 + b] ? raw[b].outs[0].dst : (shard ? nullptr : y_pool[c0 + b]);
      raw[b].in_scale = 1.0;
      raw[b].group = static_cast<int>(b);
      raw[b].outs.assign(1, Out{dst, beta, {}});
    }
    if (shard)
      tucker_raw_sharded(raw);
    else
      tucker_batch(raw);
    // the combination restricted to this chunk's Y_b (+ externals in the first chunk)
    auto real = [&](const double* key) -> const double* {
      const int64_t b = yitem(key);
      if (b < 0) return key;
      return shard ? symY(static_cast<int>(b - static_cast<int64_t>(c0))) : y_pool[b];
    };
    std::vector<const double*> srcs;
    std::vector<double*> dsts;
    std::vector<std::vector<std::pair<const double*, double>>> rows;
    for (double* dptr : order) {
      std::vector<std::pair<const double*, double>> row;
      for (auto& t : val[dptr]) {
        const int64_t b = yitem(t.first);
        const bool in_chunk = b >= static_cast<int64_t>(c0) && b < static_cast<int64_t>(c1);
        if (in_chunk || (b < 0 && c0 == 0)) row.emplace_back(real(t.first), t.second);
      }
      if (c0 > 0) {
        if (row.empty()) continue;
        row.emplace_back(dptr, 1.0);
      }
      dsts.push_back(dptr);
      rows.push_back(row);
    }
    // independent groups of outputs (no shared source or destination, e.g. the
    // blocks of a block-diagonal handle) stream separately: each reads only its
    // own sources
    std::vector<int> comp(dsts.size());
    for (size_t o = 0; o < dsts.size(); ++o) comp[o] = static_cast<int>(o);
    std::function<int(int)> root = [&](int x) { return comp[x] == x ? x : comp[x] = root(comp[x]); };
    std::map<const double*, int> owner;  // pointer -> an output touching it
    for (size_t o = 0; o < dsts.size(); ++o) {
      auto touch = [&](const double* ptr) {
        auto it = owner.find(ptr);
        if (it == owner.end())
          owner[ptr] = static_cast<int>(o);
        else
          comp[root(static_cast<int>(o))] = root(it->second);
      };
      touch(dsts[o]);
      for (auto& t : rows[o]) touch(t.first);
    }
    // outputs the next batch splits (pre_want): their digit planes come out of the combination
    // (sharded: of the chunk that completes the outputs)
    std::vector<int> want_slot(dsts.size(), -1);
    if (c1 == items.size() && !pre_want.empty() && pre_ok()) {
      const int ns = static_cast<int>(pre_want.size());
      if (pre_slots < ns) {
        const int n = h->n[0];
        const int64_t C = N / n, Kp = (n + 127) / 128 * 128;
        pre_xs = reinterpret_cast<int8_t*>(ar->alloc_doubles((static_cast<int64_t>(ns) * kOzDigits * C * Kp + 7) / 8));
        pre_xsc = ar->alloc_doubles(static_cast<int64_t>(ns) * C);
        pre_slots = ns;
      }
      for (size_t o = 0; o < dsts.size(); ++o)
        for (int k = 0; k < ns; ++k)
          if (pre_want[k] == dsts[o]) want_slot[o] = k;
    }
    std::vector<int> done(dsts.size(), 0);
    for (size_t o0 = 0; o0 < dsts.size(); ++o0) {
      const int r0 = root(static_cast<int>(o0));
      if (done[r0]) continue;
      done[r0] = 1;
      std::vector<size_t> members;
      for (size_t o = 0; o < dsts.size(); ++o)
        if (root(static_cast<int>(o)) == r0) members.push_back(o);
      for (size_t o : members)
        for (auto& t : rows[o])
          if (std::find(srcs.begin(), srcs.end(), t.first) == srcs.end()) srcs.push_back(t.first);
      std::vector<double*> cd;
      std::vector<int> cslot;
      std::vector<std::vector<double>> coef(members.size(), std::vector<double>(srcs.size(), 0.0));
      for (size_t m = 0; m < members.size(); ++m) {
        cd.push_back(dsts[members[m]]);
        cslot.push_back(want_slot[members[m]]);
        for (auto& t : rows[members[m]])
          coef[m][std::find(srcs.begin(), srcs.end(), t.first) - srcs.begin()] += t.second;
      }
      mcombine(N, srcs, cd, coef, &cslot);
      srcs.clear();
    }
  }
}

void Exec::tucker_raw_sharded_complex(const std::vector<TuckerItem>& items) {
  const int d = h->d, P = h->world, rk = h->rank;
  const size_t nb = items.size();
  const int64_t slotd = static_cast<int64_t>(h->sym_slot / sizeof(double));
  auto& scr = scr_pool;
  while (scr[0].size() < nb) scr[0].push_back(ar->alloc_doubles(slotd));
  while (scr[1].size() < nb) scr[1].push_back(ar->alloc_doubles(slotd));
  int gv[PHIKS_MAX_D + 1];
  gv[0] = 2;
  for (int mu = 0; mu < d; ++mu) gv[mu + 1] = h->gn[mu];
  // one complex μ-mode product on the local layout whose dims are dims[0..d-1]
  // with rm set (a transposition stage, μ ≥ 2): one int8 product with K = 2n (§4f) whose
  // epilogue stores straight into the owners' regions at byte offsets off0 + b·sym_slot;
  // returns false when that route does not apply (the caller then copies)
  auto cproduct_remote = [&](int mu, const int* dims, std::vector<const double*> in,
                             std::vector<const double*> mats, const Remap& rm, size_t off0) -> bool {
    if (mu == 0) return false;
    int64_t Lc = 1, Nc = 1;
    for (int k = 0; k < d; ++k) Nc *= dims[k];
    for (int k = 0; k < mu; ++k) Lc *= dims[k];
    const int n = dims[mu];
    const int64_t R = Nc / (Lc * n);
    std::vector<LaunchTerm> probe(1);
    probe[0].kcat = 1;
    probe[0].outs.push_back(Out{nullptr, 1.0, {}});
    if (!ozaki_route(2 * Lc, n, R, probe, &rm)) return false;
    std::vector<LaunchTerm> terms;
    for (size_t b = 0; b < nb; ++b) {
      LaunchTerm t;
      t.in = in[b];
      t.group = static_cast<int>(b);
      t.M = complex_parts(mats[b], n).first;
      t.kcat = 1;
      t.outs.push_back(Out{reinterpret_cast<double*>(off0 + b * h->sym_slot), 1.0, {}});
      terms.push_back(std::move(t));
    }
    mode_launch(2 * Lc, n, R, terms, &rm);
    return true;
  };
  auto cproduct = [&](int mu, const int* dims, std::vector<const double*> in, std::vector<double*> out,
                      std::vector<const double*> mats) {
    int64_t Lc = 1, Nc = 1;
    for (int k = 0; k < d; ++k) Nc *= dims[k];
    for (int k = 0; k < mu; ++k) Lc *= dims[k];
    const int n = dims[mu];
    const int64_t R = Nc / (Lc * n);
    std::vector<LaunchTerm> terms;
    for (size_t b = 0; b < nb; ++b) {
      LaunchTerm t;
      t.in = in[b];
      t.group = static_cast<int>(b);
      t.outs.push_back(Out{out[b], 1.0, {}});
      if (mu == 0) {
        t.M = mats[b];
        terms.push_back(std::move(t));
      } else {
        const auto parts = complex_parts(mats[b], n);
        LaunchTerm ti = t;
        t.M = parts.first;
        ti.M = parts.second;
        ti.cswap = 1;
        for (Out& o : ti.outs) o.srcs.assign(1, Src{o.dst, 1.0});
        terms.push_back(std::move(t));
        terms.push_back(std::move(ti));
      }
    }
    if (mu == 0)
      mode_launch(1, 2 * n, R, terms);
    else
      mode_launch(2 * Lc, n, R, terms);
  };
  auto remap_of_stage = [&](const ShardStage& s) {
    Remap r{};
    r.world = P;
    r.cq = static_cast<int>(s.n / P);
    r.crem = static_cast<int>(s.n % P);
    r.uniform = s.uniform ? 1 : 0;
    r.colstride = s.colstride;
    for (int k = 0; k < P; ++k) {
      r.kstart[k] = static_cast<int>(s.kstart[k]);
      r.kstride[k] = s.kstride[k];
      r.kroff[k] = s.kroff[k];
      r.base[k] = h->peer[k];
    }
    return r;
  };
  auto remap_copy = [&](const ShardStage& s, const double* src, size_t dst_off) {
    const Remap r = remap_of_stage(s);
    const int64_t L = s.L, R = s.R;
    const int n = static_cast<int>(s.n);
    emit("remap_copy", [src, L, n, R, dst_off, r](cudaStream_t st2) {
      return launch_remap_copy(src, L, n, R, dst_off, r, st2);
    });
  };
  // local dims of layout S_d
  int dimsS[PHIKS_MAX_D];
  for (int k = 0; k < d; ++k) dimsS[k] = h->n[k];
  std::vector<const double*> cur(nb);
  for (size_t b = 0; b < nb; ++b) cur[b] = items[b].in;
  int ping = 0;
  for (int mu = 0; mu + 2 < d; ++mu) {
    std::vector<double*> outv(nb);
    std::vector<const double*> mats(nb);
    for (size_t b = 0; b < nb; ++b) {
      outv[b] = scr[ping][b];
      mats[b] = items[b].mats[mu];
    }
    cproduct(mu, dimsS, cur, outv, mats);
    for (size_t b = 0; b < nb; ++b) cur[b] = outv[b];
    ping ^= 1;
  }
  // stage 0: mode d-1 locally, then to the owners' T pools (layout S_{d-1})
  {
    std::vector<double*> outv(nb);
    std::vector<const double*> mats(nb);
    for (size_t b = 0; b < nb; ++b) {
      outv[b] = scr[ping][b];
      mats[b] = items[b].mats[d - 2];
    }
    const ShardStage s0 = shard_stage(d + 1, gv, rk, P, 0);
    // the stage's (L, n, R) in the real view (2, n_1, …) is the K = 2n product's view
    if (!cproduct_remote(d - 2, dimsS, cur, mats, remap_of_stage(s0), kCtrlBytes)) {
      cproduct(d - 2, dimsS, cur, outv, mats);
      for (size_t b = 0; b < nb; ++b) remap_copy(s0, outv[b], kCtrlBytes + b * h->sym_slot);
    }
    ping ^= 1;
  }
  barrier();
  // stage 1: mode d locally on the transposed slab, then back to layout S_d
  {
    int dimsT[PHIKS_MAX_D];
    for (int k = 0; k < d; ++k) dimsT[k] = h->gn[k];
    dimsT[d - 2] = static_cast<int>(blk_cnt(h->gn[d - 2], P, rk));
    std::vector<const double*> in(nb);
    std::vector<double*> outv(nb);
    std::vector<const double*> mats(nb);
    for (size_t b = 0; b < nb; ++b) {
      in[b] = symT(static_cast<int>(b));
      outv[b] = scr[ping][b];
      mats[b] = items[b].mats[d - 1];
    }
    const ShardStage s1 = shard_stage(d + 1, gv, rk, P, 1);
    if (!cproduct_remote(d - 1, dimsT, in, mats, remap_of_stage(s1), kCtrlBytes + kShardChunk * h->sym_slot)) {
      cproduct(d - 1, dimsT, in, outv, mats);
      for (size_t b = 0; b < nb; ++b) remap_copy(s1, outv[b], kCtrlBytes + (kShardChunk + b) * h->sym_slot);
    }
  }
  barrier();
  int64_t nsum = 0;
  for (int mu = 0; mu < d; ++mu) nsum += h->gn[mu];
  tucker_ops += static_cast<int64_t>(nb);
  mu_flops += static_cast<double>(nb) * 8.0 * static_cast<double>(h->Nc) * static_cast<double>(nsum);
}

bool Exec::shard_digits_ok(size_t nb) const {
  const int d = h->d, P = h->world;
  (void)nb;
  if (d < 3 || !h->exch_off) return false;
  int64_t L0 = 1;
  for (int mu = 0; mu + 2 < d; ++mu) L0 *= h->gn[mu];
  const int na = h->gn[d - 2], nd = h->gn[d - 1];
  if (na % P || nd % P || (na / P) % 32 || L0 % 128) return false;
  if (L0 > h->exch_l0) return false;
  if (!ozaki_supported(L0 * (na / P), nd, 1, kOzDigits) || nd % 16) return false;
  if (h->gemm_path == PHIKS_GEMM_AUTO && nd < 128) return false;
  return true;
}

void Exec::tucker_raw_sharded(const std::vector<TuckerItem>& items) {
  if (!ok() || items.empty()) return;
  if (h->cplx) {
    tucker_raw_sharded_complex(items);
    return;
  }
  const int d = h->d, P = h->world, rk = h->rank;
  const int64_t N = h->N;
  const size_t nb = items.size();
  // int8 chain over the local modes into stage 0 (DESIGN.md §4d, §0(e)); with shard_digits_ok
  // also through stage 1 (stage 0 writes mode d's digit planes into the owners' pools)
  const bool chained = d >= 3 && ozaki_chain_route(items, 0, nb, d - 2);
  const bool digits = chained && shard_digits_ok(items.size());
  auto& scr = scr_pool;
  if (d >= 3 && !chained)
    while (scr[0].size() < nb) scr[0].push_back(ar->alloc_doubles(N));
  if (d >= 4 && !chained)
    while (scr[1].size() < nb) scr[1].push_back(ar->alloc_doubles(N));
  int64_t L = 1;
  for (int mu = 0; mu + 2 < d && !chained; ++mu) {
    const int n = h->n[mu];
    std::vector<LaunchTerm> terms;
    for (size_t b = 0; b < nb; ++b) {
      LaunchTerm t;
      t.in = (mu == 0) ? items[b].in : scr[(mu - 1) % 2][b];
      t.M = items[b].mats[mu];
      t.group = static_cast<int>(b);
      t.outs.push_back(Out{scr[mu % 2][b], 1.0, {}});
      terms.push_back(std::move(t));
    }
    mode_launch(L, n, N / (L * n), terms);
    L *= n;
  }
  const ShardStage s0 = shard_stage(d, h->gn, rk, P, 0), s1 = shard_stage(d, h->gn, rk, P, 1);
  auto remap_of = [&](const ShardStage& s) {
    Remap r{};
    r.world = P;
    r.cq = static_cast<int>(s.n / P);
    r.crem = static_cast<int>(s.n % P);
    r.uniform = s.uniform ? 1 : 0;
    r.colstride = s.colstride;
    for (int k = 0; k < P; ++k) {
      r.kstart[k] = static_cast<int>(s.kstart[k]);
      r.kstride[k] = s.kstride[k];
      r.kroff[k] = s.kroff[k];
      r.base[k] = h->peer[k];
    }
    return r;
  };
  const Remap ra = remap_of(s0), rb = remap_of(s1);
  (void)L;
  if (digits) {
    // every mode chained: stage 0 stores mode d's digit planes into the owners' T pools,
    // stage 1 (after the exchange barriers inside) reads them and stores fp64 into the Y pools
    const size_t cap = chain_cap();
    for (size_t s0c = 0; s0c < nb && ok(); s0c += cap) {  // each piece: both stages and their barriers
      tucker_chain_i8(items, s0c, std::min(nb, s0c + cap), d - 1, &ra, &rb);
      barrier();
    }
    shard_digit_ops += static_cast<int64_t>(nb);
    int64_t nsum = 0;
    for (int mu = 0; mu < d; ++mu) nsum += h->gn[mu];
    tucker_ops += static_cast<int64_t>(nb);
    mu_flops += static_cast<double>(nb) * 2.0 * static_cast<double>(N) * static_cast<double>(nsum);
    return;
  }
  if (chained) {
    // modes 1..d−2 chained on the slab, stage 0 (mode d−1) reading their digits and
    // storing fp64 into the owners' T pools
    const size_t cap = chain_cap();
    for (size_t s0c = 0; s0c < nb && ok(); s0c += cap) tucker_chain_i8(items, s0c, std::min(nb, s0c + cap), d - 2, &ra);
  } else {
    std::vector<LaunchTerm> terms;
    for (size_t b = 0; b < nb; ++b) {
      LaunchTerm t;
      t.in = (d == 2) ? items[b].in : scr[(d - 3) % 2][b];
      t.M = items[b].mats[d - 2];
      t.group = static_cast<int>(b);
      t.outs.push_back(Out{reinterpret_cast<double*>(kCtrlBytes + b * h->sym_slot), 1.0, {}});
      terms.push_back(std::move(t));
    }
    mode_launch(s0.L, static_cast<int>(s0.n), s0.R, terms, &ra);
  }
  barrier();
  {
    std::vector<LaunchTerm> terms;
    for (size_t b = 0; b < nb; ++b) {
      LaunchTerm t;
      t.in = symT(static_cast<int>(b));
      t.M = items[b].mats[d - 1];
      t.group = static_cast<int>(b);
      t.outs.push_back(Out{reinterpret_cast<double*>(kCtrlBytes + (kShardChunk + b) * h->sym_slot), 1.0, {}});
      terms.push_back(std::move(t));
    }
    mode_launch(s1.L, static_cast<int>(s1.n), s1.R, terms, &rb);
  }
  barrier();
  int64_t nsum = 0;
  for (int mu = 0; mu < d; ++mu) nsum += h->gn[mu];
  tucker_ops += static_cast<int64_t>(nb);
  mu_flops += static_cast<double>(nb) * 2.0 * static_cast<double>(N) * static_cast<double>(nsum);
}

void Exec::tucker_batch(const std::vector<TuckerItem>& items) {
  if (!ok() || items.empty()) return;
  const int d = h->d;
  const int64_t N = h->N;
  if (ozaki_chain_route(items, 0, items.size())) {  // every mode on the int8 path, no fp64 intermediates
    const size_t cap = chain_cap();
    for (size_t s0 = 0; s0 < items.size() && ok(); s0 += cap)
      tucker_chain_i8(items, s0, std::min(items.size(), s0 + cap));
    return;
  }
  // items per chunk bounded by the number of groups a non-last launch can hold
  const size_t chunk = static_cast<size_t>(kMaxGroups);
  const size_t nscr = std::min(items.size(), chunk);
  auto& scr = scr_pool;
  if (d >= 2)
    while (scr[0].size() < nscr) scr[0].push_back(ar->alloc_doubles(N));
  if (d >= 3)
    while (scr[1].size() < nscr) scr[1].push_back(ar->alloc_doubles(N));
  // complex tensors (interleaved): mode 1 contracts the merged (re/im, i_1)
  // index with the 2n×2n real form of the matrix; every other mode is two real
  // products on the (2·L, n, R) view, Mr then J(·Mi) accumulated (same group)
  const bool cx = h->cplx;
  for (size_t c0 = 0; c0 < items.size() && ok(); c0 += chunk) {
    const size_t c1 = std::min(items.size(), c0 + chunk);
    int64_t L = 1;
    for (int mu = 0; mu < d; ++mu) {
      const int n = h->n[mu];
      const int64_t R = h->Nc / (L * n);
      std::vector<LaunchTerm> terms;
      // complex μ ≥ 2 on the int8 path (plain outputs only): DESIGN.md §4f
      bool cplx_i8 = cx && mu > 0;
      if (cplx_i8) {
        std::vector<LaunchTerm> probe(1);
        probe[0].kcat = 1;
        probe[0].outs.push_back(Out{nullptr, 1.0, {}});
        cplx_i8 = ozaki_route(2 * L, n, R, probe, nullptr);
        for (size_t b = c0; b < c1 && cplx_i8; ++b) {
          const TuckerItem& it = items[b];
          if (mu == d - 1 && (it.outs.size() != 1 || !it.outs[0].srcs.empty())) cplx_i8 = false;
        }
        std::set<int> gs;
        for (size_t b = c0; b < c1 && cplx_i8; ++b)
          if (mu == d - 1 && !gs.insert(items[b].group).second) cplx_i8 = false;
      }
      for (size_t b = c0; b < c1; ++b) {
        const TuckerItem& it = items[b];
        LaunchTerm t;
        t.in = (mu == 0) ? it.in : scr[(mu - 1) % 2][b - c0];
        t.M = it.mats[mu];
        if (mu < d - 1) {
          t.group = static_cast<int>(b - c0);
          t.outs.push_back(Out{scr[mu % 2][b - c0], 1.0, {}});
        } else {
          t.group = it.group;
          t.outs = it.outs;
          if (it.in_scale != 1.0)
            for (Out& o : t.outs) o.beta *= it.in_scale;
        }
        if (cx && mu > 0 && cplx_i8) {  // one int8 product with K = 2n: [Re M | Im M]·[x ; Jx]
          t.M = complex_parts(it.mats[mu], n).first;
          t.kcat = 1;
          terms.push_back(std::move(t));
        } else if (cx && mu > 0) {
          const auto parts = complex_parts(it.mats[mu], n);
          LaunchTerm ti = t;
          t.M = parts.first;
          ti.M = parts.second;
          ti.cswap = 1;
          for (Out& o : ti.outs) {  // += β·J(acc_i): sole-source outputs only (split batches)
            o.srcs.assign(1, Src{o.dst, 1.0});
          }
          terms.push_back(std::move(t));
          terms.push_back(std::move(ti));
        } else {
          terms.push_back(std::move(t));
        }
      }
      if (cx && mu == 0)
        mode_launch(1, 2 * n, R, terms);
      else
        mode_launch(cx ? 2 * L : L, n, R, terms);
      L *= n;
    }
    int64_t nsum = 0;
    for (int mu = 0; mu < d; ++mu) nsum += h->n[mu];
    tucker_ops += static_cast<int64_t>(c1 - c0);
    mu_flops += static_cast<double>(c1 - c0) * (cx ? 8.0 : 2.0) * static_cast<double>(h->Nc) *
                static_cast<double>(nsum);
  }
}

std::pair<const double*, const double*> Exec::complex_parts(const double* Rm, int n) {
  auto itp = cparts.find(Rm);
  if (itp != cparts.end()) return itp->second;
  // contiguous: [Re M | Im M] is the n × 2n matrix of the int8 complex products (§4f)
  double* mr = ar->alloc_doubles(2 * static_cast<int64_t>(n) * n);
  double* mi = mr + static_cast<int64_t>(n) * n;
  emit("complex_parts", [Rm, n, mr, mi](cudaStream_t s) { return launch_complex_parts(Rm, n, mr, mi, s); });
  cparts[Rm] = {mr, mi};
  return {mr, mi};
}

}  // namespace host
}  // namespace phiks
