// C ABI and host orchestration of the PHIKS hot path (include/phiks.h).
//
// The host only plans and enqueues: every arithmetic step on tensors or
// matrices runs in the CUDA kernels of kernels.cu.  One apply is
//   A. small-matrix exponentials exp(c·τA_f) for the GLL nodes (Taylor degree
//      16, Paterson–Stockmeyer, scaling and squaring) and the level matrices
//      exp(τA_f/2^j) by repeated squaring,
//   B. quadrature: one batched Tucker operator per node (Eq. (10)),
//      weight-sum fused into the last mode's epilogue (Eq. (11) / Eq. (17)),
//   C. squaring levels j = s..1 (Eq. (12) / Eq. (18)), recurrence fused into the
//      last mode's epilogue, intermediate scales written on the way (Eq. (13)/(19)),
//   D. exp(τK/2^j)v actions (one Tucker operator each, l.614-616).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "phiks_internal.h"
#include "planner.h"

using namespace phiks;

namespace {

thread_local std::string g_err;

phiks_status fail(phiks_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(PHIKS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

double factorial(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}

struct Factor {
  int n = 0;
  double* dA = nullptr;   // device copy of A_f
  double norm1 = 0.0;    // ||A_f||_1
  plan::FactorRange fr{};
};

struct PlanKey {
  int mode, p, n_scales;
  double tau, tol;
  std::vector<double> norms;
  bool operator<(const PlanKey& o) const {
    return std::tie(mode, p, n_scales, tau, tol, norms) < std::tie(o.mode, o.p, o.n_scales, o.tau, o.tol, o.norms);
  }
};

}  // namespace

struct phiks_ctx {
  int d = 0;
  int n[PHIKS_MAX_D] = {0};
  int64_t N = 0;   // doubles per tensor (2·Nc for complex handles)
  int64_t Nc = 0;  // elements per tensor
  bool cplx = false;  // complex factors and tensors (interleaved re, im)
  std::vector<Factor> factors;
  int fac_of_mode[PHIKS_MAX_D] = {0};
  void* ws_own = nullptr;
  size_t ws_own_bytes = 0;
  double* h_pinned = nullptr;  // pinned host scratch (norms)
  std::map<PlanKey, plan::Plan> plan_cache;
  phiks_stats stats{};
  // profiling: event pairs around μ-mode-product launches of the last apply
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<double> ev_flops;
  std::vector<char> ev_expm;  // 1: a small-GEMM launch of the exponential stage
  int ev_used = 0;
  // ---- slab sharding along the outermost mode (phiks_create_sharded) ----
  // n[] holds the LOCAL dims of layout S_d (n[d-1] = gn[d-1]/world); the
  // transposed layout S_{d-1} has dims (n_1..n_{d-2}, gn[d-2]/world, gn[d-1]).
  int rank = 0, world = 1;
  int gn[PHIKS_MAX_D] = {0};
  char* sym = nullptr;  // own symmetric region: control block + T/Y pools
  size_t sym_bytes = 0;
  size_t sym_slot = 0;  // bytes per pooled local tensor
  char* peer[kMaxRanks] = {nullptr};
  bool peer_ipc[kMaxRanks] = {false};
  bool peers_ready = false;
  uint64_t norm_phase = 0;  // parity selects the norm-slot buffer (a fast rank may run one apply ahead)
  // CUDA graphs of whole applies (device memory, profiling off): captured on
  // s_cap the first time a request/plan/pointer set is seen, replayed after
  struct GraphEntry {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  cudaStream_t s_cap = nullptr;
  int64_t graph_replays = 0;
  // host-memory applies: copy streams and their ordering events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_h2d = nullptr, ev_d2h = nullptr, ev_cdone = nullptr, ev_ready = nullptr;
  // the exponential stage (stage A) of an apply runs on s_pre, ordered only
  // after the previous apply of this handle (ev_cdone), so it overlaps the
  // tail of whatever else is queued on the apply stream (another handle's
  // Tucker work); the stream waits on ev_pre before the first Tucker batch
  cudaStream_t s_pre = nullptr;
  cudaEvent_t ev_pre = nullptr;
  bool sharded() const { return world > 1; }
};

namespace {
// symmetric region layout (identical on every rank)
constexpr size_t kCtrlFlags = 0;                                   // uint64 flags[kMaxRanks]
constexpr size_t kCtrlErr = kMaxRanks * sizeof(uint64_t);          // int err
constexpr size_t kCtrlEpoch = 128;                                 // uint64 barrier count
constexpr size_t kCtrlNorms = 256;                                 // double norms[2][kMaxRanks][kMaxVecs]
constexpr size_t kCtrlNormsBuf = kMaxRanks * kMaxVecs * sizeof(double);
constexpr size_t kCtrlBytes = 4096;
static_assert(kCtrlNorms + 2 * kCtrlNormsBuf <= kCtrlBytes, "control block layout");
static_assert(kCtrlErr + sizeof(int) <= kCtrlEpoch && kCtrlEpoch + 8 <= kCtrlNorms, "control block layout");
constexpr int kShardChunk = 16;  // Tucker operators per sharded sub-batch (T and Y pools)
constexpr uint64_t kBarrierTimeoutNs = 60ull * 1000 * 1000 * 1000;
}  // namespace

namespace {

// ---------------------------------------------------------------------------
// Bump allocator over the workspace; in measure mode it only counts.
// ---------------------------------------------------------------------------
struct Arena {
  char* base = nullptr;
  size_t cap = 0, off = 0;
  bool measure = true;
  double* alloc_doubles(int64_t count) {
    const size_t bytes = ((static_cast<size_t>(count) * sizeof(double)) + 255) & ~size_t(255);
    char* p = measure ? nullptr : base + off;
    off += bytes;
    if (measure) return reinterpret_cast<double*>(static_cast<uintptr_t>(0x1000) + off);  // fake, never dereferenced
    return reinterpret_cast<double*>(p);
  }
};

// Geometry of the two peer-store launches of a slab-sharded Tucker operator
// (DESIGN.md §0(e)).  gn: global dims.  stage 0: the mode-(d-1) product on the
// slab (layout S_d) storing into layout S_{d-1}; stage 1: the mode-d product
// on layout S_{d-1} storing back into S_d.  Output element (l, j, r) of the
// (L, n, R) launch goes to rank k = j / cb at offset
//   l + rstride·r + roff + colstride·(j − k·cb).
struct ShardStage {
  int64_t L, n, R, cb, rstride, roff, colstride;
};
ShardStage shard_stage(int d, const int* gn, int rank, int world, int stage) {
  int64_t L0 = 1;
  for (int mu = 0; mu + 2 < d; ++mu) L0 *= gn[mu];
  const int64_t na = gn[d - 2], nd = gn[d - 1];
  const int64_t cb = na / world, cd = nd / world;
  ShardStage s{};
  if (stage == 0) {
    s = ShardStage{L0, na, cd, cb, L0 * cb, L0 * cb * rank * cd, L0};
  } else {
    s = ShardStage{L0 * cb, nd, 1, cd, 0, L0 * cb * rank, L0 * na};
  }
  return s;
}

// A source list with coefficients, kept on the host until a launch is built.
struct Src {
  const double* ptr;
  double coef;
};
struct Out {
  double* dst;
  double beta;
  std::vector<Src> srcs;
};

// One Tucker operator of a batch.
struct TuckerItem {
  const double* in = nullptr;
  double in_scale = 1.0;  // folded into every last-mode beta
  const double* mats[PHIKS_MAX_D] = {nullptr};
  int group = 0;          // last-mode accumulation group
  std::vector<Out> outs;  // last-mode epilogue
};

struct Exec {
  phiks_ctx* h;
  cudaStream_t st;
  bool measure;
  Arena* ar;
  int64_t launches = 0;
  int64_t tucker_ops = 0;
  std::vector<double*> scr_pool[2];  // N-sized scratch reused by every tucker_batch
  std::vector<double*> y_pool;       // per-item Tucker results of split batches
  int split = 0;                     // 1: quadrature sums as a separate pass, 2: also squaring
  double mu_flops = 0.0, expm_flops = 0.0;
  phiks_status status = PHIKS_OK;
  int64_t barriers = 0;

  // Recorded ops: with `rec` set, launches are appended instead of issued (the
  // phase-interleaved emulation of several ranks on one GPU replays them).
  struct Op {
    bool barrier;
    std::function<cudaError_t(cudaStream_t)> fn;
    const char* what;
  };
  std::vector<Op>* rec = nullptr;
  // host-memory applies: called (execute pass only) when the staged inputs are
  // first needed and when some outputs are final (their copy-out can start)
  std::function<void()> on_inputs;
  std::function<void(const std::vector<double*>&)> on_outputs;

  bool ok() const { return status == PHIKS_OK; }
  void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess && status == PHIKS_OK) {
      status = PHIKS_ERR_CUDA;
      g_err = std::string(what) + ": " + cudaGetErrorString(e);
    }
  }
  void emit(const char* what, std::function<cudaError_t(cudaStream_t)> fn) {
    ++launches;
    if (measure || !ok()) return;
    if (rec)
      rec->push_back(Op{false, std::move(fn), what});
    else
      check(fn(st), what);
  }
  // cross-rank barrier of a sharded handle (device-side, stream-ordered)
  void barrier() {
    ++barriers;
    if (!ok() || !h->sharded()) return;
    ++launches;
    if (measure) return;
    if (rec) {
      rec->push_back(Op{true, nullptr, "barrier"});
      return;
    }
    BarrierParams bp{};
    bp.rank = h->rank;
    bp.world = h->world;
    bp.epoch = reinterpret_cast<uint64_t*>(h->sym + kCtrlEpoch);
    bp.timeout_ns = kBarrierTimeoutNs;
    for (int k = 0; k < h->world; ++k) bp.peer_flags[k] = reinterpret_cast<uint64_t*>(h->peer[k] + kCtrlFlags);
    bp.err = reinterpret_cast<int*>(h->sym + kCtrlErr);
    check(launch_barrier(bp, st), "barrier");
  }

  // ---- one mode-product launch from host-side term lists ----
  struct LaunchTerm {
    const double* in;
    const double* M;
    int group;
    std::vector<Out> outs;
    int cswap = 0;  // complex: J applied to the accumulator (TermSpec::cswap)
  };
  void mode_launch(int64_t L, int n, int64_t R, const std::vector<LaunchTerm>& terms, const Remap* rm = nullptr) {
    if (!ok() || terms.empty()) return;
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
          rec->push_back(Op{false, [sp](cudaStream_t s) { return launch_mode_product(*sp, s); }, "mode_product"});
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

  void combine(int64_t count, const std::vector<Out>& outs) {
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

  // ---- matrix-form combination dst_o = Σ_s coef[o][s] src_s ----
  void mcombine(int64_t count, const std::vector<const double*>& srcs, const std::vector<double*>& dsts,
                const std::vector<std::vector<double>>& coef) {
    if (!ok() || dsts.empty()) return;
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

  // A batch whose last-mode epilogues run as a separate streaming pass: every
  // item writes its raw Tucker result Y_b, then the epilogue recurrences (in
  // group order, accumulations included) are evaluated symbolically into one
  // matrix-form combination over {Y_b} ∪ external sources.  Sharded handles
  // always take this path, kShardChunk items at a time (the Y_b then live in
  // the symmetric region); a later chunk accumulates into the outputs.
  void tucker_batch_split(const std::vector<TuckerItem>& items) {
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
      for (auto& row : rows)
        for (auto& t : row)
          if (std::find(srcs.begin(), srcs.end(), t.first) == srcs.end()) srcs.push_back(t.first);
      std::vector<std::vector<double>> coef(dsts.size(), std::vector<double>(srcs.size(), 0.0));
      for (size_t o = 0; o < dsts.size(); ++o)
        for (auto& t : rows[o]) coef[o][std::find(srcs.begin(), srcs.end(), t.first) - srcs.begin()] += t.second;
      mcombine(N, srcs, dsts, coef);
    }
  }

  // ---- slab-sharded raw Tucker operators (≤ kShardChunk items) ----
  // Local layout S_d: dims (n_1..n_{d-1}, n_d/P), the rank's slab of the outermost
  // mode.  Modes 1..d-2 are local; the mode-(d-1) product stores its output in
  // layout S_{d-1} (dims (n_1..n_{d-2}, n_{d-1}/P, n_d)) on the rank owning each
  // output column; after a barrier the mode-d product is local there and stores
  // back into layout S_d on the owner of each output column; a second barrier
  // makes Y_b complete.  Items write Y_b = symY(b).
  double* symT(int i) const { return reinterpret_cast<double*>(h->sym + kCtrlBytes + i * h->sym_slot); }
  double* symY(int i) const {
    return reinterpret_cast<double*>(h->sym + kCtrlBytes + (kShardChunk + i) * h->sym_slot);
  }
  void tucker_raw_sharded(const std::vector<TuckerItem>& items) {
    if (!ok() || items.empty()) return;
    const int d = h->d, P = h->world, rk = h->rank;
    const int64_t N = h->N;
    const size_t nb = items.size();
    auto& scr = scr_pool;
    if (d >= 3)
      while (scr[0].size() < nb) scr[0].push_back(ar->alloc_doubles(N));
    if (d >= 4)
      while (scr[1].size() < nb) scr[1].push_back(ar->alloc_doubles(N));
    int64_t L = 1;
    for (int mu = 0; mu + 2 < d; ++mu) {
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
      r.cb = static_cast<int>(s.cb);
      r.rstride = s.rstride;
      r.roff = s.roff;
      r.colstride = s.colstride;
      for (int k = 0; k < P; ++k) r.base[k] = h->peer[k];
      return r;
    };
    const Remap ra = remap_of(s0), rb = remap_of(s1);
    (void)L;
    {
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

  // every batch of run_job: sharded handles always split
  void batch(const std::vector<TuckerItem>& items, bool split_it) {
    if (h->sharded() || h->cplx || split_it)
      tucker_batch_split(items);
    else
      tucker_batch(items);
  }

  // ---- batched Tucker operators (Eq. (4)) ----
  void tucker_batch(const std::vector<TuckerItem>& items) {
    if (!ok() || items.empty()) return;
    const int d = h->d;
    const int64_t N = h->N;
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
          if (cx && mu > 0) {
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

  // (Mr, Mi) of a complex exponential held in its 2n×2n real form, extracted
  // once per matrix and apply (complex handles)
  std::map<const double*, std::pair<const double*, const double*>> cparts;
  std::pair<const double*, const double*> complex_parts(const double* Rm, int n) {
    auto itp = cparts.find(Rm);
    if (itp != cparts.end()) return itp->second;
    double* mr = ar->alloc_doubles(static_cast<int64_t>(n) * n);
    double* mi = ar->alloc_doubles(static_cast<int64_t>(n) * n);
    emit("complex_parts", [Rm, n, mr, mi](cudaStream_t s) { return launch_complex_parts(Rm, n, mr, mi, s); });
    cparts[Rm] = {mr, mi};
    return {mr, mi};
  }

  // out_b = A_b · B_b (+ epilogue) for n×n matrices: mode-1 product of the
  // "tensor" B (n, n) with matrix A.
  bool in_expm = false;
  void gemm_batch(int n, std::vector<LaunchTerm>& terms) {
    in_expm = true;
    mode_launch(1, n, n, terms);
    in_expm = false;
    expm_flops += 2.0 * n * static_cast<double>(n) * n * static_cast<double>(terms.size());
  }
};

// ---------------------------------------------------------------------------
// Stage A: small-matrix exponentials exp(c_k · τA_f) for a list of (f, c)
// requests.  Y = a·X (X = τA_f, a = c/2^σ, ||Y||_1 ≤ 1/2):
//   exp(Y) ≈ Σ_{k=0}^{16} Y^k/k! = B0 + Y4(B1 + Y4(B2 + Y4(B3 + Y4/16!))),
//   B_m = Σ_{r=0}^{3} Y^r/(4m+r)!  (Paterson–Stockmeyer), then σ squarings.
// The powers X^2, X^3, X^4 are shared by every request of a factor.
// ---------------------------------------------------------------------------
struct ExpReq {
  int f;
  double c;
  double* result = nullptr;  // filled in
};

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

// ---------------------------------------------------------------------------
// The whole φ-action (stages A-D) on device pointers.
// vin[ℓ] (ℓ = 0..p) device input tensors or nullptr; out_same[ℓ][j] / out_lin[j]
// device output tensors or nullptr (not requested).
// ---------------------------------------------------------------------------
struct Job {
  int mode;
  int p;
  int n_scales;
  double tau;
  int s, q;
  const double* vin[kMaxVecs] = {nullptr};
  double* out_same[kMaxVecs][PHIKS_MAX_SCALES] = {{nullptr}};
  double* out_lin[PHIKS_MAX_SCALES] = {nullptr};
};

void run_job(Exec& ex, const Job& jb) {
  phiks_ctx* h = ex.h;
  const int d = h->d;
  const int p = jb.p, s = jb.s, q = jb.q;
  const int64_t N = h->N;
  const int nf = static_cast<int>(h->factors.size());
  const bool same = jb.mode == PHIKS_MODE_SAME_VECTOR;

  // ---- which level matrices exp(τA/2^j) are needed ----
  bool want_phi0 = false;
  if (same) {
    for (int j = 0; j < jb.n_scales; ++j) want_phi0 |= jb.out_same[0][j] != nullptr;
  } else {
    want_phi0 = jb.vin[0] != nullptr;
  }
  int jmin = s;
  if (p >= 1) jmin = std::min(jmin, 1);
  if (want_phi0) jmin = 0;
  if (p >= 1 && s == 0) jmin = 0;

  std::vector<double> theta, w;
  if (p >= 1) plan::gll_rule(q, theta, w);

  // ---- Stage A ----
  std::vector<ExpReq> reqs;
  // node exponentials (θ_i ≠ 1): c_i = (1 − θ_i)/2^s; node 0 (θ = 0) gives exp(τA/2^s)
  const int n_nodes = (p >= 1) ? q - 1 : 0;
  for (int i = 0; i < n_nodes; ++i)
    for (int f = 0; f < nf; ++f) reqs.push_back({f, (1.0 - theta[i]) / std::ldexp(1.0, s)});
  if (p == 0)
    for (int f = 0; f < nf; ++f) reqs.push_back({f, 1.0 / std::ldexp(1.0, s)});
  expm_batch(ex, jb.tau, reqs);
  if (!ex.ok()) return;
  // nodeE[i][f]
  std::vector<std::vector<const double*>> nodeE(n_nodes, std::vector<const double*>(nf));
  for (int i = 0; i < n_nodes; ++i)
    for (int f = 0; f < nf; ++f) nodeE[i][f] = reqs[static_cast<size_t>(i) * nf + f].result;
  // level matrices Es[j][f], j = jmin..s
  std::vector<std::vector<double*>> Es(s + 1, std::vector<double*>(nf, nullptr));
  for (int f = 0; f < nf; ++f)
    Es[s][f] = (p >= 1) ? const_cast<double*>(nodeE[0][f]) : reqs[f].result;
  for (int j = s; j > jmin; --j) {
    std::map<int, std::vector<Exec::LaunchTerm>> byn;
    for (int f = 0; f < nf; ++f) {
      const int n = h->factors[f].n;
      Es[j - 1][f] = ex.ar->alloc_doubles(static_cast<int64_t>(n) * n);
      auto& v = byn[n];
      v.push_back({Es[j][f], Es[j][f], static_cast<int>(v.size()), {Out{Es[j - 1][f], 1.0, {}}}});
    }
    for (auto& kv : byn) ex.gemm_batch(kv.first, kv.second);
  }
  auto mats_for = [&](const std::vector<double*>& perf, const double** mats) {
    for (int mu = 0; mu < d; ++mu) mats[mu] = perf[h->fac_of_mode[mu]];
  };
  auto node_mats = [&](int i, const double** mats) {
    for (int mu = 0; mu < d; ++mu) mats[mu] = nodeE[i][h->fac_of_mode[mu]];
  };

  // inputs staged from host memory are needed from here on (stage A overlaps their copy)
  if (ex.on_inputs) ex.on_inputs();

  // ---- Stage D (same vector): exp(τK/2^j)v needs only the level matrices and
  // reads the same v as the quadrature, so with p ≥ 1 it joins the quadrature
  // batch (one launch per mode for both); a host-memory apply copies it out
  // while the squaring runs ----
  std::vector<TuckerItem> d_items;
  std::vector<double*> d_ready;
  if (same) {
    for (int j = 0; j < jb.n_scales; ++j) {
      if (!jb.out_same[0][j]) continue;
      TuckerItem it;
      it.in = jb.vin[0];
      mats_for(Es[j], it.mats);
      it.group = 1000 + j;
      it.outs.push_back(Out{jb.out_same[0][j], 1.0, {}});
      d_items.push_back(it);
      d_ready.push_back(jb.out_same[0][j]);
    }
    if (p == 0) {
      ex.batch(d_items, false);
      if (!ex.ok()) return;
      if (ex.on_outputs && !d_ready.empty()) ex.on_outputs(d_ready);
      d_items.clear();
      d_ready.clear();
    }
  }

  // ---- state buffers ----
  // state[j][ℓ] for the scale j (ℓ = 1..p)
  std::vector<std::vector<double*>> state(s + 1, std::vector<double*>(p + 1, nullptr));
  std::vector<double*> pool[2];
  auto ws_state = [&](int j, int ell) -> double* {
    auto& pl = pool[j % 2];
    while (static_cast<int>(pl.size()) <= ell) pl.push_back(nullptr);
    if (!pl[ell]) pl[ell] = ex.ar->alloc_doubles(N);
    return pl[ell];
  };
  for (int j = 0; j <= s; ++j)
    for (int ell = 1; ell <= p; ++ell) {
      double* u = (same && j < jb.n_scales) ? jb.out_same[ell][j] : nullptr;
      state[j][ell] = u ? u : ws_state(j, ell);
    }

  if (p >= 1) {
    // ---- Stage B: quadrature at scale s ----
    const double wq = w[q - 1];  // θ_q = 1 term: exp(0) = I, no Tucker operator (l.948-952)
    std::vector<TuckerItem> items;
    if (same) {
      for (int i = 0; i < n_nodes; ++i) {
        TuckerItem it;
        it.in = jb.vin[0];
        node_mats(i, it.mats);
        it.group = 0;
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
      std::vector<Out> prep;
      std::vector<std::vector<TuckerItem>> per_ell(p + 1);
      for (int ell = 1; ell <= p; ++ell) {
        bool first = true;
        for (int i = 0; i < n_nodes; ++i) {
          std::vector<Src> comb;
          for (int k = 1; k <= ell; ++k) {
            const double* v = jb.vin[p + 1 - k];
            const double c = xcoef(theta[i], ell, k);
            if (v && c != 0.0) comb.push_back(Src{v, c});
          }
          if (comb.empty()) continue;
          TuckerItem it;
          node_mats(i, it.mats);
          it.group = ell;
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
      ex.combine(N, prep);
      for (int ell = 1; ell <= p; ++ell)
        for (auto& it : per_ell[ell]) items.push_back(it);
      if (s < jb.n_scales && jb.out_lin[s]) {
        // scale s output = Ψ_p^{(s)} (+ exp term later): mirror the Ψ_p accumulation
        for (auto& it : items)
          if (it.group == p) {
            Out o = it.outs[0];
            o.dst = jb.out_lin[s];
            for (auto& sr : o.srcs)
              if (sr.ptr == state[s][p]) sr.ptr = jb.out_lin[s];
            it.outs.push_back(o);
          }
      }
    }
    for (auto& it : d_items) items.push_back(it);
    ex.batch(items, ex.split >= 1);
    if (!ex.ok()) return;
    if (ex.on_outputs && !d_ready.empty()) ex.on_outputs(d_ready);
    if (!ex.ok()) return;

    // ---- Stage C: squaring, j = s..1 ----
    for (int j = s; j >= 1; --j) {
      std::vector<TuckerItem> sq;
      for (int ell = p; ell >= 1; --ell) {
        TuckerItem it;
        it.in = state[j][ell];
        mats_for(Es[j], it.mats);
        it.group = ell;
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
      ex.batch(sq, ex.split >= 2);
      if (!ex.ok()) return;
    }
  }

  // ---- Stage D (linear combination): exp(τK/2^j)v_0 added to the result ----
  std::vector<TuckerItem> ex_items;
  if (!same) {
    for (int j = 0; j < jb.n_scales; ++j) {
      if (!jb.out_lin[j]) continue;
      if (jb.vin[0]) {
        TuckerItem it;
        it.in = jb.vin[0];
        mats_for(Es[j], it.mats);
        it.group = j;
        Out o{jb.out_lin[j], 1.0, {}};
        if (p >= 1) o.srcs.push_back(Src{jb.out_lin[j], 1.0});
        it.outs.push_back(o);
        ex_items.push_back(it);
      }
    }
  }
  ex.batch(ex_items, false);
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
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

phiks_status create_impl(int d, const int* n, const double* const* A_host, bool cplx, phiks_handle* out) {
  if (!out || !n || !A_host) return fail(PHIKS_ERR_ARG, "null argument");
  *out = nullptr;
  if (d < 1 || d > PHIKS_MAX_D) return fail(PHIKS_ERR_ARG, "d out of range");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PHIKS_ERR_CUDA, "no CUDA device");
  auto* h = new phiks_ctx();
  h->d = d;
  h->cplx = cplx;
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
  // dedupe bitwise-identical factors
  std::vector<int> rep;
  for (int mu = 0; mu < d; ++mu) {
    int found = -1;
    for (size_t f = 0; f < rep.size(); ++f) {
      const int m2 = rep[f];
      if (n[m2] == n[mu] &&
          std::memcmp(A_host[m2], A_host[mu], sizeof(double) * per * static_cast<size_t>(n[mu]) * n[mu]) == 0) {
        found = static_cast<int>(f);
        break;
      }
    }
    if (found < 0) {
      Factor F;
      // complex factors are stored (and exponentiated) in their 2n×2n real form:
      // exp of the real form is the real form of exp (an algebra homomorphism)
      std::vector<double> Rz;
      const double* A = A_host[mu];
      if (cplx) {
        Rz = realify(n[mu], A_host[mu]);
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
      F.fr = cplx ? plan::factor_range_complex(n[mu], A_host[mu]) : plan::factor_range(F.n, A);
      h->factors.push_back(F);
      rep.push_back(mu);
      found = static_cast<int>(h->factors.size()) - 1;
    }
    h->fac_of_mode[mu] = found;
  }
  if (cudaMallocHost(reinterpret_cast<void**>(&h->h_pinned), 64 * sizeof(double)) != cudaSuccess) {
    phiks_destroy(h);
    return fail(PHIKS_ERR_NOMEM, "pinned host scratch");
  }
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

phiks_status phiks_destroy(phiks_handle h) {
  if (!h) return PHIKS_OK;
  for (auto& F : h->factors)
    if (F.dA) cudaFree(F.dA);
  if (h->ws_own) cudaFree(h->ws_own);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  for (int k = 0; k < kMaxRanks; ++k)
    if (h->peer_ipc[k] && h->peer[k]) cudaIpcCloseMemHandle(h->peer[k]);
  for (cudaEvent_t e : {h->ev_h2d, h->ev_d2h, h->ev_cdone, h->ev_ready})
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

namespace {

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

phiks_status make_plan(phiks_handle h, const phiks_request* req, int p, const std::vector<double>& norms,
                       plan::Plan& out) {
  const int s_min = req->n_scales - 1;
  if (req->force_s >= 0) {
    out.s = req->force_s;
    out.q = (p >= 1) ? req->force_q : 0;
    out.T = plan::tucker_count(req->mode, out.s, req->n_scales, out.q, p);
    out.ok = true;
    return PHIKS_OK;
  }
  const double tol = req->tol > 0 ? req->tol : std::ldexp(1.0, -53);
  PlanKey key{req->mode, p, req->n_scales, req->tau, tol, norms};
  auto it = h->plan_cache.find(key);
  if (it != h->plan_cache.end()) {
    out = it->second;
    return PHIKS_OK;
  }
  plan::Rect rect{};
  double cr = 0.0, ci = 0.0, hr = 0.0, hi = 0.0;
  for (int mu = 0; mu < h->d; ++mu) {
    const auto& fr = h->factors[h->fac_of_mode[mu]].fr;
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

}  // namespace

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
  const int nodes = p >= 1 ? pl.q - 1 : 0;
  bool has0 = req->ells[0] == 0;
  out->T_executed = (req->mode == PHIKS_MODE_SAME_VECTOR) ? nodes + pl.s * p + (has0 ? req->n_scales : 0)
                                                         : nodes * p + pl.s * p + (has0 ? req->n_scales : 0);
  return PHIKS_OK;
}

// One apply on one handle, split into phases so that several emulated ranks
// can be driven phase by phase (phiks_apply_ranks_serial).
struct ApplyRun {
  phiks_handle h = nullptr;
  const phiks_request* req = nullptr;
  int p = 0, n_vecs = 0, nouts = 0;
  bool same = true, host_mem = false, host_async = false, size_only = false;
  const double* const* vecs = nullptr;
  double* const* outs = nullptr;
  cudaStream_t cs = nullptr;
  int64_t N = 0;
  size_t tbytes = 0;
  Arena ar;
  Exec ex{};
  Job jb{};
  std::vector<double*> dv, dout;
  plan::Plan pl;
  int split = 2;
  // lincomb norms
  bool need_norms = false;
  std::vector<int> which;        // index into vecs of v_1..v_p present
  double* nscratch = nullptr;    // device: 1024*kMaxVecs partials + kMaxVecs norms²
  std::vector<double*> ntmp;     // host-memory inputs staged for the norms
  int norm_launches = 0;
  size_t norm_off = kCtrlNorms;  // this apply's norm-slot buffer in the control block

  phiks_status init(phiks_handle h_, const phiks_request* req_, int n_vecs_, const double* const* vecs_,
                    double* const* outs_, void* stream, bool size_only_) {
    h = h_;
    req = req_;
    phiks_status st = validate(h, req, p);
    if (st != PHIKS_OK) return st;
    n_vecs = n_vecs_;
    vecs = vecs_;
    outs = outs_;
    size_only = size_only_;
    same = req->mode == PHIKS_MODE_SAME_VECTOR;
    nouts = same ? req->n_ells * req->n_scales : req->n_scales;
    if (!size_only) {
      if (same ? n_vecs != 1 : n_vecs != req->n_ells) return fail(PHIKS_ERR_ARG, "n_vecs");
      if (!vecs || !outs) return fail(PHIKS_ERR_ARG, "null vecs/outs");
      for (int i = 0; i < n_vecs; ++i)
        if (!vecs[i]) return fail(PHIKS_ERR_ARG, "null vector");
      for (int i = 0; i < nouts; ++i)
        if (!outs[i]) return fail(PHIKS_ERR_ARG, "null output");
    }
    if (h->sharded() && !h->peers_ready) return fail(PHIKS_ERR_ARG, "sharded handle: peers not opened");
    cs = static_cast<cudaStream_t>(stream);
    host_mem = req->mem_kind == PHIKS_MEM_HOST || req->mem_kind == PHIKS_MEM_HOST_ASYNC;
    host_async = req->mem_kind == PHIKS_MEM_HOST_ASYNC;
    N = h->N;
    tbytes = static_cast<size_t>(N) * sizeof(double);
    static const int split_mode = [] {
      // default 2: quadrature sums and squaring recurrences as a streaming pass
      // (measured faster on B200 than the fused epilogue); 0 = fused
      const char* e = getenv("PHIKS_SPLIT");
      return e ? atoi(e) : 2;
    }();
    split = split_mode;
    jb.mode = req->mode;
    jb.p = p;
    jb.n_scales = req->n_scales;
    jb.tau = req->tau;
    if (size_only) dv.assign(same ? 1 : req->n_ells, nullptr);
    else dv.assign(n_vecs > 0 ? n_vecs : 0, nullptr);
    dout.assign(nouts, nullptr);
    need_norms = !same && p >= 1 && req->force_s < 0 && !size_only;
    return PHIKS_OK;
  }

  // ---- lincomb plan input: ||v_ℓ||₂ (deterministic GPU reduction; sharded:
  // local sums of squares scattered to every rank, summed in rank order) ----
  phiks_status norms_enqueue(bool do_barrier) {
    if (!need_norms) return PHIKS_OK;
    std::vector<const double*> vv;
    for (int ell = 1; ell <= p; ++ell)
      for (int i = 0; i < req->n_ells; ++i)
        if (req->ells[i] == ell) which.push_back(i);
    if (which.empty()) return PHIKS_OK;
    const size_t sbytes = sizeof(double) * (1024 * kMaxVecs + kMaxVecs);
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&nscratch), sbytes, cs));
    for (size_t k = 0; k < which.size(); ++k) {
      if (host_mem) {
        double* t = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t), tbytes, cs));
        CUDA_TRY(cudaMemcpyAsync(t, vecs[which[k]], tbytes, cudaMemcpyHostToDevice, cs));
        ntmp.push_back(t);
        vv.push_back(t);
      } else {
        vv.push_back(vecs[which[k]]);
      }
    }
    CUDA_TRY(launch_sumsq(vv.data(), static_cast<int>(vv.size()), N, nscratch, nscratch + 1024 * kMaxVecs, cs));
    norm_launches = 2;
    if (h->sharded()) {
      norm_off = kCtrlNorms + (h->norm_phase++ & 1) * kCtrlNormsBuf;
      ScatterParams sp{};
      sp.rank = h->rank;
      sp.world = h->world;
      sp.cnt = static_cast<int>(which.size());
      sp.src = nscratch + 1024 * kMaxVecs;
      for (int k = 0; k < h->world; ++k) sp.dst[k] = reinterpret_cast<double*>(h->peer[k] + norm_off);
      CUDA_TRY(launch_scatter_small(sp, cs));
      ++norm_launches;
      if (do_barrier) {
        Arena a0;
        Exec eb{h, cs, false, &a0};
        eb.barrier();
        if (!eb.ok()) return eb.status;
        ++norm_launches;
      }
    }
    return PHIKS_OK;
  }
  // read back (synchronises the stream) and plan; `ctrl` = the control block
  // holding the gathered partial sums (sharded) — any rank's, they are equal
  phiks_status norms_finish(const char* ctrl) {
    std::vector<double> norms(p, 0.0);
    if (!which.empty()) {
      const int nv = static_cast<int>(which.size());
      const int W = h->sharded() ? h->world : 1;
      const double* srcp = h->sharded() ? reinterpret_cast<const double*>(ctrl + norm_off)
                                        : nscratch + 1024 * kMaxVecs;
      CUDA_TRY(cudaMemcpyAsync(h->h_pinned, srcp, sizeof(double) * nv * W, cudaMemcpyDeviceToHost, cs));
      for (double* t : ntmp) CUDA_TRY(cudaFreeAsync(t, cs));
      ntmp.clear();
      CUDA_TRY(cudaFreeAsync(nscratch, cs));
      nscratch = nullptr;
      CUDA_TRY(cudaStreamSynchronize(cs));
      for (int k = 0; k < nv; ++k) {
        double s2 = 0.0;
        for (int r = 0; r < W; ++r) s2 += h->h_pinned[r * nv + k];
        norms[req->ells[which[k]] - 1] = std::sqrt(s2);
      }
    }
    return make_plan(h, req, p, norms, pl);
  }

  phiks_status plan_direct(const phiks_plan_info* forced) {
    if (forced) {
      pl.s = forced->s;
      pl.q = forced->q;
      pl.ok = true;
      return PHIKS_OK;
    }
    if (!same && p >= 1 && req->force_s < 0 && size_only) return fail(PHIKS_ERR_ARG, "lincomb sizing needs a plan");
    std::vector<double> norms;
    return make_plan(h, req, p, norms, pl);
  }

  void bind(bool measure) {
    ar.off = 0;
    ar.measure = measure;
    ex.measure = measure;
    // user buffers: host memory -> device staging in the workspace; sizing
    // without pointers -> distinct fake addresses (never dereferenced)
    auto fake = [](int k) { return reinterpret_cast<double*>(static_cast<uintptr_t>(0x7f0000000000ULL) + 4096ULL * k); };
    for (int i = 0; i < static_cast<int>(dv.size()); ++i)
      dv[i] = host_mem ? ar.alloc_doubles(N) : (size_only ? fake(i) : const_cast<double*>(vecs[i]));
    for (int i = 0; i < nouts; ++i) dout[i] = host_mem ? ar.alloc_doubles(N) : (size_only ? fake(64 + i) : outs[i]);
    for (int i = 0; i < kMaxVecs; ++i) jb.vin[i] = nullptr;
    if (same) {
      jb.vin[0] = dv.empty() ? nullptr : dv[0];
      for (int j = 0; j < req->n_scales; ++j)
        for (int i = 0; i < req->n_ells; ++i) jb.out_same[req->ells[i]][j] = dout[j * req->n_ells + i];
    } else {
      for (int i = 0; i < req->n_ells; ++i) jb.vin[req->ells[i]] = dv.empty() ? nullptr : dv[i];
      for (int j = 0; j < req->n_scales; ++j) jb.out_lin[j] = dout[j];
    }
  }

  phiks_status measure(size_t* need) {
    jb.s = pl.s;
    jb.q = pl.q;
    ex = Exec{h, cs, true, &ar};
    ex.split = split;
    bind(true);
    run_job(ex, jb);
    if (!ex.ok()) return ex.status;
    *need = ar.off;
    return PHIKS_OK;
  }

  bool own_ws = false;
  phiks_status workspace(void* workspace, size_t ws_bytes, size_t need, char** base) {
    own_ws = workspace == nullptr;
    if (workspace) {
      if (ws_bytes < need) {
        h->stats.workspace_bytes = need;
        return fail(PHIKS_ERR_WORKSPACE, "workspace too small");
      }
      *base = static_cast<char*>(workspace);
      return PHIKS_OK;
    }
    if (h->ws_own_bytes < need) {
      for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);  // they reference the old workspace
      h->graphs.clear();
      if (h->ws_own) {
        CUDA_TRY(cudaStreamSynchronize(cs));
        CUDA_TRY(cudaFree(h->ws_own));
        h->ws_own = nullptr;
        h->ws_own_bytes = 0;
      }
      if (cudaMalloc(&h->ws_own, need > 0 ? need : 256) != cudaSuccess)
        return fail(PHIKS_ERR_NOMEM, "workspace cudaMalloc");
      h->ws_own_bytes = need > 0 ? need : 256;
    }
    *base = static_cast<char*>(h->ws_own);
    return PHIKS_OK;
  }

  // enqueue (rec == nullptr) or record the whole job on the bound workspace
  phiks_status execute(char* base, size_t need, std::vector<Exec::Op>* rec) {
    ar.base = base;
    ar.cap = need;
    ex = Exec{h, cs, false, &ar};
    ex.split = split;
    ex.rec = rec;
    bind(false);
    if (host_mem && rec) return fail(PHIKS_ERR_ARG, "recorded applies take device memory");
    // (never recorded yet: waiting on it is a no-op)
    if (!h->ev_cdone) CUDA_TRY(cudaEventCreateWithFlags(&h->ev_cdone, cudaEventDisableTiming));
    // stage A on the handle's pre stream: only with the library's own workspace
    // (a caller workspace may be in use on the stream until this apply starts),
    // not while capturing a graph, not for recorded (emulated-rank) applies
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(cs, &cap));
    const bool pre = !rec && own_ws && cap == cudaStreamCaptureStatusNone;
    if (pre) {
      if (!h->s_pre) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->s_pre, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&h->ev_pre, cudaEventDisableTiming));
      }
      CUDA_TRY(cudaStreamWaitEvent(h->s_pre, h->ev_cdone, 0));  // previous apply no longer reads the workspace
      ex.st = h->s_pre;
    }
    ex.on_inputs = [this, pre]() {
      if (pre) {
        ex.check(cudaEventRecord(h->ev_pre, h->s_pre), "record pre");
        ex.st = cs;
        ex.check(cudaStreamWaitEvent(cs, h->ev_pre, 0), "wait pre");
      }
      if (host_mem) ex.check(cudaStreamWaitEvent(cs, h->ev_h2d, 0), "wait h2d");
    };
    if (host_mem) {
      // copies on the handle's own streams: H2D overlaps stage A, the copy-out of
      // an output overlaps the rest of the job (and the next apply)
      if (!h->s_in) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&h->ev_h2d, &h->ev_d2h, &h->ev_ready})
          CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(h->ev_d2h, h->s_out));
      }
      CUDA_TRY(cudaStreamWaitEvent(h->s_in, h->ev_cdone, 0));  // previous apply is done with the staging
      for (size_t i = 0; i < dv.size(); ++i)
        CUDA_TRY(cudaMemcpyAsync(dv[i], vecs[i], tbytes, cudaMemcpyHostToDevice, h->s_in));
      CUDA_TRY(cudaEventRecord(h->ev_h2d, h->s_in));
      CUDA_TRY(cudaStreamWaitEvent(cs, h->ev_d2h, 0));  // previous apply's copy-out has drained
      copied.assign(nouts, false);
      ex.on_outputs = [this](const std::vector<double*>& ready) { copy_out(ready); };
    }
    run_job(ex, jb);
    ex.st = cs;
    if (!ex.ok()) return ex.status;
    if (host_mem) {
      std::vector<double*> rest;
      for (int i = 0; i < nouts; ++i)
        if (!copied[i]) rest.push_back(dout[i]);
      copy_out(rest);
      if (!ex.ok()) return ex.status;
      CUDA_TRY(cudaEventRecord(h->ev_d2h, h->s_out));
    }
    if (!rec && cap == cudaStreamCaptureStatusNone) CUDA_TRY(cudaEventRecord(h->ev_cdone, cs));
    return PHIKS_OK;
  }
  std::vector<bool> copied;
  void copy_out(const std::vector<double*>& ready) {
    if (ready.empty()) return;
    ex.check(cudaEventRecord(h->ev_ready, cs), "record ready");
    ex.check(cudaStreamWaitEvent(h->s_out, h->ev_ready, 0), "wait ready");
    for (double* p : ready)
      for (int i = 0; i < nouts; ++i)
        if (dout[i] == p && !copied[i]) {
          ex.check(cudaMemcpyAsync(outs[i], dout[i], tbytes, cudaMemcpyDeviceToHost, h->s_out), "d2h");
          copied[i] = true;
        }
  }

  void finish_stats(size_t need) {
    phiks_stats& S = h->stats;
    S.plan.s = pl.s;
    S.plan.q = pl.q;
    S.plan.T_formula = plan::tucker_count(req->mode, pl.s, req->n_scales, pl.q, p);
    S.plan.T_executed = static_cast<int>(ex.tucker_ops);
    S.kernel_launches = ex.launches + norm_launches;
    S.tucker_ops = ex.tucker_ops;
    S.mu_mode_flops = ex.mu_flops;
    S.expm_flops = ex.expm_flops;
    S.workspace_bytes = need;
    S.total_kernel_launches += S.kernel_launches;
  }
};

// error flag of the cross-rank barrier (sticky; read with a synchronous copy)
phiks_status check_barrier_flag(phiks_handle h) {
  if (!h->sharded() || !h->sym) return PHIKS_OK;
  int err = 0;
  CUDA_TRY(cudaMemcpy(&err, h->sym + kCtrlErr, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) return fail(PHIKS_ERR_CUDA, "cross-rank barrier timed out (a peer rank did not arrive)");
  return PHIKS_OK;
}

static phiks_status apply_impl(phiks_handle h, const phiks_request* req, int n_vecs, const double* const* vecs,
                               double* const* outs, void* workspace, size_t ws_bytes, void* stream,
                               bool size_only, const phiks_plan_info* forced, size_t* size_out) {
  static const bool hostprof = getenv("PHIKS_HOSTPROF") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
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
  const auto t1 = now();
  size_t need = 0;
  st = run.measure(&need);
  if (st != PHIKS_OK) return st;
  const auto t2 = now();
  struct HostProf {
    bool on;
    std::chrono::steady_clock::time_point t0, t1, t2;
    ~HostProf() {
      if (!on) return;
      const auto t3 = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      fprintf(stderr, "PHIKS_HOSTPROF plan+norms %.1f us, measure %.1f us, enqueue %.1f us\n", us(t0, t1), us(t1, t2),
              us(t2, t3));
    }
  } hostprof_guard{hostprof, t0, t1, t2};
  if (size_out) *size_out = need;
  if (size_only) return PHIKS_OK;
  char* base = nullptr;
  st = run.workspace(workspace, ws_bytes, need, &base);
  if (st != PHIKS_OK) return st;
  static const bool graphs_on = [] {
    const char* e = getenv("PHIKS_GRAPHS");
    return !(e && atoi(e) == 0);
  }();
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
                           bits(req->tol), static_cast<uint64_t>(run.pl.s), static_cast<uint64_t>(run.pl.q),
                           static_cast<uint64_t>(run.split), reinterpret_cast<uint64_t>(base), need});
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
    if (!h->ev_cdone) CUDA_TRY(cudaEventCreateWithFlags(&h->ev_cdone, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(h->ev_cdone, cs));  // orders the next apply's stage A after this replay
    run.finish_stats(need);
    return PHIKS_OK;
  }
  st = run.execute(base, need, nullptr);
  if (st != PHIKS_OK) return st;
  if (run.host_mem && !run.host_async) {
    CUDA_TRY(cudaEventSynchronize(h->ev_d2h));
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
  if (h->profiling) {
    for (int i = 0; i < h->ev_used; ++i) {
      CUDA_TRY(cudaEventSynchronize(h->ev[i].second));
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, h->ev[i].first, h->ev[i].second));
      if (h->ev_expm[i]) {
        out->expm_ms += ms;
        ++out->expm_launches;
      } else {
        out->mode_product_ms += ms;
        out->mode_product_flops += h->ev_flops[i];
        ++out->mode_product_launches;
      }
    }
  }
  return PHIKS_OK;
}

phiks_status phiks_set_profiling(phiks_handle h, int on) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  h->profiling = on != 0;
  h->ev_used = 0;
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
    h.fac_of_mode[mu] = mu;
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


// ===========================================================================
// Slab sharding across the GPUs of one box
// ===========================================================================
phiks_status phiks_create_sharded(int d, const int* n, const double* const* A_host, int rank, int world,
                                  phiks_handle* out) {
  if (!out || !n) return fail(PHIKS_ERR_ARG, "null argument");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return fail(PHIKS_ERR_ARG, "rank/world");
  if (world > 1) {
    if (d < 2) return fail(PHIKS_ERR_ARG, "sharding needs d >= 2");
    if (n[d - 1] % world != 0 || n[d - 2] % world != 0)
      return fail(PHIKS_ERR_ARG, "n_d and n_{d-1} must be divisible by world");
  }
  phiks_handle h = nullptr;
  phiks_status st = phiks_create(d, n, A_host, &h);
  if (st != PHIKS_OK) return st;
  h->rank = rank;
  h->world = world;
  if (world > 1) {
    h->n[d - 1] = n[d - 1] / world;
    h->N /= world;
    h->Nc /= world;
    h->sym_slot = (static_cast<size_t>(h->N) * sizeof(double) + 255) & ~size_t(255);
    h->sym_bytes = kCtrlBytes + 2 * kShardChunk * h->sym_slot;
    if (cudaMalloc(reinterpret_cast<void**>(&h->sym), h->sym_bytes) != cudaSuccess) {
      phiks_destroy(h);
      return fail(PHIKS_ERR_NOMEM, "symmetric region cudaMalloc");
    }
    if (cudaMemset(h->sym, 0, kCtrlBytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      phiks_destroy(h);
      return fail(PHIKS_ERR_CUDA, "symmetric region init");
    }
    h->peer[rank] = h->sym;
  } else {
    h->peers_ready = true;
  }
  *out = h;
  return PHIKS_OK;
}

phiks_status phiks_shard_info(phiks_handle h, int* rank, int* world, int64_t* local_count, size_t* sym_bytes) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  if (rank) *rank = h->rank;
  if (world) *world = h->world;
  if (local_count) *local_count = h->N;
  if (sym_bytes) *sym_bytes = h->sym_bytes;
  return PHIKS_OK;
}

phiks_status phiks_shard_ipc_handle(phiks_handle h, void* handle_out) {
  if (!h || !handle_out) return fail(PHIKS_ERR_ARG, "null argument");
  std::memset(handle_out, 0, PHIKS_IPC_HANDLE_BYTES);
  if (!h->sharded()) return PHIKS_OK;
  static_assert(sizeof(cudaIpcMemHandle_t) <= PHIKS_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t ih;
  CUDA_TRY(cudaIpcGetMemHandle(&ih, h->sym));
  std::memcpy(handle_out, &ih, sizeof(ih));
  return PHIKS_OK;
}

phiks_status phiks_shard_open_peers(phiks_handle h, const void* handles) {
  if (!h || !handles) return fail(PHIKS_ERR_ARG, "null argument");
  if (!h->sharded()) {
    h->peers_ready = true;
    return PHIKS_OK;
  }
  const char* hb = static_cast<const char*>(handles);
  for (int k = 0; k < h->world; ++k) {
    if (k == h->rank) continue;
    if (h->peer_ipc[k] && h->peer[k]) {
      cudaIpcCloseMemHandle(h->peer[k]);
      h->peer[k] = nullptr;
      h->peer_ipc[k] = false;
    }
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, hb + static_cast<size_t>(k) * PHIKS_IPC_HANDLE_BYTES, sizeof(ih));
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
    h->peer[k] = static_cast<char*>(ptr);
    h->peer_ipc[k] = true;
  }
  h->peers_ready = true;
  return PHIKS_OK;
}

phiks_status phiks_shard_base(phiks_handle h, void** base) {
  if (!h || !base) return fail(PHIKS_ERR_ARG, "null argument");
  *base = h->sym;
  return PHIKS_OK;
}

phiks_status phiks_shard_set_peer_bases(phiks_handle h, void* const* bases) {
  if (!h || !bases) return fail(PHIKS_ERR_ARG, "null argument");
  if (!h->sharded()) {
    h->peers_ready = true;
    return PHIKS_OK;
  }
  if (bases[h->rank] != h->sym) return fail(PHIKS_ERR_ARG, "bases[rank] must be this handle's region");
  for (int k = 0; k < h->world; ++k) {
    if (!bases[k]) return fail(PHIKS_ERR_ARG, "null peer base");
    h->peer[k] = static_cast<char*>(bases[k]);
  }
  h->peers_ready = true;
  return PHIKS_OK;
}

phiks_status phiks_apply_ranks_serial(const phiks_handle* hs, int world, const phiks_request* req, int n_vecs,
                                      const double* const* vecs, double* const* outs, void* stream) {
  if (!hs || world < 1 || world > kMaxRanks || !req || !vecs || !outs) return fail(PHIKS_ERR_ARG, "bad argument");
  for (int k = 0; k < world; ++k) {
    if (!hs[k] || hs[k]->world != world || hs[k]->rank != k) return fail(PHIKS_ERR_ARG, "hs[k] must be rank k of world");
    if (req->mem_kind != PHIKS_MEM_DEVICE) return fail(PHIKS_ERR_ARG, "ranks_serial takes device memory");
  }
  const bool same = req->mode == PHIKS_MODE_SAME_VECTOR;
  const int nouts = same ? req->n_ells * req->n_scales : req->n_scales;
  std::vector<ApplyRun> runs(world);
  for (int k = 0; k < world; ++k) {
    phiks_status st = runs[k].init(hs[k], req, n_vecs, vecs + static_cast<size_t>(k) * n_vecs,
                                   outs + static_cast<size_t>(k) * nouts, stream, false);
    if (st != PHIKS_OK) return st;
  }
  // plan: norms phase of every rank (no barrier: stream order), then read
  if (runs[0].need_norms) {
    for (int k = 0; k < world; ++k) {
      phiks_status st = runs[k].norms_enqueue(false);
      if (st != PHIKS_OK) return st;
    }
    for (int k = 0; k < world; ++k) {
      phiks_status st = runs[k].norms_finish(hs[0]->sym);
      if (st != PHIKS_OK) return st;
    }
  } else {
    for (int k = 0; k < world; ++k) {
      phiks_status st = runs[k].plan_direct(nullptr);
      if (st != PHIKS_OK) return st;
    }
  }
  std::vector<std::vector<Exec::Op>> ops(world);
  std::vector<size_t> need(world, 0);
  for (int k = 0; k < world; ++k) {
    phiks_status st = runs[k].measure(&need[k]);
    if (st != PHIKS_OK) return st;
    char* base = nullptr;
    st = runs[k].workspace(nullptr, 0, need[k], &base);
    if (st != PHIKS_OK) return st;
    st = runs[k].execute(base, need[k], &ops[k]);
    if (st != PHIKS_OK) return st;
  }
  // replay phase by phase: the segment between two barriers of every rank
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  std::vector<size_t> pos(world, 0);
  bool more = true;
  while (more) {
    more = false;
    for (int k = 0; k < world; ++k) {
      auto& v = ops[k];
      while (pos[k] < v.size() && !v[pos[k]].barrier) {
        cudaError_t e = v[pos[k]].fn(cs);
        if (e != cudaSuccess) return fail(PHIKS_ERR_CUDA, std::string(v[pos[k]].what) + ": " + cudaGetErrorString(e));
        ++pos[k];
      }
      if (pos[k] < v.size()) {
        ++pos[k];  // the barrier itself: implied by stream order
        more = true;
      }
    }
  }
  for (int k = 0; k < world; ++k) runs[k].finish_stats(need[k]);
  return PHIKS_OK;
}


phiks_status phiks_shard_layout(int d, const int* n, int rank, int world, int stage, int64_t* out7) {
  if (!n || !out7 || d < 2 || d > PHIKS_MAX_D || world < 1 || world > kMaxRanks || rank < 0 || rank >= world ||
      (stage != 0 && stage != 1))
    return fail(PHIKS_ERR_ARG, "bad argument");
  if (n[d - 1] % world != 0 || n[d - 2] % world != 0) return fail(PHIKS_ERR_ARG, "dims not divisible by world");
  const ShardStage s = shard_stage(d, n, rank, world, stage);
  const int64_t v[7] = {s.L, s.n, s.R, s.cb, s.rstride, s.roff, s.colstride};
  for (int i = 0; i < 7; ++i) out7[i] = v[i];
  return PHIKS_OK;
}


phiks_status phiks_wait(phiks_handle h) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  if (h->ev_d2h) CUDA_TRY(cudaEventSynchronize(h->ev_d2h));
  if (h->ev_cdone) CUDA_TRY(cudaEventSynchronize(h->ev_cdone));
  return check_barrier_flag(h);
}


phiks_status phiks_shard_peer_base(phiks_handle h, int k, void** base) {
  if (!h || !base || k < 0 || k >= h->world) return fail(PHIKS_ERR_ARG, "bad argument");
  *base = h->peer[k];
  return PHIKS_OK;
}

}  // extern "C"
