// Host orchestration of the PHIKS hot path, shared by the C-ABI translation
// units (phiks_api.cpp: create/plan/apply; orchestrate.cpp: the job of one
// apply as launches; phiks_shard.cpp: the slab-sharded handle).  Not part of
// the C ABI.
//
// The host only plans and enqueues: every arithmetic step on tensors or
// matrices runs in the CUDA kernels of kernels.cu.  One apply is
//   A. small-matrix exponentials exp(c·τA_f) for the GLL nodes (Taylor degree
//      16, Paterson–Stockmeyer, scaling and squaring) and the level matrices
//      exp(τA_f/2^j) by repeated squaring,
//   B. quadrature: one batched Tucker operator per node (Eq. (10)),
//      weight-sum (Eq. (11) / Eq. (17)) in the last mode's epilogue or a
//      streaming combination,
//   C. squaring levels j = s..1 (Eq. (12) / Eq. (18)), intermediate scales
//      written on the way (Eq. (13)/(19)),
//   D. exp(τK/2^j)v actions (one Tucker operator each, l.614-616).
#pragma once
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "phiks_internal.h"
#include "planner.h"


namespace phiks {
namespace host {

extern thread_local std::string g_err;

inline phiks_status fail(phiks_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(PHIKS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline double factorial(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}

struct Factor {
  int n = 0;
  double* dA = nullptr;   // device copy of A_f
  double norm1 = 0.0;    // ||A_f||_1
  bool metzler = false;  // real factor with every off-diagonal entry ≥ 0 (chain guard, R15)
  plan::FactorRange fr{};
};

struct PlanKey {
  int mode, p, n_scales;
  double tau, tol;
  std::vector<double> norms;
  int block;
  bool operator<(const PlanKey& o) const {
    return std::tie(mode, p, n_scales, tau, tol, norms, block) <
           std::tie(o.mode, o.p, o.n_scales, o.tau, o.tol, o.norms, o.block);
  }
};
}  // namespace host
}  // namespace phiks

using namespace phiks;
using namespace phiks::host;

struct phiks_ctx {
  int d = 0;
  int n[PHIKS_MAX_D] = {0};
  int64_t N = 0;   // doubles per tensor (2·Nc for complex handles)
  int64_t Nc = 0;  // elements per tensor
  bool cplx = false;  // complex factors and tensors (interleaved re, im)
  std::vector<Factor> factors;
  // block-diagonal K̂ = diag(K_1, …, K_nb) (§4.4): every block has
  // the dims n[] and its own factors; fac_of_block[b][μ] indexes `factors`
  int nblocks = 1;
  int fac_of_block[kMaxBlocks][PHIKS_MAX_D] = {{0}};
  void* ws_own = nullptr;
  size_t ws_own_bytes = 0;
  double* h_pinned = nullptr;  // pinned host scratch (norms)
  int* h_barrier_err = nullptr;  // pinned copy of the sharded barrier's sticky error flag (lagging check)
  std::map<PlanKey, plan::Plan> plan_cache;
  phiks_stats stats{};
  // profiling: event pairs around μ-mode-product launches of the last apply
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<double> ev_flops;
  std::vector<char> ev_expm;  // 1: small-GEMM launch of the exponential stage; 2: int8 (§4c) GEMM, 3: its digit splits
  // μ-mode-product path of the Tucker launches (phiks_set_gemm_path)
  int gemm_path = PHIKS_GEMM_AUTO;
  // execution options (phiks_set_option)
  int opt_split = 2;   // PHIKS_OPT_SPLIT
  int opt_chain = 1;   // PHIKS_OPT_CHAIN: 0 off, 1 guarded (Metzler factors), 2 forced
  int opt_graphs = 1;  // PHIKS_OPT_GRAPHS
  int opt_presplit = 1;  // PHIKS_OPT_PRESPLIT
  int opt_kskip = 1;     // PHIKS_OPT_KSKIP
  bool chain_safe() const {  // every factor Metzler: exponentials entrywise ≥ 0 (τ > 0)
    for (const auto& F : factors)
      if (!F.metzler) return false;
    return !factors.empty();
  }
  int ev_used = 0;
  unsigned long long* d_kcount = nullptr;  // profiling: the int8 GEMM's k-block counters (OzakiParams::kcount)
  // ---- slab sharding along the outermost mode (phiks_create_sharded) ----
  // n[] holds the LOCAL dims of layout S_d (n[d-1] = gn[d-1]/world); the
  // transposed layout S_{d-1} has dims (n_1..n_{d-2}, gn[d-2]/world, gn[d-1]).
  int rank = 0, world = 1;
  int gn[PHIKS_MAX_D] = {0};
  char* sym = nullptr;  // own symmetric region: control block + T/Y pools
  size_t sym_bytes = 0;
  size_t sym_slot = 0;  // bytes per pooled local tensor
  size_t exch_off = 0;  // exponent exchange buffer of the sharded digit stages ([world][16][L0] doubles)
  int64_t exch_l0 = 0;  // L0 = n_1⋯n_{d-2} it holds
  size_t xpool_off = 0, xpool_half = 0;  // sharded exponential stage: all-gathered matrices, two halves
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
  // the library-owned workspace is two halves used by alternate applies
  // (ws_parity): an apply's stage A and host copies may run ahead of the previous
  // apply, ordered only after the apply before it (same half): ev_cdone[half]
  // = compute done, ev_d2h[half] = copy-out done
  int ws_parity = 0;
  cudaEvent_t ev_h2d = nullptr, ev_ready = nullptr;
  cudaEvent_t ev_d2h[2] = {nullptr, nullptr}, ev_cdone[2] = {nullptr, nullptr};
  // the exponential stage (stage A) of an apply runs on s_pre, ordered only
  // after the previous apply of this handle (ev_cdone), so it overlaps the
  // tail of whatever else is queued on the apply stream (another handle's
  // Tucker work); the stream waits on ev_pre before the first Tucker batch
  cudaStream_t s_pre = nullptr;
  cudaEvent_t ev_pre = nullptr;
  bool sharded() const { return world > 1; }
};


namespace phiks {
namespace host {

// symmetric region layout (identical on every rank)
constexpr size_t kCtrlFlags = 0;                                   // uint64 flags[kMaxRanks]
constexpr size_t kCtrlErr = kMaxRanks * sizeof(uint64_t);          // int err
constexpr size_t kCtrlEpoch = 128;                                 // uint64 barrier count
constexpr size_t kCtrlNorms = 256;                                 // double norms[2][kMaxRanks][kMaxVecs]
constexpr size_t kCtrlNormsBuf = kMaxRanks * kMaxBlocks * kMaxVecs * sizeof(double);
constexpr size_t kCtrlFlags2 = kCtrlNorms + 2 * kCtrlNormsBuf;       // uint64 flags[kMaxRanks], barrier channel 1
constexpr size_t kCtrlEpoch2 = kCtrlFlags2 + kMaxRanks * sizeof(uint64_t);  // uint64 channel-1 barrier count
constexpr size_t kCtrlBytes = 4096;
static_assert(kCtrlEpoch2 + 8 <= kCtrlBytes, "control block layout");
static_assert(kCtrlErr + sizeof(int) <= kCtrlEpoch && kCtrlEpoch + 8 <= kCtrlNorms, "control block layout");
constexpr int kShardChunk = kShardChunkMax;  // Tucker operators per sharded sub-batch (T and Y pools)
constexpr uint64_t kBarrierTimeoutNs = 60ull * 1000 * 1000 * 1000;


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

// Block distribution of n indices over P ranks: the first n mod P ranks own
// one more.  Used for the slabs of mode d (layout S_d) and of mode d-1 (S_{d-1}).
inline int64_t blk_cnt(int64_t n, int P, int k) { return n / P + (k < n % P ? 1 : 0); }
inline int64_t blk_start(int64_t n, int P, int k) { return k * (n / P) + std::min<int64_t>(k, n % P); }

// Geometry of the two peer-store launches of a slab-sharded Tucker operator
// (DESIGN.md §0(e)).  gn: global dims.  stage 0: the mode-(d-1) product on the
// slab (layout S_d, dims (n_1..n_{d-2}, n_{d-1}, cd_r)) storing into layout
// S_{d-1} (dims (n_1..n_{d-2}, cb_k, n_d)) of the owner k of each output column;
// stage 1: the mode-d product on layout S_{d-1} storing back into S_d.  Element
// (l, j, r) of the (L, n, R) launch goes to rank k = owner(j) (block
// distribution of the n columns) at offset
//   l + kstride[k]·r + kroff[k] + colstride·(j − kstart[k]).
struct ShardStage {
  int64_t L, n, R, colstride;
  int world;
  int64_t kstart[kMaxRanks], kstride[kMaxRanks], kroff[kMaxRanks];
  bool uniform;
};
inline ShardStage shard_stage(int d, const int* gn, int rank, int world, int stage) {
  int64_t L0 = 1;
  for (int mu = 0; mu + 2 < d; ++mu) L0 *= gn[mu];
  const int64_t na = gn[d - 2], nd = gn[d - 1];
  ShardStage s{};
  s.world = world;
  s.uniform = (na % world == 0) && (nd % world == 0);
  if (stage == 0) {
    s.L = L0;
    s.n = na;
    s.R = blk_cnt(nd, world, rank);
    s.colstride = L0;
    for (int k = 0; k < world; ++k) {
      const int64_t cbk = blk_cnt(na, world, k);
      s.kstart[k] = blk_start(na, world, k);
      s.kstride[k] = L0 * cbk;
      s.kroff[k] = L0 * cbk * blk_start(nd, world, rank);
    }
  } else {
    s.L = L0 * blk_cnt(na, world, rank);
    s.n = nd;
    s.R = 1;
    s.colstride = L0 * na;
    for (int k = 0; k < world; ++k) {
      s.kstart[k] = blk_start(nd, world, k);
      s.kstride[k] = 0;
      s.kroff[k] = L0 * blk_start(na, world, rank);
    }
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
  int half = 0;                      // workspace half of the apply (sharded: the expm pool half too)
  double mu_flops = 0.0, expm_flops = 0.0;
  phiks_status status = PHIKS_OK;
  int64_t barriers = 0;

  // Recorded ops: with `rec` set, launches are appended instead of issued (the
  // phase-interleaved emulation of several ranks on one GPU replays them).
  struct Op {
    bool barrier;
    std::function<cudaError_t(cudaStream_t)> fn;
    const char* what;
    bool pre = false;  // stage A (exponentials, before on_inputs): the part a real apply runs on s_pre
  };
  bool stage_a = true;  // until on_inputs: the recorded ops belong to stage A
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
      rec->push_back(Op{false, std::move(fn), what, stage_a});
    else
      check(fn(st), what);
  }
  // cross-rank barrier of a sharded handle (device-side, stream-ordered)
  // channel 1: the exponential stage's all-gather, which runs on the handle's pre stream
  // concurrently with the previous apply's tail on the compute stream (its own flags and count,
  // so the two streams' barriers never pair up across ranks)
  void barrier(int channel = 0) {
    ++barriers;
    if (!ok() || !h->sharded()) return;
    ++launches;
    if (measure) return;
    if (rec) {
      rec->push_back(Op{true, nullptr, "barrier", stage_a});
      return;
    }
    BarrierParams bp{};
    bp.rank = h->rank;
    bp.world = h->world;
    bp.epoch = reinterpret_cast<uint64_t*>(h->sym + (channel ? kCtrlEpoch2 : kCtrlEpoch));
    bp.timeout_ns = kBarrierTimeoutNs;
    for (int k = 0; k < h->world; ++k)
      bp.peer_flags[k] = reinterpret_cast<uint64_t*>(h->peer[k] + (channel ? kCtrlFlags2 : kCtrlFlags));
    bp.err = reinterpret_cast<int*>(h->sym + kCtrlErr);
    check(launch_barrier(bp, st), "barrier");
  }

  // ---- int8 tensor-core route of plain mode products (ozaki.cu) ----
  int64_t i8_launches = 0;
  int64_t i8_chained = 0;  // Tucker operators run as chained int8 modes
  int64_t shard_digit_ops = 0;  // sharded: Tucker operators whose stage 0 wrote digit planes to the owners
  double* oz_ws = nullptr;  // grown on demand, reused by every int8 launch of the apply (one stream)
  size_t oz_ws_bytes = 0;
  static constexpr int kOzDigits = 7;
  template <class Terms>
  bool ozaki_route(int64_t L, int n, int64_t R, const Terms& terms, const Remap* rm) const {
    // slab-sharded handles (local modes and the two peer-store stages) take it too; complex
    // handles and the exponential stage's small GEMMs stay on DMMA
    if (in_expm || h->gemm_path == PHIKS_GEMM_DMMA) return false;
    if (rm && rm->world > kMaxRanks) return false;
    if (!ozaki_supported(L, n, R, kOzDigits)) return false;
    for (const auto& t : terms)
      if (t.kcat && (2 * n > kOzMaxN || !terms[0].kcat)) return false;
    // auto: where it measured faster (configs[2], n = 128: int8 chained 0.93 ms vs DMMA 0.99 ms per
    // apply; below n = 128 or 2^20 elements the launches are too small for the digit splits to pay)
    if (h->gemm_path == PHIKS_GEMM_AUTO && (n < 128 || L * R * n < (int64_t(1) << 20))) return false;
    std::set<int> groups;
    for (const auto& t : terms) {
      if (t.cswap || t.outs.size() != 1 || !t.outs[0].srcs.empty()) return false;
      if (!groups.insert(t.group).second) return false;
    }
    return true;
  }
  template <class Terms>
  void ozaki_launch(int64_t L, int n, int64_t R, const Terms& terms, const Remap* rm = nullptr) {
    constexpr int kChunkX = 8;  // distinct inputs split per launch (bounds the digit workspace)
    size_t i = 0;
    while (i < terms.size() && ok()) {
      auto pp = std::make_shared<OzakiParams>();
      OzakiParams& p = *pp;
      std::memset(&p, 0, sizeof(p));
      p.L = L;
      p.R = R;
      p.n = n;
      p.S = kOzDigits;
      p.kskip = h->opt_kskip;
      p.kcount = h->profiling ? h->d_kcount : nullptr;
      if (rm) p.remap = *rm;
      p.cplx_j = terms[i].kcat ? 1 : 0;
      size_t j = i;
      for (; j < terms.size() && p.nterms < kMaxTerms; ++j) {
        int xs = -1, es = -1;
        for (int k = 0; k < p.nx; ++k)
          if (p.x[k] == terms[j].in) xs = k;
        for (int k = 0; k < p.ne; ++k)
          if (p.e[k] == terms[j].M) es = k;
        if ((xs < 0 && p.nx == kChunkX) || (es < 0 && p.ne == kMaxTerms)) break;
        if (xs < 0) {
          xs = p.nx;
          p.x[p.nx++] = terms[j].in;
        }
        if (es < 0) {
          es = p.ne;
          p.e[p.ne++] = terms[j].M;
        }
        p.terms[p.nterms++] = OzakiTerm{xs, es, terms[j].outs[0].dst, terms[j].outs[0].beta};
      }
      const size_t need = ozaki_workspace_bytes(L, n, R, p.S, p.nx, p.ne, p.cplx_j ? 2 * n : n);
      if (need > oz_ws_bytes) {
        oz_ws = ar->alloc_doubles(static_cast<int64_t>((need + 7) / 8));
        oz_ws_bytes = need;
      }
      ozaki_bind_workspace(p, oz_ws);
      oz_emit(pp, true);
      i = j;
    }
  }
  void oz_ws_reserve(size_t need) {
    if (need > oz_ws_bytes) {
      oz_ws = ar->alloc_doubles(static_cast<int64_t>((need + 7) / 8));
      oz_ws_bytes = need;
    }
  }
  // digit splits (+ chain exponents), then the GEMM (separate event pairs: kind 3 splits, kind 2 GEMM)
  // mid: enqueued between the splits and the GEMM (the sharded stage-0 exponent exchange)
  void oz_emit(const std::shared_ptr<OzakiParams>& pp, bool split_x, const std::function<void()>& mid = nullptr);

  // ---- chained int8 Tucker operators ----
  // Every mode of the batch on the int8 path with no fp64 intermediate: the product
  // of mode μ < d writes the digits of mode μ+1 (fp64 layout, MN-major A operand of
  // the next GEMM) with fiber exponents bounded before the product (oz_chain_kernel).
  int8_t* oz_dig[2] = {nullptr, nullptr};
  double* oz_ex[2] = {nullptr, nullptr};
  double* oz_mx = nullptr;  // Mx of the current product (read by its own epilogue only)
  size_t oz_chain_cap = 0;  // Tucker operators the buffers hold
  // modes 0..mlast of the batch chained (mlast = d − 1: whole operators; sharded handles stop at
  // the mode-(d−1) stage, whose epilogue stores into the owner ranks)
  bool ozaki_chain_route(const std::vector<TuckerItem>& items, size_t c0, size_t c1, int mlast = -1) const;
  size_t chain_cap() const {  // digit buffers 2·cap·S·N bytes, at most ~8 GB
    const double per = 2.0 * kOzDigits * static_cast<double>(h->N);
    return static_cast<size_t>(std::max(1.0, std::min(24.0, std::floor(8e9 / per))));
  }
  // last mode mlast writes fp64: the items' outputs (mlast = d − 1), or with rm set the
  // sharded stage-0 peer stores into symmetric-region offset kCtrlBytes + b·sym_slot
  // With rm1 set (slab-sharded digit stages, shard_digits_ok): mode d−2 is stage 0, whose epilogue
  // writes mode d's digit planes into the owners' T pools (rm: its peer-store geometry) after the
  // cross-rank exponent exchange, then a barrier, and mode d−1 is stage 1 on the transposed slab,
  // reading those planes and storing fp64 into the owners' Y pools (rm1)
  void tucker_chain_i8(const std::vector<TuckerItem>& items, size_t c0, size_t c1, int mlast = -1,
                       const Remap* rm = nullptr, const Remap* rm1 = nullptr);

  // ---- one mode-product launch from host-side term lists ----
  struct LaunchTerm {
    const double* in;
    const double* M;
    int group;
    std::vector<Out> outs;
    int cswap = 0;  // complex: J applied to the accumulator (TermSpec::cswap)
    int kcat = 0;   // complex μ ≥ 2 on the int8 path: M = [Re | Im] (n × 2n), fibres [x ; Jx]
  };
  void mode_launch(int64_t L, int n, int64_t R, const std::vector<LaunchTerm>& terms, const Remap* rm = nullptr);

  void combine(int64_t count, const std::vector<Out>& outs);

  // ---- matrix-form combination dst_o = Σ_s coef[o][s] src_s ----
  // dslot[o] ≥ 0: output o also written as mode-1 digit planes into slot dslot[o] of pre_xs
  void mcombine(int64_t count, const std::vector<const double*>& srcs, const std::vector<double*>& dsts,
                const std::vector<std::vector<double>>& coef, const std::vector<int>* dslot = nullptr);

  // ---- next-batch digits from the streaming combination ----
  // The orchestrator names the tensors the next batch takes as inputs (pre_want, set before a
  // split batch); that batch's combination, which writes them, also writes their mode-1 digit
  // planes and fibre exponents (slots of pre_xs / pre_xsc, layout of oz_split_x_contig), and the
  // next batch's chained mode 1 reads them instead of splitting the tensors again.  pre_next
  // (filled by the combination) becomes pre_ready for exactly the following batch.
  std::vector<const double*> pre_want;
  std::map<const double*, int> pre_ready, pre_next;
  int8_t* pre_xs = nullptr;
  double* pre_xsc = nullptr;
  int pre_slots = 0;
  int64_t pre_hits = 0;
  bool pre_ok() const;  // the next batch's mode 1 can take pre-split digits

  // A batch whose last-mode epilogues run as a separate streaming pass: every
  // item writes its raw Tucker result Y_b, then the epilogue recurrences (in
  // group order, accumulations included) are evaluated symbolically into one
  // matrix-form combination over {Y_b} ∪ external sources.  Sharded handles
  // always take this path, kShardChunk items at a time (the Y_b then live in
  // the symmetric region); a later chunk accumulates into the outputs.
  void tucker_batch_split(const std::vector<TuckerItem>& items);

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
  // complex sharded handles: every product local (two accumulating real terms
  // for modes μ ≥ 2, the 2n×2n real form for μ = 1), the two transposition stages
  // as peer-store copies with the geometry of the real view (2, n_1, …, n_d)
  void tucker_raw_sharded_complex(const std::vector<TuckerItem>& items);

  // the sharded digit stages apply: uniform blocks (every warp's 32 columns of stage 0 on one
  // owner), MN-major digit tiles on both stages (L0 % 128 == 0), mode d on the int8 path, the
  // exchange buffer sized for L0, and the batch within the chain buffers
  bool shard_digits_ok(size_t nb) const;

  void tucker_raw_sharded(const std::vector<TuckerItem>& items);

  // every batch of run_job: sharded handles always split
  void batch(const std::vector<TuckerItem>& items, bool split_it) {
    pre_ready.swap(pre_next);
    pre_next.clear();
    if (h->sharded() || h->cplx || split_it)
      tucker_batch_split(items);
    else
      tucker_batch(items);
    pre_ready.clear();
    pre_want.clear();
  }

  // ---- batched Tucker operators (Eq. (4)) ----
  void tucker_batch(const std::vector<TuckerItem>& items);

  // (Mr, Mi) of a complex exponential held in its 2n×2n real form, extracted
  // once per matrix and apply (complex handles)
  std::map<const double*, std::pair<const double*, const double*>> cparts;
  std::pair<const double*, const double*> complex_parts(const double* Rm, int n);

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

void expm_batch(Exec& ex, double tau, std::vector<ExpReq>& reqs);
void expm_stage(Exec& ex, double tau, std::vector<ExpReq>& reqs);  // expm_batch, split over the ranks of a sharded handle

struct Job {
  int mode;
  int p;
  int n_scales;
  double tau;
  int s, q;
  int block = 0;  // which factor set (fac_of_block) the job's Kronecker sum uses
  const double* vin[kMaxVecs] = {nullptr};
  double* out_same[kMaxVecs][PHIKS_MAX_SCALES] = {{nullptr}};
  double* out_lin[PHIKS_MAX_SCALES] = {nullptr};
};

// the jobs of all blocks of one apply, their Tucker batches merged phase by phase
void run_jobs(Exec& ex, const std::vector<Job>& jobs);

// defined in phiks_api.cpp
phiks_status validate(phiks_handle h, const phiks_request* req, int& p);
phiks_status make_plan(phiks_handle h, const phiks_request* req, int p, const std::vector<double>& norms,
                       plan::Plan& out, int block = 0);
phiks_status check_barrier_flag(phiks_handle h);

// One apply on one handle, split into phases so that several emulated ranks
// can be driven phase by phase (phiks_apply_ranks_serial).
struct ApplyRun {
  phiks_handle h = nullptr;
  const phiks_request* req = nullptr;
  int p = 0, n_vecs = 0, nouts = 0;
  int nb = 1, vpb = 1, opb = 1;  // blocks; vectors and outputs per block (block-major arrays)
  bool same = true, host_mem = false, host_async = false, size_only = false;
  const double* const* vecs = nullptr;
  double* const* outs = nullptr;
  cudaStream_t cs = nullptr;
  int64_t N = 0;
  size_t tbytes = 0;
  Arena ar;
  Exec ex{};
  std::vector<Job> jobs;
  std::vector<double*> dv, dout;
  std::vector<plan::Plan> pls;
  int split = 2;
  // lincomb norms
  bool need_norms = false;
  std::vector<std::pair<int, int>> which;  // (block, index into the block's vectors) of v_1..v_p present
  double* nscratch = nullptr;    // device: 1024*kMaxVecs partials + the norms²
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
    nb = h->nblocks;
    vpb = same ? 1 : req->n_ells;
    opb = same ? req->n_ells * req->n_scales : req->n_scales;
    nouts = nb * opb;
    if (!size_only) {
      if (n_vecs != nb * vpb) return fail(PHIKS_ERR_ARG, "n_vecs");
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
    // default 2: quadrature sums and squaring recurrences as a streaming pass
    // (measured faster on B200 than the fused epilogue); 0 = fused
    split = h->opt_split;
    jobs.assign(nb, Job{});
    for (int b = 0; b < nb; ++b) {
      jobs[b].mode = req->mode;
      jobs[b].p = p;
      jobs[b].n_scales = req->n_scales;
      jobs[b].tau = req->tau;
      jobs[b].block = b;
    }
    pls.assign(nb, plan::Plan{});
    dv.assign(nb * vpb, nullptr);
    dout.assign(nouts, nullptr);
    need_norms = !same && p >= 1 && req->force_s < 0 && !size_only;
    return PHIKS_OK;
  }

  // ---- lincomb plan input: ||v_ℓ||₂ of every block (deterministic GPU
  // reduction; sharded: local sums of squares scattered to every rank, summed
  // in rank order) ----
  phiks_status norms_enqueue(bool do_barrier) {
    if (!need_norms) return PHIKS_OK;
    std::vector<const double*> vv;
    for (int b = 0; b < nb; ++b)
      for (int ell = 1; ell <= p; ++ell)
        for (int i = 0; i < req->n_ells; ++i)
          if (req->ells[i] == ell) which.emplace_back(b, i);
    if (which.empty()) return PHIKS_OK;
    const int nv = static_cast<int>(which.size());
    const size_t sbytes = sizeof(double) * (1024 * kMaxVecs + nv);
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&nscratch), sbytes, cs));
    for (const auto& bi : which) {
      const double* src = vecs[bi.first * vpb + bi.second];
      if (host_mem) {
        double* t = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t), tbytes, cs));
        CUDA_TRY(cudaMemcpyAsync(t, src, tbytes, cudaMemcpyHostToDevice, cs));
        ntmp.push_back(t);
        vv.push_back(t);
      } else {
        vv.push_back(src);
      }
    }
    for (int k0 = 0; k0 < nv; k0 += kMaxVecs) {
      const int cnt = std::min(kMaxVecs, nv - k0);
      CUDA_TRY(launch_sumsq(vv.data() + k0, cnt, N, nscratch, nscratch + 1024 * kMaxVecs + k0, cs));
      norm_launches += 2;
    }
    if (h->sharded()) {
      norm_off = kCtrlNorms + (h->norm_phase++ & 1) * kCtrlNormsBuf;
      ScatterParams sp{};
      sp.rank = h->rank;
      sp.world = h->world;
      sp.cnt = nv;
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
  // read back (synchronises the stream) and plan every block; `ctrl` = the
  // control block holding the gathered partial sums (sharded) — any rank's
  phiks_status norms_finish(const char* ctrl) {
    std::vector<std::vector<double>> norms(nb, std::vector<double>(p, 0.0));
    if (!which.empty()) {
      const int nv = static_cast<int>(which.size());
      const int W = h->sharded() ? h->world : 1;
      std::vector<double> host(static_cast<size_t>(nv) * W);
      const double* srcp = h->sharded() ? reinterpret_cast<const double*>(ctrl + norm_off)
                                        : nscratch + 1024 * kMaxVecs;
      CUDA_TRY(cudaMemcpyAsync(host.data(), srcp, sizeof(double) * nv * W, cudaMemcpyDeviceToHost, cs));
      for (double* t : ntmp) CUDA_TRY(cudaFreeAsync(t, cs));
      ntmp.clear();
      CUDA_TRY(cudaFreeAsync(nscratch, cs));
      nscratch = nullptr;
      CUDA_TRY(cudaStreamSynchronize(cs));
      for (int k = 0; k < nv; ++k) {
        double s2 = 0.0;
        for (int r = 0; r < W; ++r) s2 += host[static_cast<size_t>(r) * nv + k];
        norms[which[k].first][req->ells[which[k].second] - 1] = std::sqrt(s2);
      }
    }
    for (int b = 0; b < nb; ++b) {
      phiks_status st = make_plan(h, req, p, norms[b], pls[b], b);
      if (st != PHIKS_OK) return st;
    }
    return PHIKS_OK;
  }

  phiks_status plan_direct(const phiks_plan_info* forced) {
    if (forced) {
      for (auto& pl : pls) {
        pl.s = forced->s;
        pl.q = forced->q;
        pl.ok = true;
      }
      return PHIKS_OK;
    }
    if (!same && p >= 1 && req->force_s < 0 && size_only) return fail(PHIKS_ERR_ARG, "lincomb sizing needs a plan");
    std::vector<double> norms;
    for (int b = 0; b < nb; ++b) {
      phiks_status st = make_plan(h, req, p, norms, pls[b], b);
      if (st != PHIKS_OK) return st;
    }
    return PHIKS_OK;
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
    for (int i = 0; i < nouts; ++i) dout[i] = host_mem ? ar.alloc_doubles(N) : (size_only ? fake(256 + i) : outs[i]);
    for (int b = 0; b < nb; ++b) {
      Job& jb = jobs[b];
      for (int i = 0; i < kMaxVecs; ++i) jb.vin[i] = nullptr;
      const double* const* bv = dv.data() + b * vpb;
      double* const* bo = dout.data() + b * opb;
      if (same) {
        jb.vin[0] = bv[0];
        for (int j = 0; j < req->n_scales; ++j)
          for (int i = 0; i < req->n_ells; ++i) jb.out_same[req->ells[i]][j] = bo[j * req->n_ells + i];
      } else {
        for (int i = 0; i < req->n_ells; ++i) jb.vin[req->ells[i]] = bv[i];
        for (int j = 0; j < req->n_scales; ++j) jb.out_lin[j] = bo[j];
      }
    }
  }

  phiks_status measure(size_t* need) {
    for (int b = 0; b < nb; ++b) {
      jobs[b].s = pls[b].s;
      jobs[b].q = pls[b].q;
    }
    ex = Exec{h, cs, true, &ar};
    ex.split = split;
    bind(true);
    run_jobs(ex, jobs);
    if (!ex.ok()) return ex.status;
    *need = ar.off;
    return PHIKS_OK;
  }

  bool own_ws = false;
  int half = 0;
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
    const size_t halfb = ((need > 0 ? need : 256) + 4095) & ~size_t(4095);
    if (h->ws_own_bytes < 2 * halfb) {
      for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);  // they reference the old workspace
      h->graphs.clear();
      if (h->ws_own) {
        CUDA_TRY(cudaDeviceSynchronize());  // both halves may be in use on the handle's streams
        CUDA_TRY(cudaFree(h->ws_own));
        h->ws_own = nullptr;
        h->ws_own_bytes = 0;
      }
      if (cudaMalloc(&h->ws_own, 2 * halfb) != cudaSuccess) return fail(PHIKS_ERR_NOMEM, "workspace cudaMalloc");
      h->ws_own_bytes = 2 * halfb;
    }
    half = h->ws_parity;
    h->ws_parity ^= 1;
    *base = static_cast<char*>(h->ws_own) + half * (h->ws_own_bytes / 2);
    return PHIKS_OK;
  }

  // enqueue (rec == nullptr) or record the whole job on the bound workspace
  phiks_status execute(char* base, size_t need, std::vector<Exec::Op>* rec) {
    ar.base = base;
    ar.cap = need;
    ex = Exec{h, cs, false, &ar};
    ex.split = split;
    ex.half = half;
    ex.rec = rec;
    bind(false);
    if (host_mem && rec) return fail(PHIKS_ERR_ARG, "recorded applies take device memory");
    // (never recorded yet: waiting on it is a no-op)
    for (int k = 0; k < 2; ++k)
      if (!h->ev_cdone[k]) CUDA_TRY(cudaEventCreateWithFlags(&h->ev_cdone[k], cudaEventDisableTiming));
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
      // the apply before the previous one (same workspace half) no longer reads it
      CUDA_TRY(cudaStreamWaitEvent(h->s_pre, h->ev_cdone[half], 0));
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
        for (cudaEvent_t* e : {&h->ev_h2d, &h->ev_d2h[0], &h->ev_d2h[1], &h->ev_ready})
          CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
      CUDA_TRY(cudaStreamWaitEvent(h->s_in, h->ev_cdone[half], 0));  // staging half no longer read
      for (size_t i = 0; i < dv.size(); ++i)
        CUDA_TRY(cudaMemcpyAsync(dv[i], vecs[i], tbytes, cudaMemcpyHostToDevice, h->s_in));
      CUDA_TRY(cudaEventRecord(h->ev_h2d, h->s_in));
      CUDA_TRY(cudaStreamWaitEvent(cs, h->ev_d2h[half], 0));  // copy-out of this staging half has drained
      copied.assign(nouts, false);
      ex.on_outputs = [this](const std::vector<double*>& ready) { copy_out(ready); };
    }
    run_jobs(ex, jobs);
    ex.st = cs;
    if (!ex.ok()) return ex.status;
    if (host_mem) {
      std::vector<double*> rest;
      for (int i = 0; i < nouts; ++i)
        if (!copied[i]) rest.push_back(dout[i]);
      copy_out(rest);
      if (!ex.ok()) return ex.status;
      CUDA_TRY(cudaEventRecord(h->ev_d2h[half], h->s_out));
    }
    if (!rec && cap == cudaStreamCaptureStatusNone) CUDA_TRY(cudaEventRecord(h->ev_cdone[half], cs));
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
    S.plan.s = pls[0].s;
    S.plan.q = pls[0].q;
    S.plan.T_formula = plan::tucker_count(req->mode, pls[0].s, req->n_scales, pls[0].q, p);
    S.nblocks = nb;
    for (int b = 0; b < kMaxBlocks; ++b) {
      S.block_plan[b] = phiks_plan_info{};
      if (b < nb) {
        S.block_plan[b].s = pls[b].s;
        S.block_plan[b].q = pls[b].q;
        S.block_plan[b].T_formula = plan::tucker_count(req->mode, pls[b].s, req->n_scales, pls[b].q, p);
        S.block_plan[b].T_executed = -1;
      }
    }
    S.plan.T_executed = static_cast<int>(ex.tucker_ops);
    S.kernel_launches = ex.launches + norm_launches;
    S.tucker_ops = ex.tucker_ops;
    S.i8_mode_launches = ex.i8_launches;
    S.i8_chained_ops = ex.i8_chained;
    S.shard_digit_ops = ex.shard_digit_ops;
    S.presplit_inputs = ex.pre_hits;
    S.mu_mode_flops = ex.mu_flops;
    S.expm_flops = ex.expm_flops;
    S.workspace_bytes = need;
    S.total_kernel_launches += S.kernel_launches;
  }
};


}  // namespace host
}  // namespace phiks
