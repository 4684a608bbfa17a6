// Internal declarations shared by the host orchestration (phiks_api.cpp) and
// the CUDA kernels (kernels.cu).  Not part of the C ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "phiks.h"

namespace phiks {

constexpr int kMaxVecs = PHIKS_MAX_P + 1;

// ---------------------------------------------------------------------------
// Batched μ-mode product with a fused linear epilogue.
//
// A launch processes tensors viewed as (L, n, R) — L = Π_{ν<μ} n_ν (fastest),
// n = n_μ, R = Π_{ν>μ} n_ν — computing for every term t of a group
//     acc[l, j, r] = Σ_k M_t[j, k] · in_t[l, k, r]            (μ-mode product)
// and then, for every output o of the term,
//     dst_o[l, j, r] = beta_o · acc + Σ_s gamma_s · src_s[l, j, r].
// Terms of one group run sequentially in the same CTA for a given output tile,
// so a term may accumulate into a tensor an earlier term of its group wrote
// (src == dst).  Different groups must not write the same tensor.
// ---------------------------------------------------------------------------

struct SrcRef {
  const double* ptr;
  double coef;
};

struct OutSpec {
  double* dst;
  double beta;   // coefficient of the accumulator
  int src0;      // first SrcRef index
  int nsrc;      // number of SrcRefs
};

struct TermSpec {
  const double* in;
  const double* M;  // n×n column-major, element (j,k) at j + k*n
  int out0;
  int nout;
  int cswap;        // complex tensors: apply J (re ← −im, im ← re) to the accumulator first
};

struct GroupSpec {
  int t0, t1;
};

constexpr int kMaxGroups = 48;
constexpr int kMaxTerms = 48;   // also the TMA descriptor count per launch
constexpr int kMaxOuts = 128;
constexpr int kMaxSrcs = 224;
constexpr int kMaxRanks = 8;    // slab-sharded handles: ranks of one NVSwitch box
constexpr int kMaxBlocks = PHIKS_MAX_BLOCKS;  // diagonal blocks of K̂ per handle

// Remote (peer-memory) epilogue of the slab-sharded Tucker operator: when
// world > 0 every output of the launch is written to the symmetric region of
// the rank that owns its column j of the μ-mode product.  Columns are block-
// distributed: the first crem ranks own cq+1 columns, the others cq, so
//     k = j < (cq+1)·crem ? j/(cq+1) : crem + (j − (cq+1)·crem)/cq,
//     dst = base[k] + (size_t)OutSpec::dst (a byte offset)
//           + l + kstride[k]·r + kroff[k] + colstride·(j − kstart[k]),
// (l, j, r) the (L, n, R) coordinates of the element.  This folds the
// slab↔slab transposition of the mode-d product into the
// stores of the producing mode product.  Remote outputs carry no sources.
struct Remap {
  int world;    // 0: local outputs (OutSpec::dst is a pointer)
  int cq, crem; // block distribution of the n columns over the ranks
  int uniform;  // crem == 0 and every kstride / kroff equal (hoisted fast path)
  int64_t colstride;
  int kstart[kMaxRanks];
  int64_t kstride[kMaxRanks], kroff[kMaxRanks];
  char* base[kMaxRanks];
};

struct ModeParams {
  int64_t L, R;
  int n;
  int ngroups;
  Remap remap;
  GroupSpec groups[kMaxGroups];
  TermSpec terms[kMaxTerms];
  OutSpec outs[kMaxOuts];
  SrcRef srcs[kMaxSrcs];
};

// Elementwise linear combinations: for every output o,
//     dst_o[i] = Σ_s gamma_s · src_s[i],  i < count.
constexpr int kMaxCombOuts = 64;
constexpr int kMaxCombSrcs = 256;
struct CombineParams {
  int64_t count;
  int nout;
  OutSpec outs[kMaxCombOuts];  // beta unused
  SrcRef srcs[kMaxCombSrcs];
};

// Matrix-form combination: dst_o[i] = Σ_s coef[o][s] · src_s[i] for o < nout,
// every source read once per element (quadrature / squaring sums when they are
// not fused into an epilogue).
constexpr int kMcMaxSrc = 64;
constexpr int kMcMaxOut = 8;
struct MultiCombineParams {
  int64_t count;
  int nsrc, nout;
  const double* src[kMcMaxSrc];
  double* dst[kMcMaxOut];
  double coef[kMcMaxOut][kMcMaxSrc];
  // with dig[o] set (launch_multi_combine_split): output o also as the S = 7 mode-1 digit
  // planes of the next batch's int8 products, fibres of fn contiguous elements: digit s of
  // element k of fibre c at dig[o][(s·C + c)·Kp + k] (zeros for n ≤ k < Kp), the fibre exponent
  // (NaN: non-finite fibre) at dsc[o][c], C = count / fn — the layout oz_split_x_contig writes
  int8_t* dig[kMcMaxOut];
  double* dsc[kMcMaxOut];
  int fn, Kp;
};

// μ-mode products on the int8 tensor cores (ozaki.cu): every
// term t computes out_t = beta_t · (x_{xslot} ×_μ e_{eslot}) (plain outputs, no
// sources), each fiber / row written in S balanced base-256 digits.
constexpr int kOzMaxN = 512;      // mode size limit of the int8 path (E streamed per k-block above kOzMaxNRes)
constexpr int kOzMaxNRes = 256;   // E tile resident in shared memory up to this n
constexpr int kOzMaxSlices = 7;
struct OzakiTerm {
  int xslot, eslot;
  double* out;
  double beta;
  // chained Tucker modes: with dig set, the epilogue writes the
  // NEXT mode's digits instead of out: digit s of output element i at
  // dig[s·L·n·R + i] (the fp64 layout, one byte plane per digit), each next-mode
  // fiber scaled by its exponent nex[c'] (bound from the chain kernel)
  int8_t* dig;
  double* nex;
  double* nmx;  // chained: Mx(l, r') = max_i ex(l, i, r') of the input fibers (oz_chain_kernel)
};
struct OzakiParams {
  int64_t L, R;
  int n, Kp, S;
  int nx, ne, nterms;
  const double* x[kMaxTerms];  // distinct inputs (L, n, R)
  const double* e[kMaxTerms];  // distinct matrices (n×n column-major)
  OzakiTerm terms[kMaxTerms];
  int8_t* xs;    // workspace (ozaki_bind_workspace): [nx][S][L·R][Kp] slices
  double* xsc;   // [nx][L·R] fiber exponents ex (NaN: non-finite fiber)
  int8_t* es;    // [ne][S][n][Kp]
  double* esc;   // [ne][n] row exponents
  double* eb;    // [ne][n] exponents b_j with ‖e_j‖₁ < 2^{b_j} (chained modes)
  int* ecol;     // [ne][n] (ee_j − 30) − b_j (INT_MIN: non-finite row), the digit epilogue's column shift
  int* eext;     // [4][ne] min_j b_j, max_j b_j, any non-finite row (chained modes' fast-path test), and
                 // the nonzero digit blocks of each matrix: bit 4·t + kb set when some digit of rows
                 // [64t, 64t+64) × k ∈ [128kb, 128kb+128) is nonzero (the GEMM skips the others)
  int a_mn;      // 1: xs holds [nx][S][L·n·R] digit planes in the fp64 layout (MN-major A, L % 128 == 0)
  int cplx_j;    // complex μ ≥ 2 product: fibres [x ; Jx] of length K = 2n against
                 // E = [Re M | Im M] (n × 2n, column-major, Im M right after Re M), so y = Re M·x + J·Im M·x
  int n_next;    // chained: n_{μ+1} (0: plain fp64 outputs)
  Remap remap;   // slab-sharded stage (world > 0): fp64 outputs (out) or next-mode digit planes (dig,
                 // AMN only) go to the owner rank; out / dig = byte offsets in the owners' regions
  int e_ready;       // 1: es/esc/eb/ecol/eext already hold these matrices' split (the previous launch's)
  unsigned long long* kcount;  // profiling (or null): [0] += (unit, k-block) pairs, [1] += those run
  int kskip;         // 1: the GEMM skips the k-blocks whose E digits are all zero (exact: their MMAs
                     // add integer zeros) and sizes its n-tile CTA groups by the remaining work
  int shard_stage0;  // 1: the next-mode exponents come from the cross-rank exchange
                     // (launch_oz_shard_pmax / launch_oz_shard_tables), not oz_chain_kernel
};
// Slab-sharded chained stage 0: the next mode (d) runs along i_d, which the
// ranks' slabs partition, so its fibre exponents e(l, j) = b_j + Mx(l), Mx(l) = max over all i_d
// of the stage-0 input fibre exponents ex(l, i_d), need a cross-rank max.  pmax: every rank writes
// its slab's partial max of term t into slot [rank][t][l] (kShardChunkMax terms per rank) of every
// peer's exchange buffer; after a barrier, tables: Mx(l) over the ranks' slots → nmx[t][l] (the
// stage-0 epilogue's digit exponents) and the stage-1 A fibre exponents of this rank's transposed
// slab, xsc1[t][l + L0·jl] = b_{kstart + jl} + Mx(l), jl < cb (clamped like oz_chain_kernel;
// NaN if any input fibre was non-finite).
constexpr int kShardChunkMax = 24;
struct OzShardExch {
  int rank, world, nterms;
  int64_t L0, R;                       // stage-0 launch geometry (L0, n_{d-1}, R = local slab of i_d)
  const double* xsc[kMaxTerms];        // per term: its input fibre exponents, L0·R entries
  double* dst[kMaxRanks];              // peers' exchange buffers [world][kShardChunkMax][L0]
  // tables (own buffer)
  const double* exch;
  int kstart, cb;
  const double* eb[kMaxTerms];         // per term: b_j of its stage-0 matrix (n_{d-1} entries)
  double* nmx[kMaxTerms];              // per term: Mx, L0 entries
  double* xsc1[kMaxTerms];             // per term: stage-1 fibre exponents, L0·cb entries
};
cudaError_t launch_oz_shard_pmax(const OzShardExch& e, cudaStream_t st);
cudaError_t launch_oz_shard_tables(const OzShardExch& e, cudaStream_t st);

bool ozaki_supported(int64_t L, int n, int64_t R, int S);
size_t ozaki_workspace_bytes(int64_t L, int n, int64_t R, int S, int nx, int ne, int K = 0);  // K: contraction (0: n)
void ozaki_bind_workspace(OzakiParams& p, void* ws);  // sets Kp and the workspace pointers
cudaError_t launch_ozaki_mode(const OzakiParams& p, cudaStream_t st, bool split_x = true, bool split_e = true,
                              bool gemm = true);

// Kernel launchers (kernels.cu).  Return cudaError_t of the launch.
cudaError_t launch_mode_product(const ModeParams& p, cudaStream_t st);
cudaError_t launch_combine(const CombineParams& p, cudaStream_t st);
cudaError_t launch_multi_combine(const MultiCombineParams& p, cudaStream_t st);
// the same combination fused with the mode-1 digit split of the outputs that have dig[o] set
// (ozaki.cu): count % fn == 0, fn ≤ 512, Kp = fn rounded up to 128, nout ≤ the max below, 16-byte aligned
cudaError_t launch_multi_combine_split(const MultiCombineParams& p, cudaStream_t st);
int oz_multi_combine_split_max_out(int n);  // outputs per launch of the fused variant for fibres of n
// partial sums of squares of `count` doubles of each of `nvec` vectors
// -> norms2[v] (device), deterministic two-pass reduction; scratch ≥ 1024*nvec doubles
cudaError_t launch_sumsq(const double* const* vecs, int nvec, int64_t count, double* scratch,
                         double* norms2, cudaStream_t st);
cudaError_t launch_set_identity(double* E, int n, double diag, cudaStream_t st);
// dst(owner, offset) = src(l, j, r) for a local (L, n, R) tensor under a Remap
cudaError_t launch_remap_copy(const double* src, int64_t L, int n, int64_t R, size_t dst_off, const Remap& rm,
                              cudaStream_t st);
// Mr, Mi (n×n) from the interleaved real form R (2n×2n) of a complex matrix
cudaError_t launch_complex_parts(const double* R, int n, double* Mr, double* Mi, cudaStream_t st);

// Cross-rank barrier of a slab-sharded handle (one CTA): e = ++*epoch, writes e
// into slot [rank] of every peer's flag array (st.release.sys over NVLink), then
// waits until every slot of its own array is ≥ e (ld.acquire.sys).  Gives up
// after `timeout_ns` and sets *err = 1 instead of hanging.
struct BarrierParams {
  int rank, world;
  uint64_t* epoch;  // own region: the barrier count, advanced by the kernel itself (graph-replayable)
  uint64_t timeout_ns;
  uint64_t* peer_flags[kMaxRanks];  // peer k's flag array (own one at k == rank)
  int* err;                          // own region: sticky timeout flag
};
cudaError_t launch_barrier(const BarrierParams& p, cudaStream_t st);
// dst_k[rank*cnt + i] = src[i] for every peer k (small, one CTA)
struct ScatterParams {
  int rank, world, cnt;
  const double* src;
  double* dst[kMaxRanks];
};
cudaError_t launch_scatter_small(const ScatterParams& p, cudaStream_t st);
// item i: count[i] doubles from src[i] to byte offset off[i] of every rank's region base[k]
// (the sharded exponential stage's all-gather of the small matrices)
constexpr int kMaxPeerCopy = 32;
struct PeerCopyParams {
  int world, nitems;
  const double* src[kMaxPeerCopy];
  size_t off[kMaxPeerCopy];
  int64_t count[kMaxPeerCopy];
  char* base[kMaxRanks];
};
cudaError_t launch_peer_copy(const PeerCopyParams& p, cudaStream_t st);
cudaError_t launch_fp64_peak(int kind, int blocks, int64_t iters, double* sink, cudaStream_t st,
                             double* flops);

}  // namespace phiks
