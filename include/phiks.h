/*
 * phiks.h — C ABI of the B200-native PHIKS library (libphiks.so).
 *
 * PHIKS computes actions of φ-functions of a Kronecker sum
 *     K = A_d ⊕ … ⊕ A_1 = Σ_μ I_d ⊗ … ⊗ A_μ ⊗ … ⊗ I_1      (§2 Eq. (3), l.214-219)
 * without forming K, by Gauss–Lobatto–Legendre quadrature of the integral
 *     φ_ℓ(X) = ∫_0^1 θ^{ℓ-1}/(ℓ-1)! exp((1-θ)X) dθ           (Eq. (2), l.78-82)
 * at the scaled matrix τK/2^s, evaluated with Tucker operators (μ-mode
 * products with exp((1-θ_i)τA_μ/2^s), Eq. (10), l.471-477), followed
 * by the modified squaring recurrences (Eq. (12) l.554-563, Eq. (18) l.734-746).
 * The choice of s and q follows §3.3 (l.779-960).  See DESIGN.md for readings.
 *
 * Memory layout ("vec ... stacks the columns"): an order-d
 * tensor of size n_1×…×n_d is a contiguous fp64 array in column-major order,
 * element (i_1,…,i_d) at offset i_1 + n_1*(i_2 + n_2*(… + n_{d-1}*i_d)).
 * Matrices are n×n column-major fp64.
 *
 * Every compute step runs in CUDA kernels of this library (sm_100a).  There is
 * no CPU fallback: without a CUDA device every entry point that computes
 * returns PHIKS_ERR_CUDA.
 *
 * Error behaviour: every function returns a phiks_status; on error nothing is
 * written to the outputs' contents beyond what kernels already wrote, and
 * phiks_last_error() returns a human-readable message for the calling thread.
 * Handles are not thread-safe: one handle must not be used by two host
 * threads at once.  Distinct handles are independent.
 */
#ifndef PHIKS_H_
#define PHIKS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PHIKS_OK = 0,
  PHIKS_ERR_ARG = 1,        /* invalid argument (dimension, order, null pointer, ...) */
  PHIKS_ERR_CUDA = 2,       /* CUDA runtime error or no CUDA device                  */
  PHIKS_ERR_PLAN = 3,       /* §3.3 search found no admissible (s, q)                */
  PHIKS_ERR_NOMEM = 4,      /* device or pinned-host allocation failed               */
  PHIKS_ERR_WORKSPACE = 5,  /* caller workspace too small (see phiks_stats)          */
  PHIKS_ERR_LIMIT = 6       /* request exceeds a compiled limit (PHIKS_MAX_*)        */
} phiks_status;

#define PHIKS_MAX_D 8       /* tensor order d                                        */
#define PHIKS_MAX_P 6       /* highest φ order ℓ                                     */
#define PHIKS_MAX_SCALES 16 /* output time scales ŝ                                  */
#define PHIKS_MAX_N 4096    /* largest n_μ                                           */
#define PHIKS_MAX_BLOCKS 4  /* diagonal blocks of K̂ per handle (phiks_create_blocks)   */

typedef enum {
  /* φ_ℓ(τK/2^j) v for every ℓ in `ells`, j = 0..n_scales-1, one vector v
     (§3.1, formulas (6) and (13)).  ℓ = 0 means exp(τK/2^j) v. */
  PHIKS_MODE_SAME_VECTOR = 0,
  /* exp(τK/2^j) v_0 + Σ_{ℓ≥1} φ_ℓ(τK/2^j) v_ℓ / 2^{ℓj}, j = 0..n_scales-1
     (§3.2, formulas (7) and (19) with c = 1); vecs[i] pairs with ells[i]. */
  PHIKS_MODE_LINCOMB = 1
} phiks_mode;

typedef enum {
  PHIKS_MEM_DEVICE = 0, /* vecs/outs are device pointers; apply is stream-asynchronous  */
  PHIKS_MEM_HOST = 1,   /* vecs/outs are host pointers (pinned recommended); the library
                           copies them through device staging and synchronises the
                           stream before returning                                       */
  PHIKS_MEM_HOST_ASYNC = 2 /* as PHIKS_MEM_HOST but returns at once: the copies run on the
                           handle's own copy streams (inputs overlap the exponential stage,
                           exp(τK)v is copied out while the φ_ℓ≥1 part runs, and the
                           copies overlap the next apply of another handle); vecs/outs
                           MUST be pinned and stay untouched until phiks_wait(h)        */
} phiks_mem_kind;

/* Opaque handle: the factor matrices A_μ (copied to device at create), their
   per-factor numerical-range data and cached plans/workspace. */
typedef struct phiks_ctx* phiks_handle;

typedef struct {
  int mode;          /* phiks_mode                                                   */
  int n_ells;        /* number of entries of ells, 1..PHIKS_MAX_P+1                   */
  const int* ells;   /* host array of strictly increasing orders in [0, PHIKS_MAX_P]  */
  int n_scales;      /* ŝ ≥ 1: outputs at τ/2^j, j = 0..ŝ-1 (forces s ≥ ŝ-1)         */
  double tau;        /* time step τ > 0; the operator is τK                           */
  double tol;        /* relative tolerance (reading R2); ≤ 0 → 2^-53        */
  int force_s;       /* ≥ 0: use this s instead of the §3.3 search (testing); else -1 */
  int force_q;       /* ≥ 2: use this q (with force_s); else -1                       */
  int mem_kind;      /* phiks_mem_kind of vecs and outs                               */
} phiks_request;

typedef struct {
  int s;             /* scaling parameter s                                            */
  int q;             /* number of GLL quadrature nodes (0 when only ℓ = 0 requested)   */
  int T_formula;     /* Tucker count of Eq. (14) (same vector) or Eq. (19) (lincomb)   */
  int T_executed;    /* Tucker operators the library actually runs for the request     */
} phiks_plan_info;

typedef struct {
  phiks_plan_info plan;     /* plan of the last apply                               */
  int64_t kernel_launches;  /* CUDA kernels launched by the last apply              */
  int64_t tucker_ops;       /* Tucker operators executed by the last apply          */
  double mu_mode_flops;     /* 2·N·Σ_μ n_μ per Tucker operator, summed              */
  double expm_flops;        /* flops of the small-matrix exponential stage          */
  size_t workspace_bytes;   /* device workspace the last apply needed               */
  int64_t total_kernel_launches; /* since create                                    */
  /* filled only when profiling is on (phiks_set_profiling): CUDA-event timing of
     every μ-mode-product kernel launch since profiling was switched on (summed
     over the applies in between), on each apply's stream */
  int64_t mode_product_launches;  /* Tucker-operator μ-mode-product launches          */
  double mode_product_ms;         /* sum of their event-measured durations (ms)     */
  double mode_product_flops;      /* algorithmic flops of those launches (2·rows·n²) */
  int64_t expm_launches;          /* small-GEMM launches of the exponential stage   */
  double expm_ms;                 /* sum of their event-measured durations (ms)     */
  int nblocks;                    /* diagonal blocks of the handle                  */
  phiks_plan_info block_plan[PHIKS_MAX_BLOCKS]; /* plan of each block, last apply   */
  int64_t i8_mode_launches;       /* mode-product launches of the last apply that took
                                     the int8 tensor-core path (phiks_set_gemm_path)  */
  int64_t i8_launches;            /* profiling: the subset of mode_product_launches  */
  double i8_ms;                   /*   on the int8 path (digit splits + GEMM) and    */
  double i8_flops;                /*   their time and fp64-equivalent flops          */
  int64_t i8_gemm_launches;       /* profiling: the int8 GEMM launches alone         */
  double i8_gemm_ms;              /*   and their time                                */
  int64_t i8_chained_ops;         /* Tucker operators of the last apply whose modes ran
                                     chained on the int8 path (no fp64 intermediates:
                                     each product writes the next mode's digits,
                                     DESIGN.md §4d; PHIKS_OPT_CHAIN)                 */
  int64_t shard_digit_ops;        /* sharded handles: Tucker operators whose stage 0 wrote
                                     mode d's digit planes into the owners */
  int64_t presplit_inputs;        /* inputs of the last apply's chained batches whose mode-1
                                     digits the previous batch's combination wrote (no
                                     separate split pass)              */
  int64_t i8_kblocks;             /* profiling: (fibre tile × 64-row n-tile, 128-wide k-block)
                                     units of the int8 GEMM launches, and the subset  */
  int64_t i8_kblocks_run;         /*   whose MMAs ran (the rest had all-zero E digits and
                                     were skipped, PHIKS_OPT_KSKIP)                  */
} phiks_stats;

/* Create a handle for K = A_d ⊕ … ⊕ A_1.
   d: 1..PHIKS_MAX_D.  n[μ]: 1..PHIKS_MAX_N, μ = 0..d-1 (paper's μ = 1..d).
   A_host[μ]: host pointer to the n[μ]×n[μ] column-major real matrix A_μ; the
   library copies it (caller keeps ownership).  Identical factors (bitwise) are
   detected and share their exponentials.  Computes the per-factor numerical-
   range rectangle data of PAPER.md l.925-936 (reading R1) on the host.
   *out receives the handle; destroy it with phiks_destroy. */
phiks_status phiks_create(int d, const int* n, const double* const* A_host, phiks_handle* out);

/* Block until the last apply on h (its kernels and host copies) has finished;
   reports a cross-rank barrier timeout of a sharded handle as PHIKS_ERR_CUDA. */
phiks_status phiks_wait(phiks_handle h);

/* Block-diagonal K̂ = diag(K_1, …, K_nb), K_b = A_{b,d} ⊕ … ⊕ A_{b,1} (PAPER.md
   §4.4: one Kronecker sum per species of a reaction–diffusion system), all
   blocks with the dims n[0..d-1]; A_host[b*d + μ] is block b's factor A_{b,μ}
   (1 ≤ nblocks ≤ PHIKS_MAX_BLOCKS).  phiks_apply then takes the vectors of
   every block, block-major (same vector: vecs[b]; lincomb: vecs[b*n_ells + i])
   and writes every block's outputs block-major (outs[b*per_block + k], per_block
   as for one block).  Each block gets its own §3.3 plan; the blocks share the
   exponential stage and their Tucker operators run in the same launches
   (phase by phase).  phiks_stats.block_plan holds the per-block plans. */
phiks_status phiks_create_blocks(int nblocks, int d, const int* n, const double* const* A_host,
                                 phiks_handle* out);

/* phiks_create_blocks with complex factors (interleaved, as phiks_create_complex). */
phiks_status phiks_create_blocks_complex(int nblocks, int d, const int* n, const double* const* A_host,
                                         phiks_handle* out);

/* Complex K (§4.1 validates PHIKS on the complex operator
   (1+i)/100·Δ): as phiks_create, but A_host[μ] points to an n[μ]×n[μ]
   column-major complex matrix stored as interleaved (re, im) doubles
   (C99 double complex / numpy complex128 layout).  Tensors given to
   phiks_apply are then complex too: N interleaved (re, im) pairs, N = Π n_μ.
   The library works in real arithmetic on the 2n×2n real form of each factor
   (exp of the real form = real form of exp); a complex μ-mode product is the
   first-mode product with that real form (μ = 1), or two real products
   X ×_μ Re(M) + J(X ×_μ Im(M)) (μ ≥ 2, J: re ← −im, im ← re) fused in one
   launch.  The §3.3 rectangle uses the complex trace shift (reading R1).
   Sharded complex handles: phiks_create_sharded_complex. */
phiks_status phiks_create_complex(int d, const int* n, const double* const* A_host, phiks_handle* out);

/* Release the handle and every device/pinned buffer it owns.  NULL is a no-op. */
phiks_status phiks_destroy(phiks_handle h);

/* §3.3 plan for `req` without computing anything on the device.
   vec_norms: host array of ||v_ℓ||_2 for ℓ = 1..p (lincomb mode, index ℓ-1;
   0 for orders not present); ignored (may be NULL) in same-vector mode. */
phiks_status phiks_plan(phiks_handle h, const phiks_request* req, const double* vec_norms,
                        phiks_plan_info* out);

/* Apply the request.
   vecs: n_vecs pointers to input tensors (same-vector: n_vecs == 1;
         lincomb: n_vecs == n_ells, vecs[i] is v_{ells[i]}).
   outs: output tensors, caller-allocated, N doubles each, never aliasing vecs.
         same-vector: n_ells*n_scales pointers, outs[j*n_ells + i] = φ_{ells[i]}(τK/2^j)v.
         lincomb:     n_scales pointers, outs[j] = result at scale j.
   workspace: device buffer of ws_bytes, or NULL to let the library allocate and
         cache its own (grown on demand, freed by phiks_destroy).
   stream: cudaStream_t (NULL = legacy default stream).
   With PHIKS_MEM_DEVICE the call only enqueues work on `stream` (plus, in
   lincomb mode, one device→host read of the vector norms for the §3.3 plan). */
phiks_status phiks_apply(phiks_handle h, const phiks_request* req, int n_vecs,
                         const double* const* vecs, double* const* outs, void* workspace,
                         size_t ws_bytes, void* stream);

/* Device workspace (bytes) phiks_apply needs for `req` under `plan`. */
phiks_status phiks_workspace_size(phiks_handle h, const phiks_request* req,
                                  const phiks_plan_info* plan, size_t* bytes);

/* on != 0: bracket every μ-mode-product launch of subsequent applies with CUDA
   events on the apply's stream (for the roofline report); phiks_get_stats then
   waits for those events.  Off by default. */
phiks_status phiks_set_profiling(phiks_handle h, int on);

/* Path of the Tucker operators' μ-mode products:
   PHIKS_GEMM_DMMA: the fp64 DMMA kernel for every product;
   PHIKS_GEMM_I8: the int8 tensor-core kernel (7 balanced base-256 digits per
     operand, exact int32 accumulation: fp64-class error) wherever it applies
     (real handles, sharded or not, n_μ ≤ 512 — E streamed per k-block above 256 —
     plain outputs), DMMA elsewhere;
     when every mode of a Tucker batch qualifies (n_μ % 16 == 0, L_μ % 128 == 0
     for μ ≥ 2) the modes run chained: each product writes the next mode's
     digits, split with exponent bounds (reading R15) — see
     PHIKS_OPT_CHAIN below;
   PHIKS_GEMM_AUTO (default): the int8 kernel for products with n_μ ≥ 128 on
     tensors of N ≥ 2^20 elements, where it is faster.  Invalidates the handle's captured
     graphs.  PHIKS_ERR_ARG for an unknown path. */
#define PHIKS_GEMM_AUTO 0
#define PHIKS_GEMM_DMMA 1
#define PHIKS_GEMM_I8 2
phiks_status phiks_set_gemm_path(phiks_handle h, int path);

/* Per-handle execution options (the library reads no environment variables).
   Every value gives the same result up to rounding; they exist for A/B
   measurements and tests.  Setting an option invalidates the handle's captured
   graphs.  PHIKS_ERR_ARG for an unknown option or value.
   PHIKS_OPT_SPLIT   where the quadrature weight-sum (Eq. (11)/(17), l.547-552,
                     l.726-733) and the squaring recurrence (Eq. (12)/(18),
                     l.554-563, l.734-746) are evaluated: 0 = in the last mode's
                     epilogue of the Tucker launches (DMMA products; int8 batches
                     with fused outputs fall back to DMMA), 1 = quadrature as a
                     streaming pass, squaring fused, 2 (default) = both as one
                     matrix-form streaming pass over the raw Tucker results.
   PHIKS_OPT_CHAIN   int8 modes of a Tucker batch chained (R15):
                     0 = off (each mode's output split with its own maxima),
                     1 (default) = guarded: chained only when every factor τA_μ
                     of the handle is a Metzler matrix (off-diagonal ≥ 0), whose
                     exponentials are entrywise ≥ 0, so the exponent bound
                     ‖e_j‖₁·max|x| is attained (no cancellation inside a row),
                     2 = whenever the shapes allow (tests of the guard).
   PHIKS_OPT_GRAPHS  1 (default) = capture device-memory applies of tensors up to
                     2^22 elements as CUDA graphs and replay them; 0 = direct
                     launches.
   PHIKS_OPT_PRESPLIT 1 (default) = the streaming combination that produces the
                     next squaring level's inputs also writes their mode-1 int8
                     digit planes (chained batches; stats presplit_inputs); 0 = the
                     next batch splits them in a separate pass.  Same digits,
                     same results bit for bit.
   PHIKS_OPT_KSKIP   1 (default) = the int8 GEMM launches with fp64 outputs (the
                     last mode of a chained Tucker operator) skip the (64-row
                     n-tile, 128-wide k-block) blocks of E whose digits are all zero —
                     the exponentials of banded factors (the FD operators of
                     every BASELINE config) are numerically banded, and a skipped
                     block's MMAs would add exact integer zeros — and gives its
                     n-tiles CTAs in proportion to the remaining work
                     (DESIGN.md §4g); 0 = every block.  Same results bit for bit. */
#define PHIKS_OPT_SPLIT 0
#define PHIKS_OPT_CHAIN 1
#define PHIKS_OPT_GRAPHS 2
#define PHIKS_OPT_PRESPLIT 3
#define PHIKS_OPT_KSKIP 4
phiks_status phiks_set_option(phiks_handle h, int option, int value);
phiks_status phiks_get_option(phiks_handle h, int option, int* value);

/* Telemetry of the last phiks_apply on this handle. */
phiks_status phiks_get_stats(phiks_handle h, phiks_stats* out);

/* One batched μ-mode product (cost O(N n_μ)):
   out_b = in_b ×_{mu+1} M_b for b = 0..batch-1, tensors of dims n[0..d-1],
   M_b n[mu]×n[mu] column-major; all pointers device.  The building block of
   the Tucker operator, exposed for tests and benchmarks. */
phiks_status phiks_mode_product(int d, const int* n, int mu, int batch, const double* const* in,
                                const double* const* M, double* const* out, void* stream);

/* The μ-mode product of phiks_mode_product on the int8 tensor cores
   (tcgen05.mma kind::i8): every mode-μ fiber of in[b] and every
   row of M[b] is written exactly in `slices` (6 or 7) balanced base-256
   digits scaled by a power of two, and the digit products with s + t < S are
   accumulated exactly in int32; with 7 digits each operand keeps 55 bits and
   the error bound is that of an fp64 dot product (§3.1 Eq. (13) is
   the product computed).  n_μ ≤ 512.  `workspace` is device memory of at
   least phiks_mode_product_i8_workspace bytes (owned by the caller, reused
   across calls on the same stream); errors as phiks_mode_product,
   PHIKS_ERR_ARG for unsupported sizes or digit counts. */
phiks_status phiks_mode_product_i8_workspace(int d, const int* n, int mu, int slices, int batch, size_t* bytes);
phiks_status phiks_mode_product_i8(int d, const int* n, int mu, int slices, int batch, const double* const* in,
                                   const double* const* M, double* const* out, void* workspace, size_t ws_bytes,
                                   void* stream);

/* Tucker operator (Eq. (4)): out = in ×_1 M_0 ×_2 M_1 … ×_d M_{d-1},
   device pointers; scratch: 2*N doubles of device memory (NULL if d == 1). */
phiks_status phiks_tucker(int d, const int* n, const double* in, const double* const* M,
                          double* out, double* scratch, void* stream);

/* exp(c·A) for a device n×n column-major A into device E (scaling and squaring,
   degree-16 Taylor with Paterson–Stockmeyer); scratch: 8*n*n + 256 doubles. */
phiks_status phiks_expm(int n, const double* A, double c, double* E, double* scratch,
                        void* stream);

/* FP64 peak microbenchmark: launches `blocks` CTAs running `iters` iterations
   of register-resident DMMA (kind 0) or DFMA (kind 1) chains; writes a
   checksum to sink (device, one double per thread of the grid).  *flops
   receives the number of floating-point operations the launch performs. */
phiks_status phiks_fp64_peak_launch(int kind, int blocks, int64_t iters, double* sink,
                                    void* stream, double* flops);

/* Host-only §3.3 planning (no device needed): same as phiks_plan for the
   factors A_host (real, column-major, host) without creating a handle. */
phiks_status phiks_plan_host(int d, const int* n, const double* const* A_host, const phiks_request* req,
                             const double* vec_norms, phiks_plan_info* out);

/* phiks_plan_host for complex factors (interleaved, as phiks_create_complex). */
phiks_status phiks_plan_host_complex(int d, const int* n, const double* const* A_host, const phiks_request* req,
                                     const double* vec_norms, phiks_plan_info* out);

/* Host-only §3.3 search on an explicit rectangle Ξ = (center_re + i center_im)
   + [-hr, hr] + i[-hi, hi] ⊇ W(τK), absolute tolerance
   delta, norms[k-1] = ||v_k|| (lincomb) or norms[0] = ||v|| (same vector).
   s_fixed ≥ 0: only the smallest admissible q at that s is returned in out->q
   (0 if none) with out->s = s_fixed; otherwise the full search from s_min.
   Lets the planner be checked against PAPER.md Table 1 (complex operator). */
phiks_status phiks_select_plan(int mode, double center_re, double center_im, double hr, double hi, int p,
                               const double* norms, double delta, int s_hat, int s_min, int s_fixed,
                               phiks_plan_info* out);

/* ------------------------------------------------------------------------
 * Slab sharding across the GPUs of one NVSwitch box (the
 * north star of BASELINE.json: "a slab partition of the tensor ... along the
 * outermost mode, with modes 1..d-1 contracted locally and the mode-d product
 * done through an all-to-all transpose").
 *
 * Rank r of P owns the contiguous slab i_d ∈ [o_r, o_r + c_r) of every tensor
 * (block distribution: c_r = n_d/P, plus one for r < n_d mod P; o_r the sum of
 * the previous counts): column-major with dims (n_1, …, n_{d-1}, c_r), i.e.
 * elements [M·o_r, M·(o_r + c_r)) of the global column-major array, M = N/n_d.  Each Tucker
 * operator (Eq. (4); the μ-mode products commute, l.252-270) runs
 * modes 1..d-2 on the slab, then the mode-(d-1) product whose epilogue stores
 * every output column straight into the peer rank that owns it in the
 * transposed layout (slab of mode d-1, dims (n_1..n_{d-2}, c'_k, n_d)),
 * a device-side barrier, the mode-d product there (local), whose epilogue
 * stores back into the slab layout on the owner, and a second barrier: the
 * all-to-all transposition is fused into the producing kernels' stores over
 * NVLink peer memory.  The quadrature sums, squaring recurrences and scale
 * outputs are then elementwise on the slab.
 *
 * Memory: each rank allocates a symmetric region (control block + pools of
 * 2·16 slab-sized tensors) that its peers map through CUDA IPC.
 * ------------------------------------------------------------------------ */
#define PHIKS_IPC_HANDLE_BYTES 64

/* Create rank `rank` of a `world`-way slab-sharded handle for the GLOBAL
   dims n[0..d-1] and factors A_host (every rank passes the same factors).
   world = 1 gives an ordinary handle.  world > 1 needs d ≥ 2, world ≤ 8 and
   n[d-1], n[d-2] ≥ world (PHIKS_ERR_ARG otherwise); the slabs are block-
   distributed (rank r owns n_d/world indices, one more for r < n_d mod world),
   so the local slab sizes may differ between ranks (phiks_shard_info).
   Before the first apply the peers must be attached with
   phiks_shard_open_peers (one process per GPU) or phiks_shard_set_peer_bases
   (one process).  phiks_apply on the handle then takes and returns local
   slabs (phiks_shard_info's local_count doubles each); every rank must issue
   the same sequence of applies with the same request (the applies meet in
   device-side barriers; a rank that does not arrive within 60 s makes the
   barrier give up and the handle report PHIKS_ERR_CUDA from
   phiks_get_stats / host-memory applies). The timeout is sticky: every later
   barrier of the handle returns at once (no second wait), and the handle keeps
   reporting the error — destroy it and create the ranks' handles again. */
phiks_status phiks_create_sharded(int d, const int* n, const double* const* A_host, int rank, int world,
                                  phiks_handle* out);

/* Sharded handle of a block-diagonal K̂ (phiks_create_blocks × phiks_create_sharded). */
phiks_status phiks_create_sharded_blocks(int nblocks, int d, const int* n, const double* const* A_host, int rank,
                                         int world, phiks_handle* out);

/* Sharded handle of a complex K (phiks_create_complex × phiks_create_sharded):
   the complex μ-mode products run locally and the two transposition stages
   move their results with peer-store copies (real view (2, n_1, …, n_d)). */
phiks_status phiks_create_sharded_complex(int d, const int* n, const double* const* A_host, int rank, int world,
                                          phiks_handle* out);

/* Sharded block-diagonal handle with complex factors. */
phiks_status phiks_create_sharded_blocks_complex(int nblocks, int d, const int* n, const double* const* A_host,
                                                 int rank, int world, phiks_handle* out);

/* rank, world, local slab size in elements, bytes of the symmetric region
   (any output pointer may be NULL). */
phiks_status phiks_shard_info(phiks_handle h, int* rank, int* world, int64_t* local_count,
                              size_t* sym_bytes);

/* Writes PHIKS_IPC_HANDLE_BYTES bytes: the CUDA IPC handle of this rank's
   symmetric region (zeros for world = 1).  Exchange them between the ranks
   (e.g. an all-gather over torch.distributed) and pass the gathered array to
   phiks_shard_open_peers. */
phiks_status phiks_shard_ipc_handle(phiks_handle h, void* handle_out);

/* handles: world × PHIKS_IPC_HANDLE_BYTES bytes, slot k = rank k's handle
   (own slot ignored).  Maps every peer's region (cudaIpcOpenMemHandle; the
   GPUs must be peer-capable, i.e. NVLink/NVSwitch). */
phiks_status phiks_shard_open_peers(phiks_handle h, const void* handles);

/* Device base address of this rank's symmetric region (NULL for world = 1). */
phiks_status phiks_shard_base(phiks_handle h, void** base);

/* Device address under which this process sees rank k's region (after
   open_peers / set_peer_bases; k == rank gives the own region). */
phiks_status phiks_shard_peer_base(phiks_handle h, int k, void** base);

/* Same-process alternative to open_peers: bases[k] = rank k's region
   (phiks_shard_base of the handle of rank k), bases[rank] must be own. */
phiks_status phiks_shard_set_peer_bases(phiks_handle h, void* const* bases);

/* Host-only geometry of the two peer-store launches of a sharded Tucker
   operator (no device needed): n = GLOBAL dims, stage 0 = the mode-(d-1)
   product on the slab, stage 1 = the mode-d product on the transposed slab.
   out7 = {L, n, R, cb, rstride, roff, colstride}: the launch views its input
   as (L, n, R) column-major and sends output element (l, j, r) to rank
   k = j / cb at element offset l + rstride·r + roff + colstride·(j − k·cb)
   of the destination tensor.  The library's own launches use exactly this. */
phiks_status phiks_shard_layout(int d, const int* n, int rank, int world, int stage, int64_t* out7);

/* General geometry, also for ragged slabs (n_d or n_{d-1} not divisible by
   world; the first n mod world ranks own one more index).  out: 4 + 3·world
   values {L, n, R, colstride, kstart[world], kstride[world], kroff[world]};
   output element (l, j, r) goes to rank k = owner(j) (block distribution of
   the n columns) at offset l + kstride[k]·r + kroff[k] + colstride·(j − kstart[k]). */
phiks_status phiks_shard_layout_ex(int d, const int* n, int rank, int world, int stage, int64_t* out);

/* Emulation of `world` ranks on ONE GPU (tests): hs[k] is rank k (all in this
   process, peers set with phiks_shard_set_peer_bases).  Runs every rank's
   apply phase by phase on one stream — rank 0's kernels up to its next
   barrier, then rank 1's, … — so the barriers are implied by stream order and
   no kernel waits on another.  Same kernels, same peer-store epilogues and
   same plan as the multi-GPU path.  vecs: world × n_vecs device pointers
   (rank-major); outs: world × (outputs per rank) device pointers. */
phiks_status phiks_apply_ranks_serial(const phiks_handle* hs, int world, const phiks_request* req, int n_vecs,
                                      const double* const* vecs, double* const* outs, void* stream);
/* The same with a filtered replay, for the multi-GPU projection only
   (scripts/sharded_projection.py): which = 0 every kernel (= the call above),
   1 only stage A (the exponential stage and its all-gather: what a real
   apply runs on the handle's pre stream, overlapped with the previous apply),
   2 everything but stage A.  With which = 2 the applies read the exponentials
   an earlier full apply of the same handles left in their workspaces, so the
   outputs are those of a full apply only when the same request ran with
   which = 0 at least twice before (the two workspace halves).
   PHIKS_ERR_ARG for another value. */
phiks_status phiks_apply_ranks_serial_ex(const phiks_handle* hs, int world, const phiks_request* req, int n_vecs,
                                         const double* const* vecs, double* const* outs, void* stream, int which);

/* Message for the last error on the calling thread ("" if none). */
const char* phiks_last_error(void);

/* Library version string. */
const char* phiks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PHIKS_H_ */
