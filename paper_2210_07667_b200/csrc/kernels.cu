// CUDA kernels of the B200 PHIKS hot path (sm_100a).
//
//  * mode_product_kernel — batched μ-mode product (§2 l.252-270,
//    "a single μ-mode product ... can be implemented by a single matrix-matrix
//    product") on FP64 tensor cores (DMMA.8x8x4 via mma.sync m8n8k4), operands
//    staged global→shared by a multi-stage cp.async pipeline, the tensor read in
//    place (no permute: the (L, n, R) view is addressed directly), and a fused
//    linear epilogue that carries the quadrature weight-sum (Eq. (11)/(17)) and
//    the squaring-recurrence combinations (Eq. (12)/(18)).
//  * combine_kernel      — elementwise multi-output linear combinations.
//  * sumsq kernels       — deterministic ||v||_2^2 for the §3.3 plan (lincomb).
//  * fp64_peak_kernel    — DMMA / DFMA throughput microbenchmark (roofline).
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)

#include <cstdlib>

#include <algorithm>

#include "phiks_internal.h"

namespace phiks {

namespace {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 8 : 0;  // src-size 0 => zero-fill the 8 bytes
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col), fp64.  Fragments (lane = 4*g + t):
//   a = A[g][t], b = B[t][g], {c0,c1} = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Complex tensors are interleaved (re, im) doubles; for modes μ ≥ 2 the GEMM
// row index is m = c + 2l (c = 0 re, 1 im) and a complex μ-mode product is
// X ×_μ Mr + J(X ×_μ Mi) with J(t)_re = −t_im, J(t)_im = t_re.  The partner
// rows 2l, 2l+1 sit in lanes lane, lane^4 of the DMMA fragment (row = 8·mi +
// lane/4 + tile offset, tile offsets even), so J is one shuffle per element.
template <int MI, int NI>
__device__ __forceinline__ void complex_swap(double (&acc)[MI][NI][2], int lane) {
  const bool im_row = ((lane >> 2) & 1) != 0;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double partner = __shfl_xor_sync(0xffffffffu, acc[mi][ni][e], 4);
        acc[mi][ni][e] = im_row ? partner : -partner;
      }
}

// Peer-memory store of the slab-sharded epilogue (phiks_internal.h, Remap).
__device__ __forceinline__ int remap_owner(const Remap& rm, int j) {
  const int big = (rm.cq + 1) * rm.crem;
  return j < big ? j / (rm.cq + 1) : rm.crem + (j - big) / rm.cq;
}
// element (l, j, r): rowl = l (+ nothing else), r = the R index
__device__ __forceinline__ void remote_store(const Remap& rm, const OutSpec& os, int64_t l, int64_t r, int j,
                                             double v) {
  const int k = remap_owner(rm, j);
  double* base = reinterpret_cast<double*>(rm.base[k] + reinterpret_cast<uintptr_t>(os.dst));
  base[l + rm.kstride[k] * r + rm.kroff[k] + rm.colstride * static_cast<int64_t>(j - rm.kstart[k])] = v;
}

}  // namespace

// ---------------------------------------------------------------------------
// μ-mode product: GEMM rows m ∈ [0, L·R) (m = l + L·r), columns j ∈ [0, n),
// contraction k ∈ [0, n).  A operand = input tensor tile (m, k) at
// off(m,k) = (m mod L) + L·k + L·n·(m div L); B operand = M^T tile (k, j) at
// j + k·n.  KMAJ (L == 1): off(m,k) = m·n + k, the contraction index is the
// contiguous one, so the loader walks k across threads.
//
// Persistent: the grid is sized to the resident CTA count; CTA b walks the
// work units (group, tile) b, b+G, …, and inside a unit the group's terms.
// The cp.async prologue of the next (unit, term) is issued before the current
// epilogue, so global loads overlap the epilogue and the next mainloop starts
// on resident data.
// ---------------------------------------------------------------------------
// off(m) of row m: (m mod L) + L·n·(m div L); 32-bit division when it fits
__device__ __forceinline__ int64_t row_offset(int64_t m, int64_t L, int64_t Ln, bool small) {
  if (small) {
    const uint32_t mu = static_cast<uint32_t>(m), Lu = static_cast<uint32_t>(L);
    const uint32_t q = mu / Lu;
    return static_cast<int64_t>(mu - q * Lu) + Ln * q;
  }
  return (m % L) + Ln * (m / L);
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MINB, bool KMAJ>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, MINB)
    mode_product_kernel(const __grid_constant__ ModeParams p) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int MI = WM / 8, NI = WN / 8;
  constexpr int SA = BM + 4, SB = BN + 4;  // padded strides: 64-bit fragment loads conflict-free
  constexpr int A_PER_T = BM * BK / NT, B_PER_T = BK * BN / NT;
  static_assert(WM % 8 == 0 && WN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert(KMAJ || NT % BM == 0, "non-KMAJ loader assumes NT % BM == 0");
  static_assert(NT % BK == 0, "KMAJ loader assumes NT % BK == 0");
  static_assert(NT % BN == 0, "B loader assumes NT % BN == 0");
  static_assert(A_PER_T >= 1 && B_PER_T >= 1 && A_PER_T <= 32, "tile/CTA shape");

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * BK * SA;

  const int n = p.n;
  const int64_t L = p.L;
  const int64_t Mtot = L * p.R;
  const int64_t Ln = L * static_cast<int64_t>(n);
  const bool small = (Mtot < (int64_t(1) << 31)) && (L < (int64_t(1) << 31));
  const int tilesN = (n + BN - 1) / BN;
  const int64_t tilesM = (Mtot + BM - 1) / BM;
  const int64_t tiles = tilesM * tilesN;
  const int64_t units = tiles * p.ngroups;
  const int KT = (n + BK - 1) / BK;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm0 = (warp / WARPS_N) * WM;
  const int wn0 = (warp % WARPS_N) * WN;
  const int lg = lane >> 2, lt = lane & 3;

  // ---- per-(unit, term) loader context: base pointers and validity, computed once ----
  struct Ld {
    int64_t unit;
    int t;                 // absolute term index
    const double* a;       // this thread's first A element at k = 0
    const double* b;       // this thread's first B element at k = 0
    uint32_t amask;        // KMAJ: row-valid bits per i;  non-KMAJ: bit 0 = row valid
    bool bok;              // B column valid
  };
  auto make_ld = [&](int64_t unit, int t) -> Ld {
    Ld c;
    c.unit = unit;
    c.t = t;
    c.amask = 0;
    c.bok = false;
    c.a = nullptr;
    c.b = nullptr;
    if (unit >= units) return c;
    const int64_t tile = unit % tiles;
    const int64_t m0 = (tile / tilesN) * BM;
    const int j0 = static_cast<int>(tile % tilesN) * BN;
    const double* in = p.terms[t].in;
    const double* M = p.terms[t].M;
    if (KMAJ) {
      const int64_t mrow = m0 + tid / BK;
      c.a = in + mrow * n + (tid % BK);
#pragma unroll
      for (int i = 0; i < A_PER_T; ++i)
        if (mrow + i * (NT / BK) < Mtot) c.amask |= 1u << i;
    } else {
      const int64_t m = m0 + tid % BM;
      const bool ok = m < Mtot;
      c.amask = ok ? 1u : 0u;
      c.a = in + (ok ? row_offset(m, L, Ln, small) : 0) + L * (tid / BM);
    }
    const int jj = j0 + tid % BN;
    c.bok = jj < n;
    c.b = M + (c.bok ? jj : 0) + static_cast<int64_t>(tid / BN) * n;
    return c;
  };
  auto advance = [&](const Ld& c) -> Ld {
    if (c.t + 1 < p.groups[c.unit / tiles].t1) return make_ld(c.unit, c.t + 1);
    const int64_t nu = c.unit + gridDim.x;
    return make_ld(nu, nu < units ? p.groups[nu / tiles].t0 : 0);
  };
  auto load_stage = [&](const Ld& c, int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * BK * SA;
    double* bs = Bs + stage * BK * SB;
    if (KMAJ) {
      const int kk = tid % BK;
      const bool kok = (k0 + kk) < n;
#pragma unroll
      for (int i = 0; i < A_PER_T; ++i) {
        const bool v = kok && ((c.amask >> i) & 1u);
        const int mm = tid / BK + i * (NT / BK);
        cp_async8(as + kk * SA + mm, v ? c.a + k0 + static_cast<int64_t>(i) * (NT / BK) * n : c.a - (tid % BK), v);
      }
    } else {
      const int mm = tid % BM;
#pragma unroll
      for (int i = 0; i < A_PER_T; ++i) {
        const int kk = tid / BM + i * (NT / BM);
        const bool v = (c.amask & 1u) && (k0 + kk < n);
        cp_async8(as + kk * SA + mm, v ? c.a + L * (k0 + i * (NT / BM)) : p.terms[c.t].in, v);
      }
    }
    {
      const int jj = tid % BN;
#pragma unroll
      for (int i = 0; i < B_PER_T; ++i) {
        const int kk = tid / BN + i * (NT / BN);
        const bool v = c.bok && (k0 + kk < n);
        cp_async8(bs + kk * SB + jj, v ? c.b + static_cast<int64_t>(k0 + i * (NT / BN)) * n : p.terms[c.t].M, v);
      }
    }
  };
  auto prologue = [&](const Ld& c) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (c.unit < units && s < KT) load_stage(c, s, s);
      cp_async_commit();
    }
  };

  if (static_cast<int64_t>(blockIdx.x) >= units) return;
  Ld cur = make_ld(blockIdx.x, p.groups[blockIdx.x / tiles].t0);
  prologue(cur);

  double acc[MI][NI][2];
  while (cur.unit < units) {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nk = kt + STAGES - 1;
        if (nk < KT) load_stage(cur, nk % STAGES, nk);
        cp_async_commit();
      }
      const double* as = As + (kt % STAGES) * BK * SA + lt * SA + wm0 + lg;
      const double* bs = Bs + (kt % STAGES) * BK * SB + lt * SB + wn0 + lg;
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4) {
        double a[MI], b[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) a[mi] = as[k4 * 4 * SA + mi * 8];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) b[ni] = bs[k4 * 4 * SB + ni * 8];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // every warp is done with the stages: refill them for the next unit

    const Ld done = cur;
    cur = advance(cur);
    prologue(cur);  // overlaps the epilogue below

    // ---- fused linear epilogue (registers → global, loads batched per row) ----
    {
      const int64_t tile = done.unit % tiles;
      const int64_t m0 = (tile / tilesN) * BM;
      const int j0 = static_cast<int>(tile % tilesN) * BN;
      const TermSpec& term = p.terms[done.t];
      if (term.cswap) complex_swap<MI, NI>(acc, lane);
      for (int o = term.out0; o < term.out0 + term.nout; ++o) {
        const OutSpec& os = p.outs[o];
        double* dst = os.dst;
        const double beta = os.beta;
        if (p.remap.world > 0) {  // slab-sharded: stores into the owner rank's region
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) {
            const int64_t m = m0 + wm0 + mi * 8 + lg;
            if (m >= Mtot) continue;
            const int64_t l = KMAJ ? 0 : m % L, r = KMAJ ? m : m / L;
            const int jb = j0 + wn0 + 2 * lt;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int j = jb + ni * 8 + e;
                if (j < n) remote_store(p.remap, os, l, r, j, beta * acc[mi][ni][e]);
              }
          }
          continue;
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const int64_t m = m0 + wm0 + mi * 8 + lg;
          if (m >= Mtot) continue;
          const int64_t rowoff = KMAJ ? m * n : row_offset(m, L, Ln, small);
          double v[NI][2];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) v[ni][e] = beta * acc[mi][ni][e];
          const int jb = j0 + wn0 + 2 * lt;
          for (int s = os.src0; s < os.src0 + os.nsrc; ++s) {
            const double* src = p.srcs[s].ptr + rowoff;
            const double cf = p.srcs[s].coef;
            double x[NI][2];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int j = jb + ni * 8 + e;
                x[ni][e] = (j < n) ? src[KMAJ ? static_cast<int64_t>(j) : L * j] : 0.0;
              }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) v[ni][e] += cf * x[ni][e];
          }
          double* drow = dst + rowoff;
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int j = jb + ni * 8 + e;
              if (j < n) drow[KMAJ ? static_cast<int64_t>(j) : L * j] = v[ni][e];
            }
        }
      }
    }
  }
  cp_async_wait<0>();
  if (p.remap.world > 0) __threadfence_system();  // peer stores visible before the barrier kernel
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MINB>
static cudaError_t launch_cfg(const ModeParams& p, cudaStream_t st) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr size_t smem = static_cast<size_t>(STAGES) * BK * ((BM + 4) + (BN + 4)) * sizeof(double);
  static int sms = 0;
  static int occ[2] = {0, 0};
  const int64_t Mtot = p.L * p.R;
  const int64_t units = ((Mtot + BM - 1) / BM) * ((p.n + BN - 1) / BN) * p.ngroups;
  const bool kmaj = p.L == 1;
  auto k = kmaj ? mode_product_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, MINB, true>
                : mode_product_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, MINB, false>;
  if (occ[kmaj] == 0) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, NT, smem);
    if (e != cudaSuccess) return e;
    occ[kmaj] = o > 0 ? o : 1;
  }
  int64_t grid = static_cast<int64_t>(sms) * occ[kmaj];
  if (grid > units) grid = units;
  if (grid < 1) return cudaSuccess;
  k<<<static_cast<unsigned>(grid), NT, smem, st>>>(p);
  return cudaGetLastError();
}

// ===========================================================================
// TMA + mbarrier variant (the regular, large case).  One elected thread issues
// the two bulk-tensor copies of every K-chunk (A tile of the tensor, B tile of
// the matrix) into a STAGES-deep ring; all warps run DMMA and release a stage
// by arriving on its "empty" mbarrier, so the mainloop has no CTA-wide
// barrier and no per-thread address arithmetic.  The boxes are 4 elements
// wider than the tile so the smem rows come out padded (conflict-free 64-bit
// fragment loads) without a swizzle.
// ===========================================================================
struct TmaMaps {
  CUtensorMap a[kMaxTerms];
  CUtensorMap b[kMaxTerms];
};

namespace {
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

template <int BM, int BN, int BK, int KMAJ>
struct TmaGeom {
  static constexpr int SA = KMAJ ? (BK + 4) : (BM + 4);          // smem row stride of A
  static constexpr int A_ELEMS = KMAJ ? BM * (BK + 4) : BK * (BM + 4);
  static constexpr int SB = BN + 4;
  static constexpr int B_ELEMS = BK * (BN + 4);
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static_assert((A_ELEMS * 8) % 128 == 0 && (B_ELEMS * 8) % 128 == 0, "128B-aligned stage tiles");
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MINB, bool KMAJ, bool REMOTE = false,
          bool CPLX = false>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, MINB)
    mode_product_tma_kernel(const __grid_constant__ ModeParams p, const __grid_constant__ TmaMaps tm) {
  constexpr int NWARPS = WARPS_M * WARPS_N;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int MI = WM / 8, NI = WN / 8;
  using G = TmaGeom<BM, BN, BK, KMAJ>;
  constexpr unsigned STAGE_BYTES = G::STAGE_ELEMS * 8;

  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * G::STAGE_ELEMS);
  uint64_t* empty = full + STAGES;

  const int n = p.n;
  const int64_t L = p.L, R = p.R;
  const int64_t Ln = L * static_cast<int64_t>(n);
  const int tilesN = (n + BN - 1) / BN;
  const int64_t rowtilesPerSlab = KMAJ ? (R + BM - 1) / BM : (L + BM - 1) / BM;
  const int64_t rowtiles = KMAJ ? rowtilesPerSlab : rowtilesPerSlab * R;
  const int64_t tiles = rowtiles * tilesN;
  const int64_t units = tiles * p.ngroups;
  const int KT = (n + BK - 1) / BK;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm0 = (warp / WARPS_N) * WM;
  const int wn0 = (warp % WARPS_N) * WN;
  const int lg = lane >> 2, lt = lane & 3;

  if (static_cast<int64_t>(blockIdx.x) >= units) return;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // tile geometry of a unit: row origin (l0, r) or r0, column origin j0
  struct Tile {
    int64_t l0, r;  // non-KMAJ: rows l0..l0+BM of slab r; KMAJ: rows r..r+BM (l0 unused)
    int j0;
  };
  auto tile_of = [&](int64_t unit) -> Tile {
    const int64_t tile = unit % tiles;
    const int64_t rt = tile / tilesN;
    Tile T;
    T.j0 = static_cast<int>(tile % tilesN) * BN;
    if (KMAJ) {
      T.l0 = 0;
      T.r = rt * BM;
    } else {
      T.r = rt / rowtilesPerSlab;
      T.l0 = (rt % rowtilesPerSlab) * BM;
    }
    return T;
  };

  // ---- producer cursor (thread 0 only); the unit's tile coordinates and term
  // range are decoded once per unit (64-bit divisions), not per chunk ----
  int64_t p_unit = blockIdx.x;
  int p_t = p.groups[p_unit / tiles].t0, p_t1 = p.groups[p_unit / tiles].t1, p_kt = 0;
  int p_c0 = 0, p_c1 = 0, p_c2 = 0;  // TMA coordinates of the unit's A (c1 = k) and B tiles
  auto p_decode = [&]() {
    const Tile T = tile_of(p_unit);
    p_c0 = static_cast<int>(KMAJ ? T.r : T.l0);
    p_c2 = static_cast<int>(T.r);
    p_c1 = T.j0;
  };
  p_decode();
  uint32_t p_it = 0;  // chunks issued
  auto produce_one = [&]() {
    if (p_unit >= units) return;
    const uint32_t s = p_it % STAGES;
    if (p_it >= STAGES) mbar_wait(&empty[s], ((p_it / STAGES) - 1) & 1);
    double* as = smem + s * G::STAGE_ELEMS;
    double* bs = as + G::A_ELEMS;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    const int k0 = p_kt * BK;
    if (KMAJ)
      tma_load_2d(as, &tm.a[p_t], k0, p_c0, &full[s]);
    else
      tma_load_3d(as, &tm.a[p_t], p_c0, k0, p_c2, &full[s]);
    tma_load_2d(bs, &tm.b[p_t], p_c1, k0, &full[s]);
    ++p_it;
    if (++p_kt == KT) {
      p_kt = 0;
      if (p_t + 1 < p_t1) {
        ++p_t;
      } else {
        p_unit += gridDim.x;
        if (p_unit < units) {
          const GroupSpec g = p.groups[p_unit / tiles];
          p_t = g.t0;
          p_t1 = g.t1;
          p_decode();
        }
      }
    }
  };
  if (tid == 0)
    for (int s = 0; s < STAGES - 1; ++s) produce_one();

  uint32_t it = 0;  // chunks consumed
  double acc[MI][NI][2];
  for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const GroupSpec g = p.groups[unit / tiles];
    const Tile T = tile_of(unit);
    for (int t = g.t0; t < g.t1; ++t) {
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const uint32_t s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const double* as = smem + s * G::STAGE_ELEMS;
        const double* bs = as + G::A_ELEMS + lt * G::SB + wn0 + lg;
        const double* aw = KMAJ ? as + (wm0 + lg) * G::SA + lt : as + lt * G::SA + wm0 + lg;
#pragma unroll
        for (int k4 = 0; k4 < BK / 4; ++k4) {
          double a[MI], b[NI];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) a[mi] = KMAJ ? aw[mi * 8 * G::SA + k4 * 4] : aw[k4 * 4 * G::SA + mi * 8];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) b[ni] = bs[k4 * 4 * G::SB + ni * 8];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (tid == 0) produce_one();
      }

      // ---- fused linear epilogue ----
      const TermSpec& term = p.terms[t];
      if (CPLX && term.cswap) complex_swap<MI, NI>(acc, lane);
      for (int o = term.out0; o < term.out0 + term.nout; ++o) {
        const OutSpec& os = p.outs[o];
        double* dst = os.dst;
        const double beta = os.beta;
        const bool vec_ok = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
        if (REMOTE) {  // slab-sharded: stores into the owner rank's region
          const Remap& rm = p.remap;
          const int jb = T.j0 + wn0 + 2 * lt;
          if (rm.uniform && (rm.cq & 1) == 0) {
            // columns (j, j+1) share their owner: resolve owner and column base once per
            // 8-column group, then every row is one add
            double* colp[NI];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
              const int j = jb + ni * 8;
              const int k = j < n ? j / rm.cq : 0;
              colp[ni] = reinterpret_cast<double*>(rm.base[k] + reinterpret_cast<uintptr_t>(os.dst)) + rm.kroff[0] +
                         rm.colstride * static_cast<int64_t>(j - rm.kstart[k]);
            }
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              const int64_t rl = wm0 + mi * 8 + lg;
              int64_t l, r;
              if (KMAJ) {
                l = 0;
                r = T.r + rl;
                if (r >= R) continue;
              } else {
                l = T.l0 + rl;
                r = T.r;
                if (l >= L) continue;
              }
              const int64_t rowb = l + rm.kstride[0] * r;
#pragma unroll
              for (int ni = 0; ni < NI; ++ni) {
                const int j = jb + ni * 8;
                if (j < n) colp[ni][rowb] = beta * acc[mi][ni][0];
                if (j + 1 < n) colp[ni][rowb + rm.colstride] = beta * acc[mi][ni][1];
              }
            }
          } else {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              const int64_t rl = wm0 + mi * 8 + lg;
              int64_t l, r;
              if (KMAJ) {
                l = 0;
                r = T.r + rl;
                if (r >= R) continue;
              } else {
                l = T.l0 + rl;
                r = T.r;
                if (l >= L) continue;
              }
#pragma unroll
              for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int j = jb + ni * 8 + e;
                  if (j < n) remote_store(rm, os, l, r, j, beta * acc[mi][ni][e]);
                }
            }
          }
          continue;
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const int64_t rl = wm0 + mi * 8 + lg;
          int64_t rowoff;
          if (KMAJ) {
            const int64_t r = T.r + rl;
            if (r >= R) continue;
            rowoff = r * n;
          } else {
            const int64_t l = T.l0 + rl;
            if (l >= L) continue;
            rowoff = l + Ln * T.r;
          }
          double v[NI][2];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) v[ni][e] = beta * acc[mi][ni][e];
          const int jb = T.j0 + wn0 + 2 * lt;
          for (int s = os.src0; s < os.src0 + os.nsrc; ++s) {
            const double* src = p.srcs[s].ptr + rowoff;
            const double cf = p.srcs[s].coef;
            double x[NI][2];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int j = jb + ni * 8 + e;
                x[ni][e] = (j < n) ? src[KMAJ ? static_cast<int64_t>(j) : L * j] : 0.0;
              }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) v[ni][e] += cf * x[ni][e];
          }
          double* drow = dst + rowoff;
          if (KMAJ && vec_ok) {  // (j, j+1) adjacent: one 16-byte store (n even on this path)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
              const int j = jb + ni * 8;
              if (j < n) *reinterpret_cast<double2*>(drow + j) = make_double2(v[ni][0], v[ni][1]);
            }
          } else {
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int j = jb + ni * 8 + e;
                if (j < n) drow[KMAJ ? static_cast<int64_t>(j) : L * j] = v[ni][e];
              }
          }
        }
      }
    }
  }
  if (REMOTE) __threadfence_system();  // peer stores visible before the barrier kernel
}

// ---- host side: tensor-map encoding through the runtime's driver entry point ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static const EncodeTiledFn fn = [] {  // thread-safe one-time lookup
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(f);
    return static_cast<EncodeTiledFn>(nullptr);
  }();
  return fn;
}

static bool encode(CUtensorMap* m, const double* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MINB, bool REMOTE = false,
          bool CPLX = false>
static bool launch_tma(const ModeParams& p, cudaStream_t st, cudaError_t* err) {
  const bool kmaj = p.L == 1;
  const int n = p.n;
  // TMA preconditions: 16-byte strides and base addresses; rows long enough to tile
  if (n % 2 != 0) return false;
  if (!kmaj && (p.L % 2 != 0 || p.L < BM / 2)) return false;
  if (p.L * p.R > (int64_t(1) << 31) * 8) return false;
  int nterms = 0;
  for (int g = 0; g < p.ngroups; ++g) nterms = p.groups[g].t1 > nterms ? p.groups[g].t1 : nterms;
  TmaMaps maps;  // per call (12 KB on the host stack): distinct handles may launch from different threads
  for (int t = 0; t < nterms; ++t) {
    if ((reinterpret_cast<uintptr_t>(p.terms[t].in) | reinterpret_cast<uintptr_t>(p.terms[t].M)) & 15) return false;
  }
  for (int t = 0; t < nterms; ++t) {
    bool ok;
    if (kmaj) {
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(p.R)};
      const cuuint64_t str[1] = {static_cast<cuuint64_t>(n) * 8};
      const cuuint32_t box[2] = {BK + 4, BM};
      ok = encode(&maps.a[t], p.terms[t].in, 2, dims, str, box);
    } else {
      const cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.L), static_cast<cuuint64_t>(n),
                                  static_cast<cuuint64_t>(p.R)};
      const cuuint64_t str[2] = {static_cast<cuuint64_t>(p.L) * 8, static_cast<cuuint64_t>(p.L) * n * 8};
      const cuuint32_t box[3] = {BM + 4, BK, 1};
      ok = encode(&maps.a[t], p.terms[t].in, 3, dims, str, box);
    }
    const cuuint64_t bd[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(n)};
    const cuuint64_t bs[1] = {static_cast<cuuint64_t>(n) * 8};
    const cuuint32_t bb[2] = {BN + 4, BK};
    ok = ok && encode(&maps.b[t], p.terms[t].M, 2, bd, bs, bb);
    if (!ok) return false;
  }
  constexpr int NT = WARPS_M * WARPS_N * 32;
  static int sms = 0;
  static bool attr[2] = {false, false};
  const int64_t rowtiles = kmaj ? (p.R + BM - 1) / BM : ((p.L + BM - 1) / BM) * p.R;
  const int64_t units = rowtiles * ((n + BN - 1) / BN) * p.ngroups;
  if (kmaj) {
    using Gm = TmaGeom<BM, BN, BK, 1>;
    constexpr size_t smem = static_cast<size_t>(STAGES) * Gm::STAGE_ELEMS * 8 + 2 * STAGES * 8;
    auto k = mode_product_tma_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, MINB, true, REMOTE, CPLX>;
    if (!attr[1]) {
      *err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (*err != cudaSuccess) return true;
      attr[1] = true;
    }
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t grid = units < (int64_t)sms * MINB ? units : (int64_t)sms * MINB;
    k<<<static_cast<unsigned>(grid), NT, smem, st>>>(p, maps);
  } else {
    using Gm = TmaGeom<BM, BN, BK, 0>;
    constexpr size_t smem = static_cast<size_t>(STAGES) * Gm::STAGE_ELEMS * 8 + 2 * STAGES * 8;
    auto k = mode_product_tma_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, MINB, false, REMOTE, CPLX>;
    if (!attr[0]) {
      *err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (*err != cudaSuccess) return true;
      attr[0] = true;
    }
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t grid = units < (int64_t)sms * MINB ? units : (int64_t)sms * MINB;
    k<<<static_cast<unsigned>(grid), NT, smem, st>>>(p, maps);
  }
  *err = cudaGetLastError();
  return true;
}

cudaError_t launch_mode_product(const ModeParams& p, cudaStream_t st) {
  if (p.ngroups == 0) return cudaSuccess;
  const int64_t Mtot = p.L * p.R;
  if (p.remap.world > 0 && p.n > 64) {  // slab-sharded peer-store epilogue: default tile only
    cudaError_t err = cudaSuccess;
    if (launch_tma<64, 128, 16, 2, 2, 4, 2, true>(p, st, &err)) return err;
    return launch_cfg<64, 64, 16, 2, 2, 4, 3>(p, st);
  }
  bool cswap = false;
  for (int g = 0; g < p.ngroups; ++g)
    for (int t = p.groups[g].t0; t < p.groups[g].t1; ++t) cswap |= p.terms[t].cswap != 0;
  if (cswap) {  // complex modes μ ≥ 2: the J-swap instantiation (real launches keep the lean one)
    if (p.n > 64) {
      cudaError_t err = cudaSuccess;
      const int64_t units = ((Mtot + 63) / 64) * ((p.n + 127) / 128) * p.ngroups;
      const bool done = units >= 148 * 2 ? launch_tma<64, 128, 16, 2, 2, 4, 2, false, true>(p, st, &err)
                                         : launch_tma<64, 64, 16, 2, 2, 4, 3, false, true>(p, st, &err);
      if (done) return err;
    }
  } else if (p.n > 64) {
    // tile sweep (128×128 / 8 warps, 128×64 / 3 stages, cp.async only) measured slower:
    // DESIGN.md §4, profiles/r01_tile_sweep.jsonl
    cudaError_t err = cudaSuccess;
    bool done = false;
    const int64_t units = ((Mtot + 63) / 64) * ((p.n + 127) / 128) * p.ngroups;
    // far less than a wave of 64×64 tiles (the n×n GEMMs of a sharded rank's exponential stage,
    // a few matrices each): 32×32 tiles, 4× the CTAs, each a quarter of the serial K loop
    if (p.n <= 256 && ((Mtot + 63) / 64) * ((p.n + 63) / 64) * p.ngroups < 148 / 2) return launch_cfg<32, 32, 16, 2, 2, 4, 4>(p, st);
    if (units >= 148 * 2)
      done = launch_tma<64, 128, 16, 2, 2, 4, 2>(p, st, &err);  // default: 2 CTAs/SM overlap epilogues
    else  // less than a wave (e.g. the n×n GEMMs of the exponential stage): 64×64 tiles, 3 CTAs/SM
      done = launch_tma<64, 64, 16, 2, 2, 4, 3>(p, st, &err);
    if (done) return err;
  }
  // cp.async kernel: shapes TMA cannot take (odd n, odd or short L, misaligned pointers), n ≤ 64
  if (p.n > 64) {
    if (Mtot * ((p.n + 127) / 128) * p.ngroups < 148 * 4) return launch_cfg<64, 64, 16, 2, 2, 4, 3>(p, st);
    return launch_cfg<128, 128, 16, 2, 4, 4, 1>(p, st);
  }
  if (p.n > 32) return launch_cfg<128, 64, 16, 4, 2, 4, 1>(p, st);
  return launch_cfg<64, 32, 16, 4, 2, 4, 1>(p, st);
}

// ---------------------------------------------------------------------------
// Elementwise multi-output linear combination.
// ---------------------------------------------------------------------------
__global__ void combine_kernel(const __grid_constant__ CombineParams p) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < p.count; i += stride) {
    for (int o = 0; o < p.nout; ++o) {
      const OutSpec os = p.outs[o];
      double v = 0.0;
      for (int s = os.src0; s < os.src0 + os.nsrc; ++s) v += p.srcs[s].coef * p.srcs[s].ptr[i];
      os.dst[i] = v;
    }
  }
}

cudaError_t launch_combine(const CombineParams& p, cudaStream_t st) {
  if (p.nout == 0 || p.count == 0) return cudaSuccess;
  int64_t blocks = (p.count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  combine_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Matrix-form combination, two elements (16 B) per thread per step; sources
// stream once, the nout accumulators stay in registers.
// ---------------------------------------------------------------------------
template <int NOUT>
__global__ void __launch_bounds__(256) multi_combine_kernel(const __grid_constant__ MultiCombineParams p) {
  const int64_t n2 = p.count / 2;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 acc[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) acc[o] = make_double2(0.0, 0.0);
    int s = 0;
    for (; s + 4 <= p.nsrc; s += 4) {
      double2 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldcs(reinterpret_cast<const double2*>(p.src[s + u]) + i);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          const double c = p.coef[o][s + u];
          acc[o].x += c * x[u].x;
          acc[o].y += c * x[u].y;
        }
    }
    for (; s < p.nsrc; ++s) {
      const double2 x = __ldcs(reinterpret_cast<const double2*>(p.src[s]) + i);
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        acc[o].x += p.coef[o][s] * x.x;
        acc[o].y += p.coef[o][s] * x.y;
      }
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
      if (o < p.nout) reinterpret_cast<double2*>(p.dst[o])[i] = acc[o];
  }
  // odd tail element
  if (p.count & 1) {
    const int64_t i = p.count - 1;
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int o = 0; o < p.nout; ++o) {
        double v = 0.0;
        for (int s = 0; s < p.nsrc; ++s) v += p.coef[o][s] * p.src[s][i];
        p.dst[o][i] = v;
      }
  }
}

cudaError_t launch_multi_combine(const MultiCombineParams& p, cudaStream_t st) {
  if (p.nout == 0 || p.count == 0) return cudaSuccess;
  bool aligned = true;
  for (int s = 0; s < p.nsrc; ++s) aligned &= (reinterpret_cast<uintptr_t>(p.src[s]) & 15) == 0;
  for (int o = 0; o < p.nout; ++o) aligned &= (reinterpret_cast<uintptr_t>(p.dst[o]) & 15) == 0;
  if (!aligned) return cudaErrorMisalignedAddress;
  int64_t blocks = (p.count / 2 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  switch (p.nout <= 2 ? 2 : (p.nout <= 4 ? 4 : 8)) {
    case 2: multi_combine_kernel<2><<<static_cast<unsigned>(blocks), 256, 0, st>>>(p); break;
    case 4: multi_combine_kernel<4><<<static_cast<unsigned>(blocks), 256, 0, st>>>(p); break;
    default: multi_combine_kernel<8><<<static_cast<unsigned>(blocks), 256, 0, st>>>(p); break;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Deterministic sum of squares (two passes, fixed reduction order).
// ---------------------------------------------------------------------------
constexpr int kSumsqBlocks = 1024;
struct VecList {
  const double* v[kMaxVecs];
};

__device__ __forceinline__ double block_sum(double x) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = x;
  __syncthreads();
  x = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void sumsq_pass1(VecList vl, int64_t count, double* partial) {
  const double* __restrict__ v = vl.v[blockIdx.y];
  double s = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = v[i];
    s += x * x;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.y * kSumsqBlocks + blockIdx.x] = s;
}

__global__ void sumsq_pass2(const double* partial, double* norms2) {
  double s = 0.0;
  for (int i = threadIdx.x; i < kSumsqBlocks; i += blockDim.x) s += partial[blockIdx.x * kSumsqBlocks + i];
  s = block_sum(s);
  if (threadIdx.x == 0) norms2[blockIdx.x] = s;
}

cudaError_t launch_sumsq(const double* const* vecs, int nvec, int64_t count, double* scratch,
                         double* norms2, cudaStream_t st) {
  if (nvec <= 0) return cudaSuccess;
  if (nvec > kMaxVecs) return cudaErrorInvalidValue;
  VecList vl{};
  for (int i = 0; i < nvec; ++i) vl.v[i] = vecs[i];
  sumsq_pass1<<<dim3(kSumsqBlocks, nvec), 256, 0, st>>>(vl, count, scratch);
  sumsq_pass2<<<nvec, 256, 0, st>>>(scratch, norms2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Peer-store copy of a local (L, n, R) tensor with the Remap of a sharded stage
// (complex sharded handles: the complex μ-mode product is two accumulating real
// products, computed locally, then moved to the owners by this kernel).
__global__ void remap_copy_kernel(const double* __restrict__ src, int64_t L, int n, int64_t R, size_t dst_off,
                                  const __grid_constant__ Remap rm) {
  const int64_t total = L * n * R;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t l = e % L;
    const int64_t t = e / L;
    const int j = static_cast<int>(t % n);
    const int64_t r = t / n;
    const int k = remap_owner(rm, j);
    double* base = reinterpret_cast<double*>(rm.base[k] + dst_off);
    base[l + rm.kstride[k] * r + rm.kroff[k] + rm.colstride * static_cast<int64_t>(j - rm.kstart[k])] = src[e];
  }
  __syncthreads();
  __threadfence_system();
}

cudaError_t launch_remap_copy(const double* src, int64_t L, int n, int64_t R, size_t dst_off, const Remap& rm,
                              cudaStream_t st) {
  const int64_t total = L * n * R;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) return cudaSuccess;
  remap_copy_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src, L, n, R, dst_off, rm);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Real and imaginary parts of a complex n×n matrix from its interleaved real
// form R (2n×2n column-major, R[(c+2j) + (c'+2k)·2n] = [[Mr, −Mi], [Mi, Mr]]_{cc'}(j,k)).
__global__ void complex_parts_kernel(const double* R, int n, double* Mr, double* Mi) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nn;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i % n, k = i / n;
    const int64_t col = 2 * k * (2 * static_cast<int64_t>(n));
    Mr[i] = R[2 * j + col];
    Mi[i] = R[2 * j + 1 + col];
  }
}

cudaError_t launch_complex_parts(const double* R, int n, double* Mr, double* Mi, cudaStream_t st) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  int64_t blocks = (nn + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  complex_parts_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(R, n, Mr, Mi);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
__global__ void set_identity_kernel(double* E, int n, double diag) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nn;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    E[i] = (i % (n + 1) == 0) ? diag : 0.0;
}

cudaError_t launch_set_identity(double* E, int n, double diag, cudaStream_t st) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  int64_t blocks = (nn + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  set_identity_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(E, n, diag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FP64 peak microbenchmark: 16 independent register-resident chains per thread.
// ---------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(256) fp64_peak_kernel(int64_t iters, double* sink) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  double a = 1.0 + 1e-9 * (threadIdx.x & 7), b = 1.0 - 1e-9 * (threadIdx.x & 3);
  double c[16][2];
#pragma unroll
  for (int u = 0; u < 16; ++u) c[u][0] = c[u][1] = 1e-3 * u;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (KIND == 0) {
        dmma8x8x4(c[u][0], c[u][1], a, b);
      } else {
        c[u][0] = fma(a, c[u][0], b);
        c[u][1] = fma(b, c[u][1], a);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += c[u][0] + c[u][1];
  sink[tid] = s;
}

cudaError_t launch_fp64_peak(int kind, int blocks, int64_t iters, double* sink, cudaStream_t st,
                             double* flops) {
  if (kind == 0) {
    fp64_peak_kernel<0><<<blocks, 256, 0, st>>>(iters, sink);
    // per warp per iteration: 16 DMMA.8x8x4 = 16 * 8*8*4 FMA = 16 * 512 flops
    *flops = static_cast<double>(blocks) * 8.0 * static_cast<double>(iters) * 16.0 * 512.0;
  } else {
    fp64_peak_kernel<1><<<blocks, 256, 0, st>>>(iters, sink);
    *flops = static_cast<double>(blocks) * 256.0 * static_cast<double>(iters) * 32.0 * 2.0;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Cross-rank barrier and small scatter of the slab-sharded path (peer memory
// mapped through CUDA IPC; every pointer below may live on another GPU).
// ---------------------------------------------------------------------------
__global__ void barrier_kernel(const __grid_constant__ BarrierParams p) {
  const int t = threadIdx.x;
  // fail fast: once a barrier of this rank has timed out (sticky flag, reported by phiks_wait /
  // phiks_get_stats / the next apply), later barriers return at once instead of waiting out
  // their own timeouts one after another
  int failed;
  asm volatile("ld.volatile.global.s32 %0, [%1];\n" : "=r"(failed) : "l"(p.err));
  if (failed) return;
  __shared__ uint64_t epoch;
  if (t == 0) {
    epoch = *p.epoch + 1;  // only this (stream-ordered) kernel touches the counter
    *p.epoch = epoch;
  }
  __threadfence_system();
  __syncthreads();
  if (t < p.world) {
    uint64_t* slot = p.peer_flags[t] + p.rank;  // my slot in peer t's array
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(slot), "l"(epoch) : "memory");
  }
  if (t < p.world) {
    const uint64_t* mine = p.peer_flags[p.rank] + t;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t0));
    while (true) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(mine) : "memory");
      if (v >= epoch) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(now));
      if (now - t0 > p.timeout_ns) {
        atomicExch(p.err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
}

cudaError_t launch_barrier(const BarrierParams& p, cudaStream_t st) {
  if (p.world <= 1) return cudaSuccess;
  barrier_kernel<<<1, 32, 0, st>>>(p);
  return cudaGetLastError();
}

__global__ void scatter_small_kernel(const __grid_constant__ ScatterParams p) {
  for (int i = threadIdx.x; i < p.cnt * p.world; i += blockDim.x) {
    const int k = i / p.cnt, c = i % p.cnt;
    p.dst[k][p.rank * p.cnt + c] = p.src[c];
  }
  __syncthreads();
  __threadfence_system();
}

cudaError_t launch_scatter_small(const ScatterParams& p, cudaStream_t st) {
  scatter_small_kernel<<<1, 128, 0, st>>>(p);
  return cudaGetLastError();
}

__global__ void peer_copy_kernel(const __grid_constant__ PeerCopyParams p) {
  const int i = blockIdx.y;
  const int64_t cnt = p.count[i];
  const double* src = p.src[i];
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < cnt;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = src[e];
    for (int k = 0; k < p.world; ++k) reinterpret_cast<double*>(p.base[k] + p.off[i])[e] = v;
  }
  __threadfence_system();  // peer stores visible before the barrier kernel that follows
}

cudaError_t launch_peer_copy(const PeerCopyParams& p, cudaStream_t st) {
  if (p.nitems == 0) return cudaSuccess;
  int64_t mx = 0;
  for (int i = 0; i < p.nitems; ++i) mx = mx > p.count[i] ? mx : p.count[i];
  const unsigned bx = static_cast<unsigned>(std::min<int64_t>((mx + 255) / 256, 64));
  peer_copy_kernel<<<dim3(bx, p.nitems), 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace phiks
