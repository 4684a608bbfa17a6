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

}  // namespace

// ---------------------------------------------------------------------------
// μ-mode product: GEMM rows m ∈ [0, L·R) (m = l + L·r), columns j ∈ [0, n),
// contraction k ∈ [0, n).  A operand = input tensor tile (m, k) at
// off(m,k) = (m mod L) + L·k + L·n·(m div L); B operand = M^T tile (k, j) at
// j + k·n.  KMAJ (L == 1): off(m,k) = m·n + k, the contraction index is the
// contiguous one, so the loader walks k across threads.
// ---------------------------------------------------------------------------
template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool KMAJ>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, 1)
    mode_product_kernel(const __grid_constant__ ModeParams p) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int MI = WM / 8, NI = WN / 8;
  constexpr int SA = BM + 4, SB = BN + 4;  // padded strides: 64-bit fragment loads conflict-free
  constexpr int A_PER_T = BM * BK / NT, B_PER_T = BK * BN / NT;
  static_assert(WM % 8 == 0 && WN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert(NT % BM == 0 || KMAJ, "non-KMAJ loader assumes NT % BM == 0");
  static_assert(NT % BK == 0, "KMAJ loader assumes NT % BK == 0");
  static_assert(NT % BN == 0, "B loader assumes NT % BN == 0");

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * BK * SA;

  const int n = p.n;
  const int64_t L = p.L;
  const int64_t Mtot = L * p.R;
  const int64_t Ln = L * static_cast<int64_t>(n);
  const int tilesN = (n + BN - 1) / BN;
  const int64_t tile = blockIdx.x;
  const int tn = static_cast<int>(tile % tilesN);
  const int64_t m0 = (tile / tilesN) * BM;
  const int j0 = tn * BN;
  const GroupSpec g = p.groups[blockIdx.y];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm0 = (warp / WARPS_N) * WM;
  const int wn0 = (warp % WARPS_N) * WN;
  const int lg = lane >> 2, lt = lane & 3;

  // ---- per-thread loader bookkeeping (independent of the term) ----
  // A (non-KMAJ): this thread loads row mm = tid % BM at k = tid / BM + i*(NT/BM)
  // A (KMAJ):     this thread loads k = tid % BK at rows mm = tid / BK + i*(NT/BK)
  // B:            this thread loads column jj = tid % BN at k = tid / BN + i*(NT/BN)
  int64_t a_off0;      // element offset of this thread's first A element at k0 = 0
  bool a_rowok;        // non-KMAJ: row valid
  int a_k;             // k index of the first element (relative to k0)
  if (!KMAJ) {
    const int64_t m = m0 + (tid % BM);
    a_rowok = m < Mtot;
    a_k = tid / BM;
    a_off0 = a_rowok ? (m % L) + Ln * (m / L) + L * a_k : 0;
  } else {
    a_rowok = true;
    a_k = tid % BK;
    a_off0 = (m0 + tid / BK) * n + a_k;
  }
  const int b_j = j0 + tid % BN;
  const int b_k = tid / BN;
  const bool b_jok = b_j < n;

  const int KT = (n + BK - 1) / BK;

  for (int t = g.t0; t < g.t1; ++t) {
    const TermSpec term = p.terms[t];
    const double* __restrict__ in = term.in;
    const double* __restrict__ M = term.M;

    auto load_stage = [&](int stage, int kt) {
      const int k0 = kt * BK;
      double* as = As + stage * BK * SA;
      double* bs = Bs + stage * BK * SB;
      if (KMAJ) {
        const bool kok = (k0 + a_k) < n;
        const double* src = in + a_off0 + k0;
#pragma unroll
        for (int i = 0; i < A_PER_T; ++i) {
          const int mm = tid / BK + i * (NT / BK);
          const bool v = kok && (m0 + mm < Mtot);
          cp_async8(as + a_k * SA + mm, v ? src + static_cast<int64_t>(i) * (NT / BK) * n : in, v);
        }
      } else {
        const double* src = in + a_off0 + L * k0;
#pragma unroll
        for (int i = 0; i < A_PER_T; ++i) {
          const int kk = a_k + i * (NT / BM);
          const bool v = a_rowok && (k0 + kk < n);
          cp_async8(as + kk * SA + (tid % BM), v ? src + L * (i * (NT / BM)) : in, v);
        }
      }
      {
        const double* src = M + b_j + static_cast<int64_t>(k0 + b_k) * n;
#pragma unroll
        for (int i = 0; i < B_PER_T; ++i) {
          const int kk = b_k + i * (NT / BN);
          const bool v = b_jok && (k0 + kk < n);
          cp_async8(bs + kk * SB + (tid % BN), v ? src + static_cast<int64_t>(i) * (NT / BN) * n : M, v);
        }
      }
    };

    double acc[MI][NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < KT) load_stage(s, s);
      cp_async_commit();
    }

    for (int kt = 0; kt < KT; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nk = kt + STAGES - 1;
        if (nk < KT) load_stage(nk % STAGES, nk);
        cp_async_commit();
      }
      const double* as = As + (kt % STAGES) * BK * SA + lt * SA + wm0 + lg;
      const double* bs = Bs + (kt % STAGES) * BK * SB + lt * SB + wn0 + lg;
      double a[2][MI], b[2][NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[0][mi] = as[mi * 8];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[0][ni] = bs[ni * 8];
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4) {
        const int cur = k4 & 1;
        if (k4 + 1 < BK / 4) {
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) a[cur ^ 1][mi] = as[(k4 + 1) * 4 * SA + mi * 8];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) b[cur ^ 1][ni] = bs[(k4 + 1) * 4 * SB + ni * 8];
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
            dmma8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[cur][mi], b[cur][ni]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // smem is reused by the next term's prologue

    // ---- fused linear epilogue ----
    for (int o = term.out0; o < term.out0 + term.nout; ++o) {
      const OutSpec os = p.outs[o];
      double* __restrict__ dst = os.dst;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int64_t m = m0 + wm0 + mi * 8 + lg;
        if (m >= Mtot) continue;
        const int64_t rowoff = KMAJ ? m * n : (m % L) + Ln * (m / L);
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = j0 + wn0 + ni * 8 + 2 * lt + e;
            if (j >= n) continue;
            const int64_t off = rowoff + (KMAJ ? static_cast<int64_t>(j) : L * j);
            double v = os.beta * acc[mi][ni][e];
            for (int s = os.src0; s < os.src0 + os.nsrc; ++s) v += p.srcs[s].coef * p.srcs[s].ptr[off];
            dst[off] = v;
          }
        }
      }
    }
  }
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
static cudaError_t launch_cfg(const ModeParams& p, cudaStream_t st) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr size_t smem = static_cast<size_t>(STAGES) * BK * ((BM + 4) + (BN + 4)) * sizeof(double);
  const int64_t Mtot = p.L * p.R;
  const int64_t tiles = ((Mtot + BM - 1) / BM) * ((p.n + BN - 1) / BN);
  if (tiles > 0x7fffffffLL || p.ngroups > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(p.ngroups));
  if (p.L == 1) {
    auto k = mode_product_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, true>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, NT, smem, st>>>(p);
  } else {
    auto k = mode_product_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, NT, smem, st>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_mode_product(const ModeParams& p, cudaStream_t st) {
  if (p.ngroups == 0) return cudaSuccess;
  if (p.n > 64) return launch_cfg<128, 128, 16, 2, 4, 4>(p, st);
  if (p.n > 32) return launch_cfg<128, 64, 16, 4, 2, 4>(p, st);
  return launch_cfg<64, 32, 16, 4, 2, 4>(p, st);
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

}  // namespace phiks
