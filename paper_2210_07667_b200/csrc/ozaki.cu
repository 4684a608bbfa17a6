// fp64 μ-mode products on the int8 tensor cores (tcgen05.mma kind::i8).
//
// DESIGN.md §4c.  The μ-mode product Y = X ×_μ E (§3.1, Eq. (13))
// contracts every mode-μ fiber x_c (c = l + L·r of the (L, n, R) view) with the
// rows e_j of E.  Each fiber and each row is written exactly (up to a
// rounding below 2^{ex-8S}) in S balanced base-256 digits, an error-free
// splitting in the manner of Ozaki:
//     x_c = 2^{ex_c-7} Σ_{s=0..S-1} 256^{-s} a_{c,s},   e_j = 2^{ee_j-7} Σ_t 256^{-t} b_{j,t},
// a, b ∈ [-128, 127]^n integer vectors (|x| < 2^{ex-1} for the whole fiber).
// Then
//     y_{c,j} = 2^{ex_c+ee_j-14} Σ_{g=0..S-1} 256^{-g} D_g,   D_g = Σ_{s+t=g} a_{c,s}·b_{j,t},
// keeping the pairs with s + t < S (the dropped ones are below the
// representation error).  Every D_g is an exact int32 sum (|D_g| ≤ (g+1)·n·2^14
// < 2^31 for n ≤ 512; the E digits stay resident for n ≤ 256 and stream per
// k-block above) accumulated by tcgen05.mma kind::i8 in TMEM, one accumulator
// per diagonal g; the epilogue combines them exactly in 64-bit integers (one
// fp64 rounding for fp64 outputs) and applies the power-of-two scales.  With S = 7 each operand carries
// 55 bits relative to twice its fiber / row maximum, so the error is bounded
// like that of an fp64 dot product, |Δy| ≲ n·2^-52·max|e_j|·max|x_c|.
//
// Kernels: split_x (fibers → K-major int8 digits [slot][s][c][k] + 2^{ex_c}),
// split_e (rows of E → [slot][t][j][k] + 2^{ee_j}), and a persistent
// warp-specialised GEMM: each CTA owns one 64-row tile of E (its digits stay
// resident in shared memory) and walks 128-fiber tiles; TMA (SWIZZLE_32B, 4-D
// maps over (k, row, digit, slot)) streams one digit of one 32-wide k-block per
// stage; one elected thread issues, per stage s, a_s × [b_0 | … | b_{S-1-s}]
// as MMAs of N = 64(S-s) ≤ 256 whose column range is exactly the diagonal
// accumulators s … S-1 (diagonal g at TMEM columns [64g, 64g+64)); 8 epilogue
// warps drain TMEM while the next tile's MMAs run.
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "phiks_internal.h"

namespace phiks {

namespace {

constexpr int kOzBM = 128;  // fibers per tile (UMMA M, TMEM lanes)
constexpr int kOzBN = 64;   // rows of E per tile (UMMA N)
constexpr int kOzBK = 128;  // k per stage (bytes: one SWIZZLE_128B row = 4 UMMA K-steps of 32)
constexpr int kOzUK = 32;   // k per UMMA (int8)

__device__ __forceinline__ unsigned oz_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---- exact splitting into S balanced base-256 digits ----
// |v| < 2^{ex-1}: F = rint(v·2^{8S-1-ex}) (an exact power-of-two scaling and one
// fp64 → int64 conversion, rounded to nearest so that the representation errors
// of a dot product's terms have no common sign), |F| ≤ 2^{8S-2}; G = F + 0x80…80 has bytes d_i + 128,
// d_i the balanced digits of F; digit s (most significant first) = byte S-1-s
// of G ^ 0x80…80.  The scaling is split in two factors when 2^{8S-1-ex}
// overflows (fibers of subnormal magnitude).
struct OzScale {
  double a, b;
  bool two;
};
template <int S>
__device__ __forceinline__ OzScale oz_scale(int ex) {
  const int k = 8 * S - 1 - ex;
  OzScale sc;
  sc.two = k > 1000;
  sc.a = __longlong_as_double(static_cast<long long>((sc.two ? 1000 : k) + 1023) << 52);
  sc.b = __longlong_as_double(static_cast<long long>((sc.two ? k - 1000 : 0) + 1023) << 52);
  return sc;
}
template <int S>
__device__ __forceinline__ uint64_t oz_digits(double v, const OzScale& sc) {
  double t = v * sc.a;
  if (sc.two) t *= sc.b;
  const long long F = __double2ll_rn(t);
  constexpr uint64_t C = 0x8080808080808080ull >> (64 - 8 * S);
  return (static_cast<uint64_t>(F) + C) ^ C;
}
// digit s of 4 consecutive elements as one 32-bit word (element q in byte q)
template <int S>
__device__ __forceinline__ void pack4(const uint64_t (&h)[4], uint32_t (&pk)[S]) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = S - 1 - s;  // byte of the digit
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = static_cast<uint32_t>(h[q] >> (8 * (i & 4)));
    const uint32_t sel = (i & 3) | (((i & 3) + 4) << 4);
    const uint32_t x01 = __byte_perm(w[0], w[1], sel), x23 = __byte_perm(w[2], w[3], sel);
    pk[s] = __byte_perm(x01, x23, 0x5410);
  }
}
template <int S>
__device__ __forceinline__ void split4(const double (&v)[4], int ex, uint32_t (&pk)[S]) {
  const OzScale sc = oz_scale<S>(ex);
  uint64_t h[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) h[q] = oz_digits<S>(v[q], sc);
  pack4<S>(h, pk);
}

__device__ __forceinline__ double warp_max(double m) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

// exponent with |v| < 2^{ex-1} for every |v| ≤ m (m > 0 finite)
__device__ __forceinline__ int slice_exponent(double m) { return m > 0.0 ? ilogb(m) + 2 : 0; }

// ---- split_x: 32 fibers per CTA (256 threads), staged through shared memory ----
template <int S>
__global__ void __launch_bounds__(256) oz_split_x_kernel(const OzakiParams p) {
  extern __shared__ double tile[];  // [32][P], P = n | 1
  const int slot = blockIdx.y;
  const double* X = p.x[slot];
  const int64_t L = p.L, C = p.L * p.R;
  const int n = p.n, P = n | 1, Kp = p.Kp;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nf = static_cast<int>(C - c0 < 32 ? C - c0 : 32);
  if (L == 1) {  // the 32 fibers are one contiguous block of 32·n doubles
    const double* src = X + c0 * n;
    const int total = nf * n;
    for (int i = tid; i < total; i += 256) {
      const int f = i / n, k = i - f * n;
      tile[f * P + k] = __ldg(src + i);
    }
  } else {  // lane → fiber (consecutive l are contiguous), warps over k
    const int64_t c = c0 + lane;
    if (lane < nf) {
      const int64_t l = c % L, r = c / L;
      const double* src = X + l + L * n * r;
#pragma unroll 8
      for (int k = warp; k < n; k += 8) tile[lane * P + k] = __ldg(src + L * k);
    }
  }
  __syncthreads();
  int8_t* xs = p.xs + static_cast<int64_t>(slot) * S * C * Kp;
  // complex products (cplx_j): fibre f is [x_f ; (Jx)_f], (Jx)_f = −x_{f+1} for the real part
  // (f even), +x_{f−1} for the imaginary part (f odd); the blocks start at even fibres
  const int K = p.cplx_j ? 2 * n : n;
  auto val = [&](int f, int k) -> double {
    if (k < n) return tile[f * P + k];
    return (f & 1) ? tile[(f - 1) * P + k - n] : -tile[(f + 1) * P + k - n];
  };
  for (int f = warp; f < nf; f += 8) {
    const int64_t c = c0 + f;
    double m = 0.0;
    bool bad = false;
    for (int k = lane; k < K; k += 32) {
      const double v = val(f, k);
      m = fmax(m, fabs(v));
      bad |= !isfinite(v);
    }
    m = warp_max(m);
    bad = __any_sync(0xffffffffu, bad);
    const int ex = bad ? 0 : slice_exponent(m);
    for (int k0 = 4 * lane; k0 < Kp; k0 += 128) {
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (k0 + q < K && !bad) ? val(f, k0 + q) : 0.0;
      uint32_t pk[S];
      split4<S>(v, ex, pk);
#pragma unroll
      for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(xs + (s * C + c) * Kp + k0) = pk[s];
    }
    if (lane == 0)  // the fiber's exponent (NaN marks a non-finite fiber)
      p.xsc[static_cast<int64_t>(slot) * C + c] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ex;
  }
}

// ---- split_x, contiguous fibers (L = 1): one warp per fiber, values in registers ----
// Lane t holds the EPL = Kp/32 consecutive elements k ∈ [EPL·t, EPL·t + EPL) (zeros past n), so
// every digit plane row is one EPL-byte store per lane.  The fibre exponent comes from the
// maximum of the high words: for non-negative doubles the bit patterns order like the values,
// so the largest high word carries the exponent field of max|x| (ilogb(max) + 2 = field − 1021),
// and a field of 0x7ff marks a non-finite fibre (one REDUX instead of a shuffle tree of fp64
// maxima and per-element finiteness tests: this kernel was integer-ALU bound).
// Maxima of subnormal magnitude (field 0) take the exact fp64 path.
template <int S, int EPL>
__device__ __forceinline__ int oz_fibre_exponent(const double (&v)[EPL], bool& bad) {
  unsigned hm = 0;
#pragma unroll
  for (int q = 0; q < EPL; ++q) hm = max(hm, static_cast<unsigned>(__double2hiint(v[q])) & 0x7fffffffu);
  hm = __reduce_max_sync(0xffffffffu, hm);
  bad = hm >= 0x7ff00000u;
  if (bad) return 0;
  if (hm >= 0x00100000u) return static_cast<int>(hm >> 20) - 1021;
  double m = 0.0;
#pragma unroll
  for (int q = 0; q < EPL; ++q) m = fmax(m, fabs(v[q]));
  return slice_exponent(warp_max(m));
}
// the S digit planes of EPL consecutive elements (EPL % 4 == 0): pk[g][s] holds digit s of
// elements 4g..4g+3 (element q of the group in byte q)
template <int S, int EPL>
__device__ __forceinline__ void oz_split_lane(const double (&v)[EPL], int ex, bool zero, uint32_t (&pk)[EPL / 4][S]) {
  const OzScale sc = oz_scale<S>(ex);
  constexpr uint64_t Cc = 0x8080808080808080ull >> (64 - 8 * S);
#pragma unroll
  for (int g = 0; g < EPL / 4; ++g) {
    uint64_t h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double t = v[4 * g + q] * sc.a;
      if (sc.two) t *= sc.b;
      const long long F = zero ? 0ll : __double2ll_rn(t);
      h[q] = static_cast<uint64_t>(F) + Cc;  // bytes d_i + 128; the ^ 0x80 per packed word below
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = S - 1 - s;
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = static_cast<uint32_t>(h[q] >> (8 * (i & 4)));
      const uint32_t sel = (i & 3) | (((i & 3) + 4) << 4);
      pk[g][s] = __byte_perm(__byte_perm(w[0], w[1], sel), __byte_perm(w[2], w[3], sel), 0x5410) ^ 0x80808080u;
    }
  }
}
// one EPL-byte store per digit plane (dst: plane 0 of this lane's bytes, 4·EPL-aligned offsets)
template <int S, int EPL>
__device__ __forceinline__ void oz_store_lane(int8_t* dst, int64_t plane, const uint32_t (&pk)[EPL / 4][S]) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    int8_t* d = dst + s * plane;
    if constexpr (EPL == 16)
      *reinterpret_cast<uint4*>(d) = make_uint4(pk[0][s], pk[1][s], pk[2][s], pk[3][s]);
    else if constexpr (EPL == 8)
      *reinterpret_cast<uint2*>(d) = make_uint2(pk[0][s], pk[1][s]);
    else
#pragma unroll
      for (int g = 0; g < EPL / 4; ++g) reinterpret_cast<uint32_t*>(d)[g] = pk[g][s];
  }
}
template <int EPL>
__device__ __forceinline__ void oz_load_lane(const double* src, int k0, int n, bool vec, double (&v)[EPL]) {
  if (vec) {  // n == Kp, 16-byte aligned fibres
#pragma unroll
    for (int i = 0; i < EPL / 2; ++i) {
      const double2 a = __ldcs(reinterpret_cast<const double2*>(src + k0) + i);
      v[2 * i] = a.x;
      v[2 * i + 1] = a.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < EPL; ++q) v[q] = k0 + q < n ? __ldg(src + k0 + q) : 0.0;
  }
}
template <int S, int EPL>
__global__ void __launch_bounds__(256) oz_split_x_contig_kernel(const OzakiParams p) {
  const int slot = blockIdx.y;
  const int64_t C = p.R;
  const int n = p.n, Kp = p.Kp;  // Kp = 32·EPL
  const int lane = threadIdx.x & 31;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (c >= C) return;
  const int k0 = EPL * lane;
  double v[EPL];
  oz_load_lane<EPL>(p.x[slot] + c * n, k0, n, n == Kp && (reinterpret_cast<uintptr_t>(p.x[slot]) & 15) == 0, v);
  bool bad;
  const int ex = oz_fibre_exponent<S, EPL>(v, bad);
  uint32_t pk[EPL / 4][S];
  oz_split_lane<S, EPL>(v, ex, bad, pk);
  oz_store_lane<S, EPL>(p.xs + (static_cast<int64_t>(slot) * S * C + c) * Kp + k0, C * Kp, pk);
  if (lane == 0) p.xsc[static_cast<int64_t>(slot) * C + c] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ex;
}

// ---- streaming combination fused with the next batch's mode-1 split ----
// One warp per fibre of fn contiguous elements, lane t the EPL consecutive elements
// [EPL·t, EPL·t + EPL): every source is read once, the NOUT sums stay in registers (the
// accumulation order of multi_combine_kernel: sources in order, acc += c·x), the fp64 outputs
// are stored, and the outputs with dig[o] set are also split into digit planes exactly as
// oz_split_x_contig_kernel would split them after reading them back.
#ifndef OZ_MC_UNROLL
#define OZ_MC_UNROLL 2
#endif
// FS warps per fibre (1 or 2): with FS = 2 each warp sums half of the fibre (EPL = Kp/64 per lane), so
// the wide variants need half the registers and twice the warps fit per SM; the two halves meet for
// the fibre exponent in shared memory behind a named barrier of the warp pair
template <int NOUT, int EPL, int WPB = 8, int FS = 1>
__global__ void __launch_bounds__(WPB * 32) oz_multi_combine_split_kernel(const __grid_constant__ MultiCombineParams p) {
  static_assert(FS == 1 || (FS == 2 && WPB % 2 == 0 && WPB <= 30), "warp pairs");
  constexpr int S = 7;
  const int n = p.fn, Kp = p.Kp;
  const int64_t C = p.count / n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = warp % FS;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * (WPB / FS) + warp / FS;
  const bool active = c < C;  // uniform per warp pair (an idle pair still meets at its barriers)
  if (FS == 1 && !active) return;
  const int k0 = EPL * (32 * h + lane);
  __shared__ unsigned s_hm[FS == 2 ? NOUT : 1][WPB];
  __shared__ double s_m[FS == 2 ? NOUT : 1][WPB];
  auto pair_sync = [&]() {
    if constexpr (FS == 2) asm volatile("bar.sync %0, 64;\n" ::"r"(1 + (warp >> 1)) : "memory");
  };
  const bool vec = n == Kp;  // full lanes, 16-byte aligned rows (checked by the launcher)
  double acc[NOUT][EPL];
#pragma unroll
  for (int o = 0; o < NOUT; ++o)
#pragma unroll
    for (int q = 0; q < EPL; ++q) acc[o][q] = 0.0;
  // U sources per iteration, all loads issued before the sums: with NOUT·EPL accumulators in registers
  // the wide variants run one 8-warp block per SM, and one source in flight per warp left them at
  // ~0.6 of the copy peak (configs[4]: NOUT 4, EPL 16)
  constexpr int U = OZ_MC_UNROLL;
  auto load = [&](int s, double (&x)[EPL]) {
    const double* src = p.src[s] + c * n;
    if (vec) {
#pragma unroll
      for (int i = 0; i < EPL / 2; ++i) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(src + k0) + i);
        x[2 * i] = a.x;
        x[2 * i + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < EPL; ++q) x[q] = k0 + q < n ? __ldcs(src + k0 + q) : 0.0;
    }
  };
  int s0 = 0;
  const int nsrc = active ? p.nsrc : 0;
  for (; s0 + U <= nsrc; s0 += U) {
    double x[U][EPL];
#pragma unroll
    for (int u = 0; u < U; ++u) load(s0 + u, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        const double cf = p.coef[o][s0 + u];
#pragma unroll
        for (int q = 0; q < EPL; ++q) acc[o][q] += cf * x[u][q];
      }
  }
  for (int s = s0; s < nsrc; ++s) {
    double x[EPL];
    load(s, x);
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      const double cf = p.coef[o][s];
#pragma unroll
      for (int q = 0; q < EPL; ++q) acc[o][q] += cf * x[q];
    }
  }
#pragma unroll
  for (int o = 0; o < NOUT; ++o) {
    if (o >= p.nout) break;
    double* dst = p.dst[o] + c * n;
    if (!active) {
    } else if (vec) {
#pragma unroll
      for (int i = 0; i < EPL / 2; ++i)
        reinterpret_cast<double2*>(dst + k0)[i] = make_double2(acc[o][2 * i], acc[o][2 * i + 1]);
    } else {
#pragma unroll
      for (int q = 0; q < EPL; ++q)
        if (k0 + q < n) dst[k0 + q] = acc[o][q];
    }
    if (p.dig[o]) {
      bool bad;
      int ex;
      if constexpr (FS == 1) {
        ex = oz_fibre_exponent<S, EPL>(acc[o], bad);
      } else {  // oz_fibre_exponent over the two halves of the fibre
        unsigned hm = 0;
#pragma unroll
        for (int q = 0; q < EPL; ++q) hm = max(hm, static_cast<unsigned>(__double2hiint(acc[o][q])) & 0x7fffffffu);
        hm = __reduce_max_sync(0xffffffffu, hm);
        if (lane == 0) s_hm[o][warp] = hm;
        pair_sync();
        hm = max(s_hm[o][warp & ~1], s_hm[o][warp | 1]);
        bad = hm >= 0x7ff00000u;
        if (bad) {
          ex = 0;
        } else if (hm >= 0x00100000u) {
          ex = static_cast<int>(hm >> 20) - 1021;
        } else {  // subnormal maxima: the exact fp64 path (hm is the pair's, so both warps take it)
          double m = 0.0;
#pragma unroll
          for (int q = 0; q < EPL; ++q) m = fmax(m, fabs(acc[o][q]));
          m = warp_max(m);
          if (lane == 0) s_m[o][warp] = m;
          pair_sync();
          ex = slice_exponent(fmax(s_m[o][warp & ~1], s_m[o][warp | 1]));
        }
      }
      uint32_t pk[EPL / 4][S];
      oz_split_lane<S, EPL>(acc[o], ex, bad, pk);
      if (active) {
        oz_store_lane<S, EPL>(p.dig[o] + c * Kp + k0, C * Kp, pk);
        if (lane == 0 && h == 0) p.dsc[o][c] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ex;
      }
    }
  }
}

// ---- split_e: one warp per row j of E (column-major, E[j + k·n]) ----
template <int S>
__global__ void __launch_bounds__(256) oz_split_e_kernel(const OzakiParams p) {
  const int slot = blockIdx.y;
  const double* E = p.e[slot];
  const int n = p.n, Kp = p.Kp;
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= n) return;
  const int K = p.cplx_j ? 2 * n : n;  // complex products: row j of [Re M | Im M]
  double m = 0.0, a1 = 0.0;
  bool bad = false;
  for (int k = lane; k < K; k += 32) {
    const double v = E[j + static_cast<int64_t>(k) * n];
    m = fmax(m, fabs(v));
    a1 += fabs(v);
    bad |= !isfinite(v);
  }
  m = warp_max(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a1 += __shfl_xor_sync(0xffffffffu, a1, o);
  bad = __any_sync(0xffffffffu, bad);
  const int ex = bad ? 0 : slice_exponent(m);
  int8_t* es = p.es + static_cast<int64_t>(slot) * S * n * Kp;
  unsigned kbm = 0;  // k-blocks (128 k each; iteration kb of this loop) with a nonzero digit in row j
  for (int k0 = 4 * lane, kb = 0; k0 < Kp; k0 += 128, ++kb) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (k0 + q < K && !bad) ? E[j + static_cast<int64_t>(k0 + q) * n] : 0.0;
    uint32_t pk[S], nz = 0;
    split4<S>(v, ex, pk);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      *reinterpret_cast<uint32_t*>(es + (static_cast<int64_t>(s) * n + j) * Kp + k0) = pk[s];
      nz |= pk[s];
    }
    if (__any_sync(0xffffffffu, nz != 0)) kbm |= 1u << kb;
  }
  if (lane == 0 && p.eext && kbm) atomicOr(reinterpret_cast<unsigned*>(p.eext + 3 * p.ne + slot), kbm << (4 * (j / kOzBN)));
  if (lane == 0) {  // the row's scale 2^{ee-30} (the GEMM epilogue's 2^-30: 2^-14 of the digit scaling, 2^-16 of its sums)
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    p.esc[static_cast<int64_t>(slot) * n + j] = bad ? qnan : scalbn(1.0, ex - 30);
    // b_j with ‖e_j‖₁ < 2^{b_j} (a1 carries ≤ n·2^-53 relative rounding: margin 2^-40); the
    // rounded digits have |ẽ_jk| ≤ |e_jk| + 2^{ee-56}, i.e. ‖ẽ_j‖₁ ≤ ‖e_j‖₁(1 + n·2^-55) inside
    // the margin, so |Σ_k ẽ_jk x̃_k| < 2^{b_j}·max|x̃| (chained modes, §4d)
    const int b = a1 > 0.0 ? ilogb(a1 * (1.0 + 0x1p-40)) + 1 : -1100;
    if (p.eb) p.eb[static_cast<int64_t>(slot) * n + j] = bad ? qnan : b;
    if (p.ecol) {
      p.ecol[static_cast<int64_t>(slot) * n + j] = bad ? INT_MIN : (ex - 30) - b;
      if (bad) atomicOr(p.eext + 2 * p.ne + slot, 1);
      atomicMin(p.eext + slot, b);
      atomicMax(p.eext + p.ne + slot, b);
    }
  }
}

// ---- chained Tucker modes: next-mode fiber exponents as bounds ----
// For Y = X ×_μ E, |y(l, j, i, r')| ≤ ‖e_j‖₁·max_k |x(l, k, i, r')| < 2^{b_j + ex(l, i, r') − 1}
// (i = i_{μ+1}), so the mode-(μ+1) fiber c' = l + L·j + L·n·r' (over i) can be split with
// ex'(c') = b_j + max_i ex(l, i, r') before the product is computed: the product's epilogue
// writes the next mode's digits directly.  One thread per (l, r') of a term.
__global__ void __launch_bounds__(256) oz_chain_kernel(const OzakiParams p) {
  __shared__ double red[8][32];
  __shared__ double smx[32];
  const OzakiTerm term = p.terms[blockIdx.y];
  const int64_t L = p.L, C = p.L * p.R;
  const int n = p.n, nn = p.n_next;
  const int64_t M = C / nn;  // (l, r') pairs
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  // Mx(l, r') = max_i ex(l, i, r') for 32 consecutive (l, r'), the warps splitting i
  {
    const int64_t m = m0 + lane;
    double mx = -2000.0;
    bool nan = false;
    if (m < M) {
      const int64_t l = m % L, rq = m / L;
      const double* ex = p.xsc + static_cast<int64_t>(term.xslot) * C + l + L * nn * rq;
      for (int i = warp; i < nn; i += 8) {
        const double v = ex[L * i];
        nan |= isnan(v);
        mx = fmax(mx, v);
      }
    }
    red[warp][lane] = nan ? qnan : mx;
    __syncthreads();
    if (warp == 0) {
      double t = red[0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) {
        const double u = red[w][lane];
        t = (isnan(t) || isnan(u)) ? qnan : fmax(t, u);
      }
      smx[lane] = t;
      if (m < M && blockIdx.z == 0) term.nmx[m] = t;
    }
    __syncthreads();
  }
  // ex'(c') for c' = l + L·j + L·n·r' over the chunk's (l, r') and this block's 64 columns j
  const double* eb = p.eb + static_cast<int64_t>(term.eslot) * n;
  const int cnt = static_cast<int>(M - m0 < 32 ? M - m0 : 32);
  const int jb = blockIdx.z * 64, jc = n - jb < 64 ? n - jb : 64;
  for (int idx = threadIdx.x; idx < 32 * jc; idx += 256) {
    int mi, j;
    if (L == 1) {
      mi = idx / jc;
      j = jb + idx - mi * jc;
    } else {
      j = jb + (idx >> 5);
      mi = idx & 31;
    }
    if (mi >= cnt) continue;
    const int64_t m = m0 + mi, l = m % L, rq = m / L;
    // |y| < 2^1024 for finite y, and below 2^-1100 y is 0: the clamps keep the bound valid
    const double e = __ldg(eb + j) + smx[mi];
    term.nex[l + L * j + L * n * rq] = isnan(e) ? qnan : fmin(fmax(e, -1100.0), 1025.0);
  }
}

// ---- slab-sharded chained stage 0: cross-rank next-mode exponents (phiks_internal.h) ----
__global__ void __launch_bounds__(256) oz_shard_pmax_kernel(const OzShardExch e) {
  // 32 consecutive l per CTA (lanes), the 8 warps splitting the slab's R; smem reduction
  __shared__ double red[8][32];
  const int t = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t l = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  double m = -2000.0;
  bool nan = false;
  if (l < e.L0) {
    const double* x = e.xsc[t] + l;
    for (int64_t r = warp; r < e.R; r += 8) {
      const double v = x[e.L0 * r];
      nan |= isnan(v);
      m = fmax(m, v);
    }
  }
  red[warp][lane] = nan ? qnan : m;
  __syncthreads();
  if (warp != 0 || l >= e.L0) return;
  double v = red[0][lane];
#pragma unroll
  for (int w = 1; w < 8; ++w) {
    const double u = red[w][lane];
    v = (isnan(v) || isnan(u)) ? qnan : fmax(v, u);
  }
  const int64_t off = (static_cast<int64_t>(e.rank) * kShardChunkMax + t) * e.L0 + l;
  for (int k = 0; k < e.world; ++k) e.dst[k][off] = v;  // NVLink peer stores (own buffer at k == rank)
}

__global__ void __launch_bounds__(256) oz_shard_tables_kernel(const OzShardExch e) {
  const int t = blockIdx.y;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (idx >= e.L0 * e.cb) return;
  const int64_t l = idx % e.L0;
  const int jl = static_cast<int>(idx / e.L0);
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  double m = -2000.0;
  bool nan = false;
  for (int k = 0; k < e.world; ++k) {
    const double v = e.exch[(static_cast<int64_t>(k) * kShardChunkMax + t) * e.L0 + l];
    nan |= isnan(v);
    m = fmax(m, v);
  }
  if (nan) m = qnan;
  if (jl == 0) e.nmx[t][l] = m;
  const double x = __ldg(e.eb[t] + e.kstart + jl) + m;
  e.xsc1[t][idx] = isnan(x) ? qnan : fmin(fmax(x, -1100.0), 1025.0);
}

// ---- tcgen05 / TMA / mbarrier helpers ----
__device__ __forceinline__ void oz_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(oz_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void oz_mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(oz_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void oz_mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "OZ_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra OZ_WAIT_%=;\n"
      "}\n" ::"r"(oz_smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void oz_tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(oz_smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(oz_smem_u32(bar))
      : "memory");
}
// K-major SWIZZLE_128B operand: rows of 128 bytes, 8-row atoms of 1 KB (1 KB
// aligned); the k-th 32-byte UMMA slice of a row starts 32k bytes further
// (start address + 2k: the swizzle is applied to the absolute address)
__device__ __forceinline__ uint64_t oz_desc_sw128(const void* p) {
  const uint32_t a = oz_smem_u32(p);
  uint64_t d = static_cast<uint64_t>((a >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;          // leading byte offset (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // stride byte offset: 8 rows × 128 B
  d |= static_cast<uint64_t>(1) << 46;          // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;          // SWIZZLE_128B
  return d;
}
// MN-major SWIZZLE_128B operand (A of chained modes): k-rows of 128 bytes = 128
// fibers (one MN atom: the leading byte offset is unused), 8-row groups 1 KB apart
// (stride byte offset); the k-th 32-row UMMA slice starts 4 KB further
__device__ __forceinline__ uint64_t oz_desc_mn_sw128(const void* p) {
  const uint32_t a = oz_smem_u32(p);
  uint64_t d = static_cast<uint64_t>((a >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// kind::i8 instruction descriptor: D s32, A/B s8, B K-major, A K-major (or MN-major:
// bit 15), M = 128, N = BN
__host__ __device__ constexpr uint32_t oz_idesc(int bn, bool amn = false) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (amn ? (1u << 15) : 0u) | (static_cast<uint32_t>(bn >> 3) << 17) |
         ((128u >> 4) << 24);
}
__device__ __forceinline__ void oz_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   oz_smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool oz_elect() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void oz_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(oz_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void oz_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
// exact int64 → fp64 for |v| < 2^51: the bits of 1.5·2^52 + v
__device__ __forceinline__ double oz_l2d(long long v) {
  return __longlong_as_double(v + 0x4338000000000000ll) - 6755399441055744.0;
}

// ---- split_x, strided fibers (L % 32 == 0): persistent, TMA double buffer ----
// A tile is 32 consecutive fibers (l0..l0+31, r) × all n k, loaded by one TMA
// box (32, n, 1) of the (L, n, R) tensor into smem [k][32]; warp w takes
// k ∈ [32w, 32w+32) of every fiber (lane = fiber): partial maxima meet in smem,
// then each thread writes its 32 digits per slice as two 16-byte stores.
struct OzXMaps {
  CUtensorMap m[8];
};
constexpr int kOzSplitSlots = 8;

template <int S>
__global__ void __launch_bounds__(512, 1)
    oz_split_x_tma_kernel(const OzakiParams p, const __grid_constant__ OzXMaps maps,
                          const __grid_constant__ CUtensorMap dmap, int slot0, int nslots) {
  extern __shared__ __align__(1024) double oz_sx_raw[];
  double* buf = oz_sx_raw;  // indexed from the shared array itself: the compiler keeps LDS
  const int n = p.n, Kp = p.Kp;
  const int64_t L = p.L, C = p.L * p.R;
  const int tile_elems = 32 * n;
  double* red = oz_sx_raw + 2 * 32 * kOzMaxNRes + S * 2 * 4096 / 8;  // [16][32] partial maxima
  int* redbad = reinterpret_cast<int*>(red + 16 * 32);             // [16][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(redbad + 16 * 32);
  // digit staging: per digit s and 128-byte k-half h, a SWIZZLE_128B image of the
  // 32 fibers × 128 bytes box (16-byte chunk q of row r at q ^ (r & 7)), written
  // conflict-free and stored by TMA (which undoes the swizzle)
  uint8_t* stage = reinterpret_cast<uint8_t*>(oz_sx_raw) + 2 * 32 * kOzMaxNRes * 8;  // 1 KB aligned
  const int nh = Kp > 128 ? 2 : 1;  // k-halves (Kp ≤ 256)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntc = C / 32;
  const int64_t total = ntc * nslots;
  if (threadIdx.x == 0) {
    for (int b = 0; b < nslots && b < kOzSplitSlots; ++b)
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.m[b])) : "memory");
    oz_mbar_init(&full[0], 1);
    oz_mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t it, int b) {
    const int sl = static_cast<int>(it / ntc);
    const int64_t c0 = (it % ntc) * 32;
    oz_mbar_expect_tx(&full[b], static_cast<unsigned>(tile_elems * 8));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(oz_smem_u32(buf + b * tile_elems)),
        "l"(reinterpret_cast<uint64_t>(&maps.m[sl])), "r"(static_cast<int>(c0 % L)), "r"(0),
        "r"(static_cast<int>(c0 / L)), "r"(oz_smem_u32(&full[b]))
        : "memory");
  };
  if (threadIdx.x == 0 && blockIdx.x < total) issue(blockIdx.x, 0);
  int i = 0;
  for (int64_t it = blockIdx.x; it < total; it += gridDim.x, ++i) {
    const int b = i & 1;
    if (threadIdx.x == 0 && it + gridDim.x < total) issue(it + gridDim.x, b ^ 1);  // buffer b^1 is free
    oz_mbar_wait(&full[b], (i >> 1) & 1);
    const double* t = buf + b * tile_elems;
    const int sl = slot0 + static_cast<int>(it / ntc);
    const int64_t c = (it % ntc) * 32 + lane;
    const int k0 = 16 * warp;
    double m = 0.0;
    int bad = 0;
#pragma unroll 8
    for (int k = k0; k < k0 + 16 && k < n; ++k) {
      const double v = t[k * 32 + lane];
      m = fmax(m, fabs(v));
      bad |= !isfinite(v);
    }
    red[warp * 32 + lane] = m;
    redbad[warp * 32 + lane] = bad;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 16; ++w) {
      m = fmax(m, red[w * 32 + lane]);
      bad |= redbad[w * 32 + lane];
    }
    const int ex = bad ? 0 : slice_exponent(m);
    if (k0 < Kp) {
      uint32_t pk[4][S];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + 4 * g + q;
          v[q] = (k < n && !bad) ? t[k * 32 + lane] : 0.0;
        }
        split4<S>(v, ex, pk[g]);
      }
      const int h = k0 >> 7, q = (k0 & 127) >> 4;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        *reinterpret_cast<uint4*>(stage + ((s * 2 + h) * 32 + lane) * 128 + ((q ^ (lane & 7)) << 4)) =
            make_uint4(pk[0][s], pk[1][s], pk[2][s], pk[3][s]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // staging visible to the TMA store
    if (warp == 0)
      p.xsc[static_cast<int64_t>(sl) * C + c] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ex;
    __syncthreads();  // staging complete; every warp is done with buffer b and the partial maxima
    if (threadIdx.x == 0) {
      const int64_t c0 = (it % ntc) * 32;
      for (int s = 0; s < S; ++s)
        for (int h = 0; h < nh; ++h)
          asm volatile(
              "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(
                  reinterpret_cast<uint64_t>(&dmap)),
              "r"(h * 128), "r"(static_cast<int>(c0)), "r"(s), "r"(sl), "r"(oz_smem_u32(stage + (s * 2 + h) * 4096))
              : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // staging read out before reuse
    }
    __syncthreads();  // staging free for the next tile
  }
}

// One output tile of the epilogue (both GEMM kernels): fiber c (TMEM lane), columns
// j0 .. j0+31 of term term_i; waits for the accumulators (t_full, phase), drains them,
// releases TMEM through release(), then scales and stores (fp64 or the next mode's digits).
template <int S, bool OUTD, bool AMN, bool REM, int EPC, class Release>
__device__ __forceinline__ void oz_epilogue_tile(const OzakiParams& p, int term_i, int64_t c, int j0, uint32_t tl,
                                             uint64_t* t_full, unsigned phase, Release release) {
  const int lane = threadIdx.x & 31;
  const int64_t C = p.L * p.R, L = p.L;
  const OzakiTerm term = p.terms[term_i];
  const bool rvalid = c < C;
  const int64_t l = c % L, r = c / L;
  // per-tile operands issued before the accumulator wait: the fiber exponent, the
  // EPC column scales of this warp's columns (lane q holds column j0 + q, broadcast by shuffles)
  // and, for chained modes, the row-norm exponents b_j and the fiber's Mx
  const double xsv = rvalid ? p.xsc[static_cast<int64_t>(term.xslot) * C + c] : 0.0;
  const int jn = p.n - j0;  // valid columns of this half
  const double esc_l = lane < jn ? __ldg(p.esc + static_cast<int64_t>(term.eslot) * p.n + j0 + lane) : 0.0;
  double eb_l = 0.0, mx = 0.0;
  int colk[OUTD ? EPC : 1];
  bool ebad = false;
  int emin = 0, emax = 0;
  if (OUTD) {
    eb_l = lane < jn ? __ldg(p.eb + static_cast<int64_t>(term.eslot) * p.n + j0 + lane) : 0.0;
    mx = rvalid ? term.nmx[l + L * (r / p.n_next)] : 0.0;
    const int* ec = p.ecol + static_cast<int64_t>(term.eslot) * p.n + j0;
    if (jn >= EPC) {
#pragma unroll
      for (int i = 0; i < EPC / 4; ++i) {
        const int4 v4 = __ldg(reinterpret_cast<const int4*>(ec) + i);
        colk[4 * i] = v4.x;
        colk[4 * i + 1] = v4.y;
        colk[4 * i + 2] = v4.z;
        colk[4 * i + 3] = v4.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < EPC; ++q) colk[q] = q < jn ? __ldg(ec + q) : 0;
    }
    emin = __ldg(p.eext + term.eslot);
    emax = __ldg(p.eext + p.ne + term.eslot);
    ebad = __ldg(p.eext + 2 * p.ne + term.eslot) != 0;
  }
  oz_mbar_wait(t_full, phase);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // drain: per column V = 2^16 Σ_g 256^{-g} D_g from two exact int64 partial sums,
  // ta = D_0·2^16 + D_1·2^8 + D_2 (< n·2^31) and T = ((D_3·2^8 + D_4)·2^8 + D_5)·2^8 + D_6
  // (< n·2^41), V = ta + 2^-32·T (|D_g| ≤ (g+1)·n·2^14).  fp64 outputs take V with one
  // rounding; the next mode's digits (OUTD) take Pt = ⌊V·2^23⌋ = ta·2^23 + ⌊T/2^9⌋ (< 2^63
  // for n ≤ 512; the floor is below 2^-60 of the fibre bound) and stay in the integer pipes
  double acc[EPC];
  long long pt[EPC];
  // high diagonals first (T from {3, …, S-1}), then ta from {0, 1, 2}: at most 32 loaded words
  // live at a time next to the 32 partial sums
#pragma unroll
  for (int cb = 0; cb < EPC / 8; ++cb) {
    uint32_t v[S - 3][8];
#pragma unroll
    for (int g = 3; g < S; ++g) oz_ld8(tl + g * kOzBN + cb * 8, v[g - 3]);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      long long T = static_cast<long long>(static_cast<int>(v[0][q])) * 256 + static_cast<int>(v[1][q]);
      T = T * 256 + static_cast<int>(v[2][q]);
      T = T * 256 + (S == 7 ? static_cast<int>(v[S == 7 ? 3 : 0][q]) : 0);
      pt[cb * 8 + q] = T;
    }
  }
#pragma unroll
  for (int cb = 0; cb < EPC / 8; ++cb) {
    uint32_t v[3][8];
#pragma unroll
    for (int g = 0; g < 3; ++g) oz_ld8(tl + g * kOzBN + cb * 8, v[g]);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long ta = static_cast<long long>(static_cast<int>(v[0][q])) * 65536 +
                           static_cast<long long>(static_cast<int>(v[1][q])) * 256 + static_cast<int>(v[2][q]);
      const long long T = pt[cb * 8 + q];
      if constexpr (OUTD)
        pt[cb * 8 + q] = (ta << 23) + (T >> 9);
      else
        acc[cb * 8 + q] = fma(oz_l2d(T), 0x1p-32, oz_l2d(ta));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncwarp();
  release();

  // scale and store (overlaps the next tile's MMAs)
  // y = (acc · 2^{ee_j − 30}) · (β·2^{ex_c}): the power-of-two product first (no intermediate overflow)
  const int xe = isnan(xsv) ? 0 : static_cast<int>(xsv);
  const double rb = isnan(xsv) ? xsv
                    : (xe >= -1022 && xe <= 1023)
                        ? term.beta * __longlong_as_double(static_cast<long long>(xe + 1023) << 52)
                        : scalbn(term.beta, xe);
  if (OUTD) {
    // the next mode's digits of y: fiber c' = l + L·j + L·n·r' of mode μ+1
    // (r = i + n'·r') has exponent e = clamp(b_j + Mx(l, r')) (NaN marks a non-finite fiber),
    // exactly as oz_chain_kernel tabulates it; y·2^{8S-1-e} = acc·2^{(ee_j-30) + ex_c + 8S-1-e}
    // is one exact power-of-two scaling of the accumulator (β = 1 on chained modes), so the
    // digits take one DMUL and one F2I per element; digit s of element (l, j, r) goes to
    // dig[s·N + l + L·(j + n·r)]
    const int64_t N = C * p.n;  // (chained products have β = 1)
    // column pair (b_j, ee_j - 30) packed in 16-bit halves, INT_MIN for a non-finite row of E
    const int cp_l = (isnan(esc_l) || isnan(eb_l))
                         ? INT_MIN
                         : ((static_cast<int>(eb_l) + 0x4000) << 16) | (ilogb(esc_l) + 0x4000);
    const bool rbad = isnan(xsv) || isnan(mx);
    const int rk = rbad ? 0 : xe + 8 * S - 1, mxi = rbad ? 0 : static_cast<int>(mx);
    // F = rint(V·2^k) = rint(Pt·2^{k-23}): Pt shifted right by r = 23 − k with round half up,
    // or left by −r (k ≤ 27 since ee_j ≤ b_j + 2 and ex_c ≤ Mx; no overflow: |F| ≤ 2^54),
    // then balanced digits as in oz_digits
    constexpr uint64_t Cc = 0x8080808080808080ull >> (64 - 8 * S);
    auto digit_bits = [&](long long P, int k) -> uint64_t {
      // branch-free: F = ((P << ls) + 2^{rs-1}) >> rs with rs = min(max(r, 0), 63), ls = max(−r, 0)
      const int r = 23 - k;
      const int rs = min(max(r, 0), 63), ls = max(-r, 0) & 63;
      const long long half = rs > 0 ? (1ll << (rs - 1)) : 0ll;
      const long long F = ((P << ls) + half) >> rs;
      return (static_cast<uint64_t>(F) + Cc) ^ Cc;
    };
    // fast path (warp-uniform): every row of E finite and no clamp of e = b_j + Mx, so
    // k = ((ee_j − 30) − b_j) + (ex_c + 8S − 1 − Mx) = colk[q] + rowk: one add per element
    const bool fast = __all_sync(0xffffffffu, !rbad && !ebad && emin + mxi >= -1100 && emax + mxi <= 1025);
    const int rowk = rk - mxi;
    if (!fast) {
      // rare (non-finite rows or fibres, clamped exponents): fold the general exponent into
      // colk and zero the accumulators of non-finite entries (zero digits), so that the
      // per-element code below stays a single short path (the kernel's instruction footprint
      // bounds the epilogue: DESIGN.md §4e)
#pragma unroll
      for (int q = 0; q < EPC; ++q) {
        const int cpq = __shfl_sync(0xffffffffu, cp_l, q);
        const int e = min(max(((cpq >> 16) - 0x4000) + mxi, -1100), 1025);
        colk[q] = ((cpq & 0xffff) - 0x4000) + rk - e - rowk;
        if (rbad || cpq == INT_MIN) pt[q] = 0;
      }
    }
    auto digits = [&](int q) -> uint64_t { return digit_bits(pt[q], colk[q] + rowk); };
    const bool st_ok = rvalid && jn > 0;
    if (!AMN) {  // mode-1 product (L = 1): EPC consecutive bytes of each digit plane per thread
      int8_t* dg = term.dig + l + L * (j0 + static_cast<int64_t>(p.n) * r);
      const bool full = st_ok && jn >= EPC;
      const bool a32 = ((reinterpret_cast<uintptr_t>(dg) | static_cast<uintptr_t>(N)) & 31) == 0;
      uint32_t pk[EPC / 4][S];
#pragma unroll
      for (int g = 0; g < EPC / 4; ++g) {
        const uint64_t h4[4] = {digits(4 * g), digits(4 * g + 1), digits(4 * g + 2), digits(4 * g + 3)};
        pack4<S>(h4, pk[g]);
      }
#pragma unroll
      for (int sd = 0; sd < S; ++sd) {
        int8_t* ds = dg + sd * N;
        if (EPC == 32 && full && a32) {  // one 32-byte store (STG.256, a whole sector)
          asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"l"(ds), "r"(pk[0][sd]),
                       "r"(pk[1][sd]), "r"(pk[2][sd]), "r"(pk[3][sd]), "r"(pk[4][sd]), "r"(pk[5][sd]),
                       "r"(pk[6][sd]), "r"(pk[7][sd])
                       : "memory");
        } else if (full) {  // 16-byte aligned rows (n % 16 == 0 on chained modes)
#pragma unroll
          for (int h2 = 0; h2 < EPC / 16; ++h2)
            *reinterpret_cast<uint4*>(ds + 16 * h2) =
                make_uint4(pk[4 * h2][sd], pk[4 * h2 + 1][sd], pk[4 * h2 + 2][sd], pk[4 * h2 + 3][sd]);
        } else if (st_ok) {  // last n-tile of n % 64 != 0: jn is a multiple of 16
#pragma unroll
          for (int g = 0; g < EPC / 4; ++g)
            if (4 * g < jn) *reinterpret_cast<uint32_t*>(ds + 4 * g) = pk[g][sd];
        }
      }
    } else {
      // lanes hold consecutive l (MN-major next-mode digits, L % 128 == 0: row offset l + L·n·r,
      // column stride L).  Per 4 columns, the 4×4 byte blocks of each lane quad are transposed
      // by two shuffle rounds, so lane qi of a quad stores the 4 consecutive rows of column
      // q0 + qi as one 32-bit word
      const int qi = lane & 3;
      const uint32_t sel1 = (qi & 1) ? 0x3715u : 0x6240u, sel2 = (qi & 2) ? 0x3276u : 0x5410u;
      int64_t rowoff = l + L * static_cast<int64_t>(p.n) * r, cs = L;
      int8_t* dbase = term.dig;
      int jrel = j0;
      if constexpr (REM) {
        // slab-sharded stage 0: the next mode's digit planes go to the owner
        // k of column j in its transposed layout (uniform blocks of cq ≥ EPC columns, so the
        // warp's columns share one owner): plane offset l + kstride[k]·r + kroff[k] +
        // colstride·(j − kstart[k]); the owners' planes have the local plane stride N
        const Remap& rm = p.remap;
        const int k = j0 / rm.cq;
        dbase = reinterpret_cast<int8_t*>(rm.base[k] + reinterpret_cast<uintptr_t>(term.dig));
        rowoff = l + rm.kstride[k] * r + rm.kroff[k];
        cs = rm.colstride;
        jrel = j0 - rm.kstart[k];
      }
      int8_t* dq = dbase + (rowoff - qi) + cs * (jrel + qi);
      uint32_t* dqs[S];
#pragma unroll
      for (int sd = 0; sd < S; ++sd) dqs[sd] = reinterpret_cast<uint32_t*>(dq + sd * N);
      const int64_t step = cs;  // in 32-bit words: 4·cs bytes
      const bool full = st_ok && jn >= EPC;
#pragma unroll
      for (int q0 = 0; q0 < EPC; q0 += 4) {
        const uint64_t h4[4] = {digits(q0), digits(q0 + 1), digits(q0 + 2), digits(q0 + 3)};
        uint32_t pk[S];
        pack4<S>(h4, pk);
#pragma unroll
        for (int sd = 0; sd < S; ++sd) {
          const uint32_t t1 = __byte_perm(pk[sd], __shfl_xor_sync(0xffffffffu, pk[sd], 1), sel1);
          const uint32_t t2 = __byte_perm(t1, __shfl_xor_sync(0xffffffffu, t1, 2), sel2);
          if (full || (st_ok && q0 + qi < jn)) *dqs[sd] = t2;
          dqs[sd] += step;
        }
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < EPC; ++q) acc[q] = (acc[q] * __shfl_sync(0xffffffffu, esc_l, q)) * rb;  // exact, then rounded
  }
  if (!OUTD && REM && rvalid && jn > 0) {
    // slab-sharded stage: column j of the product belongs to rank k = owner(j);
    // element (l, j, r) goes to base[k] + out + l + kstride[k]·r + kroff[k] + colstride·(j − kstart[k])
    const Remap& rm = p.remap;
    const int big = (rm.cq + 1) * rm.crem;
    auto owner = [&](int j) { return j < big ? j / (rm.cq + 1) : rm.crem + (j - big) / rm.cq; };
    const int kf = owner(j0), kl = owner(j0 + (jn < EPC ? jn : EPC) - 1);
    if (kf == kl) {  // the warp's columns share one owner: one base, then a stride per column
      double* b = reinterpret_cast<double*>(rm.base[kf] + reinterpret_cast<uintptr_t>(term.out)) + rm.kroff[kf] + l +
                  rm.kstride[kf] * r + rm.colstride * static_cast<int64_t>(j0 - rm.kstart[kf]);
#pragma unroll
      for (int q = 0; q < EPC; ++q)
        if (q < jn) b[rm.colstride * q] = acc[q];
    } else {  // the owner advances by at most one rank per column (every block has ≥ 1 column)
      int k = kf;
#pragma unroll
      for (int q = 0; q < EPC; ++q) {
        const int j = j0 + q;
        if (q < jn) {
          if (k + 1 < rm.world && j >= rm.kstart[k + 1]) ++k;
          double* colp = reinterpret_cast<double*>(rm.base[k] + reinterpret_cast<uintptr_t>(term.out)) + rm.kroff[k] +
                         rm.colstride * static_cast<int64_t>(j - rm.kstart[k]);
          colp[l + rm.kstride[k] * r] = acc[q];
        }
      }
    }
  } else if (!OUTD && !REM && rvalid && jn > 0) {
    double* outp = term.out + l + L * (j0 + static_cast<int64_t>(p.n) * r);
    if (!AMN && L == 1 && jn >= EPC && (reinterpret_cast<uintptr_t>(outp) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < EPC; q += 2) *reinterpret_cast<double2*>(outp + q) = make_double2(acc[q], acc[q + 1]);
    } else {  // one predicated loop (full and partial column ranges): a small instruction footprint
#pragma unroll
      for (int q = 0; q < EPC; ++q)
        if (q < jn) outp[L * q] = acc[q];
    }
  }
}

// Persistent GEMM geometry: the E-digit tile of a (term, n-tile) stays resident
// (S × 64 rows × Kp bytes); fiber digits stream through an NST-stage ring of
// SPS-digit units (k-block kb, digit group sg).  Ring depth per variant, measured on the
// configs[3] launches (round 1, ms per 19-term batch at NST = 4 / 5 / 6 / 7): mode 1 with digit
// epilogue 2.01 / 2.02 / 2.09 / 2.14, chained mode 2 2.15 / 2.13 / 2.12 / 2.14, fp64-output
// mode 1.87 / 1.72 / 1.64 / 1.57 (the shared-memory carve-out also sizes the L1 the
// digit epilogue's stores go through).  Round 2 (integer epilogue, balanced MMA halves): mode 1
// at 5 or 6 stages 3.4 % faster than at 4, mode 2 at 7 slightly slower than at 6
#ifndef OZ_NST_KS_K
#define OZ_NST_KS_K 5
#endif
#ifndef OZ_NST_KS_D
#define OZ_NST_KS_D 7
#endif
__host__ __device__ constexpr int oz_nst(bool amn, bool outd, bool ks = false) {
  return outd ? (amn ? 6 : (ks ? OZ_NST_KS_K : 5)) : (ks ? OZ_NST_KS_D : 7);
}
#ifndef OZ_EPC_D
#define OZ_EPC_D 32
#endif
// columns per epilogue warp: 32 (16, i.e. 16 epilogue warps at 96 registers: 8 % slower on every
// kernel in r02; on the fp64-output kernels alone 7 % slower, profiles/r02_ab_kskip/ab12_epc16_fp64.txt)
__host__ __device__ constexpr int oz_epc(bool outd) { return outd ? 32 : OZ_EPC_D; }
template <int S, int NST_ = 6, int EPC_ = 32>
struct OzGeom {
  static constexpr int SPS = 1;                                // digits per stage
  static constexpr int A_BYTES = SPS * kOzBM * kOzBK;         // one stage
  static constexpr int NST = NST_;
  static constexpr int B_KB = S * kOzBN * kOzBK;              // resident E slices per k-block
  static constexpr int B_BYTES = (kOzMaxNRes / kOzBK) * B_KB; // resident (Kp ≤ 256) or a 2-block ring (SE)
  static constexpr int SMEM = NST * A_BYTES + B_BYTES + 1024 /*align*/ + 512 /*barriers*/;
  static constexpr int EPC = EPC_;
  static constexpr int EPI_WARPS = 4 * kOzBN / EPC;             // 2 per TMEM lane quarter (column halves)
  static constexpr int THREADS = 64 + EPI_WARPS * 32;
  static_assert(S * kOzBN <= 512, "TMEM holds one 64-column accumulator per diagonal");
  static_assert(SMEM <= 232448, "shared memory");
  static_assert((2 * NST + 8) * 8 + 16 + 4 * kMaxTerms <= 512, "barriers, TMEM slot and block masks");
};

// work of CTA k: n-tile nt = k % ntn, units u = q, q + Q, … over (term, m-tile),
// term-major, so the ntn CTAs sharing q read the same fiber tiles together
// work of CTA k: n-tile nt = k % ntn, units u = q, q + Q, … over (term, m-tile), term-major,
// so the ntn CTAs sharing q read the same fiber tiles together and all CTAs sweep one term's
// tiles at a time (a contiguous run of units per CTA measured slower: 2.09 -> 2.97 ms on the
// chained mode-2 launch of configs[3])
// k-blocks of term i's E digits that n-tile t multiplies: the nonzero blocks split_e recorded
// (at least one, so that every tile's accumulators are written), all of them without kskip;
// skm = the matrices' block masks, copied to shared memory at the kernel's start (a global load per
// tile on the MMA warp's path measured 9 % slower per launch)
template <bool KS>
__device__ __forceinline__ unsigned oz_kmask(const OzakiParams& p, const uint32_t* skm, int i, int t, int nk) {
  const unsigned full = (1u << nk) - 1u;
  if (!KS) return full;
  const unsigned m = (skm[p.terms[i].eslot] >> (4 * t)) & full;
  return m ? m : 1u;
}
// kskip: the n-tile groups get CTAs in proportion to their work, Σ_terms (16·#k-blocks + fix) (a tile
// of the configs[3] launches: ~4,150 cycles of MMAs per k-block and a ~2,350-cycle hand-over,
// DESIGN.md §4e; fix per launch kind, measured: §4g), so that the groups sweep the fibre tiles at the
// same rate and the L2 still serves each fibre tile once for all of them (ntn ≤ 8: n ≤ kOzMaxN)
struct OzSched {
  int ntn, nt, q, Q, nk;
  int64_t Mt, units;
  __device__ OzSched(const OzakiParams& p, const uint32_t* skm, int fix, bool ks) {
    ntn = (p.n + kOzBN - 1) / kOzBN;
    nk = p.Kp / kOzBK;
    Mt = (p.L * p.R + kOzBM - 1) / kOzBM;
    units = Mt * p.nterms;
    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    if (!ks) {
      nt = b % ntn;
      q = b / ntn;
      Q = G / ntn;
      return;
    }
    int64_t cost[8], tot = 0;
    int size[8], sum = 0;
    for (int t = 0; t < ntn; ++t) {
      cost[t] = 0;
      for (int i = 0; i < p.nterms; ++i) cost[t] += 16 * __popc(oz_kmask<true>(p, skm, i, t, nk)) + fix;
      tot += cost[t];
    }
    for (int t = 0; t < ntn; ++t) {
      size[t] = max(1, static_cast<int>(G * cost[t] / tot));
      sum += size[t];
    }
    while (sum < G) {  // largest remainder first
      int bt = 0;
      for (int t = 1; t < ntn; ++t)
        if (G * cost[t] - size[t] * tot > G * cost[bt] - size[bt] * tot) bt = t;
      ++size[bt];
      ++sum;
    }
    while (sum > G) {
      int bt = 0;
      for (int t = 1; t < ntn; ++t)
        if (size[t] > size[bt]) bt = t;
      --size[bt];
      --sum;
    }
    nt = ntn - 1;
    q = b;
    for (int t = 0, s0 = 0; t < ntn; s0 += size[t], ++t)
      if (b < s0 + size[t]) {
        nt = t;
        q = b - s0;
        break;
      }
    Q = size[nt];
  }
};

// SE: the E digits stream through a 2-block ring (one 128-k block per stage group) instead of
// staying resident per term: always for n > 256, and for short launches (kOzSeUnits)
// KS: skip the all-zero E digit blocks (PHIKS_OPT_KSKIP; oz_gemm_go picks the launches)
template <int S, bool AMN, bool OUTD, bool SE, bool REM, bool KS>
__global__ void __launch_bounds__(OzGeom<S, oz_nst(AMN, OUTD, KS), oz_epc(OUTD)>::THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ OzakiParams p, const __grid_constant__ CUtensorMap ta,
                   const __grid_constant__ CUtensorMap tb) {
  using G = OzGeom<S, oz_nst(AMN, OUTD, KS), oz_epc(OUTD)>;
  extern __shared__ uint8_t oz_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem + G::NST * G::A_BYTES;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(bres + G::B_BYTES);
  uint64_t* a_empty = a_full + G::NST;
  uint64_t* b_full = a_empty + G::NST;
  uint64_t* b_empty = b_full + 1;
  uint64_t* t_full = b_empty + 1;
  uint64_t* t_empty = t_full + 1;
  uint64_t* e_full = t_empty + 1;  // SE: [2]
  uint64_t* e_empty = e_full + 2;   // SE: [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(e_empty + 2);
  uint32_t* skm = tmem_slot + 4;  // [ne ≤ kMaxTerms] nonzero E digit blocks (kskip)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (KS) {
    if (threadIdx.x < p.ne) skm[threadIdx.x] = static_cast<uint32_t>(p.eext[3 * p.ne + threadIdx.x]);
    __syncthreads();
  }
#ifndef OZ_KS_FIX
#define OZ_KS_FIX 12
#endif
#ifndef OZ_KS_FIX_OUTD
#define OZ_KS_FIX_OUTD 32
#endif
#ifndef OZ_KS_FIX_AMN_OUTD
#define OZ_KS_FIX_AMN_OUTD 24
#endif
  const OzSched sc(p, skm, OUTD ? (AMN ? OZ_KS_FIX_AMN_OUTD : OZ_KS_FIX_OUTD) : OZ_KS_FIX, KS);
  if (sc.q >= sc.Q) return;  // idle CTA (grid not a multiple of the n-tile count)
  const int nk = p.Kp / kOzBK;
  constexpr int NSG = S / G::SPS;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    for (int s = 0; s < G::NST; ++s) {
      oz_mbar_init(&a_full[s], 1);
      oz_mbar_init(&a_empty[s], 1);
    }
    oz_mbar_init(b_full, 1);
    oz_mbar_init(b_empty, 1);
    oz_mbar_init(t_full, 1);
    oz_mbar_init(t_empty, G::EPI_WARPS);
    for (int b = 0; b < 2; ++b) {
      oz_mbar_init(&e_full[b], 1);
      oz_mbar_init(&e_empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(oz_smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer (whole warp in lockstep, one elected lane issues) ----
    int cur_term = -1, bgen = 0, it = 0, ek = 0;
    for (int64_t u = sc.q; u < sc.units; u += sc.Q) {
      const int term = static_cast<int>(u / sc.Mt);
      const int mt = static_cast<int>(u % sc.Mt);
      if (!SE && term != cur_term) {  // (re)load the resident E slices of this (term, n-tile)
        if (bgen > 0) oz_mbar_wait(b_empty, (bgen - 1) & 1);
        if (oz_elect()) {
          oz_mbar_expect_tx(b_full, static_cast<unsigned>(nk * G::B_KB));
          for (int kb = 0; kb < nk; ++kb)
            oz_tma_load_4d(bres + kb * G::B_KB, &tb, kb * kOzBK, sc.nt * kOzBN, 0, p.terms[term].eslot, b_full);
        }
        __syncwarp();
        cur_term = term;
        ++bgen;
      }
      const int xs = p.terms[term].xslot;
      const unsigned km = oz_kmask<KS>(p, skm, term, sc.nt, nk);
      for (int kb = 0; kb < nk; ++kb) {
        if (KS && !((km >> kb) & 1u)) continue;  // all E digits zero in this k-block: no MMAs, no loads
        if (SE) {  // this k-block's E digits (all S digit planes × 64 rows) into ring slot ek & 1
          const int es = ek & 1;
          if (ek >= 2) oz_mbar_wait(&e_empty[es], ((ek >> 1) & 1) ^ 1);
          if (oz_elect()) {
            oz_mbar_expect_tx(&e_full[es], static_cast<unsigned>(G::B_KB));
            oz_tma_load_4d(bres + es * G::B_KB, &tb, kb * kOzBK, sc.nt * kOzBN, 0, p.terms[term].eslot, &e_full[es]);
          }
          __syncwarp();
          ++ek;
        }
        for (int sg = 0; sg < NSG; ++sg, ++it) {
          const int st = it % G::NST;
          if (it >= G::NST) oz_mbar_wait(&a_empty[st], ((it / G::NST) & 1) ^ 1);
          if (oz_elect()) {
            oz_mbar_expect_tx(&a_full[st], G::A_BYTES);
            if (AMN) {  // (l, k, r, slot·S + digit) map over the fp64-layout digit planes; L % 128 == 0
              const int64_t c0 = static_cast<int64_t>(mt) * kOzBM;
              oz_tma_load_4d(smem + st * G::A_BYTES, &ta, static_cast<int>(c0 % p.L), kb * kOzBK,
                             static_cast<int>(c0 / p.L), xs * S + sg * G::SPS, &a_full[st]);
            } else {
              oz_tma_load_4d(smem + st * G::A_BYTES, &ta, kb * kOzBK, mt * kOzBM, sg * G::SPS, xs, &a_full[st]);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (whole warp in lockstep, one elected lane issues) ----
    // diagonal g = s + t accumulates in TMEM columns [64g, 64g + 64); descriptors
    // advance by adding (byte offset >> 4) to their start-address field
    const uint64_t a_desc0 = AMN ? oz_desc_mn_sw128(smem) : oz_desc_sw128(smem), b_desc0 = oz_desc_sw128(bres);
    constexpr uint64_t a_kstep = AMN ? (kOzUK * kOzBM) >> 4 : kOzUK >> 4;  // one UMMA k-step of A
    int cur_term = -1, bgen = 0, it = 0, tile = 0, ek = 0;
    unsigned long long kb_run = 0;
    for (int64_t u = sc.q; u < sc.units; u += sc.Q, ++tile) {
      const int term = static_cast<int>(u / sc.Mt);
      if (!SE && term != cur_term) {
        if (bgen > 0) {
          if (oz_elect()) oz_commit(b_empty);  // the previous E tile is free once its MMAs are done
          __syncwarp();
        }
        oz_mbar_wait(b_full, bgen & 1);
        cur_term = term;
        ++bgen;
      }
      if (tile > 0) oz_mbar_wait(t_empty, (tile - 1) & 1);  // epilogue drained the accumulators
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      // fully unrolled over the digits: every MMA's column offset, N and instruction
      // descriptor are compile-time constants (the issue loop is a few uniform adds per MMA).
      // Issuing the digits high to low with the accumulators released in two diagonal groups
      // (to overlap the drain) measured 14 % slower
      const unsigned km = oz_kmask<KS>(p, skm, term, sc.nt, nk);
      const int kb0 = KS ? __ffs(km) - 1 : 0;  // the first k-block initialises the accumulators
      kb_run += KS ? __popc(km) : nk;
      for (int kb = 0; kb < nk; ++kb) {
        if (KS && !((km >> kb) & 1u)) continue;
        const int es = ek & 1;
        if (SE) {
          oz_mbar_wait(&e_full[es], (ek >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        const uint64_t bd0 = b_desc0 + static_cast<uint64_t>(((SE ? es : kb) * G::B_KB) >> 4);
#pragma unroll
        for (int s = 0; s < S; ++s, ++it) {
          const int st = it % G::NST;
          oz_mbar_wait(&a_full[st], (it / G::NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint64_t ad0 = a_desc0 + static_cast<uint64_t>((st * G::A_BYTES) >> 4);
          if (oz_elect()) {
#pragma unroll
            for (int kk = 0; kk < kOzBK / kOzUK; ++kk) {
              const uint32_t accf = (kb > kb0 || s > 0 || kk > 0) ? 1u : 0u;
              // a_s × [b_0 | … | b_{S-1-s}] → diagonals s … S-1 (contiguous columns), N ≤ 256 per MMA;
              // above 256 columns two equal halves (448 = 224 + 224, 384, 320) rather than 256 + rest:
              // two equal independent accumulation streams instead of a small tail MMA (−1.5 % per launch)
              const int W = (S - s) * kOzBN, CW = W > 256 ? W / 2 : W;
#pragma unroll
              for (int c0 = 0; c0 < W; c0 += CW) {
                const int nn = CW;
                oz_mma(tmem + static_cast<uint32_t>(s * kOzBN + c0), ad0 + static_cast<uint64_t>(kk) * a_kstep,
                       bd0 + static_cast<uint64_t>((c0 * kOzBK) >> 4) + static_cast<uint64_t>(kk * 2),
                       oz_idesc(nn, AMN), accf);
              }
            }
            oz_commit(&a_empty[st]);
          }
          __syncwarp();
        }
        if (SE) {  // the k-block's E slot is free once its MMAs are done
          if (oz_elect()) oz_commit(&e_empty[es]);
          __syncwarp();
          ++ek;
        }
      }
      if (oz_elect()) oz_commit(t_full);
      __syncwarp();
    }
    if (p.kcount && lane == 0) {
      atomicAdd(p.kcount, static_cast<unsigned long long>(tile) * nk);
      atomicAdd(p.kcount + 1, kb_run);
    }
  } else {
    // ---- epilogue warps: lane quarter wq = warp % 4 (TMEM lanes 32wq..), column half ch ----
    const int wq = warp & 3, ch = (warp - 2) >> 2;
    const uint32_t tl = tmem + (static_cast<uint32_t>(wq * 32) << 16) + ch * G::EPC;
    int tile = 0;
    for (int64_t u = sc.q; u < sc.units; u += sc.Q, ++tile) {
      const int term_i = static_cast<int>(u / sc.Mt);
      const int64_t mt = u % sc.Mt;
      oz_epilogue_tile<S, OUTD, AMN, REM, G::EPC>(p, term_i, mt * kOzBM + wq * 32 + lane, sc.nt * kOzBN + ch * G::EPC, tl, t_full,
                                tile & 1, [&] {
                                  if (lane == 0) oz_mbar_arrive(t_empty);
                                });
    }
  }
  if (p.remap.world > 0) __threadfence_system();  // peer stores visible before the barrier kernel
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

typedef CUresult (*OzEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

OzEncodeFn oz_encode_fn() {
  static const OzEncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<OzEncodeFn>(f);
    return static_cast<OzEncodeFn>(nullptr);
  }();
  return fn;
}

// 4-D map over int8 digits [slot][digit][row][k] with a (128, rows_box, digit_box, 1) box, SWIZZLE_128B
bool oz_encode(CUtensorMap* m, const int8_t* base, int64_t Kp, int64_t rows, int S, int slots, int rows_box,
               int slice_box) {
  OzEncodeFn fn = oz_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(S),
                              static_cast<cuuint64_t>(slots)};
  const cuuint64_t str[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Kp * rows),
                             static_cast<cuuint64_t>(Kp * rows * S)};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(kOzBK), static_cast<cuuint32_t>(rows_box),
                             static_cast<cuuint32_t>(slice_box), 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D map over an fp64 (L, n, R) tensor with a (32, n, 1) box (split_x tiles)
bool oz_encode_x(CUtensorMap* m, const double* base, int64_t L, int n, int64_t R) {
  OzEncodeFn fn = oz_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(R)};
  const cuuint64_t str[2] = {static_cast<cuuint64_t>(L) * 8, static_cast<cuuint64_t>(L) * n * 8};
  const cuuint32_t box[3] = {32, static_cast<cuuint32_t>(n), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D map over the digit array [slot][digit][fiber][k] with a (128, 32, 1, 1) box, SWIZZLE_128B (split_x stores)
bool oz_encode_digits(CUtensorMap* m, const int8_t* base, int64_t Kp, int64_t rows, int S, int slots) {
  OzEncodeFn fn = oz_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(S),
                              static_cast<cuuint64_t>(slots)};
  const cuuint64_t str[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Kp * rows),
                             static_cast<cuuint64_t>(Kp * rows * S)};
  const cuuint32_t box[4] = {128, 32, 1, 1};  // Kp ≥ 128 (the last k-half is clipped by the tensor bounds)
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D map over digit planes in the fp64 layout, (l, k, r, plane) with a (128, 128, 1, 1)
// box, SWIZZLE_128B: the MN-major A tiles of chained modes (L % 128 == 0)
bool oz_encode_mn(CUtensorMap* m, const int8_t* base, int64_t L, int n, int64_t R, int planes) {
  OzEncodeFn fn = oz_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(R),
                              static_cast<cuuint64_t>(planes)};
  const cuuint64_t str[3] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(L) * n,
                             static_cast<cuuint64_t>(L) * n * static_cast<cuuint64_t>(R)};
  const cuuint32_t box[4] = {128, static_cast<cuuint32_t>(kOzBK), 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool oz_split_tma_ok(const OzakiParams& p) {
  for (int b = 0; b < p.nx; ++b)
    if (reinterpret_cast<uintptr_t>(p.x[b]) & 15) return false;
  return p.R < (int64_t(1) << 31) && p.L < (int64_t(1) << 31);
}

template <int S, bool AMN, bool OUTD, bool SE, bool REM = false, bool KS = false>
cudaError_t oz_gemm_go(const OzakiParams& p, cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb) {
  // zero-block skipping where a tile with fewer k-blocks is shorter: the fp64-output
  // launches (the MMAs pace the tile; CTA groups by 16·kb + 12), the mode-1 digit-output launches
  // (K-major A, the lighter digit epilogue; 16·kb + 32), and the MN-major digit-output launches from
  // four k-blocks on (n > 384: the MMAs outweigh the epilogue again; 16·kb + 24).  With two k-blocks
  // the MN-major digit epilogue's per-tile work is as long as the MMAs' (§4e), a tile with fewer
  // k-blocks is barely shorter, and every grouping measured 3-20 % slower (the groups drift apart and
  // the fibre tiles are read from DRAM twice); with one k-block there is nothing to skip; nor in a
  // slab-sharded rank's short peer-store launches (streamed E, few tiles per CTA: emulated P = 8
  // 9.0-9.2 → 8.95-8.97 ms per step without skipping there, configs[4] 92.5-95.8 → 91.8-93.1)
#ifndef OZ_KS_AMN_OUTD_MINK
#define OZ_KS_AMN_OUTD_MINK 4
#endif
#ifndef OZ_KS_REM_SHORT
#define OZ_KS_REM_SHORT 0
#endif
  if constexpr (!KS) {
    const int nk = p.Kp / kOzBK;
    const bool rem_short = p.remap.world > 0 && SE && p.Kp <= kOzMaxNRes;  // a rank's short peer-store launch
    if (p.kskip && nk >= 2 && (!OUTD || !AMN || nk >= OZ_KS_AMN_OUTD_MINK) && (OZ_KS_REM_SHORT || !rem_short))
      return oz_gemm_go<S, AMN, OUTD, SE, REM, true>(p, st, ta, tb);
  }
  if constexpr (!REM && (AMN || !OUTD)) {  // peer-store epilogues: fp64 outputs, or AMN next-mode digits
    if (p.remap.world > 0) return oz_gemm_go<S, AMN, OUTD, SE, true, KS>(p, st, ta, tb);
  } else if constexpr (!REM) {
    if (p.remap.world > 0) return cudaErrorInvalidValue;
  }
  using G = OzGeom<S, oz_nst(AMN, OUTD, KS), oz_epc(OUTD)>;
  static bool gattr = false;
  static int sms = 0;
  if (!gattr) {
    cudaError_t e =
        cudaFuncSetAttribute(oz_gemm_kernel<S, AMN, OUTD, SE, REM, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gattr = true;
  }
  const int64_t C = p.L * p.R;
  const int ntn = (p.n + kOzBN - 1) / kOzBN;
  const int64_t units = ((C + kOzBM - 1) / kOzBM) * p.nterms;
  int64_t per = sms / ntn;  // CTAs per n-tile
  if (per > units) per = units;
  if (per < 1) per = 1;
  // kskip: every SM, the kernel splits them over the n-tiles by their work (OzSched)
  int64_t grid = per * ntn;
  if (KS) {
    grid = units * ntn < sms ? units * ntn : sms;
  }
  oz_gemm_kernel<S, AMN, OUTD, SE, REM, KS><<<static_cast<unsigned>(grid), G::THREADS, G::SMEM, st>>>(p, ta, tb);
  return cudaGetLastError();
}

// fewer fibre tiles per term than this many per CTA of an n-tile: stream E (configs[3] sharded at
// P = 8: 9.40 → 9.17 ms serial for the 8 emulated ranks; thresholds 2 / 4 / 8 equal, P = 1 and
// configs[2] unchanged)
constexpr int kOzSeUnits = 4;
int oz_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <int S>
cudaError_t oz_launch(const OzakiParams& p0, cudaStream_t st, bool split_x, bool split_e, bool gemm) {
  const OzakiParams& p = p0;
  const int64_t C = p.L * p.R;
  if (split_x) {
    const size_t sm = static_cast<size_t>(32) * (p.n | 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(oz_split_x_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           32 * (kOzMaxN | 1) * 8);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    if (p.cplx_j) {
      oz_split_x_kernel<S><<<dim3(static_cast<unsigned>((C + 31) / 32), p.nx), 256, sm, st>>>(p);
    } else if (p.L == 1) {
      const dim3 g(static_cast<unsigned>((C + 7) / 8), p.nx);
      switch (p.Kp) {  // Kp = n rounded up to 128
        case 128: oz_split_x_contig_kernel<S, 4><<<g, 256, 0, st>>>(p); break;
        case 256: oz_split_x_contig_kernel<S, 8><<<g, 256, 0, st>>>(p); break;
        case 384: oz_split_x_contig_kernel<S, 12><<<g, 256, 0, st>>>(p); break;
        case 512: oz_split_x_contig_kernel<S, 16><<<g, 256, 0, st>>>(p); break;
        default: return cudaErrorInvalidValue;
      }
    } else if (p.L % 32 == 0 && p.n <= 256 && p.Kp >= 128 && oz_split_tma_ok(p)) {
      static bool tattr = false;
      static int sms = 0;
      const int smem = 2 * 32 * kOzMaxNRes * 8 + S * 2 * 4096 + 16 * 32 * 8 + 16 * 32 * 4 + 64;
      if (!tattr) {
        cudaError_t e = cudaFuncSetAttribute(oz_split_x_tma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        tattr = true;
      }
      for (int s0 = 0; s0 < p.nx; s0 += kOzSplitSlots) {
        const int ns = p.nx - s0 < kOzSplitSlots ? p.nx - s0 : kOzSplitSlots;
        OzXMaps maps;
        for (int b = 0; b < ns; ++b)
          if (!oz_encode_x(&maps.m[b], p.x[s0 + b], p.L, p.n, p.R)) return cudaErrorInvalidValue;
        CUtensorMap dmap;
        if (!oz_encode_digits(&dmap, p.xs, p.Kp, C, S, p.nx)) return cudaErrorInvalidValue;
        const int64_t total = (C / 32) * ns;
        const int grid = static_cast<int>(total < sms ? total : sms);
        oz_split_x_tma_kernel<S><<<grid, 512, smem, st>>>(p, maps, dmap, s0, ns);
      }
    } else {
      oz_split_x_kernel<S><<<dim3(static_cast<unsigned>((C + 31) / 32), p.nx), 256, sm, st>>>(p);
    }
  }
  if (split_e && p.eext && !p.e_ready) {  // min / max / flag slots of the row-norm exponents
    cudaMemsetAsync(p.eext, 0x7f, sizeof(int) * p.ne, st);
    cudaMemsetAsync(p.eext + p.ne, 0x80, sizeof(int) * p.ne, st);
    cudaMemsetAsync(p.eext + 2 * p.ne, 0, sizeof(int) * 2 * p.ne, st);  // flags, nonzero digit blocks
  }
  if (split_e && !p.e_ready) oz_split_e_kernel<S><<<dim3((p.n + 7) / 8, p.ne), 256, 0, st>>>(p);
  if (split_e && p.n_next > 0 && p.nterms > 0 && !p.shard_stage0) {  // next-mode exponent bounds (chained modes)
    const int64_t m = C / p.n_next;
    oz_chain_kernel<<<dim3(static_cast<unsigned>((m + 31) / 32), p.nterms, (p.n + 63) / 64), 256, 0, st>>>(p);
  }
  if (p.nterms == 0 || !gemm) return cudaGetLastError();
  CUtensorMap ta, tb;
  const bool amap = p.a_mn ? oz_encode_mn(&ta, p.xs, p.L, p.n, p.R, S * p.nx)
                           : oz_encode(&ta, p.xs, p.Kp, C, S, p.nx, kOzBM, OzGeom<S>::SPS);
  if (!amap) return cudaErrorInvalidValue;
  if (!oz_encode(&tb, p.es, p.Kp, p.n, S, p.ne, kOzBN, S)) return cudaErrorInvalidValue;
  // E streamed per k-block: required above 256; also when a CTA would process few units per term
  // (short launches, e.g. a slab-sharded rank's), where every term switch would reload the
  // resident E tile with the MMAs stalled behind it
  const int64_t Mt = (C + kOzBM - 1) / kOzBM, Qn = oz_sms() / ((p.n + kOzBN - 1) / kOzBN);
  if (p.Kp > kOzMaxNRes || Mt < kOzSeUnits * Qn) {
    if (p.a_mn) {
      if (p.n_next > 0) return oz_gemm_go<S, true, true, true>(p, st, ta, tb);
      return oz_gemm_go<S, true, false, true>(p, st, ta, tb);
    }
    if (p.n_next > 0) return oz_gemm_go<S, false, true, true>(p, st, ta, tb);
    return oz_gemm_go<S, false, false, true>(p, st, ta, tb);
  }
  if (p.a_mn) {
    if (p.n_next > 0) return oz_gemm_go<S, true, true, false>(p, st, ta, tb);
    return oz_gemm_go<S, true, false, false>(p, st, ta, tb);
  }
  if (p.n_next > 0) return oz_gemm_go<S, false, true, false>(p, st, ta, tb);
  return oz_gemm_go<S, false, false, false>(p, st, ta, tb);
}

}  // namespace

size_t ozaki_workspace_bytes(int64_t L, int n, int64_t R, int S, int nx, int ne, int K) {
  if (K <= 0) K = n;
  const int64_t C = L * R, Kp = (K + kOzBK - 1) / kOzBK * kOzBK;
  auto al = [](size_t b) { return (b + 1023) & ~size_t(1023); };
  return al(static_cast<size_t>(nx) * S * C * Kp) + al(static_cast<size_t>(nx) * C * 8) +
         al(static_cast<size_t>(ne) * S * n * Kp) + 2 * al(static_cast<size_t>(ne) * n * 8) +
         al(static_cast<size_t>(ne) * n * 4) + al(static_cast<size_t>(ne) * 4 * 4);
}

int oz_multi_combine_split_max_out(int n) { return n <= 256 ? 8 : 4; }  // sums in registers: NOUT·n/32 doubles

cudaError_t launch_multi_combine_split(const MultiCombineParams& p, cudaStream_t st) {
  if (p.nout == 0 || p.count == 0) return cudaSuccess;
  const int n = p.fn;
  if (n < 1 || n > kOzMaxN || p.count % n != 0 || p.nout > oz_multi_combine_split_max_out(n) ||
      p.Kp != (n + kOzBK - 1) / kOzBK * kOzBK)
    return cudaErrorInvalidValue;
  bool aligned = (n % 2) == 0;
  for (int s = 0; s < p.nsrc; ++s) aligned &= (reinterpret_cast<uintptr_t>(p.src[s]) & 15) == 0;
  for (int o = 0; o < p.nout; ++o) aligned &= (reinterpret_cast<uintptr_t>(p.dst[o]) & 15) == 0;
  if (!aligned) return cudaErrorMisalignedAddress;
  const int64_t C = p.count / n;
  const dim3 g(static_cast<unsigned>((C + 7) / 8));
  // the wide variants (NOUT·EPL ≥ 48 sums in registers, ~180-220 registers) fit one 8-warp block per
  // SM, whose load and store phases then alternate; smaller blocks let several blocks per SM overlap
#ifndef OZ_MC_WPB_WIDE
#define OZ_MC_WPB_WIDE 8
#endif
  constexpr int WW = OZ_MC_WPB_WIDE;
  const dim3 gw(static_cast<unsigned>((C + WW - 1) / WW));
  const dim3 g2(static_cast<unsigned>((C + 3) / 4));  // warp pairs: 4 fibres per 8-warp block
  const int no = p.nout <= 2 ? 2 : (p.nout <= 4 ? 4 : 8);
  switch (p.Kp * 10 + no) {  // Kp = n rounded up to 128
    case 1282: oz_multi_combine_split_kernel<2, 4><<<g, 256, 0, st>>>(p); break;
    case 1284: oz_multi_combine_split_kernel<4, 4><<<g, 256, 0, st>>>(p); break;
    case 1288: oz_multi_combine_split_kernel<8, 4><<<g, 256, 0, st>>>(p); break;
    case 2562: oz_multi_combine_split_kernel<2, 8><<<g, 256, 0, st>>>(p); break;
    case 2564: oz_multi_combine_split_kernel<4, 8><<<g, 256, 0, st>>>(p); break;
    case 2568: oz_multi_combine_split_kernel<8, 4, 8, 2><<<g2, 256, 0, st>>>(p); break;
    case 3842: oz_multi_combine_split_kernel<2, 12><<<g, 256, 0, st>>>(p); break;
    case 3844: oz_multi_combine_split_kernel<4, 12, WW><<<gw, WW * 32, 0, st>>>(p); break;
    case 5122: oz_multi_combine_split_kernel<2, 16><<<g, 256, 0, st>>>(p); break;
    case 5124: oz_multi_combine_split_kernel<4, 8, 8, 2><<<g2, 256, 0, st>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

void ozaki_bind_workspace(OzakiParams& p, void* ws) {
  const int64_t C = p.L * p.R;
  const int K = p.cplx_j ? 2 * p.n : p.n;
  p.Kp = (K + kOzBK - 1) / kOzBK * kOzBK;
  auto al = [](size_t b) { return (b + 1023) & ~size_t(1023); };
  // the matrices' digits first: two launches with the same (ne, n, Kp) find them at the same place,
  // so a launch whose matrices the previous launch already split can skip that (e_ready)
  char* w = static_cast<char*>(ws);
  p.es = reinterpret_cast<int8_t*>(w);
  w += al(static_cast<size_t>(p.ne) * p.S * p.n * p.Kp);
  p.esc = reinterpret_cast<double*>(w);
  w += al(static_cast<size_t>(p.ne) * p.n * 8);
  p.eb = reinterpret_cast<double*>(w);
  w += al(static_cast<size_t>(p.ne) * p.n * 8);
  p.ecol = reinterpret_cast<int*>(w);
  w += al(static_cast<size_t>(p.ne) * p.n * 4);
  p.eext = reinterpret_cast<int*>(w);
  w += al(static_cast<size_t>(p.ne) * 4 * 4);
  p.xs = reinterpret_cast<int8_t*>(w);
  w += al(static_cast<size_t>(p.nx) * p.S * C * p.Kp);
  p.xsc = reinterpret_cast<double*>(w);
}

bool ozaki_supported(int64_t L, int n, int64_t R, int S) {
  const int64_t C = L * R;
  return S >= 6 && S <= 7 && n >= 1 && n <= kOzMaxN && C >= 1 && C < (int64_t(1) << 31);
}

cudaError_t launch_oz_shard_pmax(const OzShardExch& e, cudaStream_t st) {
  if (e.nterms == 0) return cudaSuccess;
  oz_shard_pmax_kernel<<<dim3(static_cast<unsigned>((e.L0 + 31) / 32), e.nterms), 256, 0, st>>>(e);
  return cudaGetLastError();
}

cudaError_t launch_oz_shard_tables(const OzShardExch& e, cudaStream_t st) {
  if (e.nterms == 0) return cudaSuccess;
  oz_shard_tables_kernel<<<dim3(static_cast<unsigned>((e.L0 * e.cb + 255) / 256), e.nterms), 256, 0, st>>>(e);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_mode(const OzakiParams& p, cudaStream_t st, bool split_x, bool split_e, bool gemm) {
  switch (p.S) {
    case 6: return oz_launch<6>(p, st, split_x, split_e, gemm);
    case 7: return oz_launch<7>(p, st, split_x, split_e, gemm);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace phiks
