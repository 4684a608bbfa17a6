// Tensor-core issue probe (B200): the int8 GEMM's per-stage MMA sequence issued back to back from
// shared memory (no data movement), with one CTA per SM and 512 TMEM columns (the kernel: 64-row E
// tiles, 7 diagonals × 64 columns) against two CTAs per SM with 256 columns each (32-row E tiles,
// 7 × 32 columns: two independent accumulator pipelines per SM, each CTA's drain could hide behind
// the other's MMAs).  Aggregate MACs per SM per cycle over the whole grid.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/up2 scripts/umma_probe_2cta.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  uint64_t d = (a >> 4) & 0x3FFFu;
  d |= 1ull << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}

// BN: E rows per tile (64: the kernel, 32: the half tile); COLS: TMEM columns allocated
template <int BN, int COLS>
__global__ void __launch_bounds__(128) probe(int tiles, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 80 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(i * 2654435761u, i ^ 0x9e37, 7u * i, 0x5bd1e995u + i);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&slot)), "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint64_t a0 = desc_sw128(su32(base)), b0 = desc_sw128(su32(base + 16384));
    const long long t0 = clock64();
    for (int t = 0; t < tiles; ++t)
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int s = 0; s < 7; ++s)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            constexpr int dummy = 0;
            (void)dummy;
            const int W = (7 - s) * BN;
            const int CW = W > 256 ? W / 2 : W;
            for (int c0 = 0; c0 < W; c0 += CW)
              mma(tmem + s * BN + c0, a0 + kk * 2, b0 + kk * 2, idesc_i8(128, CW),
                  (kb | s | kk) ? 1u : 0u);
          }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&done))
                 : "memory");
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(
                     su32(&done))
                 : "memory");
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(COLS));
}

template <int BN, int COLS>
void run(const char* name, int ctas_per_sm, int tiles) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 80 * 1024 + 1024;
  cudaFuncSetAttribute(probe<BN, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = sms * ctas_per_sm;
  unsigned long long* cyc;
  cudaMalloc(&cyc, grid * sizeof(unsigned long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    probe<BN, COLS><<<grid, 128, smem>>>(tiles, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  // MACs per CTA: tiles × 2 k-blocks × 4 k-steps × Σ_s 128·(7−s)·BN·32
  double macs_cta = 0;
  for (int s = 0; s < 7; ++s) macs_cta += 128.0 * (7 - s) * BN * 32;
  macs_cta *= 8.0 * tiles;
  const double total = macs_cta * grid;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  printf("{\"variant\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f, \"macs_per_sm_per_clk_at_%d_mhz\": %.0f}\n", name,
         cudaGetErrorString(cudaGetLastError()), ms, 2 * total / (ms * 1e-3) / 1e12, clk / 1000,
         total / sms / (ms * 1e-3 * clk * 1e3));
  cudaFree(cyc);
}

int main() {
  for (int r = 0; r < 2; ++r) {
    run<64, 512>("BN64 (kernel), 1 CTA/SM, 512 cols", 1, 400);
    run<32, 256>("BN32, 1 CTA/SM, 256 cols", 1, 800);
    run<32, 256>("BN32, 2 CTAs/SM, 256 cols each", 2, 400);
  }
  return 0;
}
