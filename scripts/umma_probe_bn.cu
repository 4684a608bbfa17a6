// Tensor-core MMA rate probe (B200), BN = 64 against BN = 32 MMA sequences (round 2): back-to-back tcgen05.mma from shared memory into
// TMEM, one CTA (or CTA pair) per SM, no data movement — the ceiling an MMA-issue-bound
// kernel can reach for a given kind / shape.  Operand contents are irrelevant (zeros).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/umma_probe scripts/umma_probe.cu -lcuda
//   /tmp/umma_probe            (prints one JSON line per variant)
#include <cuda.h>
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
// kind: 0 = i8 (s8·s8 → s32), 1 = f16 (bf16·bf16 → f32)
__host__ __device__ constexpr uint32_t idesc(int kind, int m, int n) {
  return kind == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24))
                   : ((1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24));
}

template <int KIND, int PAIR>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  if (KIND == 0 && PAIR == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id));
  if (KIND == 1 && PAIR == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id));
  if (KIND == 2 && PAIR == 0)  // A operand in TMEM (column a of the allocation), int8
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(static_cast<uint32_t>(a)), "l"(b), "r"(id));
  if (KIND == 0 && PAIR == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id));
  if (KIND == 1 && PAIR == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id));
}

// one round = the MMA list (TMEM column, N) in order; K = 32 bytes per MMA
__constant__ int c_col[64], c_n[64];
template <int KIND, int PAIR>
__global__ void __launch_bounds__(128, 1) probe(int iters, int nmix, int4 ns, uint64_t* out_cycles) {
  // ns.x: commit + fence every ns.x MMAs (0: never); ns.y: random operand bytes
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x) {
    uint32_t h = ns.y ? (i * 2654435761u + blockIdx.x * 97u) : 0u;
    reinterpret_cast<uint4*>(base)[i] = make_uint4(h, h * 3u + 1u, h ^ 0x5bd1e995u, h * 7u);
  }
  __shared__ uint64_t bar2;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar2)));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  const int M = PAIR ? 256 : 128;
  uint64_t t0 = 0, t1 = 0;
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t a = desc_sw128(su32(base)), b = desc_sw128(su32(base + 16384));
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int j = 0; j < nmix; ++j) {
        if (KIND == 2)
          mma<KIND, PAIR>(tmem + c_col[j], tmem + 448 + (it & 3) * 8, b + (it & 3) * 2, idesc(0, M, c_n[j]));
        else
          mma<KIND, PAIR>(tmem + c_col[j], a + (it & 3) * 2, b + (it & 3) * 2, idesc(KIND, M, c_n[j]));
        if (ns.x && (j % ns.x) == ns.x - 1) {
          if (ns.z & 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar2))
                         : "memory");
          if (ns.z & 2) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          if (ns.z & 4) asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        }
      }
    }
    if (PAIR)
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
              su32(&bar)),
          "h"(static_cast<uint16_t>(3))
          : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                   : "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile(
        "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(su32(&bar))
        : "memory");
    t1 = clock64();
    if (rank == 0) out_cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else
    __syncthreads();
  if (warp == 0) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}


// the GEMM's MMA warp pattern: per stage (digit s of A, 4 k-steps) wait on an mbarrier
// (already complete), fence, elect one lane, issue the stage's MMAs, commit to another
// mbarrier; stages of `group` digits
__global__ void __launch_bounds__(128, 1) stage_probe(int iters, int group, uint64_t* out_cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full, empty, done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(base)[i] = make_uint4(i, 3 * i, 7, i ^ 5);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&empty)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 0) {
    // complete phase 0 of `full` so every wait on parity 0 passes at once
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&full)) : "memory");
    __syncwarp();
    const uint64_t a0 = desc_sw128(su32(base)), b0 = desc_sw128(su32(base + 16384));
    const uint64_t t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int s = 0; s < 7; ++s) {
        if (group == 1 || (s % group) == 0) {
          asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(
                           su32(&full))
                       : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        uint32_t pred = 0;
        asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
        if (pred) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int c0 = 0; c0 < (7 - s) * 64; c0 += 256) {
              const int nn = (7 - s) * 64 - c0 < 256 ? (7 - s) * 64 - c0 : 256;
              mma<0, 0>(tmem + s * 64 + c0, a0 + kk * 2, b0 + ((c0 * 128) >> 4) + kk * 2, idesc(0, 128, nn));
            }
          if (group == 1 || (s % group) == group - 1 || s == 6)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&empty))
                         : "memory");
        }
        __syncwarp();
      }
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&done))
                   : "memory");
      asm volatile("{\n.reg .pred P;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W2;\n}\n" ::"r"(
                       su32(&done))
                   : "memory");
      out_cycles[blockIdx.x] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

void run_stage(const char* name, int group, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 16 * 1024 + 56 * 1024 + 1024;
  cudaFuncSetAttribute(stage_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint64_t* cyc;
  cudaMalloc(&cyc, sms * sizeof(uint64_t));
  for (int rep = 0; rep < 2; ++rep) stage_probe<<<sms, 128, smem>>>(iters, group, cyc);
  cudaDeviceSynchronize();
  uint64_t h[256];
  cudaMemcpy(h, cyc, sms * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double macs = 128.0 * 64 * 28 * 32 * 4 * iters;  // per SM
  printf("{\"variant\": \"%s\", \"err\": \"%s\", \"macs_per_sm_per_clk\": %.0f, \"frac_of_8192\": %.3f}\n", name,
         cudaGetErrorString(cudaGetLastError()), macs / avg, macs / avg / 8192);
  cudaFree(cyc);
}

template <int KIND, int PAIR>
void run(const char* name, int nmix, const int* cols, const int* nsz, int iters, int4 ns = make_int4(0, 0, 0, 0)) {
  cudaMemcpyToSymbol(c_col, cols, nmix * sizeof(int));
  cudaMemcpyToSymbol(c_n, nsz, nmix * sizeof(int));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 48 * 1024 + 1024;
  cudaFuncSetAttribute(probe<KIND, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint64_t* cyc;
  cudaMalloc(&cyc, sms * sizeof(uint64_t));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {  // warm-up, then timed
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, probe<KIND, PAIR>, iters, nmix, ns, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  double macs = 0;
  const int M = PAIR ? 256 : 128, K = KIND != 1 ? 32 : 16;
  for (int j = 0; j < nmix; ++j) macs += double(M) * nsz[j] * K;
  macs *= double(iters) * (PAIR ? sms / 2 : sms);
  uint64_t h[256];
  cudaMemcpy(h, cyc, sms * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  double cyc_avg = 0;
  int cnt = 0;
  for (int i = 0; i < sms; i += (PAIR ? 2 : 1)) cyc_avg += h[i], ++cnt;
  cyc_avg /= cnt;
  const double macs_per_sm_clk = macs / (PAIR ? sms : sms) / cyc_avg;
  printf("{\"variant\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f, \"macs_per_sm_per_clk\": %.0f}\n", name,
         cudaGetErrorString(err), ms, 2 * macs / (ms * 1e-3) / 1e12, macs_per_sm_clk);
  cudaFree(cyc);
}

int main() {
  // per k-step MMA lists of the GEMM: BN = 64 (the kernel) and BN = 32 (two accumulator sets)
  const int c64[] = {0, 256, 64, 320, 128, 384, 192, 256, 320, 384};
  const int n64[] = {256, 192, 256, 128, 256, 64, 256, 192, 128, 64};
  const int c32[] = {0, 32, 64, 96, 128, 160, 192};
  const int n32[] = {224, 192, 160, 128, 96, 64, 32};
  const int c256[] = {0, 256, 0, 256, 0, 256, 0};
  const int n256[] = {256, 192, 256, 192, 256, 192, 256};
  for (int rnd = 0; rnd < 2; ++rnd) {
    run<2, 0>(rnd ? "BN64 seq, A in TMEM, random operands" : "BN64 seq, A in TMEM, zero operands", 10, c64, n64, 4000, make_int4(0, rnd, 0, 0));
    run<0, 0>(rnd ? "N256/192 mix, random" : "N256/192 mix, zero", 7, c256, n256, 4000, make_int4(0, rnd, 0, 0));
    run<2, 0>(rnd ? "N256/192 mix, A in TMEM, random" : "N256/192 mix, A in TMEM, zero", 7, c256, n256, 4000, make_int4(0, rnd, 0, 0));
    run<0, 0>(rnd ? "BN64 seq, random operands" : "BN64 seq, zero operands", 10, c64, n64, 4000, make_int4(0, rnd, 0, 0));
    run<0, 0>(rnd ? "BN32 seq, random operands" : "BN32 seq, zero operands", 7, c32, n32, 4000, make_int4(0, rnd, 0, 0));
  }
  return 0;
}
