// TMEM → register drain rate (B200): 8 warps (2 per TMEM lane quarter) read 448 columns
// of 128 lanes with tcgen05.ld.32x32b.x8, as the int8 GEMM epilogue does, repeatedly.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_probe scripts/tmem_drain_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int X>
__global__ void __launch_bounds__(256, 1) drain(int iters, uint64_t* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  const int wq = warp & 3, ch = warp >> 2;
  const uint32_t tl = tmem + (static_cast<uint32_t>(wq * 32) << 16) + ch * 32;
  uint32_t acc = 0;
  __syncthreads();
  const uint64_t t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int cb = 0; cb < 32 / X; ++cb) {
      uint32_t v[7][X];
#pragma unroll
      for (int g = 0; g < 7; ++g) {
        if (X == 8)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                       : "=r"(v[g][0]), "=r"(v[g][1]), "=r"(v[g][2]), "=r"(v[g][3]), "=r"(v[g][4]), "=r"(v[g][5]),
                         "=r"(v[g][6]), "=r"(v[g][7])
                       : "r"(tl + g * 64 + cb * X));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int g = 0; g < 7; ++g)
#pragma unroll
        for (int q = 0; q < X; ++q) acc += v[g][q];
    }
  }
  __syncthreads();
  const uint64_t t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 256 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* out;
  uint32_t* sink;
  cudaMalloc(&out, sms * 8);
  cudaMalloc(&sink, sms * 256 * 4);
  const int iters = 1000;
  for (int rep = 0; rep < 2; ++rep) drain<8><<<sms, 256>>>(iters, out, sink);
  cudaDeviceSynchronize();
  uint64_t h[256];
  cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double bytes = 128.0 * 448 * 4;  // one tile's accumulators
  printf("{\"probe\": \"tmem drain 128 lanes x 448 cols, 8 warps, 32x32b.x8\", \"err\": \"%s\", \"cycles_per_tile\": %.0f, "
         "\"bytes_per_cycle\": %.1f}\n",
         cudaGetErrorString(cudaGetLastError()), avg / iters, bytes * iters / avg);
  return 0;
}
