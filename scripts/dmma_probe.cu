// Standalone microbenchmark of the DMMA inner loop on sm_100a (not part of the
// library): how close to the FP64 tensor peak can an smem-fed warp tile get?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// pure register chains: W warps per block
__global__ void peak(int iters, double* sink) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0;
  double c[16][2];
  for (int u = 0; u < 16; ++u) c[u][0] = c[u][1] = u;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 16; ++u) dmma(c[u][0], c[u][1], a, b);
  double s = 0;
  for (int u = 0; u < 16; ++u) s += c[u][0] + c[u][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// smem-fed warp tile MI x NI (8x8 blocks), k loop over a smem tile of depth KD
template <int MI, int NI, int LD128>
__global__ void tile(int iters, double* sink) {
  constexpr int KD = 16;
  __shared__ double As[KD][MI * 16 + 4];  // room for two warps' rows
  __shared__ double Bs[KD][NI * 16 + 4];
  for (int i = threadIdx.x; i < KD * (MI * 16 + 4); i += blockDim.x) (&As[0][0])[i] = 1e-3 * (i % 7);
  for (int i = threadIdx.x; i < KD * (NI * 16 + 4); i += blockDim.x) (&Bs[0][0])[i] = 1e-3 * (i % 5);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lg = lane >> 2, lt = lane & 3;
  const int wm = (warp & 1) * MI * 8, wn = ((warp >> 1) & 1) * NI * 8;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k4 = 0; k4 < KD / 4; ++k4) {
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = As[k4 * 4 + lt][wm + i * 8 + lg];
#pragma unroll
      for (int j = 0; j < NI; ++j) b[j] = Bs[k4 * 4 + lt][wn + j * 8 + lg];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int blocks, int threads, int iters, double flops_per_warp_iter, double* sink) {
  kern<<<blocks, threads>>>(iters / 10, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = flops_per_warp_iter * iters * (threads / 32) * (double)blocks;
  printf("%-36s blocks=%4d threads=%4d : %6.2f TF/s  (%s)\n", name, blocks, threads, fl / (ms / 1e3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main1() {
  double* sink;
  cudaMalloc(&sink, 148 * 1024 * 8 * sizeof(double));
  for (int w : {1, 2, 3, 4, 8}) run("peak regs", peak, 148, 32 * 4 * w, 20000, 16 * 512.0, sink);
  // warp tile 64x32 (MI=8, NI=4): 32 DMMA per k4
  for (int w : {1, 2, 3, 4}) run("smem tile 64x32", tile<8, 4, 0>, 148, 32 * 4 * w, 4000, 4 * 32 * 512.0, sink);
  for (int w : {1, 2, 3, 4}) run("smem tile 32x32", tile<4, 4, 0>, 148, 32 * 4 * w, 4000, 4 * 16 * 512.0, sink);
  for (int w : {1, 2, 4}) run("smem tile 64x64", tile<8, 8, 0>, 148, 32 * 4 * w, 2000, 4 * 64 * 512.0, sink);
  for (int w : {2, 4}) run("smem tile 32x64", tile<4, 8, 0>, 148, 32 * 4 * w, 4000, 4 * 32 * 512.0, sink);
  for (int w : {2, 4}) run("smem tile 16x32", tile<2, 4, 0>, 148, 32 * 4 * w, 4000, 4 * 8 * 512.0, sink);
  return 0;
}

// ---------------------------------------------------------------------------
// GEMM-like pipeline probe: C(m, j) = Σ_k A(m,k) B(k,j) with A streamed from a
// big buffer (m contiguous, stride L per k), B a 256x256 matrix, 128x128 tile,
// 8 warps of 64x32, BK=16, 4 stages.  MODE 0 = cp.async 8B, 1 = no global loads
// (barriers only), 2 = cp.async 16B, 3 = loads but no barrier/wait (wrong
// results, timing only).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
template <int MODE>
__global__ void __launch_bounds__(256, 1) gemm_probe(const double* A, const double* B, double* C, long L, int ntiles) {
  constexpr int BM = 128, BN = 128, BK = 16, ST = 4, SA = BM + 4, SB = BN + 4, n = 256;
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + ST * BK * SA;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lg = lane >> 2, lt = lane & 3;
  const int wm0 = (warp / 4) * 64, wn0 = (warp % 4) * 32;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long m0 = (long)(tile / 2) * BM;
    const int j0 = (tile % 2) * BN;
    auto load = [&](int st, int kt) {
      if (MODE == 1) return;
      double* as = As + st * BK * SA;
      double* bs = Bs + st * BK * SB;
      if (MODE == 2) {
        for (int i = 0; i < 4; ++i) {  // A: 128x16 = 2048 doubles = 1024 x 16B, 4 per thread
          const int e = tid + i * 256, mm = (e % 64) * 2, kk = e / 64;
          cpa16(as + kk * SA + mm, A + m0 + mm + L * (kt * BK + kk));
        }
        for (int i = 0; i < 4; ++i) {
          const int e = tid + i * 256, jj = (e % 64) * 2, kk = e / 64;
          cpa16(bs + kk * SB + jj, B + j0 + jj + (long)(kt * BK + kk) * n);
        }
      } else {
        for (int i = 0; i < 8; ++i) {
          const int mm = tid % BM, kk = tid / BM + 2 * i;
          cpa8(as + kk * SA + mm, A + m0 + mm + L * (kt * BK + kk));
        }
        for (int i = 0; i < 8; ++i) {
          const int jj = tid % BN, kk = tid / BN + 2 * i;
          cpa8(bs + kk * SB + jj, B + j0 + jj + (long)(kt * BK + kk) * n);
        }
      }
    };
    double acc[8][4][2];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0;
    for (int s = 0; s < ST - 1; ++s) { load(s, s); asm volatile("cp.async.commit_group;\n"); }
    for (int kt = 0; kt < n / BK; ++kt) {
      if (MODE != 3) { asm volatile("cp.async.wait_group 2;\n" ::: "memory"); __syncthreads(); }
      if (kt + ST - 1 < n / BK) load((kt + ST - 1) % ST, kt + ST - 1);
      asm volatile("cp.async.commit_group;\n");
      const double* as = As + (kt % ST) * BK * SA + lt * SA + wm0 + lg;
      const double* bs = Bs + (kt % ST) * BK * SB + lt * SB + wn0 + lg;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        double a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = as[k4 * 4 * SA + i * 8];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = bs[k4 * 4 * SB + j * 8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j)
        for (int e = 0; e < 2; ++e)
          C[m0 + wm0 + i * 8 + lg + L * (j0 + wn0 + j * 8 + 2 * lt + e)] = acc[i][j][e];
  }
}

template <int MODE>
void run_gemm(const char* name, const double* A, const double* B, double* C, long L, int grid) {
  const int smem = 4 * 16 * (132 + 132) * 8;
  cudaFuncSetAttribute(gemm_probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int ntiles = (int)(L / 128) * 2;
  gemm_probe<MODE><<<grid, 256, smem>>>(A, B, C, L, ntiles);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) gemm_probe<MODE><<<grid, 256, smem>>>(A, B, C, L, ntiles);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s grid=%4d: %6.2f TF/s  (%s)\n", name, grid, 2.0 * L * 256 * 256 * 5 / (ms / 1e3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main2() {
  const long L = 65536;  // A: L x 256 (m contiguous) = 134 MB
  double *A, *B, *C;
  cudaMalloc(&A, L * 256 * 8);
  cudaMalloc(&B, 256 * 256 * 8);
  cudaMalloc(&C, L * 256 * 8);
  cudaMemset(A, 0, L * 256 * 8);
  cudaMemset(B, 0, 256 * 256 * 8);
  for (int grid : {148, 1024}) {
    run_gemm<0>("pipeline cp.async 8B", A, B, C, L, grid);
    run_gemm<1>("pipeline no loads (barriers)", A, B, C, L, grid);
    run_gemm<2>("pipeline cp.async 16B", A, B, C, L, grid);
    run_gemm<3>("pipeline 8B, no wait/barrier", A, B, C, L, grid);
  }
  return 0;
}

int main() { main1(); main2(); return 0; }
