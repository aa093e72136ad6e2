// Microbenchmark: throughput of the Q3H decode unit with data resident in shared
// memory (no producer, no phases).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20
#include <cstdio>
#include "../../paper_2401_08294_b200/csrc/decode_mk.cu"

template <int R, int NW, int SYNC>
__global__ void __launch_bounds__(NW * 32, 1) unit_bench(float* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ring = sm;                       // 32 KB of rows
  float4* xs = reinterpret_cast<float4*>(sm + 32768);
  float2* bs = reinterpret_cast<float2*>(xs + 16 * 73);
  float* part = reinterpret_cast<float*>(bs + 64);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(ring)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 16 * 73; i += blockDim.x) xs[i] = make_float4(1.f, 2.f, 3.f, 4.f);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) bs[i] = make_float2(1.f, 1.f);
  __syncthreads();
  const ifb::Q3HConst kc = ifb::q3h_const();
  const int w = threadIdx.x >> 5;
  for (int it = 0; it < iters; it++) {
    const int u = (w + it * NW) & 7;  // 8 units per 32 KB slot (16 rows x 2 chunks, R=4) / 4 units (R=8)
    const int units = 16 / R * 2;
    const int uu = u % units;
    const int grp = uu / 2, c = uu % 2;
    ifb::mk_unit<R, 73, true>(ring + grp * R * 2048, 2048, R, c, 64, 73, xs, bs, part + (w & 7) * 64, 2, kc);
    if (SYNC && (it % SYNC) == SYNC - 1) __syncthreads();  // waves: every warp starts together
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = part[0];
}

template <int R, int NW, int SYNC = 0>
void run(float* out) {
  auto k = unit_bench<R, NW, SYNC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int iters = 2000;
  k<<<148, NW * 32, 64 * 1024>>>(out, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, NW * 32, 64 * 1024>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double weights = 148.0 * NW * iters * R * 32 * 64;
  printf("sync=%d R=%d warps=%2d: %.3f ms  %.1f weights/clk/SM (@1.965GHz)  = %.0f GB/s Q3H-equivalent  err=%s\n", SYNC, R, NW, ms,
         weights / 148 / (ms * 1e-3 * 1.965e9), weights * 0.5 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 4);
  run<4, 16>(out); run<4, 16, 1>(out); run<4, 16, 3>(out); run<4, 15, 1>(out); run<8, 12>(out); run<8, 12, 1>(out);
  return 0;
}
