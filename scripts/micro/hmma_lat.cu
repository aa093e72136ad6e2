// mma.sync.m16n8k16 latency (one dependent chain per warp) and throughput (4 chains)
// with 1..16 warps per SM, and the same for the decode-view ALU chain.  nvcc -arch=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(float* out, int iters, long long* clk) {
  unsigned a0 = threadIdx.x * 0x3c003c00u, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 4, b1 = a0 ^ 5;
  float c[CH][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 8 / CH; r++)
#pragma unroll
    for (int j = 0; j < CH; j++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  float s = 0;
  for (int j = 0; j < CH; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  const int iters = 2048;
  for (int warps : {1, 4, 8, 16}) {
    long long c1, c4;
    k<1><<<148, warps * 32>>>(out, iters, clk); cudaDeviceSynchronize(); cudaMemcpy(&c1, clk, 8, cudaMemcpyDeviceToHost);
    k<4><<<148, warps * 32>>>(out, iters, clk); cudaDeviceSynchronize(); cudaMemcpy(&c4, clk, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d: 8 HMMA per iter: 1 chain %.1f clk/HMMA per warp, 4 chains %.1f clk/HMMA per warp\n", warps,
           (double)c1 / (iters * 8), (double)c4 / (iters * 8));
  }
  return 0;
}
