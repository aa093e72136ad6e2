// mma.sync.m16n8k16 (f16 x f16 -> f32) throughput on one B200: every warp issues
// independent MMA chains; reports FLOP/clk per SM.   nvcc -arch=sm_100a -O3 hmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters, long long* clk) {
  unsigned a0 = threadIdx.x * 0x3c003c00u, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 4, b1 = a0 ^ 5;
  float c[4][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  float s = 0;
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  for (int warps : {4, 8, 16}) {
    int iters = 4096;
    k<<<148, warps * 32>>>(out, 16, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, warps * 32>>>(out, iters, clk);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    double flop = 148.0 * warps * iters * 4 * 16 * 8 * 16 * 2;
    printf("warps/SM %2d: %.1f TFLOP/s, %.0f FLOP/clk/SM (clk %lld)\n", warps, flop / ms / 1e9, 16.0 * 8 * 16 * 2 * 4 * iters * warps / (double)c, c);
  }
  return 0;
}
