// Resolution / rate of clock64 and %globaltimer on this GPU.
#include <cstdio>
__global__ void k(unsigned long long* out) {
  unsigned long long g0, g1, c0 = clock64(), c1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  unsigned long long prevg = g0, prevc = c0;
  int gchanges = 0, cchanges = 0;
  unsigned long long mingstep = ~0ull, mincstep = ~0ull;
  for (int i = 0; i < 200000; i++) {
    unsigned long long g, c = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    if (g != prevg) { gchanges++; if (g - prevg < mingstep) mingstep = g - prevg; prevg = g; }
    if (c != prevc) { cchanges++; if (c - prevc < mincstep) mincstep = c - prevc; prevc = c; }
  }
  c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  out[0] = g1 - g0; out[1] = c1 - c0; out[2] = gchanges; out[3] = cchanges; out[4] = mingstep; out[5] = mincstep;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  k<<<1, 1>>>(d); cudaDeviceSynchronize();
  unsigned long long h[6]; cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
  printf("globaltimer delta %llu ns, clock64 delta %llu cycles -> %.3f GHz; gt changes %llu (min step %llu ns), clk changes %llu (min step %llu)\n",
         h[0], h[1], (double)h[1] / h[0], h[2], h[4], h[3], h[5]);
  return 0;
}
