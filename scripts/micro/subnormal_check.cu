// Check: for every code c in [0,127] at every bit position s in [0,17], the
// subnormal float cf = bits(c << s) times A_s = roundup(1/11) * 2^-s, rounded
// toward -inf (fma.rm, addend 0) gives exactly floor(c/11) * 2^-149 (bits = c/11),
// scalar and packed (fma.rm.f32x2); and cf * X is exact.
#include <cstdio>
#include <cstdint>
__global__ void k(int* bad, float A0) {
  int s = threadIdx.x;  // 0..17
  for (int c = 0; c < 128; c++) {
    float cf = __uint_as_float((uint32_t)c << s);
    float A = A0 * exp2f(-(float)s);
    float r;
    asm("fma.rm.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(cf), "f"(A), "f"(0.0f));
    if (__float_as_uint(r) != (uint32_t)(c / 11)) atomicAdd(bad, 1);
    unsigned long long a2, b2, d2, z = 0;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a2) : "f"(cf), "f"(__uint_as_float((uint32_t)(127 - c) << s)));
    asm("mov.b64 %0, {%1,%1};" : "=l"(b2) : "f"(A));
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(d2) : "l"(a2), "l"(b2), "l"(z));
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(d2));
    if (__float_as_uint(lo) != (uint32_t)(c / 11) || __float_as_uint(hi) != (uint32_t)((127 - c) / 11)) atomicAdd(bad + 1, 1);
    float x = 0.37251f;
    float X = x * exp2f((float)(149 - s - 64));
    float p = cf * X;
    float ref = (float)c * x * exp2f(-64.f);
    if (p != ref) atomicAdd(bad + 2, 1);
  }
}
int main() {
  int* bad; cudaMalloc(&bad, 12); cudaMemset(bad, 0, 12);
  float A0 = 1.0f / 11.0f;
  if ((double)A0 < 1.0 / 11.0) A0 = nextafterf(A0, 1.0f);
  k<<<1, 18>>>(bad, A0);
  int h[3]; cudaMemcpy(h, bad, 12, cudaMemcpyDeviceToHost);
  printf("A0=%.10e (1/11=%.10e)  scalar mismatches=%d  packed mismatches=%d  product mismatches=%d  %s\n", A0, 1.0/11, h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
