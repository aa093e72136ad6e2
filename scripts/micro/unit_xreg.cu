// Microbenchmark: the Q3H batch-1 decode unit (decode_mk.cu mk_unit) with the staged x
// read from shared memory (as the engine does) vs held in registers across units
// (x loaded once per warp): is the unit bounded by shared-memory bandwidth?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 unit_xreg.cu
#include <cstdio>
#include "../../paper_2401_08294_b200/csrc/decode_mk.cu"

using namespace ifb;
// mk_unit with the 16 x quads of this lane's block passed in registers
template <int R>
__device__ __forceinline__ void unit_xr(const unsigned char* slot_rows, int row_bytes, int c, const float4 (&xq)[16],
                                        float sx, float* part_rows, int nchunk) {
  const int lane = threadIdx.x & 31;
  const int b = c * 32 + lane;
  uint32_t wv[R][8];
#pragma unroll
  for (int i = 0; i < R; i++) {
    const uint4* a = reinterpret_cast<const uint4*>(slot_rows + i * row_bytes + b * 32);
    const uint4 lo = a[0], hi = a[1];
    wv[i][0] = lo.x; wv[i][1] = lo.y; wv[i][2] = lo.z; wv[i][3] = lo.w;
    wv[i][4] = hi.x; wv[i][5] = hi.y; wv[i][6] = hi.z; wv[i][7] = hi.w;
  }
  uint32_t vw[R][7];
#pragma unroll
  for (int i = 0; i < R; i++) {
    vw[i][0] = q3h_sview<0>(wv[i]); vw[i][1] = q3h_sview<1>(wv[i]); vw[i][2] = q3h_sview<2>(wv[i]);
    vw[i][3] = q3h_sview<3>(wv[i]); vw[i][4] = q3h_sview<4>(wv[i]); vw[i][5] = q3h_sview<5>(wv[i]);
    vw[i][6] = q3h_sview<6>(wv[i]);
  }
  u64 accc[R / 2], accq[R / 2];
#pragma unroll
  for (int i = 0; i < R / 2; i++) accc[i] = accq[i] = 0ull;
  [&]<int... J>(std::integer_sequence<int, J...>) {
    (
        [&] {
          const float4 xv = xq[J / 2];
          const float XC = (J & 1) ? xv.y : xv.x, XQ = (J & 1) ? xv.w : xv.z;
          constexpr uint32_t fmb = q3h_floor_mult_bits(kQ3hSrc[J].pos);
          const u64 fm2 = pack2(__uint_as_float(fmb), __uint_as_float(fmb));
          const u64 xc2 = pack2(XC, XC), xq2 = pack2(XQ, XQ);
#pragma unroll
          for (int ip = 0; ip < R / 2; ip++) {
            const u64 cf = pack2(__uint_as_float(q3h_scode_bits<J>(wv[2 * ip], vw[2 * ip])),
                                 __uint_as_float(q3h_scode_bits<J>(wv[2 * ip + 1], vw[2 * ip + 1])));
            const u64 qe = ffma2_rm(cf, fm2, 0ull);
            accc[ip] = ffma2(cf, xc2, accc[ip]);
            accq[ip] = ffma2(qe, xq2, accq[ip]);
          }
        }(),
        ...);
  }(std::make_integer_sequence<int, 32>{});
  float v[R];
#pragma unroll
  for (int ip = 0; ip < R / 2; ip++) {
    const float2 a = unpack2(accc[ip]), q = unpack2(accq[ip]);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int i = 2 * ip + h;
      const float lo = half_bits_to_float(wv[i][0] & 0xFFFFu), hi = half_bits_to_float(wv[i][0] >> 16);
      const float step = (hi - lo) * (0.1f * 18446744073709551616.0f);
      v[i] = fmaf(step, h ? (a.y + q.y) : (a.x + q.x), lo * sx);
    }
  }
  const float sum = warp_rows_sum<R>(v);
  constexpr int SH = R == 8 ? 2 : (R == 4 ? 3 : (R == 2 ? 4 : 5));
  if ((lane & ((1 << SH) - 1)) == 0) part_rows[(lane >> SH) * nchunk + c] = sum;
}

template <int R, int NW, int XREG>
__global__ void __launch_bounds__(NW * 32, 1) bench(float* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ring = sm;
  float4* xs = reinterpret_cast<float4*>(sm + 32768);
  float2* bs = reinterpret_cast<float2*>(xs + 16 * 73);
  float* part = reinterpret_cast<float*>(bs + 64);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(ring)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 16 * 73; i += blockDim.x) xs[i] = make_float4(1.f + i, 2.f, 3.f, 4.f);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) bs[i] = make_float2(1.f, 1.f);
  __syncthreads();
  const Q3HConst kc = q3h_const();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = w & 1;  // a warp keeps one chunk (x of its block in registers when XREG)
  float4 xq[16];
#pragma unroll
  for (int j = 0; j < 16; j++) xq[j] = xs[j * 73 + c * 32 + lane];
  const float sx = bs[c * 32 + lane].x;
  for (int it = 0; it < iters; it++) {
    const int grp = ((w >> 1) + it * (NW / 2)) % (16 / R);
    if (XREG) unit_xr<R>(ring + grp * R * 2048, 2048, c, xq, sx, part + (w & 7) * 64, 2);
    else mk_unit<R, 73, true>(ring + grp * R * 2048, 2048, R, c, 64, 73, xs, bs, part + (w & 7) * 64, 2, kc);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = part[0];
}

template <int R, int NW, int XREG>
void run(float* out) {
  auto k = bench<R, NW, XREG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 2000;
  k<<<148, NW * 32, 64 * 1024>>>(out, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, NW * 32, 64 * 1024>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double weights = 148.0 * NW * iters * R * 32 * 64;
  printf("xreg=%d R=%d warps=%2d: %.3f ms  %.1f weights/clk/SM (@1.965GHz)  err=%s\n", XREG, R, NW, ms,
         weights / 148 / (ms * 1e-3 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 4);
  run<4, 16, 0>(out); run<4, 16, 1>(out); run<2, 16, 1>(out); run<2, 16, 0>(out); run<4, 8, 1>(out); run<4, 8, 0>(out);
  return 0;
}
// link stubs for the library symbols decode_mk.cu references (host side, unused here)
namespace ifb {
if_status set_error(if_status st, const char*, ...) { return st; }
if_status check_launch(const char*) { return IF_OK; }
void count_launch(int) {}
}  // namespace ifb
