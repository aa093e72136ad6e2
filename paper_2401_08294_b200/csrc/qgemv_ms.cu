// qgemv_ms.cu — batched decode qGEMV (a4, 2 <= B <= 32, Q3H_B64) on the tensor cores
// through warp-level mma.sync.m16n8k16 (f16 x f16 -> f32), with the 3.5-bit decode
// done in registers straight into the MMA's A fragments (no shared-memory W' tile):
//
//   y[b, n] = sum_k W'[n, k] x[b, k],   W' = Eq. 2 (exact fp32) rounded once to fp16,
//   x = hi + lo (two fp16 per token, per-token power-of-two scale; Q23)
//
// Why not tcgen05 here: at decode batch sizes the UMMA N is 16..64, and the tcgen05
// path measured ~600 clk per 64-k step in the issue + commit of its four small MMAs
// alone (profiles/r1_qgemv_tc_prof.txt); a warp-level m16n8k16 costs the SM 2 clk
// (scripts/micro/hmma_bench: 2048 FLOP/clk/SM), so for N <= 64 the tensor work is
// cheap and the kernel is paced by the decode, as the batch-1 engine is.
//
// Layout.  A warp owns 16 weight rows; lane l = (r0 = l/4, c = l%4).  The MMA's k
// order inside a 64-weight block is permuted (a dot product does not care) so that
// lane c's A-fragment k-slots are the 8 consecutive pair codes [8c, 8c+8) of its two
// rows r0, r0+8 (pair j = weights 2j, 2j+1): group g (k 16g..16g+15) uses
// pairs 8c+2g (k slots 2c, 2c+1) and 8c+2g+1 (slots 2c+8, 2c+9).  The B fragments
// then read x at the ORIGINAL positions 64 kb + 16c + 4g + {0,1} and + {2,3}: one
// 8-byte shared load per (group, token tile).  The x tile of the CTA's K-range sits
// in shared memory with a row pitch of 2 (mod 32) words (conflict-free); the packed
// rows are loaded coalesced (one 16-byte load per lane per block, lane l -> row l/2)
// and redistributed through a per-warp shared buffer.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "qgemm.cuh"
#include "simd.cuh"

namespace ifb {

constexpr int MS_WARPS = 8;             // 16 rows each -> 128 rows per CTA
constexpr int MS_ROWS = 16 * MS_WARPS;
constexpr int MS_THREADS = 32 * MS_WARPS;
#ifndef IFB_MS_SMEM_KB
#define IFB_MS_SMEM_KB 100
#endif
#ifndef IFB_MS_DEPTH
#define IFB_MS_DEPTH 8
#endif
#ifndef IFB_MS_MINB
#define IFB_MS_MINB 2
#endif
constexpr int MS_SMEM_MAX = IFB_MS_SMEM_KB * 1024;  // x tile + weight rings per CTA (two CTAs per SM)
constexpr int MS_DEPTH = IFB_MS_DEPTH;              // weight blocks in flight per warp (cp.async ring)

__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__host__ __device__ constexpr float __uint_as_float_c(uint32_t u) { return __builtin_bit_cast(float, u); }
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// W' of the 8 pairs [8c, 8c+8) of TWO rows' Q3H_B64 blocks (words in shared memory),
// the two rows sharing every f32x2 instruction: Eq. 2 (w' = lo + q step, step =
// (hi - lo)/10) in fp32, rounded once to fp16.  The pair code v (7 bits) is
// masked out at bit s <= 17 of a 32-bit source, which makes it the float
// v 2^(s-149) (simd.cuh): q_e = floor(v/11) by one FMA rounding down onto
// the subnormal grid, q_o = v - 11 q_e by one exact FMA, two exact scalings
// into the normal range and one FMA each for w'.  10 instructions per 4 weights.
template <int S>
__device__ __forceinline__ void ms_pair(uint32_t src0, uint32_t src1, u64 step2, u64 lo2, uint32_t& out0,
                                        uint32_t& out1) {
  constexpr uint32_t mask = 0x7Fu << S;
  const u64 cf = pack2(__uint_as_float(src0 & mask), __uint_as_float(src1 & mask));  // v 2^(S-149)
  constexpr float fm = __uint_as_float_c(q3h_floor_mult_bits(S));
  const u64 qe = ffma2_rm(cf, pack2(fm, fm), 0ull);                                     // q_e 2^-149
  constexpr float m11 = -11.0f * (float)(1 << S);
  const u64 qo = ffma2(qe, pack2(m11, m11), cf);                                        // q_o 2^(S-149)
  const u64 qe85 = fmul2(qe, pack2(18446744073709551616.0f, 18446744073709551616.0f)); // q_e 2^-85
  constexpr float so = 18446744073709551616.0f / (float)(1 << S);
  const u64 qo85 = fmul2(qo, pack2(so, so));                                            // q_o 2^-85
  const float2 we = unpack2(ffma2(qe85, step2, lo2)), wo = unpack2(ffma2(qo85, step2, lo2));
  out0 = h2_as_u32(__floats2half2_rn(we.x, wo.x));
  out1 = h2_as_u32(__floats2half2_rn(we.y, wo.y));
}

// o1, o2, o3: word offsets of this lane's code window inside a row (constant per lane;
// o3 is clamped into the row and its word masked by m3 when the window ends at word 7)
__device__ __forceinline__ void ms_dequant2(const uint32_t* w0, const uint32_t* w1, int o1, int o2, int o3,
                                            uint32_t m3, int sh, uint32_t (&a0)[8], uint32_t (&a1)[8]) {
  const uint32_t h0 = w0[0], h1 = w1[0];
  const float lo0 = __half2float(__ushort_as_half((unsigned short)(h0 & 0xFFFFu)));
  const float hi0 = __half2float(__ushort_as_half((unsigned short)(h0 >> 16)));
  const float lo1 = __half2float(__ushort_as_half((unsigned short)(h1 & 0xFFFFu)));
  const float hi1 = __half2float(__ushort_as_half((unsigned short)(h1 >> 16)));
  constexpr float k = 0.1f * 38685626227668133590597632.0f;  // (1/10) 2^85
  const u64 step2 = pack2((hi0 - lo0) * k, (hi1 - lo1) * k), lo2 = pack2(lo0, lo1);
  const uint32_t a1w = w0[o2], b1w = w1[o2];
  const uint32_t u0lo = __funnelshift_r(w0[o1], a1w, sh), u0hi = __funnelshift_r(a1w, w0[o3] & m3, sh);
  const uint32_t u1lo = __funnelshift_r(w1[o1], b1w, sh), u1hi = __funnelshift_r(b1w, w1[o3] & m3, sh);
  const uint32_t v0 = __funnelshift_r(u0lo, u0hi, 21), v1 = __funnelshift_r(u1lo, u1hi, 21);  // pairs 3, 4
  ms_pair<0>(u0lo, u1lo, step2, lo2, a0[0], a1[0]);
  ms_pair<7>(u0lo, u1lo, step2, lo2, a0[1], a1[1]);
  ms_pair<14>(u0lo, u1lo, step2, lo2, a0[2], a1[2]);
  ms_pair<0>(v0, v1, step2, lo2, a0[3], a1[3]);
  ms_pair<7>(v0, v1, step2, lo2, a0[4], a1[4]);
  ms_pair<3>(u0hi, u1hi, step2, lo2, a0[5], a1[5]);
  ms_pair<10>(u0hi, u1hi, step2, lo2, a0[6], a1[6]);
  ms_pair<17>(u0hi, u1hi, step2, lo2, a0[7], a1[7]);
}

template <int NT>  // token tiles of 8: bp = 8 NT tokens, x rows [0, bp) hi and [bp, 2 bp) lo
__global__ void __launch_bounds__(MS_THREADS, IFB_MS_MINB) qgemv_ms_kernel(const uint8_t* __restrict__ W, int N, int K,
                                                                 const __half* __restrict__ x2,
                                                                 const float* __restrict__ sc, int B,
                                                                 float* __restrict__ y, int kper, int atomic_out) {
  constexpr int BP = 8 * NT;
  extern __shared__ __align__(16) unsigned char smem[];
  const int nb = K >> 6;
  const int kb0 = blockIdx.y * kper, kb1 = min(nb, kb0 + kper);
  const int kc = (kb1 - kb0) * 64;
  const int pitch = kc + 4;  // halves; (kc/2 + 2) words = 2 (mod 32)
  __half* xs = reinterpret_cast<__half*>(smem);
  // per-warp ring of MS_DEPTH weight blocks: [warps][MS_DEPTH][16 rows][8 words]
  uint32_t* wst = reinterpret_cast<uint32_t*>(smem + (size_t)2 * BP * pitch * 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  // weights do not depend on the predecessor: the ring fills before the wait.
  // lane l copies 16 bytes of row l/2 (half l%2) of every block: 512 coalesced bytes
  const int rbase = blockIdx.x * MS_ROWS + warp * 16;
  const int64_t row_bytes = (int64_t)nb * 32;
  const int lrow = rbase + (lane >> 1);
  const uint8_t* wrow = W + (int64_t)min(lrow, N - 1) * row_bytes + (lane & 1) * 16;
  const uint32_t src_size = lrow < N ? 16u : 0u;  // rows past N read as zeros
  uint32_t* ring = wst + warp * MS_DEPTH * 128;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + lane * 16;
#pragma unroll
  for (int i = 0; i < MS_DEPTH; i++) {
    if (kb0 + i < kb1)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ring_s + i * 512),
                   "l"(wrow + (int64_t)(kb0 + i) * 32), "r"(src_size)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  pdl_wait();
  // x tile of this CTA's K-range: 2 BP rows of kc halves, 8-byte asynchronous copies (all
  // in flight at once; the pitch keeps rows 8-byte aligned)
  {
    const int cpr = kc / 4;  // 8-byte chunks per row
    const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(xs);
    for (int i = threadIdx.x; i < 2 * BP * cpr; i += MS_THREADS) {
      const int j = i / cpr, q = i - j * cpr;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(xs_s + (uint32_t)((j * pitch + q * 4) * 2)),
                   "l"(x2 + (int64_t)j * K + (int64_t)kb0 * 64 + q * 4)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  const int r0 = lane >> 2, c = lane & 3;
  float acc[2 * NT][4];
#pragma unroll
  for (int t = 0; t < 2 * NT; t++) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  // per-lane constants hoisted out of the block loop: the code window (this lane's 56
  // bits start at byte 4 + 7c of a block), the x row of every token tile
  const int byte = 4 + 7 * c, o1 = byte >> 2, o2 = o1 + 1, o3 = o1 + 2 < 8 ? o1 + 2 : 7;
  const uint32_t m3 = o1 + 2 < 8 ? 0xFFFFFFFFu : 0u;
  const int sh = (byte & 3) * 8;
  const uint32_t* xw = reinterpret_cast<const uint32_t*>(xs) + r0 * (pitch / 2) + 8 * c;
  const int tstride = 8 * (pitch / 2);  // words between token tiles
  int slot = 0;
  for (int kb = kb0; kb < kb1; kb++) {
    asm volatile("cp.async.wait_group %0;" ::"n"(MS_DEPTH - 1) : "memory");  // block kb (this lane's part)
    __syncwarp();                                                             // ... and every lane's
    const uint32_t* wb = ring + slot * 128;
    uint32_t a_lo[8], a_hi[8];
    ms_dequant2(wb + r0 * 8, wb + (r0 + 8) * 8, o1, o2, o3, m3, sh, a_lo, a_hi);
    __syncwarp();  // the slot is read: refill it with block kb + MS_DEPTH
    if (kb + MS_DEPTH < kb1)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ring_s + slot * 512),
                   "l"(wrow + (int64_t)(kb + MS_DEPTH) * 32), "r"(src_size)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    slot = slot + 1 == MS_DEPTH ? 0 : slot + 1;
#pragma unroll
    for (int g = 0; g < 4; g++) {
#pragma unroll
      for (int t = 0; t < 2 * NT; t++) {  // token tile t: x rows 8t + r0 (hi tiles, then lo tiles)
        const uint2 b = *reinterpret_cast<const uint2*>(xw + t * tstride + 2 * g);
        mma16816(acc[t], a_lo[2 * g], a_hi[2 * g], a_lo[2 * g + 1], a_hi[2 * g + 1], b.x, b.y);
      }
    }
    xw += 32;  // next block: 64 halves
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // epilogue: C fragment rows r0, r0+8; columns 2c, 2c+1 of each 8-token tile
#pragma unroll
  for (int t = 0; t < NT; t++) {
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int tok = 8 * t + 2 * c + (e & 1);
      const int row = rbase + r0 + (e >> 1) * 8;
      if (tok < B && row < N) {
        const float v = (acc[t][e] + acc[NT + t][e]) * sc[tok];
        float* dst = y + (int64_t)tok * N + row;
        if (atomic_out) atomicAdd(dst, v);
        else *dst = v;
      }
    }
  }
}

// y (+)= W' x for a Q3H_B64 weight and the fp16 hi/lo split x2 [2 bp, K] (+ per-token
// 2^-k in sc) that qgemv_tc_launch prepared.  IF_ERR_UNSUPPORTED for other shapes.
if_status qgemv_ms_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __half* x2, const float* sc,
                          int64_t B, float* y, int accumulate, cudaStream_t st) {
  if (s.type != IF_Q3H || s.block != 64 || B < 2 || B > 32 || K % 64 || N < 1 || N > (1 << 30) || K > (1 << 24) ||
      (reinterpret_cast<uintptr_t>(W) & 15u) || (reinterpret_cast<uintptr_t>(x2) & 15u))
    return IF_ERR_UNSUPPORTED;
  const int bp = tc_bpad((int)B), NT = bp / 8;
  const int nb = (int)(K / 64);
  const int nrt = (int)((N + MS_ROWS - 1) / MS_ROWS);
  // split K until the grid covers the SMs twice and the x tile fits two CTAs per SM
  int sms = 148;
  {
    static int cached = 0;
    if (!cached) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
      if (cached <= 0) cached = 148;
    }
    sms = cached;
  }
  const int wbytes = MS_WARPS * MS_DEPTH * 128 * 4;
  const int kmax = std::max(1, (MS_SMEM_MAX - wbytes) / (2 * bp * 2 * 64 + 16));  // blocks per CTA by smem
  int splits = std::max((nb + kmax - 1) / kmax, (2 * sms + nrt - 1) / nrt);
  splits = std::min(splits, nb);
  const int kper = (nb + splits - 1) / splits;
  splits = (nb + kper - 1) / kper;
  const int kc = kper * 64;
  const size_t smem = (size_t)2 * bp * (kc + 4) * 2 + wbytes;
  const int atomic_out = splits > 1 || accumulate;
  if (splits > 1 && !accumulate) {
    if (cudaMemsetAsync(y, 0, sizeof(float) * B * N, st) != cudaSuccess) return check_launch("qgemv_ms memset");
  }
  void (*kern)(const uint8_t*, int, int, const __half*, const float*, int, float*, int, int) =
      NT == 1 ? qgemv_ms_kernel<1> : NT == 2 ? qgemv_ms_kernel<2> : qgemv_ms_kernel<4>;
  static bool configured[3] = {false, false, false};
  const int ci = NT == 1 ? 0 : NT == 2 ? 1 : 2;
  if (!configured[ci]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, MS_SMEM_MAX + 8192);
    configured[ci] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nrt, (unsigned)splits);
  cfg.blockDim = dim3(MS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = splits > 1 && !accumulate ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kern, W, (int)N, (int)K, x2, sc, (int)B, y, kper, atomic_out);
  count_launch();
  return check_launch("qgemv_ms");
}

}  // namespace ifb
