// qgemm_tc.cu — fused-dequant GEMM/GEMV on the 5th-gen tensor cores (tcgen05 +
// TMEM + TMA), P:93-94:
//     Y[m, n] (+)= sum_k W'[n, k] X[m, k]        fp32 accumulate
// Two kernels:
//  * qgemm_tc_kernel -- a5 prefill: X bf16 [M, K] by TMA (SWIZZLE_128B tensor
//    map), W' -> bf16, two 128-row UMMA M tiles per CTA (256 TMEM columns),
//    128 weight rows (UMMA N) per CTA, K in steps of 64 (one Q3H_B64 block per
//    row).  Warps: 0 TMA producer, 1 TMEM allocator + single-thread
//    tcgen05.mma issuer (kind::f16), 2-5 (Q3H_B64: 2-9, two threads per row)
//    dequantizers -- each row's packed bytes prefetched 6 stages ahead with
//    cp.async into a padded ring (odd 16-byte chunk stride: conflict-free),
//    Eq. 2 -> bf16 straight into the UMMA canonical K-major SW128
//    layout, fence.proxy.async, mbarrier arrive -- then 2-5 run the TMEM
//    epilogue (tcgen05.ld 32x32b).
//  * qgemv_tc_kernel -- a4 batched decode (2 <= B <= 64): weights on the UMMA M
//    side (128 rows), x on N = 2 Bpad columns (fp16 hi + lo, Q23);
//    see the comment above the kernel.
// Split-K over gridDim.z by a small cost model (partials combined with red.add).
#include <cuda.h>

#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "pipe.cuh"
#include "qgemm.cuh"
#include "simd.cuh"

namespace ifb {

constexpr int TC_BN = 128;     // weight rows per CTA (UMMA N)
constexpr int TC_BM = 128;     // activation rows per UMMA tile (UMMA M)
constexpr int TC_BK = 64;      // K per stage
constexpr int TC_THREADS = 256;
// fast Q3H_B64 decode variant: 8 dequant warps (2 threads per weight row, half2
// arithmetic), converters on warps 0, 10, 11 -> 12 warps
template <int QT, int BS, bool DEC>
struct TcVar {
  // prefill Q3H_B64: 8 dequant warps (two threads per weight row, exact fp32 Eq. 2)
  static constexpr bool FAST = QT == 35 && BS == 64;
  static constexpr int THREADS = FAST ? 320 : 256;
  static constexpr int NDEQ = FAST ? 256 : 128;  // dequant threads (b_full arrivals)
};
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;  // 16 KB per M tile
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;  // 16 KB
constexpr int TC_PK = 8;   // packed-weight ring slots (stages of raw bytes per row)
constexpr int TC_PD = 6;   // cp.async prefetch distance (stages)

// raw bytes of one row per stage (64 weights), and the padded ring stride:
// a multiple of 16 with an odd 16-byte chunk count (conflict-free LDS.128)
__host__ __device__ constexpr int tc_sb(int qt, int bs) { return (TC_BK / bs) * q_block_bytes(qt, bs); }
__host__ __device__ constexpr int tc_sbpad(int qt, int bs) {
  return ((tc_sb(qt, bs) + 15) / 16) % 2 ? ((tc_sb(qt, bs) + 15) / 16) * 16 : ((tc_sb(qt, bs) + 15) / 16 + 1) * 16;
}
template <bool DEC, int SBPAD = 48>
struct TcCfg {
  static constexpr int MT = DEC ? 1 : 2;          // UMMA M tiles per CTA
  static constexpr int STAGES = (DEC && SBPAD <= 48) ? 4 : 3;  // (DEC: historical decode mode, unused)
  static constexpr int STAGE_BYTES = MT * TC_A_BYTES + TC_B_BYTES;
  static constexpr int TMEM_COLS = MT * TC_BN;
};
// decode: raw fp32 x ring, 48 KB of slots of Bpad tokens x 64 k (Bpad = B rounded
// up to 8/16/32/64): 24 slots at B <= 8 ... 3 at B = 64 (deep L2 prefetch)
constexpr int TC_XRING = 48 * 1024;
constexpr int TC_XRMAX = 16;
__host__ __device__ constexpr int tc_nxr(int B) {
  return TC_XRING / (tc_bpad(B) * TC_BK * 4) < TC_XRMAX ? TC_XRING / (tc_bpad(B) * TC_BK * 4) : TC_XRMAX;
}
// wide prefill tiles (Q3H_B64, M > 256): 512 activations per weight tile, two
// 128 x 256 TMEM accumulators (all 512 columns), two stages of 80 KB -- each W'
// tile is dequantized once per 512 tokens instead of once per 256
constexpr int TC_MTW = 4;
constexpr int TC_STAGES_W = 2;
// raw-weight ring of the wide variant: 8 slots when the rows are <= 48 bytes per
// stage, else 4 (prefetch distance 2) so that two 80 KB stages still fit
__host__ __device__ constexpr int tc_pk_wide(int qt, int bs) { return tc_sbpad(qt, bs) <= 48 ? TC_PK : 4; }
__host__ __device__ constexpr int tc_smem_wide(int qt, int bs) {
  return TC_STAGES_W * (TC_MTW * TC_A_BYTES + TC_B_BYTES) + tc_pk_wide(qt, bs) * TC_BN * tc_sbpad(qt, bs) + 1024 + 512;
}
// Prefill tile shapes (weight rows x tokens per CTA):
//   TC_BASE 128 x 256, TC_WIDE 128 x 512 (M > 256), TC_TALL 256 x 256.
// The in-CTA dequantization is the limiter (a knock-out run without it halves the
// mainloop), so the more tokens share one dequantized tile the better: WIDE beats
// BASE by 1.4-1.9x.  TALL halves the X bytes per flop (L2 -> SM traffic) but
// dequantizes twice as much per flop: measured 10-25% slower than WIDE (DESIGN.md
// §6), kept compiled-out (not dispatched).
enum { TC_BASE = 0, TC_WIDE = 1, TC_TALL = 2 };
template <int QT, int BS, int SHAPE>
struct TcShape {
  static constexpr bool FAST = QT == 35 && BS == 64;
  static constexpr int MT = SHAPE == TC_WIDE ? 4 : 2;     // 128-token X tiles
  static constexpr int RT = SHAPE == TC_TALL ? 2 : 1;     // 128-row weight tiles
  static constexpr int ROWS = RT * TC_BN;
  static constexpr int STAGES = SHAPE == TC_BASE ? TcCfg<false, tc_sbpad(QT, BS)>::STAGES : 2;
  static constexpr int STAGE_BYTES = MT * TC_A_BYTES + RT * TC_B_BYTES;
  static constexpr int UN = MT * TC_BM > 256 ? 256 : MT * TC_BM;  // UMMA N
  static constexpr int NJ = MT * TC_BM / UN;                        // accumulators per row tile
  static constexpr int TMEM_COLS = RT * MT * TC_BM;
  static constexpr int PK = SHAPE == TC_BASE ? TC_PK : SHAPE == TC_WIDE ? tc_pk_wide(QT, BS) : 4;
  static constexpr int PD = PK - 2;
  static constexpr int NDEQ = 2 * ROWS;  // dequant threads: two per weight row
  static constexpr int THREADS = 64 + (NDEQ > 192 ? NDEQ : 192);
  static constexpr int NEPI = (NDEQ / 32) > 16 ? 16 : (NDEQ / 32);  // epilogue warps (multiple of 4)
  static constexpr int SMEM = STAGES * STAGE_BYTES + PK * ROWS * tc_sbpad(QT, BS) + 1024 + 512;
};
template <bool DEC>
__host__ __device__ constexpr int tc_smem(int qt, int bs) {
  return (tc_sbpad(qt, bs) <= 48 ? TcCfg<DEC, 48>::STAGES : TcCfg<DEC, 64>::STAGES) * TcCfg<DEC>::STAGE_BYTES +
         TC_PK * TC_BN * tc_sbpad(qt, bs) + (DEC ? TC_XRING : 0) + 1024 /*align*/ + 512;
}

// ---- tcgen05 / TMA PTX wrappers ----------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major SWIZZLE_128B shared-memory matrix descriptor (rows of 128 B, 8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                     // leading byte offset (ignored for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // stride byte offset: next 8-row atom
  d |= (uint64_t)1 << 46;                     // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                     // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16 (or fp16), both K-major
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);  // .x = a (low half), .y = b
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <bool F16>
__device__ __forceinline__ uint32_t pack16x2(float a, float b) {
  if constexpr (F16) return pack_f16x2(a, b);
  else return pack_bf16x2(a, b);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// small unsigned integer (< 2^23) -> float on the full-rate pipes (2^23 magic; I2F
// runs at a fraction of the FMA rate)
__device__ __forceinline__ float u2f_exact(uint32_t q) { return __uint_as_float(q | 0x4B000000u) - 8388608.0f; }

// Prefetch the SB raw bytes of weight row n for K-stage ks (64 weights) into its
// ring row (zeros are produced later by dequant_row for rows/stages out of range).
template <int QT, int BS>
__device__ __forceinline__ void prefetch_row(const uint8_t* __restrict__ W, int64_t nb, int64_t n, int64_t N,
                                             int64_t ks, int64_t K, unsigned char* dst) {
  constexpr int SB = tc_sb(QT, BS);
  if (n >= N || ks * TC_BK >= K) return;
  const uint8_t* src = W + (n * nb + ks * (TC_BK / BS)) * q_block_bytes(QT, BS);
  if (SB % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
#pragma unroll
    for (int i = 0; i < SB / 16; i++) cp_async16(dst + 16 * i, src + 16 * i);
  } else {
#pragma unroll
    for (int i = 0; i < SB / 4; i++) cp_async4(dst + 4 * i, src + 4 * i);
  }
}
// the same copy shared by two threads: part g (0/1) issues every other unit
template <int QT, int BS>
__device__ __forceinline__ void prefetch_row_part(const uint8_t* __restrict__ W, int64_t nb, int64_t n, int64_t N,
                                                  int64_t ks, int64_t K, unsigned char* dst, int g) {
  constexpr int SB = tc_sb(QT, BS);
  if (n >= N || ks * TC_BK >= K) return;
  const uint8_t* src = W + (n * nb + ks * (TC_BK / BS)) * q_block_bytes(QT, BS);
  if (SB % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
#pragma unroll
    for (int i = 0; i < SB / 16; i++)
      if ((i & 1) == g) cp_async16(dst + 16 * i, src + 16 * i);
  } else {
#pragma unroll
    for (int i = 0; i < SB / 4; i++)
      if ((i & 1) == g) cp_async4(dst + 4 * i, src + 4 * i);
  }
}

// Dequantize weight row n, weights [k0, k0 + 64), from its raw bytes in the ring
// into 128 bytes of 16-bit values in the SW128 K-major layout at row r of the
// B tile (zeros beyond N or K).
// HALF = 0 / 1: only weights [32 HALF, 32 HALF + 32) of the stage (chunks 4 HALF ..
// 4 HALF + 3 of the row); -1: all 64.
template <int QT, int BS, bool F16, int HALF = -1>
__device__ __forceinline__ void dequant_row(const unsigned char* raw, int64_t n, int64_t N, int64_t k0, int64_t K,
                                           unsigned char* btile, int r) {
  constexpr int D = q_levels(QT);
  constexpr int C = q_width(QT);
  constexpr int NC = q_ncodes(QT, BS);
  constexpr int BB = q_block_bytes(QT, BS);
  constexpr int NW = q_block_words(QT, BS);
  constexpr int SB = tc_sb(QT, BS);
  constexpr int SBW = (SB + 15) / 16 * 4;  // words read (whole 16-byte chunks)
  uint32_t out[32];  // 64 16-bit values
  if (n < N && k0 < K) {
    uint32_t words[SBW + 1];
#pragma unroll
    for (int i = 0; i < SBW / 4; i++) {
      const uint4 v = *reinterpret_cast<const uint4*>(raw + 16 * i);
      words[4 * i] = v.x, words[4 * i + 1] = v.y, words[4 * i + 2] = v.z, words[4 * i + 3] = v.w;
    }
    words[SBW] = 0u;
    constexpr int SUB0 = (HALF >= 0 && BS == 32) ? HALF : 0;
    constexpr int SUB1 = (HALF >= 0 && BS == 32) ? HALF + 1 : TC_BK / BS;
#pragma unroll
    for (int sub = SUB0; sub < SUB1; sub++) {
      // block sub starts at byte sub * BB (a multiple of 2): word-aligned or a halfword in
      const int boff = sub * BB;
      if (k0 + sub * BS >= K) {
#pragma unroll
        for (int j = 0; j < BS / 2; j++) out[sub * (BS / 2) + j] = 0u;
        continue;
      }
      uint32_t w[NW + 1];
#pragma unroll
      for (int i = 0; i <= NW; i++) {
        const int wi = boff / 4 + i;
        const uint32_t a = wi < SBW ? words[wi] : 0u, b = wi + 1 <= SBW ? words[wi + 1] : 0u;
        w[i] = (boff & 3) ? __funnelshift_r(a, b, 16) : a;
      }
      if (BB % 4) w[NW] = 0u;
      // mask the bytes past the block (BB % 4 == 2: the last word's high half)
      if constexpr (BB % 4 != 0) w[NW - 1] &= 0xFFFFu;
      const float lo = half_bits_to_float(w[0] & 0xFFFFu);
      const float hi = half_bits_to_float(w[0] >> 16);
      const float step = __fdiv_rn(__fsub_rn(hi, lo), (float)D);
      constexpr int J0 = (HALF >= 0 && BS == 64) ? HALF * NC / 2 : 0;
      constexpr int J1 = (HALF >= 0 && BS == 64) ? (HALF + 1) * NC / 2 : NC;
#pragma unroll
      for (int j = J0; j < J1; j++) {
        const uint32_t v = get_code<C, NW>(w, j);
        if constexpr (QT == 35) {
          const uint32_t q1 = (v * 187u) >> 11;  // floor(v/11) for v < 128
          const uint32_t q2 = v - 11u * q1;      // v mod 11
          out[sub * (BS / 2) + j] = pack16x2<F16>(__fmaf_rn(u2f_exact(q1), step, lo), __fmaf_rn(u2f_exact(q2), step, lo));
        } else if (j & 1) {  // pairs of consecutive weights -> one packed word
          const float w0 = __fmaf_rn(u2f_exact(get_code<C, NW>(w, j - 1)), step, lo);
          out[sub * (BS / 2) + j / 2] = pack16x2<F16>(w0, __fmaf_rn(u2f_exact(v), step, lo));
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; j++) out[j] = 0u;
  }
  // 8 chunks of 16 B; chunk c of row r lives at chunk (c ^ (r % 8)) of the row (SW128)
  unsigned char* rowp = btile + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
  for (int c = (HALF >= 0 ? 4 * HALF : 0); c < (HALF >= 0 ? 4 * HALF + 4 : 8); c++) {
    uint4 v = make_uint4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]);
    *reinterpret_cast<uint4*>(rowp + ((c ^ (r & 7)) << 4)) = v;
  }
}

// Decode mode: the raw fp32 x of K-stage ks (token m's 64 values at xr + 256 m,
// landed by bulk copies) -> fp16 hi (rows 0..63) + lo (rows 64..127) of the A
// tile, SW128 K-major.  Rows of tokens >= B stay zero (zeroed once).  TC_CONV
// warps; item = (token, 8-element chunk).
constexpr int TC_CONV = 3;  // converter warps
template <bool PERM>
__device__ __forceinline__ void convert_x_tile(const float* xr, int B, unsigned char* atile, int cidx, int lo_off = 64,
                                               const float* xmul = nullptr) {
  const int lane = threadIdx.x & 31;
  for (int t = cidx * 32 + lane; t < B * 8; t += TC_CONV * 32) {
    const int m = t >> 3, c = t & 7;
    float4 va = *reinterpret_cast<const float4*>(xr + m * TC_BK + 8 * c);
    float4 vb = *reinterpret_cast<const float4*>(xr + m * TC_BK + 8 * c + 4);
    if (xmul) {  // per-token power-of-two split scale (exact)
      const float f = xmul[m];
      va = make_float4(va.x * f, va.y * f, va.z * f, va.w * f);
      vb = make_float4(vb.x * f, vb.y * f, vb.z * f, vb.w * f);
    }
    // PERM: the fast Q3H dequant's K order (x0, x4, x1, x5, x2, x6, x3, x7) of each chunk
    const float v[8] = {va.x, PERM ? vb.x : va.y, PERM ? va.y : va.z, PERM ? vb.y : va.w,
                        PERM ? va.z : vb.x, PERM ? vb.z : vb.y, PERM ? va.w : vb.z, vb.w};
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const __half2 hh = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
      const float2 hf = __half22float2(hh);
      const __half2 ll = __floats2half2_rn(v[2 * i] - hf.x, v[2 * i + 1] - hf.y);
      h[i] = *reinterpret_cast<const uint32_t*>(&hh);
      l[i] = *reinterpret_cast<const uint32_t*>(&ll);
    }
    const int mh = m, ml = lo_off + m;
    *reinterpret_cast<uint4*>(atile + (mh >> 3) * 1024 + (mh & 7) * 128 + ((c ^ (mh & 7)) << 4)) =
        make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(atile + (ml >> 3) * 1024 + (ml & 7) * 128 + ((c ^ (ml & 7)) << 4)) =
        make_uint4(l[0], l[1], l[2], l[3]);
  }
}

// one 2D TMA of the fp32 x tile [Bpad tokens x 64 k] of K-stage ks into a raw-x
// slot (out-of-range tokens / k are zero-filled by the tensor map)
__device__ __forceinline__ void issue_x_stage(const CUtensorMap* xmap, int64_t ks, float* xr, uint64_t* bar, int bpad) {
  mbar_arrive_expect_tx(bar, (uint32_t)(bpad * TC_BK * 4));
  tma_load_2d(xr, xmap, (int)(ks * TC_BK), 0, bar);
}

// ---- Q3H_B64 half-row dequant, exact Eq. 2 in fp32 (-> fp16 / bf16), no I2F -------
// Thread half h of a row decodes pairs [16h, 16h + 16) (chunks [4h, 4h + 4)) in
// natural K order.  Per pair: c as a float via the 2^23 magic, q_e = floor(c/11)
// by an FFMA rounding down onto the 2^23 grid, q_o = c - 11 q_e,
// w' = fma(q, step, lo): all full-rate FMA/ALU ops.
template <bool BF16>
__device__ __forceinline__ void dequant_q3h64_half_f32(const unsigned char* raw, bool valid, int h, unsigned char* tile,
                                                       int r) {
  uint32_t outw[16];
  if (valid) {
    const uint4 v0 = *reinterpret_cast<const uint4*>(raw);
    const uint4 v1 = *reinterpret_cast<const uint4*>(raw + 16);
    const uint32_t hdr = v0.x;
    const uint32_t ca[9] = {v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, 0u, 0u};
    uint32_t c[6];  // code-stream bits [112 h, 112 h + 160): compile-time positions for both halves
#pragma unroll
    for (int i = 0; i < 5; i++) c[i] = h ? __funnelshift_r(ca[3 + i], ca[4 + i], 16) : ca[i];
    c[5] = 0u;
    const float lo = half_bits_to_float(hdr & 0xFFFFu), hi = half_bits_to_float(hdr >> 16);
    const float step = __fdiv_rn(__fsub_rn(hi, lo), 10.0f);
    const float M23 = 8388608.0f, r11 = 0.0909090936183929443359375f;  // 2^23, roundup(1/11)
    // two pairs per f32x2 instruction (each lane the same IEEE operation as the scalar
    // form: identical bits, half the FMA-class issue slots)
    const u64 nM2 = pack2(-M23, -M23), M2 = pack2(M23, M23), r2 = pack2(r11, r11), m2 = pack2(-11.0f, -11.0f);
    const u64 st2 = pack2(step, step), lo2 = pack2(lo, lo);
#pragma unroll
    for (int jr = 0; jr < 16; jr += 2) {
      const int p0 = 7 * jr, p1 = p0 + 7;
      const uint32_t t0 = (p0 & 31) ? __funnelshift_r(c[p0 >> 5], c[(p0 >> 5) + 1], p0 & 31) : c[p0 >> 5];
      const uint32_t t1 = (p1 & 31) ? __funnelshift_r(c[p1 >> 5], c[(p1 >> 5) + 1], p1 & 31) : c[p1 >> 5];
      const u64 cf = fadd2(pack2(__uint_as_float((t0 & 0x7Fu) | 0x4B000000u), __uint_as_float((t1 & 0x7Fu) | 0x4B000000u)),
                           nM2);                                   // c, exact
      const u64 qe = fadd2(ffma2_rm(cf, r2, M2), nM2);             // floor(c / 11)
      const u64 qo = ffma2(qe, m2, cf);                            // c mod 11
      const float2 we = unpack2(ffma2(qe, st2, lo2)), wo = unpack2(ffma2(qo, st2, lo2));
      outw[jr] = pack16x2<!BF16>(we.x, wo.x);
      outw[jr + 1] = pack16x2<!BF16>(we.y, wo.y);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; i++) outw[i] = 0u;
  }
  unsigned char* rowp = tile + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
  for (int qq = 0; qq < 4; qq++) {
    const int cch = 4 * h + qq;
    *reinterpret_cast<uint4*>(rowp + ((cch ^ (r & 7)) << 4)) =
        make_uint4(outw[4 * qq], outw[4 * qq + 1], outw[4 * qq + 2], outw[4 * qq + 3]);
  }
}

#ifdef IFB_TC_PROF
// instrumentation build only: per CTA {smid, t_start, t_mainloop_end, t_epilogue_end} (%globaltimer ns)
__device__ unsigned long long g_tc_tl[8192][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
extern "C" void ifx_tc_tl(void* host) { cudaMemcpyFromSymbol(host, g_tc_tl, sizeof(g_tc_tl)); }
#endif
template <int QT, int BS, bool DEC, int SHAPE = TC_BASE>
__global__ void __launch_bounds__(TcShape<QT, BS, SHAPE>::THREADS, 1)
    qgemm_tc_kernel(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ xdec, const uint8_t* __restrict__ W,
                    int64_t N, int64_t K, int64_t M, float* __restrict__ Y, int ksteps_per_split, int atomic_out) {
  using Var = TcShape<QT, BS, SHAPE>;
  constexpr int MT = Var::MT, RT = Var::RT, ROWS = Var::ROWS, NJ = Var::NJ, UN = Var::UN;
  constexpr int STAGES = Var::STAGES, STAGE_BYTES = Var::STAGE_BYTES, TMEM_COLS = Var::TMEM_COLS;
  constexpr int PK = Var::PK;  // raw ring slots
  constexpr int PD = Var::PD;  // cp.async prefetch distance
  constexpr int SBPAD = tc_sbpad(QT, BS);
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* pring = smem + STAGES * STAGE_BYTES;  // [PK][ROWS][SBPAD] raw weight bytes
  uint64_t* a_full = reinterpret_cast<uint64_t*>(pring + PK * ROWS * SBPAD);
  uint64_t* b_full = a_full + STAGES;
  uint64_t* empty = b_full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef IFB_TC_PROF
  const int cta_id = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0 && cta_id < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_tc_tl[cta_id][0] = smid;
    g_tc_tl[cta_id][1] = gtimer();
  }
#endif
  // grid (m tiles, n tiles, splits): the CTAs sharing a weight tile are adjacent in
  // launch order, so the second read of the tile hits L2 instead of HBM
  const int64_t n0 = (int64_t)blockIdx.y * ROWS;
  const int64_t m0 = (int64_t)blockIdx.x * (TC_BM * MT);
  const int64_t nb = K / BS;
  const int ktotal = (int)((K + TC_BK - 1) / TC_BK);
  const int ks0 = blockIdx.z * ksteps_per_split;
  const int ks1 = min(ktotal, ks0 + ksteps_per_split);
  const int nks = max(ks1 - ks0, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&a_full[s], 1);
      mbar_init(&b_full[s], Var::NDEQ / 32);  // one arrival per dequant warp
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: X tiles ----------------
      asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
      for (int i = 0; i < nks; i++) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&a_full[s], MT * TC_A_BYTES);
        unsigned char* st = smem + s * STAGE_BYTES;
        for (int mt = 0; mt < MT; mt++)
          tma_load_2d(st + mt * TC_A_BYTES, &xmap, (ks0 + i) * TC_BK, (int)(m0 + mt * TC_BM), &a_full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      // UMMA 128 x UN x 16: A = a dequantized 128-row weight tile (rows = TMEM lanes),
      // B = UN tokens of the MT X tiles (contiguous in smem: one K-major SW128 operand)
      // -> D[weight row][token]; accumulator (rt, j) at TMEM columns (rt NJ + j) UN.
      constexpr uint32_t idesc = umma_idesc_bf16(TC_BN, UN);
      for (int i = 0; i < nks; i++) {
        const int s = i % STAGES;
        const uint32_t par = (i / STAGES) & 1;
        mbar_wait(&a_full[s], par);
        mbar_wait(&b_full[s], par);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
        const uint64_t adesc0 = umma_desc_sw128(st + MT * TC_A_BYTES);
        const uint64_t bdesc0 = umma_desc_sw128(st);
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; kk++) {
          // advance 16 elements = 32 bytes along K inside the 128-byte swizzle row
#pragma unroll
          for (int rt = 0; rt < RT; rt++)
#pragma unroll
            for (int j = 0; j < NJ; j++)
              umma_bf16(tmem + (rt * NJ + j) * UN, adesc0 + (uint64_t)((rt * TC_B_BYTES) >> 4) + (uint64_t)(kk * 2),
                        bdesc0 + (uint64_t)((j * UN * 128) >> 4) + (uint64_t)(kk * 2), idesc, (i > 0) || (kk > 0));
        }
        umma_commit(&empty[s]);  // frees the stage once these MMAs completed
      }
      umma_commit(acc_full);
    }
  } else if (Var::FAST && warp < 2 + Var::NDEQ / 32) {
    // ---------------- Q3H_B64 dequantizers: two threads per row (warps 2-9 / 2-17) ----------------
    const int r = (warp - 2) * 16 + (lane >> 1), h = lane & 1;
    const int64_t n = n0 + r;
    unsigned char* myrow = pring + r * SBPAD;  // half h copies bytes [16h, 16h + 16) of the block
    auto pre = [&](int i) {
      const int64_t ks = ks0 + i;
      if (n < N && ks * TC_BK < K) cp_async16(myrow + (i % PK) * ROWS * SBPAD + 16 * h, W + (n * nb + ks) * 32 + 16 * h);
    };
#pragma unroll
    for (int i = 0; i < PD; i++) {
      if (i < nks) pre(i);
      cp_async_commit();
    }
    for (int i = 0; i < nks; i++) {
      const int s = i % STAGES;
      if (i + PD < nks) pre(i + PD);
      cp_async_commit();
      cp_async_wait<PD>();
      __syncwarp();  // the partner lane's half of the block is visible
      mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
#ifndef IFB_TC_KO_DEQ  // knock-out experiment only: W' tiles left stale
      dequant_q3h64_half_f32<true>(myrow + (i % PK) * ROWS * SBPAD, n < N && (int64_t)(ks0 + i) * TC_BK < K, h,
                                   smem + s * STAGE_BYTES + MT * TC_A_BYTES, r);
#endif
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      __syncwarp();  // the warp's W' rows (each lane fenced its own stores) ...
      if (lane == 0) mbar_arrive(&b_full[s]);  // ... one arrival per warp
      __syncwarp();  // both halves read before the ring slot is refilled
    }
    cp_async_wait<0>();
  } else if (!Var::FAST && warp < 2 + Var::NDEQ / 32) {
    // ---------------- dequantizers: two threads per weight row ----------------
    // warps 2..(2 + ROWS/32) take weights [0, 32) of the stage, the next ROWS/32 warps
    // [32, 64) of the same rows (warp-uniform halves: no divergence).  The pair shares
    // the row's ring slot, each copying every other unit; a 64-thread named barrier
    // per stage makes both halves of the copy visible to both warps.
    constexpr int RW = ROWS / 32;                  // warps per half
    const int g = (warp - 2) / RW;                 // half
    const int r = ((warp - 2) % RW) * 32 + lane;  // row
    const int bar_id = 1 + (warp - 2) % RW;       // named barrier of the warp pair
    const int64_t n = n0 + r;
    unsigned char* myring = pring + r * SBPAD;
#pragma unroll
    for (int i = 0; i < PD; i++) {
      if (i < nks) prefetch_row_part<QT, BS>(W, nb, n, N, ks0 + i, K, myring + (i % PK) * ROWS * SBPAD, g);
      cp_async_commit();
    }
    for (int i = 0; i < nks; i++) {
      const int s = i % STAGES;
      // slot (i + PD) % PK was last read at stage i + PD - PK <= i - 2: both warps have
      // passed stage i - 1's barrier since
      if (i + PD < nks)
        prefetch_row_part<QT, BS>(W, nb, n, N, ks0 + i + PD, K, myring + ((i + PD) % PK) * ROWS * SBPAD, g);
      cp_async_commit();
      cp_async_wait<PD>();
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // the partner's copies landed too
      mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
      unsigned char* btile = smem + s * STAGE_BYTES + MT * TC_A_BYTES;
      const unsigned char* raw = myring + (i % PK) * ROWS * SBPAD;
      const int64_t k0 = (int64_t)(ks0 + i) * TC_BK;
      if (g == 0)
        dequant_row<QT, BS, DEC, 0>(raw, n, N, k0, K, btile, r);
      else
        dequant_row<QT, BS, DEC, 1>(raw, n, N, k0, K, btile, r);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      __syncwarp();  // the warp's W' rows (each lane fenced its own stores) ...
      if (lane == 0) mbar_arrive(&b_full[s]);  // ... one arrival per warp
    }
    cp_async_wait<0>();
  }

  // ---------------- epilogue: TMEM -> registers -> global ----------------
  // TMEM lane = weight row, column = token.  Warp w may read lane quarter w % 4;
  // the NEPI / 4 warps of a quarter split its 32-column chunks.
  constexpr int NEPI = Var::NEPI;
  if (warp >= 2 && warp < 2 + NEPI) {
    mbar_wait(acc_full, 0);
    tc_fence_after();
#ifdef IFB_TC_PROF
    if (threadIdx.x == 64 && cta_id < 8192) g_tc_tl[cta_id][2] = gtimer();
#endif
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    constexpr int NCH = (TMEM_COLS / 32) / (NEPI / 4);  // 32-column chunks per warp
    float* sc = reinterpret_cast<float*>(smem) + (warp - 2) * 32 * 36;
#pragma unroll 1
    for (int c = 0; c < NCH; c++) {
      const int cc = half * NCH + c;
      uint32_t rr[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + cc * 32, rr);
      const int acc = (cc * 32) / UN, rt = acc / NJ;  // accumulator (rt, j)
      const int64_t mbase = m0 + (acc % NJ) * UN + (cc * 32) % UN;
      const int64_t nq = n0 + rt * TC_BN + q * 32;
      const bool vec = (N % 4 == 0) && nq + 32 <= N && !(reinterpret_cast<uintptr_t>(Y) & 15u);
      if (nks > 0 && nq < N && mbase < M) {
#pragma unroll
        for (int j = 0; j < 32; j++) sc[j * 36 + lane] = __uint_as_float(rr[j]);
        __syncwarp();
        const int nl = (lane & 7) * 4;
#pragma unroll
        for (int it = 0; it < 8; it++) {
          const int ml = it * 4 + (lane >> 3);
          const int64_t m = mbase + ml;
          if (m < M) {
            const float4 v = *reinterpret_cast<const float4*>(sc + ml * 36 + nl);
            float* yp = Y + m * N + nq + nl;
            if (vec) {
              if (atomic_out)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(yp), "f"(v.x), "f"(v.y), "f"(v.z),
                             "f"(v.w)
                             : "memory");
              else
                *reinterpret_cast<float4*>(yp) = v;
            } else {
              const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int e = 0; e < 4; e++)
                if (nq + nl + e < N) {
                  if (atomic_out)
                    atomicAdd(yp + e, vv[e]);
                  else
                    yp[e] = vv[e];
                }
            }
          }
        }
        __syncwarp();
      }
    }
    tc_fence_before();
  }
  __syncthreads();
#ifdef IFB_TC_PROF
  if (threadIdx.x == 0 && cta_id < 8192) g_tc_tl[cta_id][3] = gtimer();
#endif
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// x fp32 [B, K] -> X2 fp16 [2 bp, K]: rows [0, bp) = hi(x), rows [bp, 2 bp) = lo(x) =
// x - hi (zero rows for tokens >= B).  Run once per qGEMV when the caller provides
// scratch; the decode kernel then loads its x tiles with one SWIZZLE_128B TMA per stage
// instead of converting per CTA (every CTA would otherwise redo it).
// One CTA per token row t: max |x_t| -> per-token scale 2^k (common.cuh xsplit_k), the
// split of x_t * 2^k, and sc[t] = 2^-k for the epilogue.
__global__ void __launch_bounds__(256) x_split_kernel(const float* __restrict__ x, int B, int64_t K, int bp,
                                                      __half* __restrict__ x2, float* __restrict__ sc) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8];
  const int t = blockIdx.x;
  const float* xr = x + (int64_t)t * K;
  float m = 0.f;
  if (t < B)
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) m = fmaxf(m, fabsf(xr[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) m = fmaxf(m, red[w]);
  const int ks = xsplit_k(m);
  const float mul = pow2f(ks);
  if (threadIdx.x == 0) sc[t] = pow2f(-ks);
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const float v = t < B ? xr[k] * mul : 0.f;
    const __half h = __float2half_rn(v);
    x2[(int64_t)t * K + k] = h;
    x2[((int64_t)bp + t) * K + k] = __float2half_rn(v - __half2float(h));
  }
}

// ---------------------------------------------------------------------------
// a4 batched decode, weights on the UMMA M side: D[n, j] = sum_k W'[n, k] X[j, k]
// with M = 128 weight rows and N = 2 Bp columns (x hi of token t in column t,
// x lo in column Bp + t, Bp = B rounded up to 8/16/32/64; N >= 16).  The x tile
// is tiny (N rows), so the pipeline holds up to 8 stages; each epilogue thread
// owns one weight row and adds its hi and lo columns (no exchange), and the y
// stores are coalesced along n.
constexpr int TCD_MAXST = 4;  // measured: 8 stages are no faster (the stage loop is not depth-bound)
constexpr int TCD_WR = 16;  // weight-tile ring slots (Q3H_B64 decode), 4 KB each
constexpr int TCD_XRING = 32 * 1024;
__host__ __device__ constexpr int tcd_ncols(int B) { return 2 * tc_bpad(B) < 16 ? 16 : 2 * tc_bpad(B); }
__host__ __device__ constexpr int tcd_stage_bytes(int B) { return TC_B_BYTES + tcd_ncols(B) * 128; }
__host__ __device__ constexpr int tcd_nxr(int B) {
  return TCD_XRING / (tc_bpad(B) * TC_BK * 4) < TC_XRMAX ? TCD_XRING / (tc_bpad(B) * TC_BK * 4) : TC_XRMAX;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// epilogue of the decode kernel (warps 2-5): lane = weight row, y[t, n] = D[n, t] + D[n, bp + t]
__device__ __forceinline__ void qgemv_epilogue(uint32_t tmem, uint64_t* acc_full, float* __restrict__ Y, int64_t N,
                                               int B, int bp, int64_t n0, int nks, int atomic_out, int warp, int lane,
                                               const float* sc) {
  mbar_wait(acc_full, 0);
  tc_fence_after();
  const int q = warp & 3;  // TMEM lane quarter
  const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
  const int64_t nn = n0 + q * 32 + lane;
  for (int t0 = 0; t0 < B; t0 += 16) {
    uint32_t hv[16], lv[16];
    tmem_ld16(tbase + t0, hv);
    tmem_ld16(tbase + bp + t0, lv);  // bp = 8: columns 8..23 (16..23 unused, allocated)
    if (nn < N && nks > 0) {
#pragma unroll
      for (int j = 0; j < 16; j++) {
        if (t0 + j < B) {
          const float v = (__uint_as_float(hv[j]) + __uint_as_float(lv[j])) * sc[t0 + j];  // undo 2^k
          float* dst = Y + (int64_t)(t0 + j) * N + nn;
          if (atomic_out) atomicAdd(dst, v);
          else *dst = v;
        }
      }
    }
  }
  tc_fence_before();
}

#ifdef IFB_TCD_PROF
// instrumentation build only: per CTA clock64 sums {MMA: wait x, wait W', issue, total;
// dequant warp 2 lane 0: wait weight slot, wait free stage, dequant, total}
__device__ unsigned long long g_tcd_prof[4096][8];
extern "C" void ifx_tcd_prof(void* host) { cudaMemcpyFromSymbol(host, g_tcd_prof, sizeof(g_tcd_prof)); }
#endif
// the 8-warp Q3H_B64 dequant loop: warp w in 2..9 owns rows [16 (w - 2), +16), lane
// pair (2i, 2i + 1) = the two halves of row 16 (w - 2) + i; the weight tile of stage
// i ([128 rows x 32 B], TMA) is in ring slot i % TCD_WR
__device__ __forceinline__ void qgemv_fast_deq(int64_t N, int64_t K, int64_t n0, int ks0, int nks, int stages,
                                               int stage_bytes, unsigned char* smem, unsigned char* wring,
                                               uint64_t* wfull, uint64_t* wempty, uint64_t* empty, uint64_t* b_full,
                                               int warp, int lane) {
  const int r = (warp - 2) * 16 + (lane >> 1), h = lane & 1;
  const int64_t n = n0 + r;
  int s = 0;
  uint32_t sph = 0;  // stage slot and its phase (incremental: stages need not be a power of two)
#ifdef IFB_TCD_PROF
  unsigned long long p0 = 0, p1 = 0, p2 = 0, tstart = clock64();
#endif
  for (int i = 0; i < nks; i++, s = (s + 1 == stages) ? (sph ^= 1, 0) : s + 1) {
    const int ws = i & (TCD_WR - 1);
#ifdef IFB_TCD_PROF
    unsigned long long ta = clock64();
#endif
    mbar_wait(&wfull[ws], (i / TCD_WR) & 1);
#ifdef IFB_TCD_PROF
    unsigned long long tb = clock64();
#endif
    mbar_wait(&empty[s], sph ^ 1);
#ifdef IFB_TCD_PROF
    unsigned long long tc = clock64();
#endif
#ifndef IFB_TCD_NODEQ
    dequant_q3h64_half_f32<false>(wring + ws * 4096 + r * 32, n < N && (int64_t)(ks0 + i) * TC_BK < K, h,
                                  smem + s * stage_bytes, r);
#endif
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
    __syncwarp();  // the warp's W' rows (each lane fenced its own stores) ...
    if (lane == 0) mbar_arrive(&b_full[s]);  // ... one arrival per warp
#ifdef IFB_TCD_PROF
    unsigned long long td = clock64();
    p0 += tb - ta, p1 += tc - tb, p2 += td - tc;
    if (warp == 2 && lane == 0 && i == nks - 1 && blockIdx.x < 4096) {
      g_tcd_prof[blockIdx.x][4] = p0, g_tcd_prof[blockIdx.x][5] = p1, g_tcd_prof[blockIdx.x][6] = p2;
      g_tcd_prof[blockIdx.x][7] = td - tstart;
    }
#endif
    __syncwarp();  // both halves of every row of this warp read the ring slot
    if (lane == 0) mbar_arrive(&wempty[ws]);
  }
}

template <int QT, int BS>
struct TcdVar {
  // Q3H_B64: weight tiles [128 rows x 32 B] by 2D TMA (warp 12) into a 16-slot
  // ring, 8 dequant warps (two threads per row)
  static constexpr bool FAST = QT == 35 && BS == 64;
  static constexpr int THREADS = FAST ? 416 : 256;
  static constexpr int NDEQ = FAST ? 256 : 128;
  static constexpr int CONV1 = FAST ? 10 : 6;  // first converter warp after warp 0 (FAST: 10, 11)
};

template <int QT, int BS>
__global__ void __launch_bounds__(TcdVar<QT, BS>::THREADS, 1)
    qgemv_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                    const uint8_t* __restrict__ W, int64_t N, int64_t K, int B, float* __restrict__ Y,
                    int ksteps_per_split, int atomic_out, int stages, int xpre, const float* __restrict__ xg,
                    const float* __restrict__ xsc_g) {
  constexpr int SBPAD = tc_sbpad(QT, BS);
  using V = TcdVar<QT, BS>;
  pdl_trigger();
  const int bp = tc_bpad(B), ncols = tcd_ncols(B), stage_bytes = tcd_stage_bytes(B);
  const int nxr = tcd_nxr(B), xslot = bp * TC_BK;
  const int lxr = 31 - __clz(nxr);  // nxr is a power of two
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: W' tile (A, 128 rows) at smem + s * stage_bytes, x tile (B, ncols rows) right after
  unsigned char* pring = smem + stages * stage_bytes;  // [TC_PK][128][SBPAD] (cp.async) or [TCD_WR][128][32] (FAST, TMA)
  float* xraw = reinterpret_cast<float*>(pring + (V::FAST ? TCD_WR * 4096 : TC_PK * TC_BN * SBPAD));  // [nxr][bp][64]
  uint64_t* a_full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(xraw) + TCD_XRING);  // x ready
  uint64_t* b_full = a_full + TCD_MAXST;  // W' ready
  uint64_t* empty = b_full + TCD_MAXST;
  uint64_t* acc_full = empty + TCD_MAXST;
  uint64_t* xr_full = acc_full + 1;
  uint64_t* wfull = xr_full + TC_XRMAX;  // [TCD_WR] (FAST)
  uint64_t* wempty = wfull + TCD_WR;     // [TCD_WR]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + TCD_WR);
  // per-token split scales (converter path): max |x| bits, 2^k, 2^-k
  uint32_t* xmax_u = tmem_slot + 4;
  float* xmul_s = reinterpret_cast<float*>(xmax_u + 64);
  float* xinv_s = xmul_s + 64;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n0 = (int64_t)blockIdx.x * TC_BN;
  const int64_t nb = K / BS;
  const int ktotal = (int)((K + TC_BK - 1) / TC_BK);
  const int ks0 = blockIdx.z * ksteps_per_split;
  const int nks = max(min(ktotal, ks0 + ksteps_per_split) - ks0, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&a_full[s], xpre ? 1 : TC_CONV);
      mbar_init(&b_full[s], V::NDEQ / 32);  // one arrival per dequant warp
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    for (int i = 0; i < TC_XRMAX; i++) mbar_init(&xr_full[i], 1);
    for (int i = 0; i < TCD_WR; i++) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 8);  // the 8 dequant warps
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) xmax_u[i] = 0u;
  // x tiles: rows of tokens >= B (hi and lo) are never written -> zero them once
  for (int s = 0; s < stages; s++)
    for (int i = threadIdx.x; i < ncols * 8; i += blockDim.x)
      reinterpret_cast<uint4*>(smem + s * stage_bytes + TC_B_BYTES)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the predecessor (PDL) wrote x / y: every role but the weight stream waits for it
  if (!(V::FAST && warp == 12)) pdl_wait();

  if (V::FAST && warp == 12) {
    // ---------------- weight tiles: one 2D TMA per stage, 16 slots ahead ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
      for (int i = 0; i < nks; i++) {
        const int ws = i & (TCD_WR - 1);
        mbar_wait(&wempty[ws], ((i / TCD_WR) & 1) ^ 1);
        mbar_arrive_expect_tx(&wfull[ws], 4096u);
        tma_load_2d(pring + ws * 4096, &wmap, (ks0 + i) * 32, (int)n0, &wfull[ws]);
      }
    }
  } else if (xpre && warp == 0) {
    // ---------------- x tiles pre-split by x_split_kernel: one SWIZZLE_128B TMA per stage ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
      for (int i = 0; i < nks; i++) {
        const int s = i % stages;
        mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&a_full[s], (uint32_t)(ncols * 128));
        tma_load_2d(smem + s * stage_bytes + TC_B_BYTES, &xmap, (ks0 + i) * TC_BK, 0, &a_full[s]);
      }
    }
  } else if (!xpre && (warp == 0 || (warp >= V::CONV1 && warp < V::CONV1 + 2))) {
    // ---------------- converters: raw fp32 x (2D TMA ring) -> fp16 hi/lo x tiles ----------------
    const int cidx = warp == 0 ? 0 : warp - V::CONV1 + 1;
    const bool issuer = warp == 0 && lane == 0;
    {
      // per-token max |x| over this CTA's k range -> power-of-two split scale; the
      // epilogue of this CTA undoes it before its (split-K) partial is added
      const int cthr = cidx * 32 + lane;
      const int64_t k0 = (int64_t)ks0 * TC_BK;
      const int64_t k1 = min(K, (int64_t)(ks0 + nks) * TC_BK);
      const int n4 = k1 > k0 ? (int)((k1 - k0) >> 2) : 0;  // K % 8 == 0
      float m = 0.f;
      int tc = -1;
      for (int j = cthr; j < B * n4; j += TC_CONV * 32) {
        const int t = j / n4;
        if (t != tc) {
          if (tc >= 0) atomicMax(&xmax_u[tc], __float_as_uint(m));
          tc = t;
          m = 0.f;
        }
        const float4 v = reinterpret_cast<const float4*>(xg + (int64_t)t * K + k0)[j - t * n4];
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
      if (tc >= 0) atomicMax(&xmax_u[tc], __float_as_uint(m));
      named_bar_sync(3, TC_CONV * 32);
      for (int t = cthr; t < 64; t += TC_CONV * 32) {
        const int kx = xsplit_k(__uint_as_float(xmax_u[t]));
        xmul_s[t] = pow2f(kx);
        xinv_s[t] = pow2f(-kx);
      }
      named_bar_sync(3, TC_CONV * 32);
      asm volatile("bar.arrive 5, %0;" ::"n"((TC_CONV + 4) * 32) : "memory");  // scales ready for the epilogue
    }
    if (issuer)
      for (int i = 0; i < nxr && i < nks; i++) issue_x_stage(&xmap, ks0 + i, xraw + i * xslot, &xr_full[i], bp);
    for (int i = 0; i < nks; i++) {
      const int s = i % stages, xs = (i & (nxr - 1));
      mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
      mbar_wait(&xr_full[xs], (i >> lxr) & 1);
#ifndef IFB_TCD_NOCONV
      convert_x_tile<false>(xraw + xs * xslot, B, smem + s * stage_bytes + TC_B_BYTES, cidx, bp, xmul_s);
#endif
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[s]);
      named_bar_sync(3, TC_CONV * 32);  // every converter is done with this raw-x slot
      if (issuer && i + nxr < nks) issue_x_stage(&xmap, ks0 + i + nxr, xraw + xs * xslot, &xr_full[xs], bp);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread): A = W' (M = 128), B = x (N = ncols) ----------------
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_f16(TC_BN, ncols);
#ifdef IFB_TCD_PROF
      unsigned long long q0 = 0, q1 = 0, q2 = 0, tstart = clock64(), tprev = 0;
#endif
      for (int i = 0; i < nks; i++) {
        const int s = i % stages;
        const uint32_t par = (i / stages) & 1;
#ifdef IFB_TCD_PROF
        unsigned long long ta = clock64();
        if (i > 0) q2 += ta - tprev;
#endif
        mbar_wait(&a_full[s], par);
#ifdef IFB_TCD_PROF
        unsigned long long tb = clock64();
        q0 += tb - ta;
#endif
        mbar_wait(&b_full[s], par);
#ifdef IFB_TCD_PROF
        unsigned long long tc = clock64();
        q1 += tc - tb;
        tprev = tc;
        if (i == nks - 1 && blockIdx.x < 4096) {
          g_tcd_prof[blockIdx.x][0] = q0, g_tcd_prof[blockIdx.x][1] = q1, g_tcd_prof[blockIdx.x][2] = q2;
          g_tcd_prof[blockIdx.x][3] = tc - tstart;
        }
#endif
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * stage_bytes);
        const uint64_t adesc0 = umma_desc_sw128(st), bdesc0 = umma_desc_sw128(st + TC_B_BYTES);
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; kk++)
#ifndef IFB_TCD_NOMMA
          umma_bf16(tmem, adesc0 + (uint64_t)(kk * 2), bdesc0 + (uint64_t)(kk * 2), idesc, (i > 0) || (kk > 0));
#endif
        umma_commit(&empty[s]);
      }
      umma_commit(acc_full);
    }
  } else if (V::FAST && warp >= 6 && warp < 10) {
    // ---------------- Q3H_B64 dequantizers, second half of the 8 warps ----------------
    // (warps 2-9: 16 rows each, lane pairs = the two halves of a row; warps 2-5
    //  run the epilogue below after the same loop)
    qgemv_fast_deq(N, K, n0, ks0, nks, stages, stage_bytes, smem, pring, wfull, wempty, empty, b_full, warp, lane);
  } else if (V::FAST && warp >= 2 && warp < 6) {
    qgemv_fast_deq(N, K, n0, ks0, nks, stages, stage_bytes, smem, pring, wfull, wempty, empty, b_full, warp, lane);
    if (!xpre) named_bar_sync(5, (TC_CONV + 4) * 32);  // the converters' per-CTA scales are in smem
    qgemv_epilogue(tmem, acc_full, Y, N, B, bp, n0, nks, atomic_out, warp, lane, xpre ? xsc_g : xinv_s);
  } else if (!V::FAST && warp >= 2 && warp < 6) {
    // ---------------- dequantizers: one weight row per thread (Eq. 2 in fp32, -> fp16) ----------------
    const int r = threadIdx.x - 64;  // 0..127
    const int64_t n = n0 + r;
    unsigned char* myring = pring + r * SBPAD;
#pragma unroll
    for (int i = 0; i < TC_PD; i++) {
      if (i < nks) prefetch_row<QT, BS>(W, nb, n, N, ks0 + i, K, myring + (i % TC_PK) * TC_BN * SBPAD);
      cp_async_commit();
    }
    for (int i = 0; i < nks; i++) {
      const int s = i % stages;
      if (i + TC_PD < nks) prefetch_row<QT, BS>(W, nb, n, N, ks0 + i + TC_PD, K, myring + ((i + TC_PD) % TC_PK) * TC_BN * SBPAD);
      cp_async_commit();
      cp_async_wait<TC_PD>();
      mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
      dequant_row<QT, BS, true>(myring + (i % TC_PK) * TC_BN * SBPAD, n, N, (int64_t)(ks0 + i) * TC_BK, K,
                                smem + s * stage_bytes, r);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      __syncwarp();  // the warp's W' rows (each lane fenced its own stores) ...
      if (lane == 0) mbar_arrive(&b_full[s]);  // ... one arrival per warp
    }
    cp_async_wait<0>();
    if (!xpre) named_bar_sync(5, (TC_CONV + 4) * 32);  // the converters' per-CTA scales are in smem
    qgemv_epilogue(tmem, acc_full, Y, N, B, bp, n0, nks, atomic_out, warp, lane, xpre ? xsc_g : xinv_s);
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128) : "memory");
  }
}

// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool get_encoder() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

static int tc_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// split K to minimise  waves * (F + k-steps per split): whole waves of SMs against
// the fixed per-CTA cost (prologue, pipeline fill, atomic epilogue ~ F k-steps,
// measured); partials combined with red.add
static int tc_splits(int tiles, int ktotal) {
  const int sms = tc_sms();
  constexpr int F = 12;
  int best = 1;
  long bcost = -1;
  for (int sp = 1; sp <= 8; sp++) {
    if (sp > 1 && ktotal / sp < 4) break;
    const long waves = (tiles * sp + sms - 1) / sms;
    const long cost = waves * (F + (ktotal + sp - 1) / sp);
    if (bcost < 0 || cost < bcost) {
      bcost = cost;
      best = sp;
    }
  }
  return best;
}

template <bool DEC>
static if_status tc_run(if_scheme s, const CUtensorMap& map, const float* xdec, const uint8_t* W, int64_t N, int64_t K,
                        int64_t M, float* Y, int accumulate, cudaStream_t st) {
  // the cp.async weight prefetch needs 4-byte aligned rows (Q3H_B32 with an odd
  // number of blocks per row is 2-byte aligned: SIMT path)
  const int64_t row_bytes = K / s.block * q_block_bytes(s.type, s.block);
  if ((row_bytes & 3) || (reinterpret_cast<uintptr_t>(W) & 3u)) return IF_ERR_UNSUPPORTED;
  const int ktotal = (int)((K + TC_BK - 1) / TC_BK);
  return dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    auto go = [&]<int SHAPE>() -> if_status {
      using V = TcShape<QT, BS, SHAPE>;
      const int ntile = (int)((N + V::ROWS - 1) / V::ROWS);
      const int mtile = (int)((M + TC_BM * V::MT - 1) / (TC_BM * V::MT));
      const int splits = tc_splits(ntile * mtile, ktotal);
      const int kper = (ktotal + splits - 1) / splits;
      const int atomic_out = (splits > 1) || accumulate;
      if (splits > 1 && !accumulate) {
        if (cudaMemsetAsync(Y, 0, sizeof(float) * M * N, st) != cudaSuccess) return check_launch("qgemm_tc memset");
      }
      auto kern = qgemm_tc_kernel<QT, BS, DEC, SHAPE>;
      constexpr int smem = V::SMEM;
      static_assert(smem <= 227 * 1024, "shared memory");
      static bool configured = false;
      if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        configured = true;
      }
      dim3 grid(mtile, ntile, splits);
      kern<<<grid, V::THREADS, smem, st>>>(map, xdec, W, N, K, M, Y, kper, atomic_out);
      count_launch();
      return IF_OK;
    };
    // M > 256: 512-token tiles (each weight dequantized once per 512 tokens)
    if_status r = M > 256 ? go.template operator()<TC_WIDE>() : go.template operator()<TC_BASE>();
    if (r != IF_OK) return r;
    return check_launch(DEC ? "qgemv_tc" : "qgemm_tc");
  });
}

if_status qgemm_tc_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __nv_bfloat16* X, int64_t M,
                          float* Y, int accumulate, cudaStream_t st) {
  // TMA needs the X row pitch (K * 2 bytes) to be a multiple of 16 and a 16-byte aligned base
  if (K % 8 != 0 || (reinterpret_cast<uintptr_t>(X) & 15u) || M > (int64_t)1 << 30 || N > (int64_t)1 << 30)
    return IF_ERR_UNSUPPORTED;
  if (!get_encoder()) return IF_ERR_UNSUPPORTED;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)TC_BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(X), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(IF_ERR_CUDA, "qgemm_tc: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  return tc_run<false>(s, map, nullptr, W, N, K, M, Y, accumulate, st);
}

if_status qgemv_tc_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B, float* Y,
                          int accumulate, cudaStream_t st, void* x2_scratch, size_t x2_bytes, int x2_ready) {
  if (B < 1 || B > 64 || K % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15u) || N > (int64_t)1 << 30)
    return IF_ERR_UNSUPPORTED;
  const int64_t row_bytes = K / s.block * q_block_bytes(s.type, s.block);
  if ((row_bytes & 3) || (reinterpret_cast<uintptr_t>(W) & 3u)) return IF_ERR_UNSUPPORTED;
  if (!get_encoder()) return IF_ERR_UNSUPPORTED;
  CUtensorMap map;  // x fp32 [B, K], tiles of Bpad tokens x 64 k, no swizzle (the converter reads it)
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)B};
  cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)tc_bpad((int)B)};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(IF_ERR_CUDA, "qgemv_tc: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  // caller scratch for fp16 hi/lo x: split once, TMA-load the tiles (no per-CTA conversion)
  const int bp = tc_bpad((int)B), ncols = tcd_ncols((int)B);
  // scratch: [64 floats 2^-k per token][x2 fp16 [2 bp, K]] (common.cuh X2_SC_BYTES)
  const int xpre = x2_scratch && x2_bytes >= (size_t)X2_SC_BYTES + (size_t)ncols * K * 2 &&
                   !(reinterpret_cast<uintptr_t>(x2_scratch) & 15u);
  float* x2sc = xpre ? reinterpret_cast<float*>(x2_scratch) : nullptr;
  if (xpre) {
    __half* x2 = reinterpret_cast<__half*>(reinterpret_cast<char*>(x2_scratch) + X2_SC_BYTES);
    if (!x2_ready) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)bp);  // one CTA per token row (per-token scale)
    lc.blockDim = dim3(256);
    lc.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = la;
    lc.numAttrs = 1;
    const float* xa = x;
    int Bi = (int)B, bpi = bp;
    int64_t Ki = K;
    __half* x2a = x2;
    float* sca = x2sc;
    void* args[] = {(void*)&xa, (void*)&Bi, (void*)&Ki, (void*)&bpi, (void*)&x2a, (void*)&sca};
    cudaLaunchKernelExC(&lc, (const void*)x_split_kernel, args);
    count_launch();
    }
    cuuint64_t xd[2] = {(cuuint64_t)K, (cuuint64_t)ncols};
    cuuint64_t xs[1] = {(cuuint64_t)K * 2};
    cuuint32_t xb[2] = {(cuuint32_t)TC_BK, (cuuint32_t)ncols};
    cr = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x2, xd, xs, xb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_error(IF_ERR_CUDA, "qgemv_tc: x2 tensor map failed (%d)", (int)cr);
#ifndef IFB_NO_MS
    // small batches of 3.5-bit weights: the warp-level MMA kernel (decode in registers)
    const if_status rm = qgemv_ms_launch(s, W, N, K, x2, x2sc, B, Y, accumulate, st);
    if (rm != IF_ERR_UNSUPPORTED) return rm;
#endif
  }
  const int ntile = (int)((N + TC_BN - 1) / TC_BN);
  const int ktotal = (int)((K + TC_BK - 1) / TC_BK);
  const int splits = tc_splits(ntile, ktotal);
  const int kper = (ktotal + splits - 1) / splits;
  const int atomic_out = (splits > 1) || accumulate;
  if (splits > 1 && !accumulate) {
    if (cudaMemsetAsync(Y, 0, sizeof(float) * B * N, st) != cudaSuccess) return check_launch("qgemv_tc memset");
  }
  CUtensorMap wmap;  // Q3H_B64 packed weights as bytes [N rows x row_bytes], tiles of 128 rows x 32 B
  memset(&wmap, 0, sizeof(wmap));
  if (s.type == IF_Q3H && s.block == 64) {
    if ((row_bytes & 15) || (reinterpret_cast<uintptr_t>(W) & 15u)) return IF_ERR_UNSUPPORTED;
    cuuint64_t wd[2] = {(cuuint64_t)row_bytes, (cuuint64_t)N};
    cuuint64_t ws[1] = {(cuuint64_t)row_bytes};
    cuuint32_t wb[2] = {32u, (cuuint32_t)TC_BN};
    cr = g_encode(&wmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(W), wd, ws, wb, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_error(IF_ERR_CUDA, "qgemv_tc: weight tensor map failed (%d)", (int)cr);
  }
  return dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    auto kern = qgemv_tc_kernel<QT, BS>;
    constexpr int fixed = (TcdVar<QT, BS>::FAST ? TCD_WR * 4096 : TC_PK * TC_BN * tc_sbpad(QT, BS)) + TCD_XRING + 1024 + 768 +
                          768;  // + per-token split scales
    const int sb = tcd_stage_bytes((int)B);
    int stages = std::min(TCD_MAXST, (227 * 1024 - fixed) / sb);
    if (stages < 2) return IF_ERR_UNSUPPORTED;
    const int smem = stages * sb + fixed;
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntile, 1, splits);
    cfg.blockDim = dim3(TcdVar<QT, BS>::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue + weight prefetch overlap the predecessor
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = splits > 1 && !accumulate ? 0 : 1;  // (after the split-K memset: plain stream order)
    cudaLaunchKernelEx(&cfg, kern, map, wmap, W, N, K, (int)B, Y, kper, atomic_out, stages, xpre, x, (const float*)x2sc);
    count_launch();
    return check_launch("qgemv_tc");
  });
}

}  // namespace ifb
