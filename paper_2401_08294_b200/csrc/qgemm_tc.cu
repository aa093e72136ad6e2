// qgemm_tc.cu — a5: prefill GEMM with fused dequantization on the 5th-gen
// tensor cores (tcgen05 + TMEM + TMA), P:94:
//     Y[m, n] (+)= sum_k W'[n, k] X[m, k]       X bf16, W' -> bf16, fp32 accumulate
//
// CTA tile: 128 output columns (weight rows n) x 256 output rows (activations m,
// two 128-row UMMA tiles, i.e. two 128x128 fp32 accumulators = 256 TMEM
// columns), K in steps of 64 (one Q3H_B64 block per weight row).  Optional
// split-K over gridDim.z (partials combined with red.global.add.v4.f32).
// Warp roles (8 warps):
//   warp 0  TMA producer: X tiles [128 rows x 64 k] bf16, SWIZZLE_128B tensor map
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer (kind::f16, bf16)
//   warps 2-5  dequantizers: weight row r = thread, Eq. 2 -> bf16,
//           written straight into the UMMA canonical K-major SW128 layout,
//           fence.proxy.async, mbarrier arrive
//   warps 2-5  epilogue: tcgen05.ld 32x32b (TMEM lane quarter = warp % 4)
// Pipeline: 4 stages, full barriers (A: TMA tx bytes; B: 128 dequant arrivals),
// empty barriers armed by tcgen05.commit.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "pipe.cuh"
#include "qgemm.cuh"

namespace ifb {

constexpr int TC_BN = 128;     // weight rows per CTA (UMMA N)
constexpr int TC_BM = 128;     // activation rows per UMMA tile (UMMA M)
constexpr int TC_MT = 2;       // UMMA M tiles per CTA
constexpr int TC_BK = 64;      // K per stage
constexpr int TC_STAGES = 4;
constexpr int TC_THREADS = 256;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;  // 16 KB per M tile
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;  // 16 KB
constexpr int TC_STAGE_BYTES = TC_MT * TC_A_BYTES + TC_B_BYTES;
constexpr int TC_SMEM = TC_STAGES * TC_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TC_TMEM_COLS = TC_MT * TC_BN;  // 256

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

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M = 128, N = 128
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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

// Dequantize weight row n, weights [k0, k0 + 64), into 128 bytes of bf16 in the
// SW128 K-major layout at row r of the B tile (zeros beyond N or K).
template <int QT, int BS>
__device__ __forceinline__ void dequant_row(const uint8_t* __restrict__ W, int64_t nb, int64_t n, int64_t N,
                                           int64_t k0, int64_t K, unsigned char* btile, int r) {
  constexpr int D = q_levels(QT);
  constexpr int C = q_width(QT);
  constexpr int NC = q_ncodes(QT, BS);
  constexpr int BB = q_block_bytes(QT, BS);
  constexpr int NW = q_block_words(QT, BS);
  uint32_t out[32];  // 64 bf16
#pragma unroll
  for (int sub = 0; sub < TC_BK / BS; sub++) {
    const int64_t kk = k0 + sub * BS;
    if (n < N && kk < K) {
      uint32_t w[NW + 1];
      load_block_words<BB, NW>(W + (n * nb + kk / BS) * BB, w);
      const float lo = half_bits_to_float(w[0] & 0xFFFFu);
      const float hi = half_bits_to_float(w[0] >> 16);
      const float step = __fdiv_rn(__fsub_rn(hi, lo), (float)D);
#pragma unroll
      for (int j = 0; j < NC; j++) {
        const uint32_t v = get_code<C, NW>(w, j);
        if constexpr (QT == 35) {
          const uint32_t q1 = (v * 187u) >> 11;  // floor(v/11) for v < 128
          const uint32_t q2 = v - 11u * q1;      // v mod 11
          out[sub * (BS / 2) + j] = pack_bf16x2(__fmaf_rn((float)q1, step, lo), __fmaf_rn((float)q2, step, lo));
        } else {
          const float wp = __fmaf_rn((float)v, step, lo);
          if (j & 1)
            out[sub * (BS / 2) + j / 2] |= pack_bf16x2(0.f, wp) & 0xFFFF0000u;
          else
            out[sub * (BS / 2) + j / 2] = pack_bf16x2(wp, 0.f) & 0x0000FFFFu;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < BS / 2; j++) out[sub * (BS / 2) + j] = 0u;
    }
  }
  // 8 chunks of 16 B; chunk c of row r lives at chunk (c ^ (r % 8)) of the row (SW128)
  unsigned char* rowp = btile + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
  for (int c = 0; c < 8; c++) {
    uint4 v = make_uint4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]);
    *reinterpret_cast<uint4*>(rowp + ((c ^ (r & 7)) << 4)) = v;
  }
}

template <int QT, int BS>
__global__ void __launch_bounds__(TC_THREADS, 1)
    qgemm_tc_kernel(const __grid_constant__ CUtensorMap xmap, const uint8_t* __restrict__ W, int64_t N, int64_t K,
                    int64_t M, float* __restrict__ Y, int ksteps_per_split, int atomic_out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * TC_STAGE_BYTES);
  uint64_t* b_full = a_full + TC_STAGES;
  uint64_t* empty = b_full + TC_STAGES;
  uint64_t* acc_full = empty + TC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n0 = (int64_t)blockIdx.x * TC_BN;
  const int64_t m0 = (int64_t)blockIdx.y * (TC_BM * TC_MT);
  const int64_t nb = K / BS;
  const int ktotal = (int)((K + TC_BK - 1) / TC_BK);
  const int ks0 = blockIdx.z * ksteps_per_split;
  const int ks1 = min(ktotal, ks0 + ksteps_per_split);
  const int nks = ks1 - ks0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; s++) {
      mbar_init(&a_full[s], 1);
      mbar_init(&b_full[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: X tiles ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
      for (int i = 0; i < nks; i++) {
        const int s = i % TC_STAGES;
        mbar_wait(&empty[s], ((i / TC_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&a_full[s], TC_MT * TC_A_BYTES);
        unsigned char* st = smem + s * TC_STAGE_BYTES;
        for (int mt = 0; mt < TC_MT; mt++)
          tma_load_2d(st + mt * TC_A_BYTES, &xmap, (ks0 + i) * TC_BK, (int)(m0 + mt * TC_BM), &a_full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(TC_BM, TC_BN);
      for (int i = 0; i < nks; i++) {
        const int s = i % TC_STAGES;
        const uint32_t par = (i / TC_STAGES) & 1;
        mbar_wait(&a_full[s], par);
        mbar_wait(&b_full[s], par);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * TC_STAGE_BYTES);
        const uint64_t bdesc0 = umma_desc_sw128(st + TC_MT * TC_A_BYTES);
#pragma unroll
        for (int mt = 0; mt < TC_MT; mt++) {
          const uint64_t adesc0 = umma_desc_sw128(st + mt * TC_A_BYTES);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; kk++) {
            // advance 16 bf16 = 32 bytes along K inside the 128-byte swizzle row
            umma_bf16(tmem + mt * TC_BN, adesc0 + (uint64_t)(kk * 2), bdesc0 + (uint64_t)(kk * 2), idesc,
                      (i > 0) || (kk > 0));
          }
        }
        umma_commit(&empty[s]);  // frees the stage once these MMAs completed
      }
      umma_commit(acc_full);
    }
  } else if (warp < 6) {
    // ---------------- dequantizers: one weight row per thread ----------------
    const int r = threadIdx.x - 64;  // 0..127
    for (int i = 0; i < nks; i++) {
      const int s = i % TC_STAGES;
      mbar_wait(&empty[s], ((i / TC_STAGES) & 1) ^ 1);
      unsigned char* btile = smem + s * TC_STAGE_BYTES + TC_MT * TC_A_BYTES;
      dequant_row<QT, BS>(W, nb, n0 + r, N, (int64_t)(ks0 + i) * TC_BK, K, btile, r);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      mbar_arrive(&b_full[s]);
    }
  }

  // ---------------- epilogue: TMEM -> registers -> global ----------------
  if (warp >= 2 && warp < 6) {
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
#pragma unroll
    for (int mt = 0; mt < TC_MT; mt++) {
      const int64_t m = m0 + mt * TC_BM + q * 32 + lane;
#pragma unroll
      for (int cc = 0; cc < TC_BN / 32; cc++) {
        uint32_t rr[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + mt * TC_BN + cc * 32, rr);
        const int64_t nbase = n0 + cc * 32;
        if (m < M && nks > 0) {
          float* yrow = Y + m * N + nbase;
          if (nbase + 32 <= N && (N % 4) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              if (atomic_out) {
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(yrow + j), "f"(__uint_as_float(rr[j])),
                             "f"(__uint_as_float(rr[j + 1])), "f"(__uint_as_float(rr[j + 2])), "f"(__uint_as_float(rr[j + 3]))
                             : "memory");
              } else {
                *reinterpret_cast<float4*>(yrow + j) = make_float4(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1]),
                                                                   __uint_as_float(rr[j + 2]), __uint_as_float(rr[j + 3]));
              }
            }
          } else {
            for (int j = 0; j < 32; j++)
              if (nbase + j < N) {
                if (atomic_out)
                  atomicAdd(yrow + j, __uint_as_float(rr[j]));
                else
                  yrow[j] = __uint_as_float(rr[j]);
              }
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS) : "memory");
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
  const int ntile = (int)((N + TC_BN - 1) / TC_BN);
  const int mtile = (int)((M + TC_BM * TC_MT - 1) / (TC_BM * TC_MT));
  const int ktotal = (int)((K + TC_BK - 1) / TC_BK);
  // split K until the grid covers the SMs (partials combined with red.add)
  int splits = 1;
  while (ntile * mtile * splits < tc_sms() && ktotal / (splits * 2) >= 8) splits *= 2;
  const int kper = (ktotal + splits - 1) / splits;
  const int atomic_out = (splits > 1) || accumulate;
  if (splits > 1 && !accumulate) {
    if (cudaMemsetAsync(Y, 0, sizeof(float) * M * N, st) != cudaSuccess) return check_launch("qgemm_tc memset");
  }
  return dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    auto kern = qgemm_tc_kernel<QT, BS>;
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
      configured = true;
    }
    dim3 grid(ntile, mtile, splits);
    kern<<<grid, TC_THREADS, TC_SMEM, st>>>(map, W, N, K, M, Y, kper, atomic_out);
    count_launch();
    return check_launch("qgemm_tc");
  });
}

}  // namespace ifb
