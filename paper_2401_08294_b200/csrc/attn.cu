// attn.cu — grouped-query decode attention over a per-slot KV cache (SURVEY NEXT-1,
// DESIGN.md Q24): the step between the qkv and o projections of every layer.
//
//   head_i = Attention(Q_i, K^j, V^j),  j = floor(i / (H/G))
//   Attention = scaled dot-product, causal over the slot's positions 0..p
//   RoPE on q and k: pair (2m, 2m+1) turned by p * 10000^(-2m/hd)    (Table 1)
//
// Two kernels per layer (T tokens, token t = (slot s_t, position p_t)):
//  1. rope_append_kernel — one warp per (token, head): cos/sin of p*theta_m evaluated in
//     fp64 (an fp32 angle loses ~p*2^-24 rad), q/k rotated in place in the qkv buffer, k
//     and v appended to the cache at (s_t, p_t).  All tokens append before any attends,
//     so a chunk of consecutive positions of one slot is causal prefill.
//  2. attn_kernel — one CTA per (token, kv group, position split): the group's H/G query
//     heads share every K/V row the CTA loads (the GQA saving); 4 warps take the split's
//     positions ATT_U at a time (ATT_U rows of K and V in flight per warp) with an online
//     softmax (flash-decoding); lanes own head_dim/32 dimensions.  The partial
//     (max, sum, acc) of each head goes to the workspace; the LAST split CTA of a
//     (token, group) to arrive (a self-resetting counter) merges the splits (log-sum-exp)
//     into the context: fp32 (decode), bf16 (prefill GEMM input).  For the batched
//     tensor-core decode the last GROUP of a token to arrive also writes the row's fp16
//     hi/lo split with its per-token scale.  (Round 1 ran rope / partial / combine as
//     three launches whose single-CTA-per-token kernels were latency-bound: ~100 us per
//     layer at batch 1; profiles/r2_kv_decode.txt.)
// The cache is the caller's device memory, fp32 [layers][slots][max_ctx][lkv][hd]
// (rank-local kv heads); K/V bytes join the decode roofline (2 * 4 * lkv * hd per position
// per layer read).
#include <stdlib.h>

#include <cuda_bf16.h>

#include "attn.cuh"
#include "ms_rec.cuh"
#include "common.cuh"

namespace ifb {

constexpr int ATT_MAXPER = 8;  // query heads per kv group handled by one CTA (Llama-2 70B: 8)
constexpr int ATT_NW = 4;      // warps per attention CTA
constexpr int ATT_U = 4;       // positions per warp iteration (loads in flight)

template <int EPL>
struct VecF;
template <>
struct VecF<2> {
  using T = float2;
};
template <>
struct VecF<4> {
  using T = float4;
};

template <int EPL>
__device__ __forceinline__ void ld_vec(const float* p, float (&v)[EPL]) {
  const typename VecF<EPL>::T x = *reinterpret_cast<const typename VecF<EPL>::T*>(p);
  const float* f = reinterpret_cast<const float*>(&x);
#pragma unroll
  for (int e = 0; e < EPL; e++) v[e] = f[e];
}
template <int EPL>
__device__ __forceinline__ void st_vec(float* p, const float (&v)[EPL]) {
  typename VecF<EPL>::T x;
  float* f = reinterpret_cast<float*>(&x);
#pragma unroll
  for (int e = 0; e < EPL; e++) f[e] = v[e];
  *reinterpret_cast<typename VecF<EPL>::T*>(p) = x;
}

// grid (T + npad, ceil((lh + 2 lkv) / 4)), 128 threads: warp = one head of token t.
// Rows t >= T (npad > 0, batched decode) zero the x2 split's padding rows.
template <int EPL>
__global__ void __launch_bounds__(128) rope_append_kernel(float* __restrict__ qkv, int T, int lh, int lkv,
                                                          const int32_t* __restrict__ slot_ids,
                                                          const int32_t* __restrict__ positions, float* __restrict__ kc,
                                                          float* __restrict__ vc, int slots, int max_ctx,
                                                          int32_t* __restrict__ status, __half* __restrict__ x2,
                                                          int bp, float* __restrict__ x2sc) {
  pdl_trigger();
  pdl_wait();
  constexpr int hd = 32 * EPL;
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (t >= T) {  // padding row of the fp16 split: zero hi and lo, scale of a zero row
    const int nq = lh * hd;
    for (int i = blockIdx.y * 128 + threadIdx.x; i < nq; i += gridDim.y * 128) {
      x2[(int64_t)t * nq + i] = __float2half_rn(0.f);
      x2[((int64_t)bp + t) * nq + i] = __float2half_rn(0.f);
    }
    if (blockIdx.y == 0 && threadIdx.x == 0) x2sc[t] = pow2f(-xsplit_k(0.f));
    return;
  }
  const int s = slot_ids[t], p = positions[t];
  if (s < 0 || s >= slots || p < 0 || p >= max_ctx) {
    if (threadIdx.x == 0 && blockIdx.y == 0) report_status(status, IF_ERR_ARG);
    return;
  }
  const int head = blockIdx.y * 4 + warp;  // q heads 0..lh-1, k lh.., v lh+lkv..
  if (head >= lh + 2 * lkv) return;
  const int nqkv = (lh + 2 * lkv) * hd;
  float* src = qkv + (int64_t)t * nqkv + (int64_t)head * hd + lane * EPL;
  float v[EPL];
  ld_vec<EPL>(src, v);
  if (head < lh + lkv) {  // q or k: rotate the lane's pairs (2m, 2m+1), m = lane*EPL/2 + j
#pragma unroll
    for (int j = 0; j < EPL / 2; j++) {
      const int m = lane * (EPL / 2) + j;
      const double theta = exp(-2.0 * (double)m / (double)hd * 9.210340371976184);  // 10000^(-2m/hd), ln 10000
      double sn, c;
      sincos((double)p * theta, &sn, &c);
      const float cf = (float)c, sf = (float)sn;
      const float x = v[2 * j], y = v[2 * j + 1];
      v[2 * j] = x * cf - y * sf;
      v[2 * j + 1] = x * sf + y * cf;
    }
    st_vec<EPL>(src, v);
  }
  if (head >= lh) {  // append k (rotated) / v at (s, p)
    const bool isk = head < lh + lkv;
    const int j = isk ? head - lh : head - lh - lkv;
    float* dst = (isk ? kc : vc) + ((int64_t)s * max_ctx + p) * lkv * hd + (int64_t)j * hd + lane * EPL;
    st_vec<EPL>(dst, v);
  }
}

// RoPE of one lane's EPL values (pairs (2m, 2m+1), m = lane EPL/2 + j) at position p:
// the rope_append_kernel formula (angles in fp64)
template <int EPL>
__device__ __forceinline__ void rope_pairs(float (&v)[EPL], int p, int lane) {
  constexpr int hd = 32 * EPL;
#pragma unroll
  for (int j = 0; j < EPL / 2; j++) {
    const int m = lane * (EPL / 2) + j;
    const double theta = exp(-2.0 * (double)m / (double)hd * 9.210340371976184);  // 10000^(-2m/hd), ln 10000
    double sn, c;
    sincos((double)p * theta, &sn, &c);
    const float cf = (float)c, sf = (float)sn;
    const float x = v[2 * j], y = v[2 * j + 1];
    v[2 * j] = x * cf - y * sf;
    v[2 * j + 1] = x * sf + y * cf;
  }
}

// partial record per (token, local head, split): [m, l, acc[hd]] (hd + 2 floats)
// grid (T * lkv, nsplit), 128 threads.  gcnt[t * lkv + jl] / tcnt[t]: zero between calls
// (the last arriver resets its counter).
template <int EPL>
__global__ void __launch_bounds__(128) attn_kernel(const float* __restrict__ qkv, int T, int lh, int lkv,
                                                   const int32_t* __restrict__ slot_ids,
                                                   const int32_t* __restrict__ positions, const float* __restrict__ kc,
                                                   const float* __restrict__ vc, int slots, int max_ctx, int nsplit,
                                                   float* part, uint32_t* gcnt, uint32_t* tcnt, float* ctx,
                                                   __nv_bfloat16* __restrict__ ctx16, __half* __restrict__ x2, int bp,
                                                   float* __restrict__ x2sc, uint8_t* __restrict__ rec, int rec_nt,
                                                   int fused, float* __restrict__ rot_out, int32_t* __restrict__ status) {
  pdl_trigger();
  pdl_wait();
  constexpr int NW = ATT_NW, U = ATT_U, hd = 32 * EPL;
  __shared__ float sm_m[NW][ATT_MAXPER], sm_l[NW][ATT_MAXPER];
  __shared__ float sm_acc[NW][ATT_MAXPER][hd];
  __shared__ float red[NW];
  __shared__ int s_last;
  const int t = blockIdx.x / lkv, jl = blockIdx.x % lkv, sp = blockIdx.y;
  const int per = lh / lkv;  // local query heads of this group: jl*per .. jl*per + per - 1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = slot_ids[t], p = positions[t];
  const bool ok = s >= 0 && s < slots && p >= 0 && p < max_ctx;
  const int n = ok ? p + 1 : 0;
  const int chunk = (n + nsplit - 1) / nsplit;
  const int tau0 = sp * chunk, tau1 = min(n, tau0 + chunk);
  const int nqkv = (lh + 2 * lkv) * hd, nq = lh * hd;
  const float scale = rsqrtf((float)hd);
  float q[ATT_MAXPER][EPL], acc[ATT_MAXPER][EPL], m[ATT_MAXPER], l[ATT_MAXPER];
#pragma unroll
  for (int h = 0; h < ATT_MAXPER; h++) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; e++) acc[h][e] = 0.f;
    if (h < per) {
      ld_vec<EPL>(qkv + (int64_t)t * nqkv + (jl * per + h) * hd + lane * EPL, q[h]);
      if (fused && ok) {
        rope_pairs<EPL>(q[h], p, lane);  // q after RoPE (the rope kernel's turn, in registers)
        if (rot_out && sp == 0) st_vec<EPL>(rot_out + (int64_t)t * nqkv + (jl * per + h) * hd + lane * EPL, q[h]);
      }
#pragma unroll
      for (int e = 0; e < EPL; e++) q[h][e] *= scale;
    } else {
#pragma unroll
      for (int e = 0; e < EPL; e++) q[h][e] = 0.f;
    }
  }
  const int64_t base = (int64_t)s * max_ctx * lkv * hd + (int64_t)jl * hd + lane * EPL;
  // fused RoPE/append (T = 1): k_p, v_p of this group from the projections, k rotated;
  // position p is read from registers (the append below is for later steps), and the
  // split holding p appends them
  float kp[EPL], vp[EPL];
  if (fused && ok) {
    ld_vec<EPL>(qkv + (int64_t)t * nqkv + (lh + jl) * hd + lane * EPL, kp);
    ld_vec<EPL>(qkv + (int64_t)t * nqkv + (lh + lkv + jl) * hd + lane * EPL, vp);
    rope_pairs<EPL>(kp, p, lane);
    if (warp == 0 && p >= tau0 && p < tau1) {
      st_vec<EPL>(const_cast<float*>(kc) + base + (int64_t)p * lkv * hd, kp);
      st_vec<EPL>(const_cast<float*>(vc) + base + (int64_t)p * lkv * hd, vp);
    }
    if (rot_out && sp == 0 && warp == 0) {
      st_vec<EPL>(rot_out + (int64_t)t * nqkv + (lh + jl) * hd + lane * EPL, kp);
      st_vec<EPL>(rot_out + (int64_t)t * nqkv + (lh + lkv + jl) * hd + lane * EPL, vp);
    }
  } else if (fused && !ok && sp == 0 && jl == 0 && threadIdx.x == 0) {
    report_status(status, IF_ERR_ARG);
  }
  for (int tau = tau0 + warp * U; tau < tau1; tau += NW * U) {
    float kv[U][EPL], vv[U][EPL];
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (tau + u < tau1) {
        if (fused && tau + u == p) {
#pragma unroll
          for (int e = 0; e < EPL; e++) kv[u][e] = kp[e], vv[u][e] = vp[e];
        } else {
          ld_vec<EPL>(kc + base + (int64_t)(tau + u) * lkv * hd, kv[u]);
          ld_vec<EPL>(vc + base + (int64_t)(tau + u) * lkv * hd, vv[u]);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < ATT_MAXPER; h++) {
      if (h >= per) break;
      float d[U];
      float mn = m[h];
#pragma unroll
      for (int u = 0; u < U; u++) {
        float x = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; e++) x = fmaf(q[h][e], kv[u][e], x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        d[u] = tau + u < tau1 ? x : -INFINITY;
        mn = fmaxf(mn, d[u]);
      }
      const float a = expf(m[h] - mn);  // m = -inf (first rows): 0
      l[h] *= a;
#pragma unroll
      for (int e = 0; e < EPL; e++) acc[h][e] *= a;
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (tau + u < tau1) {
          const float b = expf(d[u] - mn);
          l[h] += b;
#pragma unroll
          for (int e = 0; e < EPL; e++) acc[h][e] = fmaf(b, vv[u][e], acc[h][e]);
        }
      }
      m[h] = mn;
    }
  }
  // merge the 4 warps (log-sum-exp)
#pragma unroll
  for (int h = 0; h < ATT_MAXPER; h++) {
    if (h >= per) break;
    if (lane == 0) {
      sm_m[warp][h] = m[h];
      sm_l[warp][h] = l[h];
    }
#pragma unroll
    for (int e = 0; e < EPL; e++) sm_acc[warp][h][lane * EPL + e] = acc[h][e];
  }
  __syncthreads();
  // threads own (head, dim) elements of the group: i = h * hd + e
  for (int i = threadIdx.x; i < per * hd; i += blockDim.x) {
    const int h = i / hd, e = i - h * hd;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; w++) M = fmaxf(M, sm_m[w][h]);
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < NW; w++) {
      const float f = sm_m[w][h] == -INFINITY ? 0.f : expf(sm_m[w][h] - M);
      L = fmaf(sm_l[w][h], f, L);
      A = fmaf(sm_acc[w][h][e], f, A);
    }
    if (nsplit == 1) {  // the split is the whole context: final value
      const float v = L > 0.f ? A / L : 0.f;
      const int64_t o = (int64_t)t * nq + (jl * per + h) * hd + e;
      if (ctx) ctx[o] = v;
      if (ctx16) ctx16[o] = __float2bfloat16(v);
    } else {
      float* rec = part + (((int64_t)t * lh + jl * per + h) * nsplit + sp) * (hd + 2);
      if (e == 0) {
        rec[0] = M;
        rec[1] = L;
      }
      rec[2 + e] = A;
    }
  }
  if (nsplit > 1) {
    // the last split CTA of (t, jl) to arrive merges the splits
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t old = atomicAdd(&gcnt[t * lkv + jl], 1u);
      s_last = old == (uint32_t)nsplit - 1;
      if (s_last) gcnt[t * lkv + jl] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int i = threadIdx.x; i < per * hd; i += blockDim.x) {
      const int h = i / hd, e = i - h * hd;
      const float* rec = part + ((int64_t)t * lh + jl * per + h) * nsplit * (hd + 2);
      // every split's (m, l, acc_e) in flight at once (a serial loop paid one L2 latency
      // per split and per pass: ~10 us of a 14.5 us kernel at 19 splits), then the
      // log-sum-exp merge in split order
      float mk[ATT_MAXSPLIT], lk[ATT_MAXSPLIT], ak[ATT_MAXSPLIT];
#pragma unroll
      for (int k = 0; k < ATT_MAXSPLIT; k++) {
        mk[k] = k < nsplit ? __ldcg(rec + k * (hd + 2)) : -INFINITY;
        lk[k] = k < nsplit ? __ldcg(rec + k * (hd + 2) + 1) : 0.f;
        ak[k] = k < nsplit ? __ldcg(rec + k * (hd + 2) + 2 + e) : 0.f;
      }
      float M = -INFINITY;
#pragma unroll
      for (int k = 0; k < ATT_MAXSPLIT; k++) M = fmaxf(M, mk[k]);
      float L = 0.f, A = 0.f;
#pragma unroll
      for (int k = 0; k < ATT_MAXSPLIT; k++) {
        if (k >= nsplit) break;
        const float f = mk[k] == -INFINITY ? 0.f : expf(mk[k] - M);
        L = fmaf(lk[k], f, L);
        A = fmaf(ak[k], f, A);
      }
      const float v = L > 0.f ? A / L : 0.f;
      const int64_t o = (int64_t)t * nq + (jl * per + h) * hd + e;
      if (ctx) ctx[o] = v;
      if (ctx16) ctx16[o] = __float2bfloat16(v);
    }
  }
  if (rec) {
    // this CTA wrote the final ctx of (t, group jl): per * hd values = nblk 64-blocks,
    // re-read (same CTA, after the barrier) into the chain's fragment records
    __syncthreads();
    const int nblk = per * hd / 64, gb0 = jl * per * hd / 64, nit = nblk * 4;
    for (int it0 = threadIdx.x & ~31; it0 < ((nit + 31) & ~31); it0 += blockDim.x) {
      const int it = it0 + lane, blk = it >> 2, c = it & 3;
      const bool ok = it < nit;
      float x[16];
      const float* src = ctx + (int64_t)t * nq + (int64_t)(gb0 + blk) * 64 + 16 * c;
#pragma unroll
      for (int i = 0; i < 16; i++) x[i] = ok ? src[i] : 0.f;
      ms_put_item(rec + ((size_t)(gb0 + (ok ? blk : 0)) * rec_nt + (t >> 3)) * FR_REC, t, c, x, ok);
    }
  }
  if (!x2) return;
  // the last group of token t to arrive writes the row's fp16 hi/lo split (common.cuh)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t old = atomicAdd(&tcnt[t], 1u);
    s_last = old == (uint32_t)lkv - 1;
    if (s_last) tcnt[t] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* row = ctx + (int64_t)t * nq;
  float mx = 0.f;
  for (int i = threadIdx.x; i < nq; i += blockDim.x) mx = fmaxf(mx, fabsf(__ldcg(row + i)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = 0.f;
#pragma unroll
  for (int w = 0; w < NW; w++) mx = fmaxf(mx, red[w]);
  const int k = xsplit_k(mx);
  const float mul = pow2f(k);
  if (threadIdx.x == 0) x2sc[t] = pow2f(-k);
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    const float v = __ldcg(row + i) * mul;
    const __half hh = __float2half_rn(v);
    x2[(int64_t)t * nq + i] = hh;
    x2[((int64_t)bp + t) * nq + i] = __float2half_rn(v - __half2float(hh));
  }
}

template <typename... KArgs, typename... Args>
static void launch_attn(void (*kern)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t st, bool pdl,
                        Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, (KArgs)args...);
  count_launch();
}

int attn_nsplit(int64_t T, int lkv, int max_ctx) {
  if (T > ATT_MAXT) return 1;  // prefill chunks: one CTA per (token, group) covers its context
  int64_t want = (4 * 148 + T * lkv - 1) / (T * lkv);
  if (want > ATT_MAXSPLIT) want = ATT_MAXSPLIT;
  if (want > max_ctx) want = max_ctx;
  return want < 1 ? 1 : (int)want;
}

size_t attn_cnt_words(int lkv) { return (size_t)ATT_MAXT * lkv + ATT_MAXT; }

template <int EPL>
static void attn_launch(const AttnArgs& a, float* kc, float* vc, int ns, cudaStream_t st) {
  // one token, no fp16 split / records: RoPE and the append fused into the attention
  // kernel (one launch instead of two per layer)
  static const int no_fuse = getenv("IFB_NO_ROPE_FUSE") != nullptr;  // A/B experiments only
  const int fused = a.T == 1 && !a.x2 && !a.rec && !no_fuse;
  if (!fused) {
    const int npad = a.x2 ? a.bp - (int)a.T : 0;
    const dim3 ga((unsigned)(a.T + npad), (unsigned)((a.lh + 2 * a.lkv + 3) / 4));
    launch_attn(rope_append_kernel<EPL>, ga, 128, 0, st, a.pdl, a.qkv, (int)a.T, a.lh, a.lkv, a.slot_ids, a.positions,
                kc, vc, a.slots, a.max_ctx, a.status, a.x2, a.bp, a.x2sc);
  }
  const dim3 gb((unsigned)(a.T * a.lkv), (unsigned)ns);
  launch_attn(attn_kernel<EPL>, gb, 128, 0, st, a.pdl, (const float*)a.qkv, (int)a.T, a.lh, a.lkv, a.slot_ids,
              a.positions, (const float*)kc, (const float*)vc, a.slots, a.max_ctx, ns, a.part, a.cnt,
              a.cnt ? a.cnt + (size_t)ATT_MAXT * a.lkv : nullptr, a.ctx, a.ctx16, a.x2, a.bp, a.x2sc, a.rec, a.rec_nt,
              fused, fused ? a.rot_out : nullptr, a.status);
  if (!fused && a.rot_out)  // the rope kernel rotated q, k in place
    cudaMemcpyAsync(a.rot_out, a.qkv, (size_t)a.T * (a.lh + 2 * a.lkv) * a.hd * 4, cudaMemcpyDeviceToDevice, st);
}

if_status attn_run(const AttnArgs& a, cudaStream_t st) {
  if ((a.hd != 64 && a.hd != 128) || a.lh % a.lkv || a.lh / a.lkv > ATT_MAXPER)
    return set_error(IF_ERR_UNSUPPORTED, "attention: head_dim %d (64/128), heads per kv group %d (<= %d)", a.hd,
                     a.lh / (a.lkv ? a.lkv : 1), ATT_MAXPER);
  const int ns = attn_nsplit(a.T, a.lkv, a.max_ctx);
  if ((ns > 1 || a.x2) && (!a.cnt || a.T > ATT_MAXT || !a.part))
    return set_error(IF_ERR_ARG, "attention: split merge needs the counter / partial workspace (T=%lld)", (long long)a.T);
  if (a.x2 && (!a.ctx || a.bp < a.T)) return set_error(IF_ERR_ARG, "attention: fp16 split needs the fp32 context");
  if (a.rec && (!a.ctx || a.hd % 64 || a.rec_nt * 8 < a.T)) return set_error(IF_ERR_ARG, "attention: records need the fp32 context");
  const size_t layer_elems = (size_t)a.slots * a.max_ctx * a.lkv * a.hd;
  float* kc = a.k + (size_t)a.layer * layer_elems;
  float* vc = a.v + (size_t)a.layer * layer_elems;
  if (a.hd == 128)
    attn_launch<4>(a, kc, vc, ns, st);
  else
    attn_launch<2>(a, kc, vc, ns, st);
  return check_launch("attention");
}

}  // namespace ifb
