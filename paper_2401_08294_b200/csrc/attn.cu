// attn.cu — grouped-query decode attention over a per-slot KV cache (SURVEY NEXT-1,
// DESIGN.md Q24): the step between the qkv and o projections of every layer.
//
//   head_i = Attention(Q_i, K^j, V^j),  j = floor(i / (H/G))
//   Attention = scaled dot-product, causal over the slot's positions 0..p
//   RoPE on q and k: pair (2m, 2m+1) turned by p * 10000^(-2m/hd)    (Table 1)
//
// Three kernels per layer (T tokens, token t = (slot s_t, position p_t)):
//  1. rope_append_kernel  — one CTA per token: cos/sin of p*theta_m evaluated in fp64
//     (an fp32 angle loses ~p*2^-24 rad), q/k rotated in place in the qkv buffer, k and
//     v appended to the cache at (s_t, p_t).  All tokens append before any attends, so
//     a chunk of consecutive positions of one slot is causal prefill.
//  2. attn_partial_kernel — one CTA per (token, kv group, position split): the group's
//     H/G query heads share every K/V row the CTA loads (the GQA saving); 4 warps
//     stride over the split's positions with an online softmax (flash-decoding), lanes
//     own head_dim/32 dimensions; partial (max, sum, acc) per head to the workspace.
//  3. attn_combine_kernel — one CTA per token: merges the splits (log-sum-exp) into the
//     context row: fp32 (decode), bf16 (prefill GEMM input) and, for the batched
//     tensor-core decode, the fp16 hi/lo split with its per-token scale.
// The cache is the caller's device memory, fp32 [layers][slots][max_ctx][lkv][hd]
// (rank-local kv heads); K/V bytes join the decode roofline (2 * 4 * lkv * hd per position
// per layer read).
#include <cuda_bf16.h>

#include "attn.cuh"
#include "common.cuh"

namespace ifb {

constexpr int ATT_MAXPER = 8;  // query heads per kv group handled by one CTA (Llama-2 70B: 8)

__global__ void __launch_bounds__(128) rope_append_kernel(float* __restrict__ qkv, int T, int lh, int lkv, int hd,
                                                          const int32_t* __restrict__ slot_ids,
                                                          const int32_t* __restrict__ positions, float* __restrict__ kc,
                                                          float* __restrict__ vc, int slots, int max_ctx,
                                                          int32_t* __restrict__ status) {
  pdl_trigger();
  pdl_wait();
  __shared__ float cs[2][256];  // hd/2 <= 256
  const int t = blockIdx.x;
  const int s = slot_ids[t], p = positions[t];
  if (s < 0 || s >= slots || p < 0 || p >= max_ctx) {
    if (threadIdx.x == 0) report_status(status, IF_ERR_ARG);
    return;
  }
  const int half = hd / 2;
  for (int m = threadIdx.x; m < half; m += blockDim.x) {
    const double theta = exp(-2.0 * (double)m / (double)hd * 9.210340371976184);  // 10000^(-2m/hd), ln 10000
    double sn, c;
    sincos((double)p * theta, &sn, &c);
    cs[0][m] = (float)c;
    cs[1][m] = (float)sn;
  }
  __syncthreads();
  const int nqkv = (lh + 2 * lkv) * hd;
  float* row = qkv + (int64_t)t * nqkv;
  // q heads and k heads: rotate consecutive pairs in place
  const int npairs = (lh + lkv) * half;
  for (int i = threadIdx.x; i < npairs; i += blockDim.x) {
    const int m = i % half;
    float2* pr = reinterpret_cast<float2*>(row) + i;
    const float2 x = *pr;
    *pr = make_float2(x.x * cs[0][m] - x.y * cs[1][m], x.x * cs[1][m] + x.y * cs[0][m]);
  }
  __syncthreads();
  // append k (rotated) and v at (s, p)
  const int64_t off = ((int64_t)s * max_ctx + p) * lkv * hd;
  for (int e = threadIdx.x; e < lkv * hd; e += blockDim.x) {
    kc[off + e] = row[lh * hd + e];
    vc[off + e] = row[(lh + lkv) * hd + e];
  }
}

// partial record per (token, local head, split): [m, l, acc[hd]] (hd + 2 floats)
template <int EPL>
__global__ void __launch_bounds__(128) attn_partial_kernel(const float* __restrict__ qkv, int lh, int lkv, int hd,
                                                           const int32_t* __restrict__ slot_ids,
                                                           const int32_t* __restrict__ positions,
                                                           const float* __restrict__ kc, const float* __restrict__ vc,
                                                           int slots, int max_ctx, int nsplit,
                                                           float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  constexpr int NW = 4;
  __shared__ float sm_m[NW][ATT_MAXPER], sm_l[NW][ATT_MAXPER];
  __shared__ float sm_acc[NW][ATT_MAXPER][32 * EPL];
  const int t = blockIdx.x / lkv, jl = blockIdx.x % lkv, sp = blockIdx.y;
  const int per = lh / lkv;  // local query heads of this group: jl*per .. jl*per + per - 1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = slot_ids[t], p = positions[t];
  const bool ok = s >= 0 && s < slots && p >= 0 && p < max_ctx;
  const int n = ok ? p + 1 : 0;
  const int chunk = (n + nsplit - 1) / nsplit;
  const int tau0 = sp * chunk, tau1 = min(n, tau0 + chunk);
  const int nqkv = (lh + 2 * lkv) * hd;
  const float scale = rsqrtf((float)hd);
  float q[ATT_MAXPER][EPL], acc[ATT_MAXPER][EPL], m[ATT_MAXPER], l[ATT_MAXPER];
#pragma unroll
  for (int h = 0; h < ATT_MAXPER; h++) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; e++) {
      acc[h][e] = 0.f;
      q[h][e] = h < per ? qkv[(int64_t)t * nqkv + (jl * per + h) * hd + lane * EPL + e] * scale : 0.f;
    }
  }
  const int64_t base = (int64_t)s * max_ctx * lkv * hd + (int64_t)jl * hd + lane * EPL;
  for (int tau = tau0 + warp; tau < tau1; tau += NW) {
    const float* kr = kc + base + (int64_t)tau * lkv * hd;
    const float* vr = vc + base + (int64_t)tau * lkv * hd;
    float kv[EPL], vv[EPL];
#pragma unroll
    for (int e = 0; e < EPL; e++) {
      kv[e] = kr[e];
      vv[e] = vr[e];
    }
#pragma unroll
    for (int h = 0; h < ATT_MAXPER; h++) {
      if (h >= per) break;
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; e++) d = fmaf(q[h][e], kv[e], d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const float mn = fmaxf(m[h], d);
      const float a = expf(m[h] - mn), b = expf(d - mn);
      l[h] = l[h] * a + b;
#pragma unroll
      for (int e = 0; e < EPL; e++) acc[h][e] = fmaf(acc[h][e], a, b * vv[e]);
      m[h] = mn;
    }
  }
  // merge the 4 warps (log-sum-exp), warp 0 writes the split's record per head
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
  if (warp == 0) {
    for (int h = 0; h < per; h++) {
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; w++) M = fmaxf(M, sm_m[w][h]);
      float L = 0.f, A[EPL];
#pragma unroll
      for (int e = 0; e < EPL; e++) A[e] = 0.f;
#pragma unroll
      for (int w = 0; w < NW; w++) {
        const float f = sm_m[w][h] == -INFINITY ? 0.f : expf(sm_m[w][h] - M);
        L = fmaf(sm_l[w][h], f, L);
#pragma unroll
        for (int e = 0; e < EPL; e++) A[e] = fmaf(sm_acc[w][h][lane * EPL + e], f, A[e]);
      }
      float* rec = part + (((int64_t)t * lh + jl * per + h) * nsplit + sp) * (hd + 2);
      if (lane == 0) {
        rec[0] = M;
        rec[1] = L;
      }
#pragma unroll
      for (int e = 0; e < EPL; e++) rec[2 + lane * EPL + e] = A[e];
    }
  }
}

// one CTA per token row t < rows (rows >= T: padding rows of the x2 split are zero)
__global__ void __launch_bounds__(256) attn_combine_kernel(const float* __restrict__ part, int T, int lh, int hd,
                                                           int nsplit, float* __restrict__ ctx,
                                                           __nv_bfloat16* __restrict__ ctx16, __half* __restrict__ x2,
                                                           int bp, float* __restrict__ x2sc) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float row[];  // [lh * hd]
  __shared__ float red[8];
  const int t = blockIdx.x;
  const int nq = lh * hd;
  float mx = 0.f;
  if (t < T) {
    for (int i = threadIdx.x; i < nq; i += blockDim.x) {
      const int h = i / hd, e = i - h * hd;
      const float* rec = part + ((int64_t)t * lh + h) * nsplit * (hd + 2);
      float M = -INFINITY;
      for (int s = 0; s < nsplit; s++) M = fmaxf(M, rec[s * (hd + 2)]);
      float L = 0.f, A = 0.f;
      for (int s = 0; s < nsplit; s++) {
        const float ms = rec[s * (hd + 2)];
        const float f = ms == -INFINITY ? 0.f : expf(ms - M);
        L = fmaf(rec[s * (hd + 2) + 1], f, L);
        A = fmaf(rec[s * (hd + 2) + 2 + e], f, A);
      }
      const float v = L > 0.f ? A / L : 0.f;
      row[i] = v;
      mx = fmaxf(mx, fabsf(v));
      if (ctx) ctx[(int64_t)t * nq + i] = v;
      if (ctx16) ctx16[(int64_t)t * nq + i] = __float2bfloat16(v);
    }
  }
  if (!x2) return;
  // fp16 hi/lo split of the row with its per-token power-of-two scale (common.cuh)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) mx = fmaxf(mx, red[w]);
  const int k = xsplit_k(mx);
  const float mul = pow2f(k);
  if (threadIdx.x == 0) x2sc[t] = pow2f(-k);
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    const float v = t < T ? row[i] * mul : 0.f;
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
  int64_t want = (2 * 148 + T * lkv - 1) / (T * lkv);
  if (want > ATT_MAXSPLIT) want = ATT_MAXSPLIT;
  if (want > max_ctx) want = max_ctx;
  return want < 1 ? 1 : (int)want;
}

if_status attn_run(const AttnArgs& a, cudaStream_t st) {
  if (a.hd % 32 || a.hd > 256 || (a.hd != 64 && a.hd != 128) || a.lh % a.lkv || a.lh / a.lkv > ATT_MAXPER)
    return set_error(IF_ERR_UNSUPPORTED, "attention: head_dim %d (64/128), heads per kv group %d (<= %d)", a.hd,
                     a.lh / (a.lkv ? a.lkv : 1), ATT_MAXPER);
  const size_t layer_elems = (size_t)a.slots * a.max_ctx * a.lkv * a.hd;
  float* kc = a.k + (size_t)a.layer * layer_elems;
  float* vc = a.v + (size_t)a.layer * layer_elems;
  launch_attn(rope_append_kernel, dim3((unsigned)a.T), 128, 0, st, a.pdl, a.qkv, (int)a.T, a.lh, a.lkv, a.hd,
              a.slot_ids, a.positions, kc, vc, a.slots, a.max_ctx, a.status);
  const int ns = attn_nsplit(a.T, a.lkv, a.max_ctx);
  const dim3 g((unsigned)(a.T * a.lkv), (unsigned)ns);
  if (a.hd == 128)
    launch_attn(attn_partial_kernel<4>, g, 128, 0, st, a.pdl, (const float*)a.qkv, a.lh, a.lkv, a.hd, a.slot_ids,
                a.positions, (const float*)kc, (const float*)vc, a.slots, a.max_ctx, ns, a.part);
  else
    launch_attn(attn_partial_kernel<2>, g, 128, 0, st, a.pdl, (const float*)a.qkv, a.lh, a.lkv, a.hd, a.slot_ids,
                a.positions, (const float*)kc, (const float*)vc, a.slots, a.max_ctx, ns, a.part);
  const size_t smem = (size_t)a.lh * a.hd * 4;
  static bool cfg_done = false;
  if (!cfg_done) {
    cudaFuncSetAttribute(attn_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cfg_done = true;
  }
  if (smem > 64 * 1024) return set_error(IF_ERR_UNSUPPORTED, "attention: %d local heads x %d too wide", a.lh, a.hd);
  const int rows = a.x2 ? a.bp : (int)a.T;
  launch_attn(attn_combine_kernel, dim3((unsigned)rows), 256, smem, st, a.pdl, (const float*)a.part, (int)a.T, a.lh,
              a.hd, ns, a.ctx, a.ctx16, a.x2, a.bp, a.x2sc);
  return check_launch("attention");
}

}  // namespace ifb
