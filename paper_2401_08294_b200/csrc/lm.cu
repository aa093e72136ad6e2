// lm.cu — the language-model head around the stack (Q27) and the
// speculative-sampling verification of Algorithm 1 (NEXT-3):
//   if_embed        h[t] = E[token_t]                        (the stack's input)
//   if_lm_logits    logits[t] = rms(h[t]) . W'_lm            (final RMSNorm, S:325,
//                   then the block-quantized output projection through if_qgemv:
//                   B = T rows, the batched tensor-core path for 2 <= T <= 64)
//   if_argmax       greedy next token (first maximum)
//   if_spec_verify  one verification round: accept draft t when (is_top and it lies
//                   in the target's top-k/top-p pool) or a < min(1, q/p),
//                   else resample from (q - p)_+ and stop; all accepted -> an extra
//                   token from q at position K (Algorithm 1).
// The verification works in fp64 (the oracle's precision, so both sides take the
// accept/reject and sampling decisions in the same precision, Q26): one CTA,
// softmax statistics by block reductions, inverse-CDF sampling by a block scan.
#include <float.h>

#include "common.cuh"

namespace ifb {

if_status qgemv_dispatch(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x,
                         int64_t B, float* y, int acc, cudaStream_t st, void* x2_scratch, size_t x2_bytes,
                         int x2_ready);

// ---- embedding gather: one CTA per token row, 128-bit copies ---------------------
__global__ void __launch_bounds__(256) embed_kernel(const float* __restrict__ E, int V, int d,
                                                    const int32_t* __restrict__ tok, float* __restrict__ h,
                                                    int32_t* __restrict__ status) {
  const int t = blockIdx.x;
  const int v = tok[t];
  const bool ok = v >= 0 && v < V;
  if (!ok && threadIdx.x == 0) report_status(status, IF_ERR_ARG);
  const float4* src = reinterpret_cast<const float4*>(E + (int64_t)(ok ? v : 0) * d);
  float4* dst = reinterpret_cast<float4*>(h + (int64_t)t * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) dst[i] = ok ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---- final RMSNorm of selected rows: a[b] = rms(h[rows[b]]) (rows nullable = identity)
__global__ void __launch_bounds__(256) lm_rmsnorm_kernel(const float* __restrict__ h, const int32_t* __restrict__ rows,
                                                         int d, float* __restrict__ a) {
  __shared__ float red[8];
  const int b = blockIdx.x;
  const float* hr = h + (int64_t)(rows ? rows[b] : b) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(hr[i], hr[i], ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) tot += red[w];
  const float inv = 1.0f / sqrtf(tot / (float)d + 1e-5f);
  float* ar = a + (int64_t)b * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ar[i] = hr[i] * inv;
}

// ---- greedy choice: first index of the row maximum (one CTA per row) ----------------
__global__ void __launch_bounds__(512) argmax_kernel(const float* __restrict__ logits, int64_t V,
                                                     int32_t* __restrict__ tok) {
  __shared__ float sv[16];
  __shared__ int64_t si[16];
  const float* r = logits + (int64_t)blockIdx.x * V;
  float bv = -INFINITY;
  int64_t bi = V;  // NaN-only rows fall through to index 0 below
  for (int64_t i = threadIdx.x; i < V; i += blockDim.x) {
    const float x = r[i];
    if (x > bv) {  // strictly greater: a thread keeps its first maximum
      bv = x;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = sv[0];
    bi = si[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
        bv = sv[w];
        bi = si[w];
      }
    tok[blockIdx.x] = (int32_t)(bi < V ? bi : 0);
  }
}

// ---- speculative verification (one CTA of SV_THREADS) ---------------------------------
constexpr int SV_THREADS = 1024;

struct SvShared {
  double red[SV_THREADS / 32];
  double scan[SV_THREADS / 32];
  int ired[SV_THREADS / 32];
  int pick;
  int last_pos;
};

__device__ __forceinline__ double sv_sum(double v, SvShared& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < SV_THREADS / 32; w++) t += s.red[w];  // fixed order: same on every thread
  return t;
}
__device__ __forceinline__ float sv_max(float v, SvShared& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = (double)v;
  __syncthreads();
  double t = -INFINITY;
  for (int w = 0; w < SV_THREADS / 32; w++) t = fmax(t, s.red[w]);
  return (float)t;
}
__device__ __forceinline__ int sv_count(int v, SvShared& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.ired[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
  for (int w = 0; w < SV_THREADS / 32; w++) t += s.ired[w];
  return t;
}

// Weight of index i for the sampling pass: (q - p)_+ (residual) or q (target).
struct SvWeights {
  const float* l;  // target logits row
  const float* p;  // draft probabilities row (residual only)
  float m;
  double inv_sum;
  bool residual;
  __device__ __forceinline__ double q(int64_t i) const { return exp((double)l[i] - (double)m) * inv_sum; }
  __device__ __forceinline__ double w(int64_t i) const {
    const double qi = q(i);
    if (!residual) return qi;
    const double r = qi - (double)p[i];
    return r > 0.0 ? r : 0.0;
  }
};

// Inverse-CDF draw: the smallest i whose running sum (index order) exceeds u * total;
// -1 when the total is not positive.  Thread j owns the contiguous chunk
// [j*C, (j+1)*C): chunk sums, a block scan of them, then the owning thread walks its
// chunk.  (u -> 1 rounding: the last index with positive weight.)
__device__ int sv_sample(const SvWeights& W, int64_t V, double u, SvShared& s) {
  const int64_t C = (V + SV_THREADS - 1) / SV_THREADS;
  const int64_t i0 = (int64_t)threadIdx.x * C, i1 = min(V, i0 + C);
  double loc = 0.0;
  int64_t lastpos = -1;
  for (int64_t i = i0; i < i1; i++) {
    const double wi = W.w(i);
    loc += wi;
    if (wi > 0.0) lastpos = i;
  }
  // exclusive scan of the chunk sums in thread order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  __syncthreads();
  if (lane == 31) s.scan[wid] = inc;
  if (threadIdx.x == 0) {
    s.pick = INT_MAX;
    s.last_pos = -1;
  }
  __syncthreads();
  double base = 0.0, total = 0.0;
  for (int w = 0; w < SV_THREADS / 32; w++) {
    if (w < wid) base += s.scan[w];
    total += s.scan[w];
  }
  const double excl = base + inc - loc;
  if (lastpos >= 0) atomicMax(&s.last_pos, (int)lastpos);
  if (!(total > 0.0)) {
    __syncthreads();
    return -1;
  }
  const double target = u * total;
  if (i0 < i1 && excl + loc > target) {  // this chunk may hold the crossing
    double run = excl;
    for (int64_t i = i0; i < i1; i++) {
      run += W.w(i);
      if (run > target) {
        atomicMin(&s.pick, (int)i);
        break;
      }
    }
  }
  __syncthreads();
  const int r = s.pick != INT_MAX ? s.pick : s.last_pos;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SV_THREADS) spec_verify_kernel(int K, int64_t V, const float* __restrict__ tgt,
                                                                 const float* __restrict__ draft_probs,
                                                                 const int32_t* __restrict__ draft_tok,
                                                                 const float* __restrict__ u_acc, float u_smp,
                                                                 int is_top, int top_k, float top_p,
                                                                 int32_t* __restrict__ out_tok,
                                                                 int32_t* __restrict__ n_out) {
  __shared__ SvShared s;
  int bad = 0;  // every draft token is checked before any decision (as the oracle does)
  for (int t = threadIdx.x; t < K; t += SV_THREADS) bad |= (draft_tok[t] < 0 || draft_tok[t] >= V);
  if (sv_count(bad, s)) {
    if (threadIdx.x == 0) *n_out = -IF_ERR_ARG;
    return;
  }
  int n = 0;
  for (int t = 0; t <= K; t++) {
    const float* l = tgt + (int64_t)t * V;
    float m = -INFINITY;
    for (int64_t i = threadIdx.x; i < V; i += SV_THREADS) m = fmaxf(m, l[i]);
    m = sv_max(m, s);
    double e = 0.0;
    for (int64_t i = threadIdx.x; i < V; i += SV_THREADS) e += exp((double)l[i] - (double)m);
    const double sum = sv_sum(e, s);
    SvWeights W{l, draft_probs + (int64_t)t * V, m, 1.0 / sum, false};
    if (t == K) {  // all K accepted: one extra token from the target at position K
      const int y = sv_sample(W, V, (double)u_smp, s);
      if (threadIdx.x == 0) {
        out_tok[n] = y;
        *n_out = n + 1;
      }
      return;
    }
    const int x = draft_tok[t];
    const double qx = W.q(x);
    const double px = (double)W.p[x];
    double ratio = px > 0.0 ? qx / px : 1.0;
    if (ratio > 1.0) ratio = 1.0;
    bool pool = false;
    if (is_top) {
      int more = 0;
      double mass = 0.0;
      for (int64_t i = threadIdx.x; i < V; i += SV_THREADS) {
        const double qi = W.q(i);
        if (qi > qx) {
          more++;
          mass += qi;
        }
      }
      more = sv_count(more, s);
      mass = sv_sum(mass, s);
      pool = !(top_k > 0 && more >= top_k) && !(top_p < 1.f && mass >= (double)top_p) && (top_k > 0 || top_p < 1.f);
    }
    if (pool || (double)u_acc[t] < ratio) {  // x_{n+t} <- draft, n <- n+1
      if (threadIdx.x == 0) out_tok[n] = x;
      n++;
      continue;
    }
    // reject: sample x_{n+t} ~ (q - p)_+ and exit the loop
    W.residual = true;
    int y = sv_sample(W, V, (double)u_smp, s);
    if (y < 0) {
      W.residual = false;
      y = sv_sample(W, V, (double)u_smp, s);
    }
    if (threadIdx.x == 0) {
      out_tok[n] = y;
      *n_out = n + 1;
    }
    return;
  }
}

}  // namespace ifb

using namespace ifb;

extern "C" if_status if_embed(const float* table, int32_t V, int32_t d, const int32_t* tokens, int64_t T, float* h,
                              int32_t* dev_status, if_stream_t stream) {
  if (V < 1 || d < 4 || d % 4 || T < 0 || T > (1 << 30)) return set_error(IF_ERR_SHAPE, "if_embed: V=%d d=%d T=%lld", V, d, (long long)T);
  if (T == 0) return IF_OK;
  if (!table || !tokens || !h) return set_error(IF_ERR_ARG, "if_embed: null pointer");
  if ((reinterpret_cast<uintptr_t>(table) | reinterpret_cast<uintptr_t>(h)) & 15u)
    return set_error(IF_ERR_ARG, "if_embed: table and h must be 16-byte aligned");
  embed_kernel<<<(unsigned)T, 256, 0, (cudaStream_t)stream>>>(table, V, d, tokens, h, dev_status);
  count_launch();
  return check_launch("if_embed");
}

extern "C" if_status if_lm_logits(if_scheme s, const uint8_t* lm, int64_t V, int64_t d, const float* h, int64_t T,
                                  const int32_t* rows, float* logits, float* scratch, if_stream_t stream) {
  if (!scheme_ok(s)) return set_error(IF_ERR_SCHEME, "if_lm_logits: invalid scheme");
  if (V < 1 || d < 1 || d % s.block || T < 1 || T > 64)
    return set_error(IF_ERR_SHAPE, "if_lm_logits: V=%lld d=%lld T=%lld", (long long)V, (long long)d, (long long)T);
  if (!lm || !h || !logits || !scratch) return set_error(IF_ERR_ARG, "if_lm_logits: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  lm_rmsnorm_kernel<<<(unsigned)T, 256, 0, st>>>(h, rows, (int)d, scratch);
  count_launch();
  if_status r = check_launch("if_lm_logits");
  if (r) return r;
  return qgemv_dispatch("if_lm_logits", s, lm, V, d, scratch, T, logits, 0, st, nullptr, 0, 0);
}

extern "C" if_status if_argmax(const float* logits, int64_t T, int64_t V, int32_t* tokens, if_stream_t stream) {
  if (T < 0 || V < 1) return set_error(IF_ERR_SHAPE, "if_argmax: T=%lld V=%lld", (long long)T, (long long)V);
  if (T == 0) return IF_OK;
  if (!logits || !tokens) return set_error(IF_ERR_ARG, "if_argmax: null pointer");
  argmax_kernel<<<(unsigned)T, 512, 0, (cudaStream_t)stream>>>(logits, V, tokens);
  count_launch();
  return check_launch("if_argmax");
}

extern "C" if_status if_spec_verify(int32_t K, int64_t V, const float* tgt_logits, const float* draft_probs,
                                    const int32_t* draft_tok, const float* u_acc, float u_smp, int32_t is_top,
                                    int32_t top_k, float top_p, int32_t* out_tok, int32_t* n_out,
                                    if_stream_t stream) {
  if (K < 0 || K > 64 || V < 1 || V > INT32_MAX)
    return set_error(IF_ERR_SHAPE, "if_spec_verify: K=%d V=%lld", K, (long long)V);
  if (!tgt_logits || !out_tok || !n_out || (K > 0 && (!draft_probs || !draft_tok || !u_acc)))
    return set_error(IF_ERR_ARG, "if_spec_verify: null pointer");
  if (!(u_smp >= 0.f && u_smp < 1.f)) return set_error(IF_ERR_ARG, "if_spec_verify: u_smp outside [0, 1)");
  spec_verify_kernel<<<1, SV_THREADS, 0, (cudaStream_t)stream>>>(K, V, tgt_logits, draft_probs, draft_tok, u_acc,
                                                                 u_smp, is_top, top_k, top_p, out_tok, n_out);
  count_launch();
  return check_launch("if_spec_verify");
}
