// stack.cu — the Llama-shaped linear stack on one rank (Q18) and its
// glue (a6): RMSNorm (eps 1e-5, unit gain), single-position GQA
// attention (softmax over one key = the v row of head i's kv group
// floor(i/(H/G)), contiguous groups S:393), SiLU(g)*u,
// residual adds; plus the TP merges and pipeline hand-off (a7/a8)
// through comm.cu.
#include <cuda_bf16.h>

#include <algorithm>
#include <vector>

#include "attn.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "decode_mk.cuh"
#include "qgemm.cuh"

namespace ifb {
extern unsigned long long* g_mk_dbg;

template <typename T>
__device__ __forceinline__ T to_out(float v);
template <>
__device__ __forceinline__ float to_out<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float v) {
  return __float2bfloat16(v);
}

// optional fp16 hi/lo split of a glue kernel's output for the tensor-core qGEMV that
// reads it (x2 [2 bp, K]: row t = hi, row bp + t = lo, of x_t * 2^k_t; sc[t] = 2^-k_t,
// common.cuh xsplit_k), so no separate split launch.  The x2 variants run one CTA per
// token row: the row's max |x| fixes its scale before any element is split.
__device__ __forceinline__ void put_x2(__half* x2, int bp, int64_t K, int64_t t, int64_t k, float v) {
  const __half h = __float2half_rn(v);
  x2[t * K + k] = h;
  x2[((int64_t)bp + t) * K + k] = __float2half_rn(v - __half2float(h));
}

// ---- x2 glue of the batched decode chain: one CTA of 1024 threads per token row, the
// row held in registers (<= 32 values per thread: rows up to 32768), so every global
// load of the row is in flight at once (a strided loop that stores between its loads
// pays one global latency per element: 13-32 us per launch in round 1's chain).
constexpr int GX_THREADS = 1024, GX_VMAX = 32;

__device__ __forceinline__ float gx_block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < GX_THREADS / 32; w++) t += red[w];
  return t;
}
__device__ __forceinline__ float gx_block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < GX_THREADS / 32; w++) t = fmaxf(t, red[w]);
  return t;
}
// the split of the row (values v[], count n) with its per-token scale, plus the fp32 row
__device__ __forceinline__ void gx_store_split(const float (&v)[GX_VMAX], int n, int t, int bp, float mx, float* out,
                                               __half* x2, float* sc) {
  const int k = xsplit_k(mx);
  const float mul = pow2f(k);
  if (threadIdx.x == 0) sc[t] = pow2f(-k);
#pragma unroll
  for (int i = 0; i < GX_VMAX; i++) {
    const int e = threadIdx.x + i * GX_THREADS;
    if (e < n) {
      if (out) out[(int64_t)t * n + e] = v[i];
      put_x2(x2, bp, n, t, e, v[i] * mul);
    }
  }
}
__device__ __forceinline__ void gx_pad_row(int n, int t, int bp, __half* x2, float* sc) {
  for (int e = threadIdx.x; e < n; e += GX_THREADS) put_x2(x2, bp, n, t, e, 0.f);
  if (threadIdx.x == 0) sc[t] = 1.f;
}

// a[t] = rms(h[t]) and its split; zeroes zbuf[zn] (the next qGEMV accumulates)
__global__ void __launch_bounds__(GX_THREADS) rmsnorm_x2_kernel(const float* __restrict__ h, float* __restrict__ a, int d,
                                                                float* __restrict__ zbuf, int64_t zn,
                                                                __half* __restrict__ x2, int T, int bp,
                                                                float* __restrict__ sc) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[GX_THREADS / 32];
  for (int64_t i = (int64_t)blockIdx.x * GX_THREADS + threadIdx.x; i < zn; i += (int64_t)gridDim.x * GX_THREADS)
    zbuf[i] = 0.f;
  const int t = blockIdx.x;
  if (t >= T) return gx_pad_row(d, t, bp, x2, sc);
  const float* hr = h + (int64_t)t * d;
  float v[GX_VMAX];
  float ss = 0.f, mx = 0.f;
#pragma unroll
  for (int i = 0; i < GX_VMAX; i++) {
    const int e = threadIdx.x + i * GX_THREADS;
    v[i] = e < d ? hr[e] : 0.f;
    ss = fmaf(v[i], v[i], ss);
    mx = fmaxf(mx, fabsf(v[i]));
  }
  const float inv = 1.0f / sqrtf(gx_block_sum(ss, red) / (float)d + 1e-5f);
  mx = gx_block_max(mx, red) * inv;
#pragma unroll
  for (int i = 0; i < GX_VMAX; i++) v[i] *= inv;
  gx_store_split(v, d, t, bp, mx, a, x2, sc);
}

// ctx[t, i hd + e] = v[t, j hd + e], j = floor((h0 + i)/(H/G)) - k0, and its split
__global__ void __launch_bounds__(GX_THREADS) vbcast_x2_kernel(const float* __restrict__ qkv, float* __restrict__ ctx,
                                                               int T, int lh, int lkv, int hd, int h0, int k0, int per,
                                                               __half* __restrict__ x2, int bp,
                                                               float* __restrict__ sc) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[GX_THREADS / 32];
  const int t = blockIdx.x;
  const int nq = lh * hd, nqkv = (lh + 2 * lkv) * hd;
  if (t >= T) return gx_pad_row(nq, t, bp, x2, sc);
  const float* vr = qkv + (int64_t)t * nqkv + (int64_t)(lh + lkv) * hd;
  float v[GX_VMAX];
  float mx = 0.f;
#pragma unroll
  for (int i = 0; i < GX_VMAX; i++) {
    const int r = threadIdx.x + i * GX_THREADS;
    v[i] = 0.f;
    if (r < nq) {
      const int hi = r / hd, e = r - hi * hd;
      v[i] = vr[(int64_t)((h0 + hi) / per - k0) * hd + e];
      mx = fmaxf(mx, fabsf(v[i]));
    }
  }
  gx_store_split(v, nq, t, bp, gx_block_max(mx, red), ctx, x2, sc);
}

// act[t, f] = silu(g) u (gate/up rows interleaved: g = gu[t, 2f], u = gu[t, 2f+1]) and its split
__global__ void __launch_bounds__(GX_THREADS) silu_mul_x2_kernel(const float* __restrict__ gu, float* __restrict__ act,
                                                                 int T, int lf, __half* __restrict__ x2, int bp,
                                                                 float* __restrict__ sc) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[GX_THREADS / 32];
  const int t = blockIdx.x;
  if (t >= T) return gx_pad_row(lf, t, bp, x2, sc);
  const float2* gr = reinterpret_cast<const float2*>(gu + (int64_t)t * 2 * lf);
  float v[GX_VMAX];
  float mx = 0.f;
#pragma unroll
  for (int i = 0; i < GX_VMAX; i++) {
    const int f = threadIdx.x + i * GX_THREADS;
    v[i] = 0.f;
    if (f < lf) {
      const float2 p = gr[f];
      v[i] = p.x / (1.0f + expf(-p.x)) * p.y;
      mx = fmaxf(mx, fabsf(v[i]));
    }
  }
  gx_store_split(v, lf, t, bp, gx_block_max(mx, red), act, x2, sc);
}

// a[t] = h[t] / sqrt(mean(h[t]^2) + 1e-5)
// (zbuf, zn: optionally zero the next qGEMV's output, which then accumulates --
//  no memset node, so the chain stays programmatic)
template <typename OutT>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ h, OutT* __restrict__ a, int d,
                                                      float* __restrict__ zbuf = nullptr, int64_t zn = 0) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < zn; i += (int64_t)gridDim.x * blockDim.x)
    zbuf[i] = 0.f;
  __shared__ float red[8];
  const float* hr = h + (int64_t)blockIdx.x * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(hr[i], hr[i], ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) tot += red[w];
  const float inv = 1.0f / sqrtf(tot / (float)d + 1e-5f);
  OutT* ar = a + (int64_t)blockIdx.x * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ar[i] = to_out<OutT>(hr[i] * inv);
}

// ctx[t, i*hd + e] = v[t, j*hd + e],  j = floor((h0 + i)/(H/G)) - k0  (local heads/kv-heads)
template <typename OutT>
__global__ void vbcast_kernel(const float* __restrict__ qkv, OutT* __restrict__ ctx, int T, int lh, int lkv, int hd,
                              int h0, int k0, int per) {
  pdl_trigger();
  pdl_wait();
  const int64_t nq = (int64_t)lh * hd, nqkv = (int64_t)(lh + 2 * lkv) * hd;
  const int64_t total = (int64_t)T * nq;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / nq, r = idx - t * nq;
    const int i = (int)(r / hd), e = (int)(r - (int64_t)i * hd);
    const int j = (h0 + i) / per - k0;
    ctx[idx] = to_out<OutT>(qkv[t * nqkv + (int64_t)(lh + lkv) * hd + (int64_t)j * hd + e]);
  }
}

// act[t, f] = silu(g) * u with gate/up rows interleaved: g = gu[t, 2f], u = gu[t, 2f+1]
template <typename OutT>
__global__ void silu_mul_kernel(const float* __restrict__ gu, OutT* __restrict__ act, int T, int lf) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = (int64_t)T * lf;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / lf, f = idx - t * lf;
    const float g = gu[t * 2 * lf + 2 * f], u = gu[t * 2 * lf + 2 * f + 1];
    act[idx] = to_out<OutT>(g / (1.0f + expf(-g)) * u);
  }
}

// x2 variant, one CTA per token row: pass 1 the row max of silu(g) u, pass 2 the split
// launch with the programmatic-dependent-launch attribute (decode chain)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, (KArgs)args...);
}

static int ew_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  return (int)g;
}

struct Local {
  int lh, lkv, lf, nq, nqkv, d, hd, layers;
};

static if_status local_dims(const if_stack_shape* s, const if_plan* p, int rank, Local* L) {
  if (!s || !p) return set_error(IF_ERR_ARG, "stack: null shape/plan");
  if (!scheme_ok(s->scheme)) return set_error(IF_ERR_SCHEME, "stack: invalid scheme");
  if (rank < 0 || rank >= p->devices || p->devices > 8) return set_error(IF_ERR_ARG, "stack: rank %d", rank);
  if (s->hidden % 64 || (s->heads * s->head_dim) % 64 || s->ffn % 64 || s->kv_heads < 1 || s->heads % s->kv_heads)
    return set_error(IF_ERR_SHAPE, "stack: bad shape");
  const if_assignment& a = p->a[rank];
  if (a.head_begin < 0 || a.head_end > s->heads || a.kv_end > s->kv_heads || a.ffn_blk_end > s->ffn / 64 ||
      a.layer_end > s->layers || a.layer_begin < 0 || a.head_end <= a.head_begin || a.kv_end <= a.kv_begin ||
      a.ffn_blk_end <= a.ffn_blk_begin)
    return set_error(IF_ERR_PLAN, "stack: assignment of rank %d inconsistent with shape", rank);
  L->lh = a.head_end - a.head_begin;
  L->lkv = a.kv_end - a.kv_begin;
  L->lf = (a.ffn_blk_end - a.ffn_blk_begin) * 64;
  L->hd = s->head_dim;
  L->d = s->hidden;
  L->nq = L->lh * s->head_dim;
  L->nqkv = (L->lh + 2 * L->lkv) * s->head_dim;
  L->layers = a.layer_end - a.layer_begin;
  return IF_OK;
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct WS {
  float* a;
  float* qkv;
  float* ctx;
  float* gu;
  float* act;
  float* part;
  float* attn;  // KV-cache attention partials [min(T, ATT_MAXT)][lh][ATT_MAXSPLIT][hd + 2]
  uint32_t* acnt;  // attention merge counters (self-resetting; fixed offset)
  int* done;  // decode engine: phase counters [4 * MK_MAXL] + epoch
  float* xsimg;  // 3 transformed-input images + sum-h^2 partials (decode engine)
  void* x2;      // batched decode: fp16 hi/lo split of a qGEMV input (2 x 64 x maxK halves)
  void* msrec;   // fused batched chain (qgemv_ms.cu): fragment records + sum-h^2 partials
  size_t x2_bytes;
  size_t bytes;
};

// Workspace layout.  The decode engine's persistent state (phase counters, step
// epoch, parity-tagged input images) and the fp16 split buffer sit FIRST, at
// offsets that depend only on (shape, plan, rank) -- never on the call's T -- so
// one zero-filled workspace serves calls with any T <= max_tokens (ADVICE r1:
// a T-dependent carve let a later call with another T read stale images as its
// epoch).  The T-sized activation scratch follows.
static WS carve(void* base, const Local& L, int64_t T) {
  WS w;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t elems) {
    float* r = reinterpret_cast<float*>(p ? p + off : nullptr);
    off += al256(elems * 4);
    return r;
  };
  w.done = reinterpret_cast<int*>(take((size_t)4 * MK_MAXL + 32));
  // 3 images of 16 x xstride float4 (xstride <= nbp_max + 9) + 256 floats
  const size_t nbp_max = (size_t)((std::max(std::max(L.d, L.nq), L.lf) / 64 + 31) / 32) * 32;
  w.xsimg = take(3 * 16 * (nbp_max + 16) * 4 + 256);
  const size_t maxK = (size_t)std::max(std::max(L.d, L.nq), L.lf);
  w.x2 = take(64 * maxK + X2_SC_BYTES / 4);  // [64 per-token scales][2 x 64 x maxK fp16]
  w.x2_bytes = 64 * maxK * 4 + X2_SC_BYTES;
  w.acnt = reinterpret_cast<uint32_t*>(take(attn_cnt_words(L.lkv)));
  w.msrec = take(ms_chain_ws_bytes(L.d, L.nq, L.lf) / 4 + 1);
  w.a = take((size_t)T * L.d);
  w.qkv = take((size_t)T * L.nqkv);
  w.ctx = take((size_t)T * L.nq);
  w.gu = take((size_t)T * 2 * L.lf);
  w.act = take((size_t)T * L.lf);
  w.part = take((size_t)T * L.d);
  w.attn = take((size_t)std::min<int64_t>(T, ATT_MAXT) * L.lh * ATT_MAXSPLIT * (L.hd + 2));
  w.bytes = off;
  return w;
}

}  // namespace ifb

using namespace ifb;

extern "C" if_status if_stack_workspace_bytes(const if_stack_shape* shape, const if_plan* plan, int32_t rank,
                                              int64_t max_tokens, int32_t mode, size_t* bytes) {
  Local L;
  if_status st = local_dims(shape, plan, rank, &L);
  if (st) return st;
  if (!bytes) return set_error(IF_ERR_ARG, "if_stack_workspace_bytes: null");
  if (max_tokens < 1 || (mode == IF_DECODE && max_tokens > 64) || max_tokens > 4096)
    return set_error(IF_ERR_ARG, "if_stack_workspace_bytes: max_tokens=%lld", (long long)max_tokens);
  *bytes = carve(nullptr, L, max_tokens).bytes;
  return IF_OK;
}

struct KvRun;
static AttnArgs attn_args(const Local& L, const KvRun* kvr, const WS& w, int64_t T, int nlayers, int l);

struct KvRun {
  const if_kv_cache* kv;
  const int32_t* slot_ids;
  const int32_t* positions;
};

static if_status run_stack(const if_stack_shape* shape, const if_plan* plan, int32_t rank, if_comm comm,
                           const if_layer_weights* stage_layers, const float* h_in, int64_t T, int32_t mode,
                           float* h_out, float* last_qkv, void* workspace, if_stream_t stream, const KvRun* kvr) {
  Local L;
  if_status st = local_dims(shape, plan, rank, &L);
  if (st) return st;
  if (mode != IF_DECODE && mode != IF_PREFILL) return set_error(IF_ERR_ARG, "if_run_stack: mode %d", mode);
  if (T < 1 || (mode == IF_DECODE && T > 64) || T > 4096) return set_error(IF_ERR_ARG, "if_run_stack: T=%lld", (long long)T);
  if (!h_out || !workspace || !stage_layers) return set_error(IF_ERR_ARG, "if_run_stack: null pointer");
  const if_assignment& asg = plan->a[rank];
  const bool first = asg.stage == 0, last = asg.stage == plan->stages - 1;
  if (first && !h_in) return set_error(IF_ERR_ARG, "if_run_stack: null h_in on stage 0");
  if ((plan->devices > 1) && !comm) return set_error(IF_ERR_ARG, "if_run_stack: comm required for %d devices", plan->devices);
  const int groups = plan->groups;
  cudaStream_t cs = (cudaStream_t)stream;
  const if_scheme sc = shape->scheme;
  WS w = carve(workspace, L, T);
  const int64_t nh = T * (int64_t)L.d;
  const int per = shape->heads / shape->kv_heads;

  // stage input: h_in on stage 0, hand-off from stage-1 otherwise
  if (first) {
    if (h_out != h_in && cudaMemcpyAsync(h_out, h_in, nh * 4, cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
      return check_launch("if_run_stack: copy h_in");
  } else {
    if ((st = comm_recv(comm, h_out, nh, cs))) return st;
  }
  const int nlayers = asg.layer_end - asg.layer_begin;
  // batch-1 Q3H_B64 decode on one TP rank: the whole stage in ONE persistent launch
  // (batch 2..6: one engine launch per token beats the tensor-core path, whose
  //  per-launch cost dominates at small B; both stream the weights from HBM)
  // tensor parallelism: the engine merges the o / down partials itself over the
  // communicator's exchange regions (peer memory); NCCL communicators take the
  // per-layer path below
  float* tp_boxes[8] = {nullptr};
  int tp_n = 1, tp_me = 0, tp_hidden = 0, tp_grid = 0;
  const bool tp_ok = groups == 1 || (comm_engine(comm, tp_boxes, &tp_n, &tp_me, &tp_hidden, &tp_grid) && tp_hidden >= L.d);
  // batch sizes that run one engine launch per token: 3.5-bit from B = 2 takes the fused
  // batched chain instead (measured 7B: B = 2 934 tok/s vs 909 with the engine per token,
  // B = 3 1396); the k-bit schemes up to B = 6 (their batched path is tcgen05)
  static const char* tenv = getenv("IFB_MK_TMAX");  // experiments only
  const int mk_tmax = tenv ? atoi(tenv) : (sc.type == IF_Q3H && sc.block == 64 ? 1 : 6);
  // with a KV cache (NEXT-1) the 3.5-bit engine runs in partial launches per token:
  // [qkv_0] attn_0 [o_0 gu_0 down_0 qkv_1] attn_1 ... [o_L-1 gu down] (one rank)
  const bool mk_kv = kvr && T <= (getenv("IFB_NO_MSCHAIN_KV") ? 2 : 1) && sc.type == IF_Q3H && sc.block == 64 && groups == 1 && !getenv("IFB_NO_MK_KV");
  const bool mk = mode == IF_DECODE && T <= mk_tmax && !(sc.type == IF_Q3H && sc.block == 32) && tp_ok &&
                  nlayers <= MK_MAXL && nlayers > 0 && (!kvr || mk_kv);
  if (mk) {
    static thread_local MkParams P;
    P.mode = MK_MODE_STACK;
    P.qt = sc.type;
    P.bs = sc.block;
    P.layers = nlayers;
    P.d = L.d;
    P.nq = L.nq;
    P.nqkv = L.nqkv;
    P.lf = L.lf;
    P.hd = L.hd;
    P.lh = L.lh;
    P.lkv = L.lkv;
    P.h0 = asg.head_begin;
    P.k0 = asg.kv_begin;
    P.per = per;
    P.h = h_out;
    P.qkv = w.qkv;
    P.act = w.act;
    P.last_qkv = last_qkv;
    P.done = w.done;
    P.epoch = reinterpret_cast<uint32_t*>(w.done + 4 * MK_MAXL);
    {
      const int nbp_max = ((std::max(std::max(L.d, L.nq), L.lf) / 64 + 31) / 32) * 32;
      const size_t img = (size_t)16 * (nbp_max + 16);
      P.xs_h = reinterpret_cast<float4*>(w.xsimg);
      P.xs_ctx = P.xs_h + img;
      P.xs_act = P.xs_ctx + img;
      P.ssq = reinterpret_cast<float*>(P.xs_act + img);
    }
    P.dbg = g_mk_dbg;
    P.tp = groups > 1 ? tp_n : 1;
    P.tp_me = tp_me;
    P.tp_hidden = tp_hidden;
    for (int q = 0; q < 8; q++) P.tp_box[q] = tp_boxes[q];
    P.grid = comm ? tp_grid : 0;
    for (int l = 0; l < nlayers; l++) {
      const if_layer_weights& Wl = stage_layers[l];
      if (!Wl.wqkv || !Wl.wo || !Wl.wgu || !Wl.wdown) return set_error(IF_ERR_ARG, "if_run_stack: null weights, layer %d", l);
      P.w[l][0] = Wl.wqkv;
      P.w[l][1] = Wl.wo;
      P.w[l][2] = Wl.wgu;
      P.w[l][3] = Wl.wdown;
    }
    P.part = 0;
    P.x_first = nullptr;
    P.qkv_out = nullptr;
    for (int64_t t = 0; t < T && !st; t++) {
      P.h = h_out + t * L.d;
      P.last_qkv = last_qkv ? last_qkv + t * L.nqkv : nullptr;
      if (!kvr) {
        st = mk_launch(P, cs);
        continue;
      }
      // KV attention between each layer's qkv and o phases (attn.cu on this token)
      P.part = 1;
      P.last_qkv = nullptr;  // q, k are returned after RoPE: copied after the last attention
      P.x_first = w.ctx;
      P.qkv_out = w.qkv;
      for (int k = 0; k <= nlayers && !st; k++) {
        P.p_begin = k == 0 ? 0 : 4 * (k - 1) + 1;
        P.p_end = k == nlayers ? 4 * nlayers : 4 * k + 1;
        st = mk_launch(P, cs);
        if (st || k == nlayers) break;
        KvRun one = *kvr;
        one.slot_ids = kvr->slot_ids + t;
        one.positions = kvr->positions + t;
        AttnArgs aa = attn_args(L, &one, w, 1, nlayers, k);
        aa.ctx = w.ctx;
        aa.rot_out = (k == nlayers - 1 && last_qkv) ? last_qkv + t * L.nqkv : nullptr;  // q, k after RoPE
        st = attn_run(aa, cs);
      }
    }
    if (st != IF_ERR_UNSUPPORTED) {
      if (st) return st;
      if (!last) {
        if ((st = comm_send(comm, h_out, nh, cs))) return st;
      }
      return check_launch("if_run_stack");
    }
  }
  // batched 3.5-bit decode (T <= 16, one TP rank): the fused chain, 4 launches per layer
  // with the glue in the GEMV epilogues (qgemv_ms.cu)
  if (mode == IF_DECODE && T >= 2 && groups == 1 && sc.type == IF_Q3H && sc.block == 64 && nlayers > 0 &&
      (!kvr || !getenv("IFB_NO_MSCHAIN_KV"))) {
    std::vector<MsChainLayer> ml((size_t)nlayers);
    for (int l = 0; l < nlayers; l++) {
      const if_layer_weights& Wl = stage_layers[l];
      if (!Wl.wqkv || !Wl.wo || !Wl.wgu || !Wl.wdown) return set_error(IF_ERR_ARG, "if_run_stack: null weights, layer %d", l);
      ml[(size_t)l] = {Wl.wqkv, Wl.wo, Wl.wgu, Wl.wdown};
    }
    // with a KV cache: attention between each layer's qkv and o kernels; its merge
    // writes the ctx records; q, k are returned after RoPE (copied after the last layer)
    struct KvChain {
      const Local* L;
      const KvRun* kvr;
      const WS* w;
      int64_t T;
      int nlayers;
      float* last_qkv;
      cudaStream_t cs;
    } kc = {&L, kvr, &w, T, nlayers, last_qkv, cs};
    MsAttnFn fn = nullptr;
    if (kvr)
      fn = [](void* p, int l, uint8_t* rec, int nt) -> if_status {
        const KvChain& k = *static_cast<const KvChain*>(p);
        AttnArgs aa = attn_args(*k.L, k.kvr, *k.w, k.T, k.nlayers, l);
        aa.ctx = k.w->ctx;
        aa.rec = rec;
        aa.rec_nt = nt;
        aa.pdl = true;
        aa.rot_out = (l == k.nlayers - 1) ? k.last_qkv : nullptr;  // q, k after RoPE
        return attn_run(aa, k.cs);
      };
    st = ms_chain_run(ml.data(), nlayers, L.d, L.lh, L.lkv, L.hd, L.lf, per, T, h_out, last_qkv, w.msrec, cs, fn, &kc, w.qkv);
    if (st != IF_ERR_UNSUPPORTED) {
      if (st) return st;
      if (!last) {
        if ((st = comm_send(comm, h_out, nh, cs))) return st;
      }
      return check_launch("if_run_stack");
    }
  }
  // batched decode (2 <= T <= 64): the glue kernels also write the fp16 hi/lo split of
  // the next qGEMV's input into the workspace (x2r: no separate split launch)
  const bool use_x2 = mode == IF_DECODE && T >= 2;
  __half* x2h = use_x2 ? reinterpret_cast<__half*>(reinterpret_cast<char*>(w.x2) + X2_SC_BYTES) : nullptr;
  float* x2s = use_x2 ? reinterpret_cast<float*>(w.x2) : nullptr;
  const int bpx = use_x2 ? tc_bpad((int)T) : 0;
  const int x2r = use_x2 ? 1 : 0;
  for (int l = 0; l < nlayers; l++) {
    const if_layer_weights& Wl = stage_layers[l];
    if (!Wl.wqkv || !Wl.wo || !Wl.wgu || !Wl.wdown) return set_error(IF_ERR_ARG, "if_run_stack: null weights, layer %d", l);
    if (mode == IF_DECODE) {
      // ---- attention sub-layer ----
      if (use_x2)
        launch_pdl(rmsnorm_x2_kernel, (unsigned)bpx, GX_THREADS, cs, (const float*)h_out, w.a, (int)L.d, w.qkv,
                   (int64_t)T * L.nqkv, x2h, (int)T, bpx, x2s);
      else
        launch_pdl(rmsnorm_kernel<float>, (unsigned)T, 256, cs, (const float*)h_out, w.a, (int)L.d, w.qkv,
                   (int64_t)T * L.nqkv);
      count_launch();
      if ((st = qgemv_dispatch("if_run_stack(qkv)", sc, Wl.wqkv, L.nqkv, L.d, w.a, T, w.qkv, 1, cs, w.x2, w.x2_bytes, x2r)))
        return st;
      if (kvr) {
        // GQA attention over the KV cache (attn.cu, NEXT-1): RoPE + append, split
        // partials, combine -> ctx (and its fp16 split for the batched qGEMV)
        AttnArgs aa = attn_args(L, kvr, w, T, nlayers, l);
        aa.rot_out = (l == nlayers - 1) ? last_qkv : nullptr;  // q, k after RoPE
        aa.ctx = w.ctx;
        aa.x2 = x2h;
        aa.bp = bpx;
        aa.x2sc = x2s;
        aa.pdl = true;
        if ((st = attn_run(aa, cs))) return st;
      } else if (use_x2)
        launch_pdl(vbcast_x2_kernel, (unsigned)bpx, GX_THREADS, cs, (const float*)w.qkv, w.ctx, (int)T, (int)L.lh, (int)L.lkv,
                   (int)L.hd, (int)asg.head_begin, (int)asg.kv_begin, (int)per, x2h, bpx, x2s);
      else
        launch_pdl(vbcast_kernel<float>, (unsigned)ew_grid(T * L.nq), 256, cs, (const float*)w.qkv, w.ctx, (int)T,
                   (int)L.lh, (int)L.lkv, (int)L.hd, (int)asg.head_begin, (int)asg.kv_begin, (int)per);
      count_launch();
      if (groups == 1) {
        if ((st = qgemv_dispatch("if_run_stack(o)", sc, Wl.wo, L.d, L.nq, w.ctx, T, h_out, 1, cs, w.x2, w.x2_bytes, x2r)))
          return st;
      } else {
        if ((st = qgemv_dispatch("if_run_stack(o)", sc, Wl.wo, L.d, L.nq, w.ctx, T, w.part, 0, cs, w.x2, w.x2_bytes, x2r)))
          return st;
        if ((st = comm_allreduce_into(comm, w.part, h_out, nh, 1, cs))) return st;  // merge #1
      }
      // ---- feed-forward sub-layer ----
      if (use_x2)
        launch_pdl(rmsnorm_x2_kernel, (unsigned)bpx, GX_THREADS, cs, (const float*)h_out, w.a, (int)L.d, w.gu,
                   (int64_t)T * 2 * L.lf, x2h, (int)T, bpx, x2s);
      else
        launch_pdl(rmsnorm_kernel<float>, (unsigned)T, 256, cs, (const float*)h_out, w.a, (int)L.d, w.gu,
                   (int64_t)T * 2 * L.lf);
      count_launch();
      if ((st = qgemv_dispatch("if_run_stack(gu)", sc, Wl.wgu, 2 * L.lf, L.d, w.a, T, w.gu, 1, cs, w.x2, w.x2_bytes, x2r)))
        return st;
      if (use_x2)
        launch_pdl(silu_mul_x2_kernel, (unsigned)bpx, GX_THREADS, cs, (const float*)w.gu, w.act, (int)T, (int)L.lf, x2h, bpx,
                   x2s);
      else
        launch_pdl(silu_mul_kernel<float>, (unsigned)ew_grid(T * L.lf), 256, cs, (const float*)w.gu, w.act, (int)T,
                   (int)L.lf);
      count_launch();
      if (groups == 1) {
        if ((st = qgemv_dispatch("if_run_stack(down)", sc, Wl.wdown, L.d, L.lf, w.act, T, h_out, 1, cs, w.x2, w.x2_bytes, x2r)))
          return st;
      } else {
        if ((st = qgemv_dispatch("if_run_stack(down)", sc, Wl.wdown, L.d, L.lf, w.act, T, w.part, 0, cs, w.x2, w.x2_bytes, x2r)))
          return st;
        if ((st = comm_allreduce_into(comm, w.part, h_out, nh, 1, cs))) return st;  // merge #2
      }
    } else {
      __nv_bfloat16* a16 = reinterpret_cast<__nv_bfloat16*>(w.a);
      __nv_bfloat16* c16 = reinterpret_cast<__nv_bfloat16*>(w.ctx);
      __nv_bfloat16* f16 = reinterpret_cast<__nv_bfloat16*>(w.act);
      rmsnorm_kernel<__nv_bfloat16><<<(unsigned)T, 256, 0, cs>>>(h_out, a16, L.d);
      count_launch();
      if ((st = qgemm_impl("if_run_stack(qkv)", sc, Wl.wqkv, L.nqkv, L.d, reinterpret_cast<uint16_t*>(a16), T, w.qkv, 0, cs)))
        return st;
      if (kvr) {  // causal attention of the chunk over the cache (all tokens append first)
        AttnArgs aa = attn_args(L, kvr, w, T, nlayers, l);
        aa.rot_out = (l == nlayers - 1) ? last_qkv : nullptr;  // q, k after RoPE
        aa.ctx16 = c16;
        if ((st = attn_run(aa, cs))) return st;
      } else {
        vbcast_kernel<__nv_bfloat16><<<ew_grid(T * L.nq), 256, 0, cs>>>(w.qkv, c16, (int)T, L.lh, L.lkv, L.hd,
                                                                       asg.head_begin, asg.kv_begin, per);
        count_launch();
      }
      if (groups == 1) {
        if ((st = qgemm_impl("if_run_stack(o)", sc, Wl.wo, L.d, L.nq, reinterpret_cast<uint16_t*>(c16), T, h_out, 1, cs)))
          return st;
      } else {
        if ((st = qgemm_impl("if_run_stack(o)", sc, Wl.wo, L.d, L.nq, reinterpret_cast<uint16_t*>(c16), T, w.part, 0, cs)))
          return st;
        if ((st = comm_allreduce_into(comm, w.part, h_out, nh, 1, cs))) return st;
      }
      rmsnorm_kernel<__nv_bfloat16><<<(unsigned)T, 256, 0, cs>>>(h_out, a16, L.d);
      count_launch();
      if ((st = qgemm_impl("if_run_stack(gu)", sc, Wl.wgu, 2 * L.lf, L.d, reinterpret_cast<uint16_t*>(a16), T, w.gu, 0, cs)))
        return st;
      silu_mul_kernel<__nv_bfloat16><<<ew_grid(T * L.lf), 256, 0, cs>>>(w.gu, f16, (int)T, L.lf);
      count_launch();
      if (groups == 1) {
        if ((st = qgemm_impl("if_run_stack(down)", sc, Wl.wdown, L.d, L.lf, reinterpret_cast<uint16_t*>(f16), T, h_out, 1, cs)))
          return st;
      } else {
        if ((st = qgemm_impl("if_run_stack(down)", sc, Wl.wdown, L.d, L.lf, reinterpret_cast<uint16_t*>(f16), T, w.part, 0, cs)))
          return st;
        if ((st = comm_allreduce_into(comm, w.part, h_out, nh, 1, cs))) return st;
      }
    }
    if (l == nlayers - 1 && last_qkv && !kvr) {  // (with a cache, the attention returns q, k after RoPE)
      if (cudaMemcpyAsync(last_qkv, w.qkv, (size_t)T * L.nqkv * 4, cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
        return check_launch("if_run_stack: last_qkv");
    }
  }
  if (!last) {
    if ((st = comm_send(comm, h_out, nh, cs))) return st;
  }
  return check_launch("if_run_stack");
}

static AttnArgs attn_args(const Local& L, const KvRun* kvr, const WS& w, int64_t T, int nlayers, int l) {
  (void)nlayers;
  AttnArgs a = {};
  a.qkv = w.qkv;
  a.T = T;
  a.lh = L.lh;
  a.lkv = L.lkv;
  a.hd = L.hd;
  a.slot_ids = kvr->slot_ids;
  a.positions = kvr->positions;
  a.k = kvr->kv->k;
  a.v = kvr->kv->v;
  a.slots = kvr->kv->slots;
  a.max_ctx = kvr->kv->max_ctx;
  a.layer = l;
  a.status = kvr->kv->status;
  a.part = w.attn;
  a.cnt = w.acnt;
  return a;
}

extern "C" if_status if_run_stack(const if_stack_shape* shape, const if_plan* plan, int32_t rank, if_comm comm,
                                  const if_layer_weights* stage_layers, const float* h_in, int64_t T, int32_t mode,
                                  float* h_out, float* last_qkv, void* workspace, if_stream_t stream) {
  return run_stack(shape, plan, rank, comm, stage_layers, h_in, T, mode, h_out, last_qkv, workspace, stream, nullptr);
}

extern "C" if_status if_kv_cache_bytes(const if_stack_shape* shape, const if_plan* plan, int32_t rank, int32_t slots,
                                       int32_t max_ctx, size_t* bytes_each) {
  Local L;
  if_status st = local_dims(shape, plan, rank, &L);
  if (st) return st;
  if (!bytes_each || slots < 1 || max_ctx < 1) return set_error(IF_ERR_ARG, "if_kv_cache_bytes: slots/max_ctx/null");
  *bytes_each = (size_t)L.layers * slots * max_ctx * L.lkv * L.hd * sizeof(float);
  return IF_OK;
}

extern "C" if_status if_run_stack_kv(const if_stack_shape* shape, const if_plan* plan, int32_t rank, if_comm comm,
                                     const if_layer_weights* stage_layers, const float* h_in, int64_t T, int32_t mode,
                                     float* h_out, float* last_qkv, const if_kv_cache* kv, const int32_t* slot_ids,
                                     const int32_t* positions, void* workspace, if_stream_t stream) {
  if (!kv || !kv->k || !kv->v || !slot_ids || !positions || kv->slots < 1 || kv->max_ctx < 1)
    return set_error(IF_ERR_ARG, "if_run_stack_kv: null cache / slot ids / positions");
  if (shape && shape->head_dim % 2) return set_error(IF_ERR_SHAPE, "if_run_stack_kv: RoPE needs an even head_dim");
  const KvRun kvr = {kv, slot_ids, positions};
  return run_stack(shape, plan, rank, comm, stage_layers, h_in, T, mode, h_out, last_qkv, workspace, stream, &kvr);
}
