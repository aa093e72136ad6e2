/*
 * if_b200.h — C ABI of the B200-native block-quantized GEMV/GEMM library for
 * Inferflow's hot path (arxiv 2401.08294).
 *
 * Citations: "P:n" = line n of PAPER.md (the Inferflow report); "S:n" = line n
 * of SPEC.md; "Qn" = reading n in DESIGN.md §Readings.
 *
 * Conventions for every entry point
 *  - Pointers named W, x, y, X, Y, packed, h_*, workspace are DEVICE pointers
 *    (cudaMalloc / torch CUDA tensors) unless stated otherwise.  The library owns
 *    no tensor memory and never allocates on the hot path; the only internal
 *    state is inside an if_comm.
 *  - Calls are stream-ordered and asynchronous on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  No entry point synchronises except
 *    if_comm_* set-up calls.  All compute entry points are CUDA-graph capturable.
 *  - Host-detectable errors (argument, shape, scheme, plan, grid) return
 *    immediately and launch nothing.  Data-dependent errors are written to an
 *    optional device int32 `dev_status` (0 = OK; the first error wins), which
 *    the caller reads after synchronising.  Launch failures return IF_ERR_CUDA.
 *    if_last_error() returns a thread-local message for the last non-OK status.
 *  - Packed tensors: W is [N, K] row-major with quantization blocks running
 *    along K (the reduction dimension; Q9).  Block (n, b) covers
 *    W[n, b*block .. (b+1)*block) and is stored at byte offset
 *    (n*(K/block) + b) * if_block_bytes(s) as
 *        [lo fp16 LE][hi fp16 LE][codes, tightly bit-packed LSB-first]
 *    (two FP16 numbers per block P:191; Q2/Q11/Q12).  K % block == 0.
 */
#ifndef IF_B200_H
#define IF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* if_stream_t; /* identical to cudaStream_t */

typedef enum {
  IF_OK = 0,
  IF_ERR_ARG = 1,     /* null pointer, bad enum, bad batch, misaligned pointer       */
  IF_ERR_SHAPE = 2,   /* K % block != 0, negative or inconsistent sizes              */
  IF_ERR_SCHEME = 3,  /* qtype/block outside Table 3's family      */
  IF_ERR_INPUT = 4,   /* (device) non-finite weight or |w| beyond fp16 range (Q8)    */
  IF_ERR_DECODE = 5,  /* (device) Q3H pair code > 120 (Q14)              */
  IF_ERR_PLAN = 6,    /* indivisible heads/kv-heads/FFN, layers < stages     */
  IF_ERR_GRID = 7,    /* devices != stages x groups                          */
  IF_ERR_CUDA = 8,    /* CUDA launch / runtime failure                               */
  IF_ERR_COMM = 9,    /* communicator failure (peer memory or NCCL; SURVEY's IF_ERR_NCCL) */
  IF_ERR_UNSUPPORTED = 10,
  IF_ERR_IO = 11      /* container file: cannot open/read/write, malformed, truncated */
} if_status;

/* Schemes ("2, 3, 4, 5, 6, and 8" bits plus 3.5-bit Q3H). */
typedef enum { IF_Q2 = 2, IF_Q3 = 3, IF_Q3H = 35, IF_Q4 = 4, IF_Q5 = 5, IF_Q6 = 6, IF_Q8 = 8 } if_qtype;

/* block in {32, 64} for every type (Table 3 defaults). */
typedef struct {
  int32_t type;  /* if_qtype */
  int32_t block; /* weights per block */
} if_scheme;

/* ---------------------------------------------------------------------------
 * Sizes (host only, no device work)
 * ------------------------------------------------------------------------- */

/* Bytes of one block: 4 (two fp16) + ceil(block*bits/8).
 * Returns -1 for an invalid scheme. */
int64_t if_block_bytes(if_scheme s);

/* N*(K/block)*if_block_bytes(s); -1 if the scheme is invalid, N<0, K<0 or K%block. */
int64_t if_packed_bytes(if_scheme s, int64_t N, int64_t K);

/* Actual bits per weight as a reduced fraction num/den = (block*bits + 32)/block
 * (Table 3).  IF_ERR_SCHEME for an invalid scheme. */
if_status if_bits_per_weight(if_scheme s, int64_t* num, int64_t* den);

/* ---------------------------------------------------------------------------
 * Synthetic inputs: out[i] = float(s(idx)) * scale with
 * idx = offset + i and the counter-based Irwin-Hall(4) generator of synth/.
 * Device out[n], fp32.  Not part of the method; used to fill HBM with weights
 * and activations without a host round trip.
 * ------------------------------------------------------------------------- */
if_status if_synth_fill(uint64_t seed, uint64_t tensor_id, float scale, float* out, int64_t n,
                        int64_t offset, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * a1 + a2: quantize (Eq. 1; 3.5-bit P:120-127; pair code P:124-127)
 * W       device fp32 [N, K] row-major, read only.
 * packed  device uint8 [if_packed_bytes(s, N, K)], written.
 * Per block: min/max (−0 -> +0), lo = fp16 round-down(min), hi = fp16
 * round-up(max) (Q3), q = roundf(((w - lo) / (hi - lo)) * D) in binary32 (Q1,
 * Q4), D = 2^k-1 or 10; Q3H codes v = q_{2i}*11 + q_{2i+1}.  Bit-exact with
 * the oracle.  Non-finite inputs or min/max beyond fp16 -> dev_status = 4 (the
 * block is still written with undefined content).
 * ------------------------------------------------------------------------- */
if_status if_quantize(if_scheme s, const float* W, int64_t N, int64_t K, uint8_t* packed,
                      int32_t* dev_status /* nullable */, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * a3: dequantize (Eq. 2; Q3H decode P:129-136)
 * packed  device uint8 [if_packed_bytes], W_out device fp32 [N, K].
 * w' = fma32(q, (hi - lo)/D, lo) (Q5).  Q3H codes > 120 -> dev_status = 5.
 * ------------------------------------------------------------------------- */
if_status if_dequantize(if_scheme s, const uint8_t* packed, int64_t N, int64_t K, float* W_out,
                        int32_t* dev_status /* nullable */, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * a4: decode GEMV with fused dequantization
 *   y[b, n] = sum_k W'[n, k] * x[b, k]       (fp32 accumulation)
 * W  device packed [N, K]; x device fp32 [B, K]; y device fp32 [B, N].
 * 1 <= B <= 64.  x and y 16-byte aligned, W 16-byte aligned (cudaMalloc /
 * torch allocations are).  Codes are not validated (invalid Q3H codes give
 * unspecified values, memory-safe).  Result within 1e-3 normwise of the fp64
 * definition (BASELINE.json north_star).
 * B = 1: fp32 CUDA-core path (Q3H_B64: the persistent engine of decode_mk.cu),
 *   deterministic (same bits every call).
 * B >= 2: tcgen05 tensor cores (qgemm_tc.cu): W' formed exactly (Eq. 2, fp32)
 *   then rounded to fp16, x split into fp16 hi + lo, fp32 accumulation
 *   (Q23); split-K partials are combined with atomic adds, so the
 *   low bits may differ between calls.  Shapes the TMA path cannot take
 *   (unaligned rows) fall back to the CUDA-core kernels.
 * ------------------------------------------------------------------------- */
if_status if_qgemv(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B,
                   float* y, if_stream_t stream);

/* Same, y[b, n] += sum_k W'[n,k] x[b,k]  (residual add fused; y read then written). */
if_status if_qgemv_acc(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x,
                       int64_t B, float* y, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * a5: prefill GEMM with fused dequantization on tcgen05 tensor cores
 *   Y[m, n] = sum_k W'[n, k] * X[m, k]       (bf16 x bf16 -> fp32 accumulate)
 * W device packed [N, K]; X device bf16 [M, K] (raw uint16 bit patterns);
 * Y device fp32 [M, N].  W' is rounded to bf16 inside the kernel (the
 * dequantized tile is staged in shared memory as bf16).  Within 2e-2 normwise
 * of the fp64 definition evaluated on the same bf16 X (north_star).
 * ------------------------------------------------------------------------- */
if_status if_qgemm(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const uint16_t* X_bf16,
                   int64_t M, float* Y, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * a7/a8: partition planner (Table 4; Q20)
 * ------------------------------------------------------------------------- */
typedef enum { IF_BY_LAYER = 0, IF_BY_TENSOR = 1, IF_HYBRID = 2 } if_strategy;

/* Llama-shaped stack (Q18): d = hidden, H heads, G kv heads,
 * head_dim, F = ffn.  Requirements: d, H*head_dim, F multiples of 64;
 * H % G == 0. */
typedef struct {
  int32_t layers, hidden, heads, kv_heads, head_dim, ffn;
  if_scheme scheme;
} if_stack_shape;

/* One device's share.  0-based half-open ranges (reports print them 1-based
 * inclusive).  FFN ranges are in units of 64 weights (Q20). */
typedef struct {
  int32_t rank, stage, group_rank;
  int32_t layer_begin, layer_end;
  int32_t head_begin, head_end;
  int32_t kv_begin, kv_end;
  int32_t ffn_blk_begin, ffn_blk_end;
} if_assignment;

typedef struct {
  int32_t strategy; /* if_strategy */
  int32_t devices, stages, groups;
  if_assignment a[8];
} if_plan;

/* Balanced contiguous ranges, remainder to earlier stages/ranks.
 * by_layer: stages = devices, groups = 1; by_tensor: stages = 1,
 * groups = devices; hybrid: stages x groups = devices (IF_ERR_GRID otherwise),
 * devices of one stage are adjacent ranks (Table 4).  heads, kv_heads
 * divisible by groups, F/64 >= groups, layers >= stages (IF_ERR_PLAN).
 * 1 <= devices <= 8. */
if_status if_plan_partition(int32_t strategy, const if_stack_shape* shape, int32_t devices,
                            int32_t stages, int32_t groups, if_plan* out);

/* ---------------------------------------------------------------------------
 * Communicators for the TP merges (a7, "merged twice") and the pipeline
 * hand-off (a8).  One process per GPU.  Two kinds behind one handle:
 *
 * NCCL (the library-collective baseline):
 *   if_comm_nccl_unique_id(id128)                 rank 0 creates the id (host, 128 B);
 *   (caller broadcasts it, e.g. torch.distributed.broadcast_object_list)
 *   if_comm_init(plan, rank, id128, &c)           ncclCommInitRank over plan->devices
 *       ranks + ncclCommSplit by stage (the TP group).  The device is the caller's
 *       current CUDA device.  all-reduce = ncclAllReduce (sum; NCCL's reduction
 *       order, Q21), send/recv = ncclSend/ncclRecv.  libnccl.so.2 is dlopen'ed (a
 *       process that already loaded torch's copy reuses it); IF_ERR_COMM when absent.
 *
 * Peer memory (B200-native, deterministic):
 *   if_comm_create(plan, rank, max_tokens, &c)   allocates this rank's
 *       symmetric mailbox (device memory owned by the communicator);
 *   if_comm_ipc_handle(c, out64)                 64-byte CUDA IPC handle of it;
 *   (caller all-gathers the handles, e.g. torch.distributed.all_gather_object)
 *   if_comm_open_peers(c, handles)              handles: host, devices x 64 bytes
 *   if_comm_destroy(c).
 * Set-up calls synchronise the device.  devices == 1 needs no peers.
 * ------------------------------------------------------------------------- */
typedef struct if_comm_s* if_comm;
if_status if_comm_nccl_unique_id(uint8_t* id128 /* host, 128 bytes */);
if_status if_comm_init(const if_plan* plan, int32_t rank, const uint8_t* nccl_unique_id /* host, 128 B */,
                       if_comm* out);
if_status if_comm_create(const if_plan* plan, int32_t rank, int64_t max_tokens, int32_t hidden,
                         if_comm* out);
if_status if_comm_ipc_handle(if_comm c, uint8_t* handle64 /* host, 64 bytes */);
if_status if_comm_open_peers(if_comm c, const uint8_t* handles /* host, devices*64 bytes */);
if_status if_comm_destroy(if_comm c);
/* All plan->devices ranks' peer-memory communicators inside ONE process on the
 * current device (outs: plan->devices handles), peers wired with plain pointers.
 * For running a multi-rank plan on one GPU as concurrent streams (tests, single-GPU
 * functional checks): each rank's decode engine then uses SMs / devices CTAs so
 * that every rank's engine is co-resident (the in-engine TP merges wait on peers). */
if_status if_comm_create_local(const if_plan* plan, int64_t max_tokens, int32_t hidden, if_comm* outs);

/* In-place all-reduce(sum) of buf[n] fp32 over this rank's TP group.  Peer
 * memory: every rank of the group ends with bit-identical sums (fixed rank
 * order); NCCL: ncclAllReduce.  Stream-ordered, graph capturable. */
if_status if_comm_allreduce(if_comm c, float* buf, int64_t n, if_stream_t stream);
/* Pipeline hand-off: send buf[n] to the same group rank of stage+1 / receive
 * from stage-1 into buf.  The stages form a ring: on the last stage send_next
 * goes to stage 0, and on stage 0 recv_prev receives from the last stage (the
 * autoregressive feedback of a decode step's output).  Needs stages > 1. */
if_status if_comm_send_next(if_comm c, const float* buf, int64_t n, if_stream_t stream);
if_status if_comm_recv_prev(if_comm c, float* buf, int64_t n, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * The Llama-shaped linear stack on this rank (Q18), decode or prefill.
 * Per layer of this rank's stage (rank-local shards, see if_plan):
 *   a = rms(h); [q|k|v] = a W_qkv^T; ctx_i = v_{floor(i/(H/G))};
 *   h += all_reduce(ctx W_o^T); a = rms(h); [g|u] = a W_gu^T;
 *   h += all_reduce((silu(g)*u) W_down^T)
 * stage_layers[i] holds the packed shards of layer layer_begin+i:
 *   wqkv  [(lh + 2 lkv) head_dim, d] : q rows of my heads, then k, then v rows
 *   wo    [d, lh head_dim]           : K-columns of my heads
 *   wgu   [2 lf, d]                  : gate and up rows of my FFN range INTERLEAVED:
 *                                      row 2f = gate row f, row 2f+1 = up row f
 *   wdown [d, lf]                    : K-columns of my FFN range
 * h_in  device fp32 [T, d] (ignored on stages > 0, which receive from stage-1),
 * h_out device fp32 [T, d] (valid on the last stage), last_qkv device fp32
 * [T, (lh + 2 lkv) head_dim] of the stage's last layer (nullable).
 * mode IF_DECODE (1 <= T <= 64, fp32 activations: T = 1 (3.5-bit) or T <= 6 (k-bit
 * schemes) runs the persistent engine -- one launch per token for the whole stage, with the TP
 * merges inside it when comm is a peer-memory communicator; 3.5-bit 2 <= T <= 16 on one
 * tensor-parallel rank runs the fused batched chain (qgemv_ms.cu: 4 launches per layer, the
 * glue in the GEMV epilogues, results bit-identical run to run); otherwise per-layer
 * qGEMVs (3.5-bit T <= 32: the warp-MMA kernel, else as in if_qgemv) or IF_PREFILL (T <= 4096,
 * qGEMM on tcgen05 with bf16 activations).
 * workspace: device, if_stack_workspace_bytes(); ZERO-FILL IT ONCE before the
 * first call (cudaMemset) and keep it with this (shape, plan, rank): it carries
 * the decode engine's step epoch and the chain's self-resetting split-K counters across
 * calls.  comm may be NULL when
 * plan->devices == 1.  Never synchronises; graph capturable.
 * ------------------------------------------------------------------------- */
enum { IF_DECODE = 0, IF_PREFILL = 1 };
typedef struct {
  const uint8_t* wqkv;
  const uint8_t* wo;
  const uint8_t* wgu;
  const uint8_t* wdown;
} if_layer_weights;

if_status if_stack_workspace_bytes(const if_stack_shape* shape, const if_plan* plan, int32_t rank,
                                   int64_t max_tokens, int32_t mode, size_t* bytes);
if_status if_run_stack(const if_stack_shape* shape, const if_plan* plan, int32_t rank, if_comm comm,
                       const if_layer_weights* stage_layers, const float* h_in, int64_t T,
                       int32_t mode, float* h_out, float* last_qkv, void* workspace,
                       if_stream_t stream);

/* ---------------------------------------------------------------------------
 * The stack with grouped-query decode attention over a KV cache (SURVEY NEXT-1,
 * DESIGN.md Q24).  Same as if_run_stack, except the single-position stand-in
 * (ctx_i = v of its kv group) is replaced by, per layer and token t:
 *   q_i, k_j <- RoPE(., p_t): pair (2m, 2m+1) turned by p_t * 10000^(-2m/hd)
 *                                          (Table 1 P:71 "rope")
 *   K[slot_t][p_t] = k, V[slot_t][p_t] = v (every token of the call appends first)
 *   ctx_i = sum_{tau <= p_t} softmax(q_i . K^j[tau] / sqrt(hd)) V^j[tau],
 *           j = floor(i / (H/G))
 * so a decode batch is T independent queries (T distinct slots) and a chunk of
 * consecutive positions of one slot is causal prefill.  At p_t = 0 it equals
 * if_run_stack.  last_qkv holds q and k after RoPE.
 * kv: caller-owned device cache, fp32 k and v arrays of if_kv_cache_bytes() each,
 *     layout [stage layers][slots][max_ctx][lkv][head_dim] (this rank's kv heads);
 *     zero-filling is not needed (positions > p_t are never read).
 * slot_ids, positions: DEVICE int32 [T] (graph replays may change them in place).
 * An out-of-range slot or position writes IF_ERR_ARG to kv->status (nullable) and
 * that token's context is zero; the call itself returns IF_OK.
 * head_dim 64 or 128, heads per kv group <= 8.  Persistent-engine batches (Q3H_B64,
 * T <= 6, one TP rank) take the per-layer path when a cache is given.
 * ------------------------------------------------------------------------- */
typedef struct {
  float* k;
  float* v;
  int32_t slots, max_ctx;
  int32_t* status; /* device, nullable */
} if_kv_cache;

if_status if_kv_cache_bytes(const if_stack_shape* shape, const if_plan* plan, int32_t rank, int32_t slots,
                            int32_t max_ctx, size_t* bytes_each);
if_status if_run_stack_kv(const if_stack_shape* shape, const if_plan* plan, int32_t rank, if_comm comm,
                          const if_layer_weights* stage_layers, const float* h_in, int64_t T, int32_t mode,
                          float* h_out, float* last_qkv, const if_kv_cache* kv, const int32_t* slot_ids,
                          const int32_t* positions, void* workspace, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * Language-model head (Q27): what turns the stack's output into "a set of
 * next tokens" and gives the target logits of speculative decoding
 * (Algorithm 1).  All pointers device, stream-ordered, graph capturable.
 *
 * if_embed:      h[t] = table[tokens[t]]   table fp32 [V, d] (16-B aligned, d % 4 == 0),
 *                tokens int32 [T], h fp32 [T, d].  A token outside [0, V) writes
 *                IF_ERR_ARG to dev_status (nullable) and a zero row.
 * if_lm_logits:  logits[b] = rms(h[rows[b]]) . W'_lm^T   (final RMSNorm, unit gain,
 *                eps 1e-5; then if_qgemv with B = T, 1 <= T <= 64: same
 *                precision contract, 1e-3 normwise).  lm packed [V, d] in scheme s;
 *                rows int32 [T] (nullable = 0..T-1) index h's rows; scratch fp32 [T, d].
 * if_argmax:     tokens[t] = first index of the maximum of logits[t] (greedy).
 * ------------------------------------------------------------------------- */
if_status if_embed(const float* table, int32_t V, int32_t d, const int32_t* tokens, int64_t T, float* h,
                   int32_t* dev_status, if_stream_t stream);
if_status if_lm_logits(if_scheme s, const uint8_t* lm, int64_t V, int64_t d, const float* h, int64_t T,
                       const int32_t* rows, float* logits, float* scratch, if_stream_t stream);
if_status if_argmax(const float* logits, int64_t T, int64_t V, int32_t* tokens, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * Speculative sampling, one verification round (Algorithm 1; SURVEY
 * NEXT-3; readings Q25/Q26).  Algorithm 1's notation: the draft model p proposed
 * draft_tok [K] with distributions draft_probs [K, V]; the target q was evaluated at
 * the K+1 positions in parallel, tgt_logits [K+1, V] (q = softmax, temperature 1).
 * For t < K: accept draft t when (is_top and it lies in q's top-k / top-p pool,
 * fewer than top_k tokens, and less than top_p mass, strictly more
 * probable) or u_acc[t] < min(1, q(x)/p(x)); else draw from (q - p)_+ with u_smp
 * and stop.  All K accepted: draw an extra token from q at position K with u_smp.
 * Draws are inverse-CDF in index order (the smallest i whose running sum exceeds
 * u * total).  top_k <= 0 / top_p >= 1 disable that pool.  Decisions in fp64.
 * All arrays device; out_tok [K+1], *n_out = accepted + 1, or -IF_ERR_ARG when a
 * draft token lies outside [0, V).  0 <= K <= 64; u_smp in [0, 1).
 * ------------------------------------------------------------------------- */
if_status if_spec_verify(int32_t K, int64_t V, const float* tgt_logits, const float* draft_probs,
                         const int32_t* draft_tok, const float* u_acc, float u_smp, int32_t is_top, int32_t top_k,
                         float top_p, int32_t* out_tok, int32_t* n_out, if_stream_t stream);

/* ---------------------------------------------------------------------------
 * Dynamic batching (Fig. 3): an inference engine with the
 * paper's two-function interface over one rank's stack (plan by_layer, 1 device).
 *   if_engine_add_query(S)  add query S (host prompt tokens) to the query pool;
 *                           FIFO admission when a KV slot is free
 *   if_engine_infer()       ONE step over the pool: admits queued queries, runs the
 *                           prompts of new queries (causal chunks, continued over
 *                           later steps when they exceed the token budget) and one
 *                           decode token of every running query in a single
 *                           if_run_stack_kv batch, then the LM head and the greedy
 *                           choice -> (query id, next token) for every query whose
 *                           prompt is complete.  A query finishes at eos, after
 *                           max_new tokens, or at max_ctx; its slot is released.
 * Example (Fig. 3): S1, S2 decoding, AddQuery(S3) at T3 -> Infer() returns
 * S1_3, S2_3 and S3's first token in the same step.
 * if_engine_verify()        speculative decoding's target pass for one running query
 *                           (NEXT-3): [last token, draft_tok[0..K)] as one causal
 *                           chunk, logits at all K+1 positions (small-M qGEMV), then
 *                           if_spec_verify; the accepted tokens + 1 are appended.
 * The engine owns its device state (KV cache, workspace, logits; allocated at create)
 * and runs on the caller's stream; infer/verify synchronise it (results are host).
 * Weights, embedding table and LM head stay caller-owned and must outlive it.
 * ------------------------------------------------------------------------- */
typedef struct if_engine_s* if_engine;
typedef struct {
  if_stack_shape shape;            /* the stack (scheme = the LM head's too) */
  const if_layer_weights* layers;  /* host array of shape.layers device weight sets */
  const float* embed;              /* device fp32 [vocab, hidden] */
  const uint8_t* lm_head;          /* device packed [vocab, hidden] */
  int32_t vocab;
  int32_t slots;                   /* pool capacity (concurrent queries), 1..64 */
  int32_t max_ctx;                 /* positions per slot */
  int32_t step_tokens;             /* token budget of one Infer() step, slots..64 */
} if_engine_config;

if_status if_engine_create(const if_engine_config* cfg, if_engine* out);
if_status if_engine_add_query(if_engine e, const int32_t* prompt /* host */, int32_t n, int32_t max_new,
                              int32_t eos /* < 0: none */, int64_t* query_id);
if_status if_engine_infer(if_engine e, int64_t* ids /* host [cap] */, int32_t* tokens /* host [cap] */, int32_t cap,
                          int32_t* n_out, if_stream_t stream);
if_status if_engine_verify(if_engine e, int64_t query_id, int32_t K, const int32_t* draft_tok /* host [K] */,
                           const float* draft_probs /* device [K, vocab] */, const float* u_acc /* host [K] */,
                           float u_smp, int32_t is_top, int32_t top_k, float top_p, int32_t* out_tok /* host [K+1] */,
                           int32_t* n_out, if_stream_t stream);
/* phase: 0 queued, 1 prefill, 2 decoding, 3 finished, -1 unknown id */
if_status if_engine_query(if_engine e, int64_t query_id, int32_t* phase, int32_t* generated, int32_t* position);
/* device logits of the last infer/verify step, [rows, vocab] (engine-owned, valid
 * until the next call) and the query id of each row */
if_status if_engine_last_logits(if_engine e, const float** logits, int32_t* rows, int64_t* ids /* host [64] */);
if_status if_engine_destroy(if_engine e);

/* ---------------------------------------------------------------------------
 * Packed-tensor container (S:122-123 section layout; Q28).
 * File: "IFQC", u32 version 1, u32 tensor count, then per tensor: u16 name length,
 * name, u8 scheme id (if_qtype), u16 block, u8 ndim, u32 dims[ndim], u32 block count
 * (= prod(dims) / block; blocks run along the last dim), the packed blocks exactly as
 * if_quantize writes them.  Integers little-endian.
 *   if_container_save   dims: n x 8 int64 (row i = tensor i's dims); data[i] host or
 *                       device (data_on_device) packed bytes; device data goes through
 *                       a pinned bounce buffer on `stream` (synchronised).
 *   if_container_open   parses and checks every header (magic, version, scheme, block
 *                       count vs dims, payload extents, no trailing bytes): IF_ERR_IO
 *                       with the byte offset in if_last_error() otherwise.
 *   if_container_load   tensor i -> device memory: pipelined pread into pinned staging
 *                       buffers by 4 reader threads, async H2D on `stream`.  Returns
 *                       once every copy is enqueued (stream-ordered completion).
 *   if_container_read_host  tensor i -> host memory (synchronous).
 * ------------------------------------------------------------------------- */
typedef struct if_container_s* if_container;
if_status if_container_save(const char* path, int32_t n, const char* const* names, const if_scheme* schemes,
                            const int32_t* ndims, const int64_t* dims, const void* const* data, int32_t data_on_device,
                            if_stream_t stream);
if_status if_container_open(const char* path, if_container* out);
int32_t if_container_count(if_container c);
if_status if_container_info(if_container c, int32_t i, char* name, int32_t name_cap, if_scheme* s, int32_t* ndim,
                            int64_t* dims /* [8] */, int64_t* bytes);
if_status if_container_find(if_container c, const char* name, int32_t* index);
if_status if_container_load(if_container c, int32_t i, void* dst_device, if_stream_t stream);
if_status if_container_read_host(if_container c, int32_t i, void* dst_host);
if_status if_container_close(if_container c);

/* ---------------------------------------------------------------------------
 * Partition cost model and auto-planner (Table 5
 * P:224-237; Q29).  Per-token latency of one decode stream:
 *   L (t_fixed + layer_bytes / groups / bw)           every layer on a 1/groups shard
 *   + 2 L t_merge[groups]   (groups > 1)              "merged twice" per layer
 *   + (stages - 1) t_hop                              stage hand-offs
 * decode = 1 / latency (tokens/s of one stream); throughput = decode x min(stages,
 * micro_batches) (a filled pipeline, Q22).  layer_bytes = the packed bytes of one
 * layer in shape's scheme.  The calibrated parameters come from measured B200 runs
 * (profiles/r2_cost_calibration.json).  if_plan_auto: over every grid stages x groups
 * = devices that if_plan_partition accepts, the plan maximising decode (objective 0)
 * or throughput (1); ties keep fewer TP ranks.
 * ------------------------------------------------------------------------- */
typedef struct {
  double t_fixed_s;     /* per layer and token, independent of the shard size */
  double bw_bytes_s;    /* effective weight-streaming bandwidth of one device */
  double t_merge_s[9];  /* one all-reduce within a TP group of g ranks, index g */
  double t_hop_s;       /* one stage-to-stage hand-off */
} if_cost_model;
if_status if_cost_estimate(const if_stack_shape* shape, int32_t stages, int32_t groups, const if_cost_model* cm,
                           int32_t micro_batches, double* decode, double* throughput);
if_status if_plan_auto(int32_t objective, const if_stack_shape* shape, int32_t devices, const if_cost_model* cm,
                       int32_t micro_batches, if_plan* out, double* decode, double* throughput);

/* Thread-local message for the last non-OK status returned on this thread. */
const char* if_last_error(void);

/* Number of kernels this library launched on this host thread since the last
 * reset (instrumentation for bench.py's gpu_launches). */
int64_t if_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* IF_B200_H */
