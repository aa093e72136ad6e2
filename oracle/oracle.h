/*
 * oracle.h — plain, slow, obviously-correct CPU oracle for the Inferflow
 * block-quantized GEMV/GEMM hot path (arxiv 2401.08294).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with the CUDA path in
 * paper_2401_08294_b200/csrc (and never includes anything from there).
 *
 * Citations: "P:n" = line n of PAPER.md (the Inferflow report), "S:n" = line
 * n of SPEC.md; "Q<n>" = reading n in DESIGN.md §Readings.
 *
 * Status codes (numerically equal to the product ABI's by design decision, but
 * declared independently here):
 *   0 OK, 1 ARG, 2 SHAPE, 3 SCHEME, 4 INPUT (non-finite / beyond fp16 range),
 *   5 DECODE (Q3H pair code > 120), 6 PLAN, 7 GRID.
 */
#ifndef INFERFLOW_ORACLE_H
#define INFERFLOW_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- scheme (P:118 schemes, Table 3) ---------------------------- */
/* qtype: 2,3,4,5,6,8 = k-bit (Eq.1);  35 = Q3H 3.5-bit. */
int     ref_scheme_valid(int qtype, int block);
int     ref_levels(int qtype);                 /* D = 2^k-1, or 10 for Q3H */
int64_t ref_code_bytes(int qtype, int n);      /* ceil(n*bits/8)   */
int64_t ref_block_bytes(int qtype, int block); /* code bytes + two fp16    */
void    ref_bits_per_weight(int qtype, int block, int64_t* num, int64_t* den);

/* ---- binary16 helpers (two FP16 numbers per block; Q3) ------------- */
uint16_t ref_f32_to_f16_rd(float f);   /* round toward -inf */
uint16_t ref_f32_to_f16_ru(float f);   /* round toward +inf */
float    ref_f16_to_f32(uint16_t h);   /* exact */

/* ---- 3.5-bit pair code ---------------------------------------- */
int ref_pack_pair(int q_even, int q_odd);            /* q_{2i}*11 + q_{2i+1}; -1 if a digit > 10 */
int ref_unpack_pair(int v, int* q_first, int* q_second); /* floor(v/11), v mod 11; 5 if v>120 */

/* ---- one block (Eq.1 P:102 / 3.5-bit P:122-127 / Eq.2) --------------- */
/* n = number of weights in the block (32/64; any n>=1 in test mode, even for Q3H). */
int ref_quantize_block(int qtype, int n, const float* w, uint8_t* out);
int ref_dequantize_block(int qtype, int n, const uint8_t* in, float* w_out);
/* codes as integers (per weight digits 0..D) — for Table 2 checks */
int ref_block_codes(int qtype, int n, const uint8_t* in, int32_t* q_out);

/* ---- tensors: W [N,K] row-major, blocks along K (Q9) ---------------------- */
int ref_quantize(int qtype, int block, const float* W, int64_t N, int64_t K, uint8_t* packed);
int ref_dequantize(int qtype, int block, const uint8_t* packed, int64_t N, int64_t K, float* W_out);

/* ---- products: the plain definition y = x W'^T evaluated in fp64 */
/* X [M,K] fp32, Y [M,N] fp64.  Dequantizes each row to fp32 W' first (Eq.2). */
int ref_matmul_f64(int qtype, int block, const uint8_t* packed, int64_t N, int64_t K,
                   const float* X, int64_t M, double* Y);

/* ---- the Llama-shaped linear stack (Q18) ------------------------- */
typedef struct {
  int32_t layers, hidden, heads, kv_heads, head_dim, ffn;
  int32_t qtype, block;
} ref_stack_shape;

/* Per layer packed weights: wqkv [(H+2G)hd, d], wo [d, H hd], wgu [2F, d] (gate rows
 * then up rows), wdown [d, F].  h_in [T,d] fp32.  h_out [T,d] fp64,
 * last_qkv [T,(H+2G)hd] fp64 (nullable).  Entirely in fp64 from the exact fp32 W'. */
int ref_stack_f64(const ref_stack_shape* s, const uint8_t* const* wqkv, const uint8_t* const* wo,
                  const uint8_t* const* wgu, const uint8_t* const* wdown,
                  const float* h_in, int64_t T, double* h_out, double* last_qkv);

/* ---- the stack with decode attention over a KV cache (Q24) ----
 * As ref_stack_f64, except the single-position stand-in is replaced by scaled
 * dot-product grouped-query attention over a per-slot KV cache (P:332-337,
 * P:341-347), with RoPE on q and k (Table 1 P:71 "position_embedding rope";
 * S:343 consecutive pairs, theta_m = 10000^(-2m/hd)).  Token t of the batch has
 * cache slot slot_ids[t] and position positions[t]; per layer all T tokens append
 * their k, v first, then each attends causally to positions 0..positions[t] of its
 * slot.  kcache/vcache: fp64 [layers][slots][max_ctx][G][hd], caller-owned state.
 * Returns 2 for a slot or position out of range.  At positions[t] = 0 this equals
 * ref_stack_f64 (softmax over one key; RoPE at position 0 is the identity). */
int ref_stack_kv_f64(const ref_stack_shape* s, const uint8_t* const* wqkv, const uint8_t* const* wo,
                     const uint8_t* const* wgu, const uint8_t* const* wdown, const float* h_in, int64_t T,
                     const int32_t* slot_ids, const int32_t* positions, int32_t slots, int32_t max_ctx,
                     double* kcache, double* vcache, double* h_out, double* last_qkv);

/* ---- speculative sampling, one verification round (Algorithm 1, P:351-384;
 * SURVEY NEXT-3; readings Q25/Q26) ------------------------------------------
 * Algorithm 1's own notation: the draft model p proposes draft_tok[0..K) with
 * distributions draft_probs [K][V]; the target q is evaluated "in parallel" at the
 * K+1 positions, tgt_logits [K+1][V] (q = softmax, temperature 1).  For t < K:
 * accept draft t when (is_top and it lies in the target's top-k/top-p pool) or
 * u_acc[t] < min(1, q(x)/p(x)); else sample from (q - p)_+ with u_smp and stop.
 * All K accepted: sample an extra token from q at position K with u_smp.
 * Sampling with a uniform u: the smallest index i whose running sum (index order)
 * exceeds u * total.  top_k <= 0 / top_p >= 1 disable that pool.
 * out_tok [K+1]; *n_out = accepted + 1.  Returns 2 on bad sizes or tokens. */
int ref_spec_verify(int K, int V, const float* tgt_logits, const float* draft_probs, const int32_t* draft_tok,
                    const float* u_acc, float u_smp, int is_top, int top_k, float top_p, int32_t* out_tok,
                    int32_t* n_out);

/* ---- language-model head (reading Q27) ---------------
 * logits [T][V] = rms(h[t]) . W'_lm[v]  (final RMSNorm, unit gain, eps 1e-5; the
 * output projection lm [V, d] block-quantized).  h fp64 [T][d]. */
int ref_lm_logits_f64(int qtype, int block, const uint8_t* lm, int64_t V, int64_t d, const double* h, int64_t T,
                      double* logits);
/* greedy choice: first index of the maximum; -1 for n = 0 */
int64_t ref_argmax_f64(const double* x, int64_t n);

/* ---- partition cost model (Table 5; Q29) --------
 * latency = L (t_fixed + layer_bytes / groups / bw) + 2 L t_merge[groups] [groups > 1]
 *         + (stages - 1) t_hop;  decode = 1 / latency;
 * throughput = decode x min(stages, micro_batches).  t_merge indexed by group size. */
int ref_cost_estimate(int layers, int stages, int groups, double t_fixed, double layer_bytes, double bw,
                      const double* t_merge, double t_hop, int micro_batches, double* decode, double* throughput);

/* ---- partition planner (Table 4; Q20) ----------------- */
/* strategy: 0 by-layer, 1 by-tensor, 2 hybrid.  Output arrays have `devices`
 * entries, 0-based half-open ranges: layer [lb,le), head [hb,he), kv-head [kb,ke),
 * FFN 64-block [fb,fe).  ffn_blocks = F / block-granule. */
int ref_plan(int strategy, int layers, int heads, int kv_heads, int ffn_blocks,
             int devices, int stages, int groups,
             int32_t* stage_of, int32_t* group_rank_of,
             int32_t* lb, int32_t* le, int32_t* hb, int32_t* he,
             int32_t* kb, int32_t* ke, int32_t* fb, int32_t* fe);

/* Virtual-partition replay of the stack (SURVEY §4 "How we test multi-GPU"):
 * every rank's shard math replayed on CPU in fp64 — column shards of qkv/gate/up,
 * row (K) shards of o/down, partial sums reduced by addition over the TP group,
 * stage-to-stage hand-off.  Same outputs as ref_stack_f64 up to fp64 rounding. */
int ref_stack_partitioned_f64(const ref_stack_shape* s, int strategy, int devices, int stages,
                              int groups, const uint8_t* const* wqkv, const uint8_t* const* wo,
                              const uint8_t* const* wgu, const uint8_t* const* wdown,
                              const float* h_in, int64_t T, double* h_out);

#ifdef __cplusplus
}
#endif
#endif
