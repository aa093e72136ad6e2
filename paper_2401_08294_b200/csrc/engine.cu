// engine.cu — dynamic batching (Fig. 3) and the
// speculative-decoding target pass (Algorithm 1; NEXT-3) as a native
// query-pool runtime over one rank's stack.
// ifb-build: -std=c++17
//   (host-only file; nvcc 12.9's C++20 front end aborts on <deque>/<vector> here)
//
// AddQuery(S) puts S in a FIFO admission queue; Infer() is one iteration-level
// step (the Orca-style scheduling the paper cites): admit queued queries
// while KV slots are free, give every decoding query one token and fill the rest
// of the step's token budget with prompt chunks of prefilling queries (FIFO; a
// prompt longer than the remaining budget continues next step), run them as ONE
// if_run_stack_kv batch (decode tokens and causal prompt chunks side by side: each
// token carries its own slot and position), then the LM head on the rows that end
// a query's input and the greedy choice.  The host side is plain bookkeeping; the
// per-step device work is: one packed H2D of the step's index arrays, embed, the
// stack, RMSNorm + LM-head qGEMV, argmax, one D2H of the chosen tokens.
#include <deque>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace ifb {

enum { PH_QUEUED = 0, PH_PREFILL = 1, PH_DECODE = 2, PH_DONE = 3 };

struct Query {
  int64_t id;
  std::vector<int32_t> prompt;
  std::vector<int32_t> out;
  int32_t consumed = 0;  // prompt tokens already in the KV cache
  int32_t pos = 0;       // position of the pending token (decode phase)
  int32_t last = 0;      // pending token (the last emitted one), not yet in the cache
  int32_t slot = -1;
  int32_t max_new = 0;
  int32_t eos = -1;
  int phase = PH_QUEUED;
};

}  // namespace ifb

struct if_engine_s {
  if_engine_config cfg;
  if_plan plan;
  std::vector<if_layer_weights> layers;
  // device state (owned)
  float* kv_k = nullptr;
  float* kv_v = nullptr;
  int32_t* status = nullptr;
  void* ws = nullptr;
  float* h_in = nullptr;
  float* h_out = nullptr;
  float* scratch = nullptr;
  float* logits = nullptr;
  int32_t* idx = nullptr;   // [4][step_tokens]: tokens | slots | positions | emit rows
  int32_t* tok = nullptr;   // [65] chosen tokens (+ n_out of a verification)
  float* u_dev = nullptr;   // [64] verification uniforms
  int32_t* hidx = nullptr;  // pinned host mirrors
  int32_t* htok = nullptr;
  float* hu = nullptr;
  if_kv_cache kv;
  // pool
  std::deque<ifb::Query*> queued;
  std::vector<ifb::Query*> active;
  std::unordered_map<int64_t, ifb::Query*> all;
  std::vector<int32_t> free_slots;
  int64_t next_id = 1;
  int32_t last_rows = 0;
  int64_t last_ids[64];
};

using namespace ifb;

static void engine_free(if_engine e) {
  cudaFree(e->kv_k);
  cudaFree(e->kv_v);
  cudaFree(e->status);
  cudaFree(e->ws);
  cudaFree(e->h_in);
  cudaFree(e->h_out);
  cudaFree(e->scratch);
  cudaFree(e->logits);
  cudaFree(e->idx);
  cudaFree(e->tok);
  cudaFree(e->u_dev);
  cudaFreeHost(e->hidx);
  cudaFreeHost(e->htok);
  cudaFreeHost(e->hu);
  for (auto& kv : e->all) delete kv.second;
  delete e;
}

extern "C" if_status if_engine_create(const if_engine_config* cfg, if_engine* out) {
  if (!cfg || !out || !cfg->layers || !cfg->embed || !cfg->lm_head) return set_error(IF_ERR_ARG, "if_engine_create: null pointer");
  *out = nullptr;
  const if_engine_config& c = *cfg;
  if (c.vocab < 2 || c.slots < 1 || c.slots > 64 || c.max_ctx < 2 || c.step_tokens < c.slots || c.step_tokens > 64)
    return set_error(IF_ERR_ARG, "if_engine_create: vocab=%d slots=%d max_ctx=%d step_tokens=%d", c.vocab, c.slots,
                     c.max_ctx, c.step_tokens);
  if (c.shape.hidden % c.shape.scheme.block || c.shape.hidden % 4)
    return set_error(IF_ERR_SHAPE, "if_engine_create: hidden %d", c.shape.hidden);
  if_engine e = new if_engine_s();
  e->cfg = c;
  if_status st = if_plan_partition(IF_BY_LAYER, &c.shape, 1, 0, 0, &e->plan);
  if (st) {
    delete e;
    return st;
  }
  e->layers.assign(c.layers, c.layers + c.shape.layers);
  size_t kvb = 0, wsb = 0;
  if ((st = if_kv_cache_bytes(&c.shape, &e->plan, 0, c.slots, c.max_ctx, &kvb)) ||
      (st = if_stack_workspace_bytes(&c.shape, &e->plan, 0, c.step_tokens, IF_DECODE, &wsb))) {
    delete e;
    return st;
  }
  const int64_t T = c.step_tokens, d = c.shape.hidden;
  bool ok = cudaMalloc(&e->kv_k, kvb) == cudaSuccess && cudaMalloc(&e->kv_v, kvb) == cudaSuccess &&
            cudaMalloc(&e->status, 16) == cudaSuccess && cudaMalloc(&e->ws, wsb) == cudaSuccess &&
            cudaMalloc(&e->h_in, T * d * 4) == cudaSuccess && cudaMalloc(&e->h_out, T * d * 4) == cudaSuccess &&
            cudaMalloc(&e->scratch, T * d * 4) == cudaSuccess &&
            cudaMalloc(&e->logits, (size_t)T * c.vocab * 4) == cudaSuccess &&
            cudaMalloc(&e->idx, 4 * T * 4) == cudaSuccess && cudaMalloc(&e->tok, 80 * 4) == cudaSuccess &&
            cudaMalloc(&e->u_dev, 64 * 4) == cudaSuccess && cudaMallocHost(&e->hidx, 4 * T * 4) == cudaSuccess &&
            cudaMallocHost(&e->htok, 80 * 4) == cudaSuccess && cudaMallocHost(&e->hu, 64 * 4) == cudaSuccess;
  ok = ok && cudaMemset(e->ws, 0, wsb) == cudaSuccess && cudaMemset(e->status, 0, 16) == cudaSuccess &&
       cudaDeviceSynchronize() == cudaSuccess;
  if (!ok) {
    engine_free(e);
    return set_error(IF_ERR_CUDA, "if_engine_create: device allocation failed (%s)", cudaGetErrorString(cudaGetLastError()));
  }
  e->kv = if_kv_cache{e->kv_k, e->kv_v, c.slots, c.max_ctx, e->status};
  for (int32_t s = c.slots - 1; s >= 0; s--) e->free_slots.push_back(s);
  *out = e;
  return IF_OK;
}

extern "C" if_status if_engine_destroy(if_engine e) {
  if (!e) return set_error(IF_ERR_ARG, "if_engine_destroy: null engine");
  cudaDeviceSynchronize();
  engine_free(e);
  return IF_OK;
}

extern "C" if_status if_engine_add_query(if_engine e, const int32_t* prompt, int32_t n, int32_t max_new, int32_t eos,
                                         int64_t* query_id) {
  if (!e || !prompt || !query_id) return set_error(IF_ERR_ARG, "if_engine_add_query: null pointer");
  if (n < 1 || n >= e->cfg.max_ctx || max_new < 1)
    return set_error(IF_ERR_ARG, "if_engine_add_query: prompt of %d tokens (max_ctx %d), max_new %d", n, e->cfg.max_ctx, max_new);
  for (int32_t i = 0; i < n; i++)
    if (prompt[i] < 0 || prompt[i] >= e->cfg.vocab) return set_error(IF_ERR_ARG, "if_engine_add_query: token %d at %d", prompt[i], i);
  Query* q = new Query();
  q->id = e->next_id++;
  q->prompt.assign(prompt, prompt + n);
  q->max_new = max_new;
  q->eos = eos;
  e->queued.push_back(q);
  e->all[q->id] = q;
  *query_id = q->id;
  return IF_OK;
}

extern "C" if_status if_engine_query(if_engine e, int64_t id, int32_t* phase, int32_t* generated, int32_t* position) {
  if (!e) return set_error(IF_ERR_ARG, "if_engine_query: null engine");
  auto it = e->all.find(id);
  const Query* q = it == e->all.end() ? nullptr : it->second;
  if (phase) *phase = q ? q->phase : -1;
  if (generated) *generated = q ? (int32_t)q->out.size() : 0;
  if (position) *position = q ? (q->phase == PH_DECODE || q->phase == PH_DONE ? q->pos : q->consumed) : 0;
  return IF_OK;
}

extern "C" if_status if_engine_last_logits(if_engine e, const float** logits, int32_t* rows, int64_t* ids) {
  if (!e) return set_error(IF_ERR_ARG, "if_engine_last_logits: null engine");
  if (logits) *logits = e->logits;
  if (rows) *rows = e->last_rows;
  if (ids)
    for (int32_t i = 0; i < e->last_rows; i++) ids[i] = e->last_ids[i];
  return IF_OK;
}

// Run T tokens (host index arrays already in e->hidx: tokens | slots | positions |
// emit rows) through embed -> stack -> LM head over `rows` emitting rows.  verify: the
// K+1 logits feed if_spec_verify instead of the argmax.
static if_status engine_forward(if_engine e, int32_t T, int32_t rows, cudaStream_t st) {
  const int32_t S = e->cfg.step_tokens;
  if (cudaMemcpyAsync(e->idx, e->hidx, 4 * S * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return check_launch("if_engine: index upload");
  const int32_t* d_tok = e->idx;
  const int32_t* d_slot = e->idx + S;
  const int32_t* d_pos = e->idx + 2 * S;
  const int32_t* d_rows = e->idx + 3 * S;
  const if_engine_config& c = e->cfg;
  if_status r = if_embed(c.embed, c.vocab, c.shape.hidden, d_tok, T, e->h_in, e->status, (if_stream_t)st);
  if (r) return r;
  r = if_run_stack_kv(&c.shape, &e->plan, 0, nullptr, e->layers.data(), e->h_in, T, IF_DECODE, e->h_out, nullptr,
                      &e->kv, d_slot, d_pos, e->ws, (if_stream_t)st);
  if (r) return r;
  return if_lm_logits(c.shape.scheme, c.lm_head, c.vocab, c.shape.hidden, e->h_out, rows, d_rows, e->logits,
                      e->scratch, (if_stream_t)st);
}

static void finish_if_done(if_engine e, Query* q) {
  const int32_t t = q->out.back();
  if ((q->eos >= 0 && t == q->eos) || (int32_t)q->out.size() >= q->max_new || q->pos + 1 >= e->cfg.max_ctx) {
    q->phase = PH_DONE;
    e->free_slots.push_back(q->slot);
    q->slot = -1;
  }
}

extern "C" if_status if_engine_infer(if_engine e, int64_t* ids, int32_t* tokens, int32_t cap, int32_t* n_out,
                                     if_stream_t stream) {
  if (!e || !n_out || (cap > 0 && (!ids || !tokens))) return set_error(IF_ERR_ARG, "if_engine_infer: null pointer");
  *n_out = 0;
  cudaStream_t st = (cudaStream_t)stream;
  // admission (FIFO, capacity = KV slots)
  while (!e->queued.empty() && !e->free_slots.empty()) {
    Query* q = e->queued.front();
    e->queued.pop_front();
    q->slot = e->free_slots.back();
    e->free_slots.pop_back();
    q->phase = PH_PREFILL;
    e->active.push_back(q);
  }
  const int32_t S = e->cfg.step_tokens;
  int32_t* htok = e->hidx;
  int32_t* hslot = e->hidx + S;
  int32_t* hpos = e->hidx + 2 * S;
  int32_t* hrow = e->hidx + 3 * S;
  std::vector<Query*> emit;
  int32_t T = 0;
  for (Query* q : e->active)  // one decode token per running query
    if (q->phase == PH_DECODE) {
      htok[T] = q->last;
      hslot[T] = q->slot;
      hpos[T] = q->pos;
      hrow[emit.size()] = T;
      emit.push_back(q);
      T++;
    }
  std::vector<std::pair<Query*, int32_t>> chunks;
  for (Query* q : e->active)  // prompt chunks in admission order, within the budget
    if (q->phase == PH_PREFILL && T < S) {
      const int32_t n = std::min<int32_t>((int32_t)q->prompt.size() - q->consumed, S - T);
      for (int32_t i = 0; i < n; i++) {
        htok[T + i] = q->prompt[q->consumed + i];
        hslot[T + i] = q->slot;
        hpos[T + i] = q->consumed + i;
      }
      T += n;
      chunks.push_back({q, n});
      if (q->consumed + n == (int32_t)q->prompt.size()) {
        hrow[emit.size()] = T - 1;
        emit.push_back(q);
      }
    }
  if (T == 0) return IF_OK;
  const int32_t rows = (int32_t)emit.size();
  if_status r;
  if (rows > cap) return set_error(IF_ERR_ARG, "if_engine_infer: %d results exceed cap %d", rows, cap);
  if (rows == 0) {  // only prompt chunks that do not finish their prompt: no LM head
    if (cudaMemcpyAsync(e->idx, e->hidx, 4 * S * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return check_launch("if_engine_infer: index upload");
    const if_engine_config& c = e->cfg;
    if ((r = if_embed(c.embed, c.vocab, c.shape.hidden, e->idx, T, e->h_in, e->status, stream))) return r;
    if ((r = if_run_stack_kv(&c.shape, &e->plan, 0, nullptr, e->layers.data(), e->h_in, T, IF_DECODE, e->h_out,
                             nullptr, &e->kv, e->idx + S, e->idx + 2 * S, e->ws, stream)))
      return r;
  } else {
    if ((r = engine_forward(e, T, rows, st))) return r;
    if ((r = if_argmax(e->logits, rows, e->cfg.vocab, e->tok, stream))) return r;
    if (cudaMemcpyAsync(e->htok, e->tok, rows * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return check_launch("if_engine_infer: token download");
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("if_engine_infer: step");
  for (auto& ch : chunks) ch.first->consumed += ch.second;
  e->last_rows = rows;
  for (int32_t i = 0; i < rows; i++) {
    Query* q = emit[i];
    const int32_t t = e->htok[i];
    e->last_ids[i] = q->id;
    ids[i] = q->id;
    tokens[i] = t;
    if (q->phase == PH_DECODE) {
      q->pos++;
    } else {  // prompt complete: the first generated token
      q->phase = PH_DECODE;
      q->pos = (int32_t)q->prompt.size();
    }
    q->last = t;
    q->out.push_back(t);
    finish_if_done(e, q);
  }
  std::vector<Query*> keep;
  for (Query* q : e->active)
    if (q->phase != PH_DONE) keep.push_back(q);
  e->active.swap(keep);
  *n_out = rows;
  return IF_OK;
}

extern "C" if_status if_engine_verify(if_engine e, int64_t id, int32_t K, const int32_t* draft_tok,
                                      const float* draft_probs, const float* u_acc, float u_smp, int32_t is_top,
                                      int32_t top_k, float top_p, int32_t* out_tok, int32_t* n_out,
                                      if_stream_t stream) {
  if (!e || !out_tok || !n_out || (K > 0 && (!draft_tok || !draft_probs || !u_acc)))
    return set_error(IF_ERR_ARG, "if_engine_verify: null pointer");
  *n_out = 0;
  auto it = e->all.find(id);
  if (it == e->all.end() || it->second->phase != PH_DECODE)
    return set_error(IF_ERR_ARG, "if_engine_verify: query %lld is not decoding", (long long)id);
  Query* q = it->second;
  const int32_t S = e->cfg.step_tokens;
  if (K < 0 || K + 1 > S || q->pos + K >= e->cfg.max_ctx)
    return set_error(IF_ERR_ARG, "if_engine_verify: K=%d at position %d (budget %d, max_ctx %d)", K, q->pos, S, e->cfg.max_ctx);
  for (int32_t t = 0; t < K; t++)
    if (draft_tok[t] < 0 || draft_tok[t] >= e->cfg.vocab) return set_error(IF_ERR_ARG, "if_engine_verify: draft token %d", draft_tok[t]);
  // [last, d_1 .. d_K] at positions pos .. pos+K of the query's slot: K+1 target
  // distributions q(x | x_1..x_n), q(x | .., d_1), .., q(x | .., d_K) (Algorithm 1)
  int32_t* htok = e->hidx;
  for (int32_t t = 0; t <= K; t++) {
    htok[t] = t == 0 ? q->last : draft_tok[t - 1];
    e->hidx[S + t] = q->slot;
    e->hidx[2 * S + t] = q->pos + t;
    e->hidx[3 * S + t] = t;
  }
  for (int32_t t = 0; t < K; t++) e->hu[t] = u_acc[t];
  cudaStream_t st = (cudaStream_t)stream;
  if_status r = engine_forward(e, K + 1, K + 1, st);
  if (r) return r;
  if (K > 0 && cudaMemcpyAsync(e->u_dev, e->hu, K * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return check_launch("if_engine_verify: uniforms");
  // draft tokens: rows 0..K-1 of the index block hold [last, d_1..] -> d_t is idx[t+1]
  r = if_spec_verify(K, e->cfg.vocab, e->logits, draft_probs, e->idx + 1, e->u_dev, u_smp, is_top, top_k, top_p,
                     e->tok, e->tok + 72, stream);
  if (r) return r;
  if (cudaMemcpyAsync(e->htok, e->tok, 80 * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return check_launch("if_engine_verify: download");
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("if_engine_verify: step");
  const int32_t n = e->htok[72];
  if (n < 1 || n > K + 1) return set_error(IF_ERR_CUDA, "if_engine_verify: verification returned %d", n);
  e->last_rows = K + 1;
  for (int32_t i = 0; i <= K; i++) e->last_ids[i] = q->id;
  for (int32_t i = 0; i < n; i++) {
    out_tok[i] = e->htok[i];
    q->out.push_back(e->htok[i]);
  }
  // accepted drafts d_1..d_{n-1} are in the cache at pos+1..pos+n-1 (with `last` at
  // pos); the new pending token is the resampled / extra one at pos + n
  q->pos += n;
  q->last = e->htok[n - 1];
  *n_out = n;
  finish_if_done(e, q);
  if (q->phase == PH_DONE) {
    std::vector<Query*> keep;
    for (Query* a : e->active)
      if (a != q) keep.push_back(a);
    e->active.swap(keep);
  }
  return IF_OK;
}
