// api.cu — host-side C-ABI helpers: status/error plumbing, sizes, and the
// partition planner (Table 4; Q20).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>

#include "common.cuh"

namespace ifb {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

if_status set_error(if_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

if_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(IF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return IF_OK;
}

void count_launch(int n) { g_launches += n; }

}  // namespace ifb

using namespace ifb;

extern "C" const char* if_last_error(void) { return g_err; }

extern "C" int64_t if_launch_count(int32_t reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

extern "C" int64_t if_block_bytes(if_scheme s) {
  if (!scheme_ok(s)) return -1;
  return q_block_bytes(s.type, s.block);
}

extern "C" int64_t if_packed_bytes(if_scheme s, int64_t N, int64_t K) {
  if (!scheme_ok(s) || N < 0 || K < 0 || K % s.block) return -1;
  return N * (K / s.block) * (int64_t)q_block_bytes(s.type, s.block);
}

extern "C" if_status if_bits_per_weight(if_scheme s, int64_t* num, int64_t* den) {
  if (!scheme_ok(s)) return set_error(IF_ERR_SCHEME, "if_bits_per_weight: invalid scheme");
  if (!num || !den) return set_error(IF_ERR_ARG, "if_bits_per_weight: null pointer");
  // (block * bits + 2*16) / block, bits = 3.5 for Q3H stored as 7 bits per pair
  int64_t n = (int64_t)q_ncodes(s.type, s.block) * q_width(s.type) + 32, d = s.block;
  int64_t a = n, b = d;
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  *num = n / a;
  *den = d / a;
  return IF_OK;
}

// ---------------------------------------------------------------------------
// partition planner
// ---------------------------------------------------------------------------
static void balanced(int n, int p, int i, int32_t* b, int32_t* e) {
  // contiguous balanced ranges, remainder to the earlier parts
  const int base = n / p, rem = n % p;
  *b = i * base + (i < rem ? i : rem);
  *e = *b + base + (i < rem ? 1 : 0);
}

extern "C" if_status if_plan_partition(int32_t strategy, const if_stack_shape* shape, int32_t devices,
                                       int32_t stages, int32_t groups, if_plan* out) {
  if (!shape || !out) return set_error(IF_ERR_ARG, "if_plan_partition: null pointer");
  if (devices < 1 || devices > 8) return set_error(IF_ERR_ARG, "if_plan_partition: devices=%d outside 1..8", devices);
  const if_stack_shape& s = *shape;
  if (!scheme_ok(s.scheme)) return set_error(IF_ERR_SCHEME, "if_plan_partition: invalid scheme");
  if (s.layers < 1 || s.hidden < 1 || s.heads < 1 || s.kv_heads < 1 || s.head_dim < 1 || s.ffn < 1)
    return set_error(IF_ERR_SHAPE, "if_plan_partition: non-positive dimension");
  if (s.heads % s.kv_heads || s.hidden % 64 || (s.heads * s.head_dim) % 64 || s.ffn % 64)
    return set_error(IF_ERR_SHAPE, "if_plan_partition: dims must be multiples of 64 and H %% G == 0");
  if (strategy == IF_BY_LAYER) {
    stages = devices;  // each device a layer range, all heads
    groups = 1;
  } else if (strategy == IF_BY_TENSOR) {
    stages = 1;  // every device all layers, tensors split
    groups = devices;
  } else if (strategy == IF_HYBRID) {
    if (stages < 1 || groups < 1 || stages * groups != devices)  // S:615 grid error
      return set_error(IF_ERR_GRID, "if_plan_partition: stages(%d) x groups(%d) != devices(%d)", stages, groups, devices);
  } else {
    return set_error(IF_ERR_ARG, "if_plan_partition: unknown strategy %d", strategy);
  }
  const int ffn_blocks = s.ffn / 64;
  if (s.layers < stages) return set_error(IF_ERR_PLAN, "if_plan_partition: layers(%d) < stages(%d)", s.layers, stages);
  if (s.heads % groups || s.kv_heads % groups || ffn_blocks < groups)
    return set_error(IF_ERR_PLAN, "if_plan_partition: heads(%d)/kv_heads(%d) not divisible by groups(%d)", s.heads,
                     s.kv_heads, groups);
  memset(out, 0, sizeof(*out));
  out->strategy = strategy;
  out->devices = devices;
  out->stages = stages;
  out->groups = groups;
  for (int d = 0; d < devices; d++) {
    if_assignment& a = out->a[d];
    a.rank = d;
    a.stage = d / groups;  // Table 4: ranks of a stage are adjacent
    a.group_rank = d % groups;
    balanced(s.layers, stages, a.stage, &a.layer_begin, &a.layer_end);
    balanced(s.heads, groups, a.group_rank, &a.head_begin, &a.head_end);
    balanced(s.kv_heads, groups, a.group_rank, &a.kv_begin, &a.kv_end);
    balanced(ffn_blocks, groups, a.group_rank, &a.ffn_blk_begin, &a.ffn_blk_end);
    // W_o is split along K by heads (row-parallel): each rank's column
    // range must start and end on a quantization-block boundary, or its shard
    // would not be a whole-block slice of the packed tensor
    if (((int64_t)a.head_begin * s.head_dim) % s.scheme.block || ((int64_t)a.head_end * s.head_dim) % s.scheme.block)
      return set_error(IF_ERR_PLAN,
                       "if_plan_partition: rank %d head range [%d,%d) x head_dim %d is not a multiple of block %d", d,
                       a.head_begin, a.head_end, s.head_dim, s.scheme.block);
  }
  return IF_OK;
}
