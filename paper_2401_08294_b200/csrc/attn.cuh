// attn.cuh — internal interface of the KV-cache decode attention (attn.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/if_b200.h"

namespace ifb {

constexpr int ATT_MAXSPLIT = 32;  // position splits per (token, kv group)
constexpr int ATT_MAXT = 64;      // split merging (and the fp16 split) up to this many tokens

struct AttnArgs {
  float* qkv;  // [T, (lh + 2 lkv) hd] this rank's projections; q/k rotated in place
  int64_t T;
  int lh, lkv, hd;
  const int32_t* slot_ids;  // device [T]
  const int32_t* positions; // device [T]
  float* k;                 // cache base, [layers][slots][max_ctx][lkv][hd]
  float* v;
  int slots, max_ctx, layer;
  int32_t* status;          // nullable device status (IF_ERR_ARG on an out-of-range slot/position)
  float* part;              // workspace [min(T, ATT_MAXT)][lh][ATT_MAXSPLIT][hd + 2]
  uint32_t* cnt;            // workspace, zero between calls: attn_cnt_words(lkv) counters
  float* ctx;               // nullable fp32 [T, lh hd]
  __nv_bfloat16* ctx16;     // nullable bf16 [T, lh hd] (prefill)
  __half* x2;               // nullable fp16 hi/lo split [2 bp, lh hd] (batched decode)
  int bp;
  float* x2sc;              // per-token 2^-k of the split
  uint8_t* rec;             // nullable: fragment records of ctx for the fused batched chain (ms_rec.cuh)
  int rec_nt;               // token tiles of 8 per record block (1 or 2)
  float* rot_out;           // nullable [T, (lh + 2 lkv) hd]: q, k after RoPE and v (the stack's last_qkv)
  bool pdl;
};

if_status attn_run(const AttnArgs& a, cudaStream_t st);
int attn_nsplit(int64_t T, int lkv, int max_ctx);
size_t attn_cnt_words(int lkv);

}  // namespace ifb
