// decode_mk.cuh — interface of the persistent Q3H_B64 batch-1 decode engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/if_b200.h"

namespace ifb {

constexpr int MK_MAXL = 128;  // layers per stage handled by one launch
constexpr int MK_MAXG = 160;  // >= CTAs in the grid (one per SM)
enum { MK_MODE_STACK = 0, MK_MODE_GEMV = 1 };

struct MkParams {
  int mode;
  int layers;
  int d, nq, nqkv, lf, hd, lh, lkv, h0, k0, per;
  float* h;         // [d] residual stream, updated in place
  float* qkv;       // [nqkv]
  float* act;       // [lf] silu(g)*u, written by the gate/up epilogue
  float* last_qkv;  // nullable
  // Phase dependencies without fences (see decode_mk.cu, "images"): done[p]
  // counts CTAs past phase p over all launches (G per launch), epoch = completed
  // launches.  Both live in the caller's workspace, zero-filled once before use.
  int* done;  // [4 * MK_MAXL]
  uint32_t* epoch;
  // phase inputs pre-transformed by the producing epilogues (xs layout, float4
  // [16][xstride]) and the per-CTA sum-h^2 partials for RMSNorm
  float4* xs_h;
  float4* xs_ctx;
  float4* xs_act;
  float* ssq;
  // standalone GEMV (MK_MODE_GEMV): y (+)= W x
  const float* x_in;
  float* y_out;
  int gemv_N, gemv_K, acc;
  // filled by mk_launch
  int nslot, nbp_max, raw_max, xstride;  // nbp_max / xstride: the staged input in shared memory (one K-segment)
  int xg;      // float4 row stride of the global phase images (whole K)
  // tensor parallelism inside the engine ("merged twice"): the o / down
  // epilogues push their partial rows to every group peer's exchange region and sum
  // the group's partials in rank order (bit-identical on every rank).  tp = 1: off.
  int tp, tp_me, tp_hidden;
  float* tp_box[8];  // exchange regions of the group members (group-rank order; [me] = own)
  int grid;          // CTAs per launch (0 = one per SM); ranks sharing one GPU split the SMs
  int qt, bs;        // scheme (if_qtype, block): 35/64 = the 3.5-bit engine; k-bit schemes too
  // partial launches (KV attention between the qkv and o phases, stack.cu): phases
  // [p_begin, p_end) of the stack; the first one stages its input from x_first (or h),
  // a final qkv phase writes its rows to qkv_out, o/down always write h, and only the
  // launch that ends the stack advances the epoch.  part = 0: the whole stack.
  int part, p_begin, p_end;
  const float* x_first;
  float* qkv_out;
  int seg_nb;  // K-segment length in 64-blocks (multiple of 32); 0 = whole rows
  // readers start staging a phase input once all but `early` CTAs signalled the previous
  // phase (the parity tags catch the late words; no writer can be a version ahead, see
  // decode_mk.cu); 0 = wait for every CTA
  int early;
  unsigned long long* dbg;  // nullable: per-CTA %globaltimer stamps [G][nphase][8] (instrumentation)
  const uint8_t* w[MK_MAXL][4];  // qkv, o, gu (gate/up rows interleaved), down per layer
};

if_status mk_launch(MkParams& P, cudaStream_t st);

}  // namespace ifb
