/*
 * oracle.c — plain, slow, obviously-correct CPU oracle (C99, single thread).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * bench.py cpu_baseline / --impl reference leg, never by the product path.
 * Built with  -O2 -ffp-contract=off -fno-fast-math  so every float operation
 * below is one IEEE binary32 operation in round-to-nearest-even, exactly as
 * written (Q4).  Shares no code with the CUDA path.
 *
 * Every function follows the paper step by step:
 *   Eq. 1  q = Round((w - min)/(max - min) * (2^k - 1))
 *   Eq. 2  w' = q/(2^k - 1) * (max - min) + min
 *   3.5-bit D = 10, pair code q_{2i}*11 + q_{2i+1}, decode
 *                       floor(q/11), q mod 11
 *   two FP16 numbers per block, block sizes
 *   partition strategies (Table 4)
 *   grouped-query attention over a KV cache with RoPE (Table 1)
 * Readings where the paper is silent are numbered Q1..Q24 in DESIGN.md.
 *
 * Parity pins (tests/test_oracle_*.py): Table 2 codes/w'/averages, Table 3
 * bits/weight, exhaustive pair code, half-step bound, containment, brute-force
 * integer matmuls, Table 4 plan, virtual-partition equivalence.  The stack
 * composition (ref_stack_f64, Q18) has no printed values in the paper:
 * "parity unpinned" by the paper; pinned only by special cases (zero weights
 * → identity, 1-layer hand composition, partition replay equivalence).
 * ref_stack_kv_f64 (Q24) is pinned by tests/test_oracle_attention.py: position 0
 * == ref_stack_f64 bitwise, RoPE rotation law, uniform keys -> mean of values,
 * chunk == token-by-token, batching transparency.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define REF_MAX_BLOCK 4096 /* longest block accepted (tensor blocks are 32/64; test mode any) */

/* ------------------------------------------------------------------------ */
/* scheme                                                                   */
/* ------------------------------------------------------------------------ */

/* k-bit schemes of P:118 ("2, 3, 4, 5, 6, and 8") plus Q3H ("3.5-bit"). */
int ref_scheme_valid(int qtype, int block) {
  int ok_type = (qtype == 2 || qtype == 3 || qtype == 4 || qtype == 5 || qtype == 6 ||
                 qtype == 8 || qtype == 35);
  int ok_block = (block == 32 || block == 64);
  return ok_type && ok_block;
}

/* Levels D: 2^k - 1 (Eq. 1); 10 for 3.5-bit. */
int ref_levels(int qtype) {
  if (qtype == 35) return 10;
  return (1 << qtype) - 1;
}

/* Width in bits of one stored code: k for k-bit; 7 per *pair* for Q3H. */
static int code_width(int qtype) { return qtype == 35 ? 7 : qtype; }
/* Number of stored codes for n weights. */
static int n_codes(int qtype, int n) { return qtype == 35 ? n / 2 : n; }

/* ceil(n * bits / 8): tight packing. For Q3H: (n/2)*7 bits. */
int64_t ref_code_bytes(int qtype, int n) {
  int64_t bits = (int64_t)n_codes(qtype, n) * code_width(qtype);
  return (bits + 7) / 8;
}

/* two FP16 numbers stored per block = 4 bytes. */
int64_t ref_block_bytes(int qtype, int block) { return ref_code_bytes(qtype, block) + 4; }

/* Actual bits/weight = (block*bits + 2*16) / block; reduced fraction. */
void ref_bits_per_weight(int qtype, int block, int64_t* num, int64_t* den) {
  int64_t n = (int64_t)n_codes(qtype, block) * code_width(qtype) + 32;
  int64_t d = block;
  int64_t a = n, b = d;
  while (b) { int64_t t = a % b; a = b; b = t; }
  *num = n / a;
  *den = d / a;
}

/* ------------------------------------------------------------------------ */
/* binary16, written out by hand (Q3: directed rounding of min/max)          */
/* ------------------------------------------------------------------------ */

/* Convert binary32 -> binary16, rounding the *value* down (dir<0) or up (dir>0). */
static uint16_t f32_to_f16_directed(float f, int dir) {
  uint32_t u;
  memcpy(&u, &f, 4);
  uint32_t sign = u >> 31;
  uint32_t e8 = (u >> 23) & 0xFFu;
  uint32_t man = u & 0x7FFFFFu;
  uint16_t s16 = (uint16_t)(sign << 15);
  if (e8 == 0xFFu) { /* inf / nan */
    if (man) return 0x7E00u;
    return (uint16_t)(s16 | 0x7C00u);
  }
  if (e8 == 0 && man == 0) return s16; /* signed zero kept */
  /* magnitude rounded up iff (round-up and positive) or (round-down and negative) */
  int mag_up = (dir > 0) ? !sign : sign;
  /* |f| = M * 2^E with integer M */
  uint32_t M = e8 ? (man | 0x800000u) : man;
  int E = e8 ? (int)e8 - 150 : -149;
  /* floor(log2 |f|) */
  int top = 31;
  while (!((M >> top) & 1u)) top--;
  int ef = E + top;
  if (ef > 15) { /* beyond binary16 range */
    return (uint16_t)(s16 | (mag_up ? 0x7C00u : 0x7BFFu));
  }
  int ulp = (ef < -14 ? -14 : ef) - 10; /* exponent of one binary16 ulp at |f| */
  uint32_t q;
  int exact;
  int sh = ulp - E;
  if (sh <= 0) {
    q = M << (-sh);
    exact = 1;
  } else if (sh >= 32) {
    q = 0;
    exact = 0; /* M != 0 */
  } else {
    q = M >> sh;
    exact = (M & ((1u << sh) - 1u)) == 0;
  }
  if (!exact && mag_up) q += 1;
  uint32_t bits;
  if (ef < -14) {
    bits = q; /* subnormal (q == 1024 carries into the smallest normal) */
  } else {
    bits = ((uint32_t)(ef + 15) << 10) + q - 1024u; /* carry of q==2048 bumps exponent */
  }
  return (uint16_t)(s16 | bits);
}

uint16_t ref_f32_to_f16_rd(float f) { return f32_to_f16_directed(f, -1); }
uint16_t ref_f32_to_f16_ru(float f) { return f32_to_f16_directed(f, +1); }

float ref_f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h >> 15);
  uint32_t e5 = (h >> 10) & 0x1Fu;
  uint32_t m10 = h & 0x3FFu;
  double mag;
  if (e5 == 0x1Fu) {
    mag = m10 ? NAN : INFINITY;
  } else if (e5 == 0) {
    mag = ldexp((double)m10, -24);
  } else {
    mag = ldexp((double)(m10 + 1024u), (int)e5 - 25);
  }
  return (float)(sign ? -mag : mag); /* exact: binary16 ⊂ binary32 */
}

/* ------------------------------------------------------------------------ */
/* 3.5-bit pair code                                             */
/* ------------------------------------------------------------------------ */

int ref_pack_pair(int q_even, int q_odd) {
  if (q_even < 0 || q_even > 10 || q_odd < 0 || q_odd > 10) return -1;
  return q_even * 11 + q_odd; /* q = q_{2i} x 11 + q_{2i+1} */
}

int ref_unpack_pair(int v, int* q_first, int* q_second) {
  if (v < 0 || v > 120) return 5; /* value beyond the 121 valid codes */
  *q_first = v / 11;  /* floor(q/11) */
  *q_second = v % 11; /* q mod 11 */
  return 0;
}

/* ------------------------------------------------------------------------ */
/* bit stream: code j occupies bits [j*c, (j+1)*c), LSB-first (Q11)   */
/* ------------------------------------------------------------------------ */

static void put_bits(uint8_t* area, int64_t bitpos, int width, uint32_t value) {
  /* width <= 8: the field lies in byte bitpos/8 and possibly the next one */
  int64_t byte = bitpos / 8;
  int off = (int)(bitpos % 8);
  uint32_t window = (value & ((1u << width) - 1u)) << off;
  area[byte] |= (uint8_t)(window & 0xFFu);
  if (off + width > 8) area[byte + 1] |= (uint8_t)(window >> 8);
}

static uint32_t get_bits(const uint8_t* area, int64_t bitpos, int width) {
  /* width <= 8: the field lies in byte bitpos/8 and possibly the next one */
  int64_t byte = bitpos / 8;
  int off = (int)(bitpos % 8);
  uint32_t window = area[byte];
  if (off + width > 8) window |= (uint32_t)area[byte + 1] << 8;
  return (window >> off) & ((1u << width) - 1u);
}

/* ------------------------------------------------------------------------ */
/* one block                                                                */
/* ------------------------------------------------------------------------ */

/* Eq. 1; 3.5-bit variant.  Reading of every silent
 * point: Q1 round-half-away (roundf), Q2 (min,max) as the two fp16, Q3 RD/RU,
 * Q4 binary32 ((w-lo)/r)*D, Q6 r==0 -> q=0, Q7 -0 -> +0, Q8 non-finite error,
 * Q12 header [lo16][hi16] then codes. */
int ref_quantize_block(int qtype, int n, const float* w, uint8_t* out) {
  if (!(qtype == 2 || qtype == 3 || qtype == 4 || qtype == 5 || qtype == 6 || qtype == 8 ||
        qtype == 35))
    return 3;
  if (n < 1 || n > REF_MAX_BLOCK || (qtype == 35 && (n % 2) != 0)) return 3;
  const int D = ref_levels(qtype);
  /* step 1: finite inputs only */
  for (int i = 0; i < n; i++)
    if (!isfinite(w[i])) return 4;
  /* step 2: min(w), max(w) of the block, -0 canonicalised to +0 (Q7) */
  float m = w[0], M = w[0];
  for (int i = 1; i < n; i++) {
    if (w[i] < m) m = w[i];
    if (w[i] > M) M = w[i];
  }
  m = m + 0.0f;
  M = M + 0.0f;
  /* step 3: the two FP16 numbers, directed so that lo <= w <= hi (Q3) */
  uint16_t lo16 = ref_f32_to_f16_rd(m);
  uint16_t hi16 = ref_f32_to_f16_ru(M);
  if ((lo16 & 0x7C00u) == 0x7C00u || (hi16 & 0x7C00u) == 0x7C00u) return 4;
  const float lo = ref_f16_to_f32(lo16);
  const float hi = ref_f16_to_f32(hi16);
  const float r = hi - lo;
  /* step 4: q_i = Round((w_i - min)/(max - min) * D) */
  int32_t q[REF_MAX_BLOCK];
  for (int i = 0; i < n; i++) {
    if (r == 0.0f) {
      q[i] = 0; /* Q6: degenerate block */
    } else {
      float t = ((w[i] - lo) / r) * (float)D;
      float rq = roundf(t); /* Q1: half away from zero */
      if (rq < 0.0f) rq = 0.0f; /* defensive; unreachable under Q3 */
      if (rq > (float)D) rq = (float)D;
      q[i] = (int32_t)rq;
    }
  }
  /* step 5: serialise [lo16 LE][hi16 LE][codes] */
  int64_t cb = ref_code_bytes(qtype, n);
  memset(out, 0, (size_t)(4 + cb));
  out[0] = (uint8_t)(lo16 & 0xFFu);
  out[1] = (uint8_t)(lo16 >> 8);
  out[2] = (uint8_t)(hi16 & 0xFFu);
  out[3] = (uint8_t)(hi16 >> 8);
  uint8_t* area = out + 4;
  if (qtype == 35) {
    for (int j = 0; j < n / 2; j++) {
      int v = ref_pack_pair(q[2 * j], q[2 * j + 1]);
      put_bits(area, (int64_t)j * 7, 7, (uint32_t)v);
    }
  } else {
    for (int i = 0; i < n; i++) put_bits(area, (int64_t)i * qtype, qtype, (uint32_t)q[i]);
  }
  return 0;
}

int ref_block_codes(int qtype, int n, const uint8_t* in, int32_t* q_out) {
  if (n < 1 || (qtype == 35 && (n % 2) != 0)) return 3;
  const uint8_t* area = in + 4;
  if (qtype == 35) {
    for (int j = 0; j < n / 2; j++) {
      int a, b;
      int st = ref_unpack_pair((int)get_bits(area, (int64_t)j * 7, 7), &a, &b);
      if (st) return st;
      q_out[2 * j] = a;
      q_out[2 * j + 1] = b;
    }
  } else {
    for (int i = 0; i < n; i++) q_out[i] = (int32_t)get_bits(area, (int64_t)i * qtype, qtype);
  }
  return 0;
}

/* Eq. 2, as fma32(q, (hi - lo)/D, lo) (Q5). */
int ref_dequantize_block(int qtype, int n, const uint8_t* in, float* w_out) {
  if (!(qtype == 2 || qtype == 3 || qtype == 4 || qtype == 5 || qtype == 6 || qtype == 8 ||
        qtype == 35))
    return 3;
  if (n < 1 || n > REF_MAX_BLOCK) return 3;
  int32_t q[REF_MAX_BLOCK];
  int st = ref_block_codes(qtype, n, in, q);
  if (st) return st;
  uint16_t lo16 = (uint16_t)(in[0] | (in[1] << 8));
  uint16_t hi16 = (uint16_t)(in[2] | (in[3] << 8));
  const float lo = ref_f16_to_f32(lo16);
  const float hi = ref_f16_to_f32(hi16);
  const float step = (hi - lo) / (float)ref_levels(qtype);
  for (int i = 0; i < n; i++) w_out[i] = fmaf((float)q[i], step, lo);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* tensors                                                                  */
/* ------------------------------------------------------------------------ */

int ref_quantize(int qtype, int block, const float* W, int64_t N, int64_t K, uint8_t* packed) {
  if (!ref_scheme_valid(qtype, block)) return 3;
  if (N < 0 || K < 0 || K % block) return 2;
  const int64_t bb = ref_block_bytes(qtype, block);
  const int64_t nb = K / block;
  for (int64_t n = 0; n < N; n++)
    for (int64_t b = 0; b < nb; b++) {
      int st = ref_quantize_block(qtype, block, W + n * K + b * block, packed + (n * nb + b) * bb);
      if (st) return st;
    }
  return 0;
}

int ref_dequantize(int qtype, int block, const uint8_t* packed, int64_t N, int64_t K, float* W_out) {
  if (!ref_scheme_valid(qtype, block)) return 3;
  if (N < 0 || K < 0 || K % block) return 2;
  const int64_t bb = ref_block_bytes(qtype, block);
  const int64_t nb = K / block;
  for (int64_t n = 0; n < N; n++)
    for (int64_t b = 0; b < nb; b++) {
      int st = ref_dequantize_block(qtype, block, packed + (n * nb + b) * bb, W_out + n * K + b * block);
      if (st) return st;
    }
  return 0;
}

/* Y[m,n] = sum_k W'[n,k] X[m,k] in fp64 (plain definition). Rows of W'
 * are dequantized (Eq. 2, fp32) one at a time to bound memory. */
static int matmul_rows_f64(int qtype, int block, const uint8_t* packed, int64_t N, int64_t K,
                           const double* X, int64_t M, double* Y) {
  const int64_t bb = ref_block_bytes(qtype, block);
  const int64_t nb = K / block;
  float* row = (float*)malloc(sizeof(float) * (size_t)(K ? K : 1));
  for (int64_t n = 0; n < N; n++) {
    for (int64_t b = 0; b < nb; b++) {
      int st = ref_dequantize_block(qtype, block, packed + (n * nb + b) * bb, row + b * block);
      if (st) {
        free(row);
        return st;
      }
    }
    for (int64_t m = 0; m < M; m++) {
      double acc = 0.0;
      const double* x = X + m * K;
      for (int64_t k = 0; k < K; k++) acc += (double)row[k] * x[k];
      Y[m * N + n] = acc;
    }
  }
  free(row);
  return 0;
}

int ref_matmul_f64(int qtype, int block, const uint8_t* packed, int64_t N, int64_t K,
                   const float* X, int64_t M, double* Y) {
  if (!ref_scheme_valid(qtype, block)) return 3;
  if (N < 0 || K < 0 || M < 0 || K % block) return 2;
  double* Xd = (double*)malloc(sizeof(double) * (size_t)(M * K > 0 ? M * K : 1));
  for (int64_t i = 0; i < M * K; i++) Xd[i] = (double)X[i];
  int st = matmul_rows_f64(qtype, block, packed, N, K, Xd, M, Y);
  free(Xd);
  return st;
}

/* ------------------------------------------------------------------------ */
/* the stack (Q18): RMSNorm -> qkv -> single-position GQA -> o + residual ->   */
/* RMSNorm -> gate/up -> SiLU(g)*u -> down + residual                        */
/* ------------------------------------------------------------------------ */

/* rms(h) = h / sqrt(mean(h^2) + 1e-5)  (unit gain) */
static void rmsnorm_f64(const double* h, int64_t d, double* a) {
  double ss = 0.0;
  for (int64_t i = 0; i < d; i++) ss += h[i] * h[i];
  double inv = 1.0 / sqrt(ss / (double)d + 1e-5);
  for (int64_t i = 0; i < d; i++) a[i] = h[i] * inv;
}

static double silu_f64(double g) { return g / (1.0 + exp(-g)); }

static int check_shape(const ref_stack_shape* s) {
  if (!ref_scheme_valid(s->qtype, s->block)) return 3;
  if (s->layers < 0 || s->hidden <= 0 || s->heads <= 0 || s->kv_heads <= 0 || s->head_dim <= 0 ||
      s->ffn <= 0)
    return 2;
  if (s->heads % s->kv_heads) return 2;
  if (s->hidden % s->block || (s->heads * s->head_dim) % s->block || s->ffn % s->block) return 2;
  return 0;
}

int ref_stack_f64(const ref_stack_shape* s, const uint8_t* const* wqkv, const uint8_t* const* wo,
                  const uint8_t* const* wgu, const uint8_t* const* wdown, const float* h_in,
                  int64_t T, double* h_out, double* last_qkv) {
  int st = check_shape(s);
  if (st) return st;
  const int64_t d = s->hidden, H = s->heads, G = s->kv_heads, hd = s->head_dim, F = s->ffn;
  const int64_t nq = H * hd, nkv = G * hd, nqkv = nq + 2 * nkv;
  double* h = h_out;
  for (int64_t i = 0; i < T * d; i++) h[i] = (double)h_in[i];
  double* a = (double*)malloc(sizeof(double) * (size_t)(T * d));
  double* qkv = (double*)malloc(sizeof(double) * (size_t)(T * nqkv));
  double* ctx = (double*)malloc(sizeof(double) * (size_t)(T * nq));
  double* gu = (double*)malloc(sizeof(double) * (size_t)(T * 2 * F));
  double* act = (double*)malloc(sizeof(double) * (size_t)(T * F));
  double* dh = (double*)malloc(sizeof(double) * (size_t)(T * d));
  for (int l = 0; l < s->layers && !st; l++) {
    /* attention sub-layer */
    for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
    st = matmul_rows_f64(s->qtype, s->block, wqkv[l], nqkv, d, a, T, qkv);
    if (st) break;
    /* single position: softmax over one key = 1, so head i's context is the v of
     * its kv group j = floor(i / (H/G)) (contiguous groups S:393) */
    for (int64_t t = 0; t < T; t++)
      for (int64_t i = 0; i < H; i++) {
        int64_t j = i / (H / G);
        for (int64_t e = 0; e < hd; e++)
          ctx[t * nq + i * hd + e] = qkv[t * nqkv + nq + nkv + j * hd + e];
      }
    st = matmul_rows_f64(s->qtype, s->block, wo[l], d, nq, ctx, T, dh);
    if (st) break;
    for (int64_t i = 0; i < T * d; i++) h[i] += dh[i];
    /* feed-forward sub-layer */
    for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
    st = matmul_rows_f64(s->qtype, s->block, wgu[l], 2 * F, d, a, T, gu);
    if (st) break;
    for (int64_t t = 0; t < T; t++)
      for (int64_t f = 0; f < F; f++)
        act[t * F + f] = silu_f64(gu[t * 2 * F + f]) * gu[t * 2 * F + F + f];
    st = matmul_rows_f64(s->qtype, s->block, wdown[l], d, F, act, T, dh);
    if (st) break;
    for (int64_t i = 0; i < T * d; i++) h[i] += dh[i];
    if (last_qkv && l == s->layers - 1)
      memcpy(last_qkv, qkv, sizeof(double) * (size_t)(T * nqkv));
  }
  free(a);
  free(qkv);
  free(ctx);
  free(gu);
  free(act);
  free(dh);
  return st;
}

/* ------------------------------------------------------------------------ */
/* the stack with GQA decode attention over a KV cache (NEXT-1, Q24)          */
/* ------------------------------------------------------------------------ */

/* RoPE (Table 1): rotate consecutive pairs (2m, 2m+1) of one head
 * vector by the angle pos * theta_m, theta_m = 10000^(-2m/hd) */
static void rope_f64(double* x, int64_t hd, int64_t pos) {
  for (int64_t m = 0; m < hd / 2; m++) {
    double theta = pow(10000.0, -2.0 * (double)m / (double)hd);
    double ang = (double)pos * theta;
    double c = cos(ang), sn = sin(ang);
    double x0 = x[2 * m], x1 = x[2 * m + 1];
    x[2 * m] = x0 * c - x1 * sn;
    x[2 * m + 1] = x0 * sn + x1 * c;
  }
}

int ref_stack_kv_f64(const ref_stack_shape* s, const uint8_t* const* wqkv, const uint8_t* const* wo,
                     const uint8_t* const* wgu, const uint8_t* const* wdown, const float* h_in, int64_t T,
                     const int32_t* slot_ids, const int32_t* positions, int32_t slots, int32_t max_ctx,
                     double* kcache, double* vcache, double* h_out, double* last_qkv) {
  int st = check_shape(s);
  if (st) return st;
  if (s->head_dim % 2) return 2;
  for (int64_t t = 0; t < T; t++)
    if (slot_ids[t] < 0 || slot_ids[t] >= slots || positions[t] < 0 || positions[t] >= max_ctx) return 2;
  const int64_t d = s->hidden, H = s->heads, G = s->kv_heads, hd = s->head_dim, F = s->ffn;
  const int64_t nq = H * hd, nkv = G * hd, nqkv = nq + 2 * nkv;
  const int64_t per_pos = G * hd, per_slot = (int64_t)max_ctx * per_pos, per_layer = (int64_t)slots * per_slot;
  double* h = h_out;
  for (int64_t i = 0; i < T * d; i++) h[i] = (double)h_in[i];
  double* a = (double*)malloc(sizeof(double) * (size_t)(T * d));
  double* qkv = (double*)malloc(sizeof(double) * (size_t)(T * nqkv));
  double* ctx = (double*)malloc(sizeof(double) * (size_t)(T * nq));
  double* gu = (double*)malloc(sizeof(double) * (size_t)(T * 2 * F));
  double* act = (double*)malloc(sizeof(double) * (size_t)(T * F));
  double* dh = (double*)malloc(sizeof(double) * (size_t)(T * d));
  double* sc = (double*)malloc(sizeof(double) * (size_t)max_ctx);
  for (int l = 0; l < s->layers && !st; l++) {
    double* K = kcache + (int64_t)l * per_layer;
    double* V = vcache + (int64_t)l * per_layer;
    /* attention sub-layer: projections */
    for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
    st = matmul_rows_f64(s->qtype, s->block, wqkv[l], nqkv, d, a, T, qkv);
    if (st) break;
    /* RoPE on every q and k head at the token's position; append k, v to the cache */
    for (int64_t t = 0; t < T; t++) {
      double* q = qkv + t * nqkv;
      for (int64_t i = 0; i < H; i++) rope_f64(q + i * hd, hd, positions[t]);
      for (int64_t j = 0; j < G; j++) rope_f64(q + nq + j * hd, hd, positions[t]);
      double* kd = K + slot_ids[t] * per_slot + (int64_t)positions[t] * per_pos;
      double* vd = V + slot_ids[t] * per_slot + (int64_t)positions[t] * per_pos;
      for (int64_t e = 0; e < nkv; e++) {
        kd[e] = q[nq + e];
        vd[e] = q[nq + nkv + e];
      }
    }
    /* scaled dot-product attention of head i against kv group j = floor(i/(H/G)),
     * causal over the slot's positions 0..p */
    for (int64_t t = 0; t < T; t++) {
      const int64_t p = positions[t];
      const double* Ks = K + slot_ids[t] * per_slot;
      const double* Vs = V + slot_ids[t] * per_slot;
      for (int64_t i = 0; i < H; i++) {
        const int64_t j = i / (H / G);
        const double* q = qkv + t * nqkv + i * hd;
        double mx = -INFINITY;
        for (int64_t tau = 0; tau <= p; tau++) {
          double dot = 0.0;
          for (int64_t e = 0; e < hd; e++) dot += q[e] * Ks[tau * per_pos + j * hd + e];
          sc[tau] = dot / sqrt((double)hd);
          if (sc[tau] > mx) mx = sc[tau];
        }
        double den = 0.0;
        for (int64_t tau = 0; tau <= p; tau++) {
          sc[tau] = exp(sc[tau] - mx);
          den += sc[tau];
        }
        for (int64_t e = 0; e < hd; e++) {
          double acc = 0.0;
          for (int64_t tau = 0; tau <= p; tau++) acc += sc[tau] * Vs[tau * per_pos + j * hd + e];
          ctx[t * nq + i * hd + e] = acc / den;
        }
      }
    }
    st = matmul_rows_f64(s->qtype, s->block, wo[l], d, nq, ctx, T, dh);
    if (st) break;
    for (int64_t i = 0; i < T * d; i++) h[i] += dh[i];
    /* feed-forward sub-layer (as ref_stack_f64) */
    for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
    st = matmul_rows_f64(s->qtype, s->block, wgu[l], 2 * F, d, a, T, gu);
    if (st) break;
    for (int64_t t = 0; t < T; t++)
      for (int64_t f = 0; f < F; f++)
        act[t * F + f] = silu_f64(gu[t * 2 * F + f]) * gu[t * 2 * F + F + f];
    st = matmul_rows_f64(s->qtype, s->block, wdown[l], d, F, act, T, dh);
    if (st) break;
    for (int64_t i = 0; i < T * d; i++) h[i] += dh[i];
    if (last_qkv && l == s->layers - 1)
      memcpy(last_qkv, qkv, sizeof(double) * (size_t)(T * nqkv));
  }
  free(a);
  free(qkv);
  free(ctx);
  free(gu);
  free(act);
  free(dh);
  free(sc);
  return st;
}

/* ------------------------------------------------------------------------ */
/* speculative sampling: one verification round of Algorithm 1     */
/* ------------------------------------------------------------------------ */

/* q = softmax(logits) in fp64 (temperature 1) */
static void softmax_f64(const float* logits, int V, double* q) {
  double mx = -INFINITY, sum = 0.0;
  for (int i = 0; i < V; i++)
    if ((double)logits[i] > mx) mx = (double)logits[i];
  for (int i = 0; i < V; i++) {
    q[i] = exp((double)logits[i] - mx);
    sum += q[i];
  }
  for (int i = 0; i < V; i++) q[i] /= sum;
}

/* smallest index whose running sum (index order) exceeds u * total; -1 if total == 0 */
static int sample_index(const double* w, int V, double u) {
  double total = 0.0;
  for (int i = 0; i < V; i++) total += w[i];
  if (!(total > 0.0)) return -1;
  double target = u * total, run = 0.0;
  for (int i = 0; i < V; i++) {
    run += w[i];
    if (run > target) return i;
  }
  for (int i = V - 1; i >= 0; i--)
    if (w[i] > 0.0) return i; /* u -> 1 rounding: the last token with weight */
  return -1;
}

/* "the draft token is present in the top-k / top-p pools": fewer than k tokens
 * are strictly more probable, and the mass strictly more probable is below top_p */
static int in_pool(const double* q, int V, int x, int top_k, double top_p) {
  int more = 0;
  double mass = 0.0;
  for (int i = 0; i < V; i++)
    if (q[i] > q[x]) {
      more++;
      mass += q[i];
    }
  if (top_k > 0 && more >= top_k) return 0;
  if (top_p < 1.0 && mass >= top_p) return 0;
  return top_k > 0 || top_p < 1.0;
}

int ref_spec_verify(int K, int V, const float* tgt_logits, const float* draft_probs, const int32_t* draft_tok,
                    const float* u_acc, float u_smp, int is_top, int top_k, float top_p, int32_t* out_tok,
                    int32_t* n_out) {
  if (K < 0 || V < 1) return 2;
  for (int t = 0; t < K; t++)
    if (draft_tok[t] < 0 || draft_tok[t] >= V) return 2;
  double* q = (double*)malloc(sizeof(double) * (size_t)V);
  double* r = (double*)malloc(sizeof(double) * (size_t)V);
  int n = 0;
  for (int t = 0; t < K; t++) {
    softmax_f64(tgt_logits + (int64_t)t * V, V, q);
    const float* p = draft_probs + (int64_t)t * V;
    const int x = draft_tok[t];
    double ratio = (double)p[x] > 0.0 ? q[x] / (double)p[x] : 1.0;
    if (ratio > 1.0) ratio = 1.0;
    if ((is_top && in_pool(q, V, x, top_k, (double)top_p)) || (double)u_acc[t] < ratio) {
      out_tok[n++] = x; /* x_{n+t} <- draft, n <- n+1 */
      continue;
    }
    /* reject: sample x_{n+t} ~ (q - p)_+ and exit the loop */
    for (int i = 0; i < V; i++) r[i] = q[i] - (double)p[i] > 0.0 ? q[i] - (double)p[i] : 0.0;
    int y = sample_index(r, V, (double)u_smp);
    if (y < 0) y = sample_index(q, V, (double)u_smp);
    out_tok[n++] = y;
    *n_out = n;
    free(q);
    free(r);
    return 0;
  }
  /* all K accepted: one extra token from the target at position K */
  softmax_f64(tgt_logits + (int64_t)K * V, V, q);
  out_tok[n++] = sample_index(q, V, (double)u_smp);
  *n_out = n;
  free(q);
  free(r);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* language-model head: the step that turns the stack's output into the next  */
/* token (NEXT-2 "a set of next tokens"; NEXT-3 target logits,     */
/* P:362-365; reading Q27)                                                   */
/* ------------------------------------------------------------------------ */

/* logits[t, v] = sum_i W'_lm[v, i] * rms(h[t])_i: the final RMSNorm (unit gain,
 * eps 1e-5) then the output projection, block-quantized like every other
 * matrix (Eq. 2 dequantized in fp32, products and sums in fp64). */
int ref_lm_logits_f64(int qtype, int block, const uint8_t* lm, int64_t V, int64_t d, const double* h, int64_t T,
                      double* logits) {
  if (!ref_scheme_valid(qtype, block)) return 3;
  if (V < 1 || d < 1 || T < 0 || d % block) return 2;
  double* a = (double*)malloc(sizeof(double) * (size_t)(T * d > 0 ? T * d : 1));
  for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
  int st = matmul_rows_f64(qtype, block, lm, V, d, a, T, logits);
  free(a);
  return st;
}

/* greedy decoding: the first index holding the largest value */
int64_t ref_argmax_f64(const double* x, int64_t n) {
  int64_t best = 0;
  for (int64_t i = 1; i < n; i++)
    if (x[i] > x[best]) best = i;
  return n > 0 ? best : -1;
}

/* ------------------------------------------------------------------------ */
/* partition cost model (S:629-637 estimate; "merged twice"; Table 5      */
/* P:224-237; reading Q29)                                                   */
/* ------------------------------------------------------------------------ */

/* Per-token latency of one decode stream under a (stages x groups) partition:
 *   L layers, each on a 1/groups shard: t_fixed + (layer_bytes / groups) / bw
 *   + 2 merges per layer when groups > 1 ("merged twice"): t_merge[groups]
 *   + (stages - 1) stage hand-offs: t_hop
 * decode speed = 1 / latency; throughput = decode speed x min(stages, micro_batches)
 * (a filled pipeline keeps every stage busy, Q22).  Seconds, bytes, bytes/s. */
int ref_cost_estimate(int layers, int stages, int groups, double t_fixed, double layer_bytes, double bw,
                      const double* t_merge, double t_hop, int micro_batches, double* decode, double* throughput) {
  if (layers < 1 || stages < 1 || groups < 1 || groups > 8 || micro_batches < 1 || bw <= 0.0) return 2;
  double lat = (double)layers * (t_fixed + (layer_bytes / (double)groups) / bw);
  if (groups > 1) lat += 2.0 * (double)layers * t_merge[groups];
  lat += (double)(stages - 1) * t_hop;
  *decode = 1.0 / lat;
  *throughput = *decode * (double)(micro_batches < stages ? micro_batches : stages);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* partition planner (Table 4; Q20)           */
/* ------------------------------------------------------------------------ */

/* balanced contiguous split of n items into p parts, remainder to earlier parts */
static void split_range(int n, int p, int i, int32_t* b, int32_t* e) {
  int base = n / p, rem = n % p;
  int start = i * base + (i < rem ? i : rem);
  *b = start;
  *e = start + base + (i < rem ? 1 : 0);
}

int ref_plan(int strategy, int layers, int heads, int kv_heads, int ffn_blocks, int devices,
             int stages, int groups, int32_t* stage_of, int32_t* group_rank_of, int32_t* lb,
             int32_t* le, int32_t* hb, int32_t* he, int32_t* kb, int32_t* ke, int32_t* fb,
             int32_t* fe) {
  if (devices < 1 || layers < 1 || heads < 1 || kv_heads < 1 || ffn_blocks < 1) return 1;
  if (strategy == 0) { /* layer-wise: each device a layer range, all heads */
    stages = devices;
    groups = 1;
  } else if (strategy == 1) { /* tensor-wise: all layers, split tensors */
    stages = 1;
    groups = devices;
  } else if (strategy == 2) { /* hybrid: stages x groups (Table 4) */
    if (stages < 1 || groups < 1 || stages * groups != devices) return 7;
  } else {
    return 1;
  }
  if (layers < stages) return 6;
  if (heads % groups || kv_heads % groups || ffn_blocks < groups) return 6;
  for (int dev = 0; dev < devices; dev++) {
    int s = dev / groups, g = dev % groups; /* Table 4: devices of a stage are adjacent */
    stage_of[dev] = s;
    group_rank_of[dev] = g;
    split_range(layers, stages, s, &lb[dev], &le[dev]);
    split_range(heads, groups, g, &hb[dev], &he[dev]);
    split_range(kv_heads, groups, g, &kb[dev], &ke[dev]);
    split_range(ffn_blocks, groups, g, &fb[dev], &fe[dev]);
  }
  return 0;
}

/* Copy rows [r0, r1) of a packed [N, K] tensor. */
static void slice_rows(const uint8_t* p, int64_t K, int64_t bb, int block, int64_t r0, int64_t r1,
                       uint8_t* out) {
  int64_t rowb = (K / block) * bb;
  memcpy(out, p + r0 * rowb, (size_t)((r1 - r0) * rowb));
}
/* Copy column blocks [c0, c1) (in units of weights, multiples of block) of all N rows. */
static void slice_cols(const uint8_t* p, int64_t N, int64_t K, int64_t bb, int block, int64_t c0,
                       int64_t c1, uint8_t* out) {
  int64_t nb = K / block, b0 = c0 / block, b1 = c1 / block;
  for (int64_t n = 0; n < N; n++)
    memcpy(out + n * (b1 - b0) * bb, p + (n * nb + b0) * bb, (size_t)((b1 - b0) * bb));
}

int ref_stack_partitioned_f64(const ref_stack_shape* s, int strategy, int devices, int stages,
                              int groups, const uint8_t* const* wqkv, const uint8_t* const* wo,
                              const uint8_t* const* wgu, const uint8_t* const* wdown,
                              const float* h_in, int64_t T, double* h_out) {
  int st = check_shape(s);
  if (st) return st;
  const int64_t d = s->hidden, H = s->heads, G = s->kv_heads, hd = s->head_dim, F = s->ffn;
  const int64_t nq = H * hd, nkv = G * hd, nqkv = nq + 2 * nkv;
  const int GR = 64; /* FFN split granule (whole 64-weight blocks, Q20) */
  if (F % GR) return 2;
  int32_t so[8], gro[8], lb[8], le[8], hb[8], he[8], kb[8], ke[8], fb[8], fe[8];
  if (devices > 8) return 1;
  st = ref_plan(strategy, s->layers, (int)H, (int)G, (int)(F / GR), devices, stages, groups, so,
                gro, lb, le, hb, he, kb, ke, fb, fe);
  if (st) return st;
  if (strategy == 0) { stages = devices; groups = 1; }
  if (strategy == 1) { stages = 1; groups = devices; }
  const int64_t bb = ref_block_bytes(s->qtype, s->block);
  double* h = h_out;
  for (int64_t i = 0; i < T * d; i++) h[i] = (double)h_in[i];
  double* a = (double*)malloc(sizeof(double) * (size_t)(T * d));
  double* dh = (double*)malloc(sizeof(double) * (size_t)(T * d));
  double* part = (double*)malloc(sizeof(double) * (size_t)(T * d));
  size_t maxw = (size_t)((nqkv * d > 2 * F * d ? nqkv * d : 2 * F * d) / s->block * bb);
  uint8_t* shard = (uint8_t*)malloc(maxw);
  uint8_t* shard2 = (uint8_t*)malloc(maxw);
  double* qkv = (double*)malloc(sizeof(double) * (size_t)(T * nqkv));
  double* ctx = (double*)malloc(sizeof(double) * (size_t)(T * nq));
  double* gu = (double*)malloc(sizeof(double) * (size_t)(T * 2 * F));
  double* act = (double*)malloc(sizeof(double) * (size_t)(T * F));
  for (int sg = 0; sg < stages && !st; sg++) {
    int dev0 = sg * groups;
    /* stage hand-off: h simply flows into the next stage's layers */
    for (int l = lb[dev0]; l < le[dev0] && !st; l++) {
      /* ---- attention sub-layer: every TP rank computes a partial of W_o ctx ---- */
      for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
      for (int64_t i = 0; i < T * d; i++) dh[i] = 0.0;
      for (int g = 0; g < groups && !st; g++) {
        int dev = dev0 + g;
        int64_t h0 = hb[dev], h1 = he[dev], k0 = kb[dev], k1 = ke[dev];
        int64_t lq = (h1 - h0) * hd, lkv = (k1 - k0) * hd, lqkv = lq + 2 * lkv;
        /* column shard of qkv: q rows of my heads, k and v rows of my kv heads */
        int64_t rowb = (d / s->block) * bb;
        slice_rows(wqkv[l], d, bb, s->block, h0 * hd, h1 * hd, shard);
        slice_rows(wqkv[l], d, bb, s->block, nq + k0 * hd, nq + k1 * hd, shard + lq * rowb);
        slice_rows(wqkv[l], d, bb, s->block, nq + nkv + k0 * hd, nq + nkv + k1 * hd,
                   shard + (lq + lkv) * rowb);
        double* lqkvb = (double*)malloc(sizeof(double) * (size_t)(T * lqkv));
        st = matmul_rows_f64(s->qtype, s->block, shard, lqkv, d, a, T, lqkvb);
        if (st) { free(lqkvb); break; }
        /* local heads read local kv heads (contiguous groups align with the split) */
        int64_t per = H / G;
        double* lctx = (double*)malloc(sizeof(double) * (size_t)(T * lq));
        for (int64_t t = 0; t < T; t++)
          for (int64_t i = h0; i < h1; i++) {
            int64_t j = i / per - k0;
            for (int64_t e = 0; e < hd; e++)
              lctx[t * lq + (i - h0) * hd + e] = lqkvb[t * lqkv + lq + lkv + j * hd + e];
          }
        /* row (K) shard of o: columns of my heads */
        slice_cols(wo[l], d, nq, bb, s->block, h0 * hd, h1 * hd, shard2);
        st = matmul_rows_f64(s->qtype, s->block, shard2, d, lq, lctx, T, part);
        for (int64_t i = 0; i < T * d; i++) dh[i] += part[i]; /* merge #1 */
        free(lctx);
        free(lqkvb);
      }
      if (st) break;
      for (int64_t i = 0; i < T * d; i++) h[i] += dh[i];
      /* ---- feed-forward sub-layer ---- */
      for (int64_t t = 0; t < T; t++) rmsnorm_f64(h + t * d, d, a + t * d);
      for (int64_t i = 0; i < T * d; i++) dh[i] = 0.0;
      for (int g = 0; g < groups && !st; g++) {
        int dev = dev0 + g;
        int64_t f0 = (int64_t)fb[dev] * GR, f1 = (int64_t)fe[dev] * GR, lf = f1 - f0;
        int64_t rowb = (d / s->block) * bb;
        slice_rows(wgu[l], d, bb, s->block, f0, f1, shard);
        slice_rows(wgu[l], d, bb, s->block, F + f0, F + f1, shard + lf * rowb);
        st = matmul_rows_f64(s->qtype, s->block, shard, 2 * lf, d, a, T, gu);
        if (st) break;
        for (int64_t t = 0; t < T; t++)
          for (int64_t f = 0; f < lf; f++)
            act[t * lf + f] = silu_f64(gu[t * 2 * lf + f]) * gu[t * 2 * lf + lf + f];
        slice_cols(wdown[l], d, F, bb, s->block, f0, f1, shard2);
        st = matmul_rows_f64(s->qtype, s->block, shard2, d, lf, act, T, part);
        for (int64_t i = 0; i < T * d; i++) dh[i] += part[i]; /* merge #2 */
      }
      if (st) break;
      for (int64_t i = 0; i < T * d; i++) h[i] += dh[i];
    }
  }
  free(a);
  free(dh);
  free(part);
  free(shard);
  free(shard2);
  free(qkv);
  free(ctx);
  free(gu);
  free(act);
  return st;
}
