// mk_scheme.cuh — the k-bit schemes ("2, 3, 4, 5, 6, and 8" bits; block sizes
// 32/64) in the persistent decode engine (decode_mk.cu).  The engine's phase
// structure (ring, images, hand-offs, epilogues) is scheme-independent; what depends on
// the scheme is how a block's codes meet the staged input:
//
//   code k of a block (w bits, LSB-first from bit k*w of the code area) is masked
//   out of a 32-bit source -- a code word, or a funnel-shifted view of two -- at bit
//   position s_k <= 24 - w, where the masked bits ARE the float c_k * 2^(s_k - 149)
//   (exponent field 0 or 1: subnormal / smallest normal, the value is continuous).  With
//   the staged input X_k = x_k * 2^(85 - s_k) one FFMA accumulates c_k x_k * 2^-64, and
//   w' = lo + c * (hi - lo) / D (Eq. 2) gives  y = lo * sum(x) + step * sum(c x).
//
// Cost per weight and row: one LOP3 (mask) + half an FFMA2 (two rows per FFMA2), plus
// one funnel shift per view (codes that straddle or sit above bit 24 - w).
#pragma once
#include <stdint.h>

#include "simd.cuh"

namespace ifb {

template <int W, int BS>
struct GkTab {
  int view[BS];      // -1: the code sits in code word `word`; else the index of its view
  int word[BS];      // code-area word (0-based) of a direct code
  int pos[BS];       // bit position s_k of the code in its source
  int view_bit[BS];  // stream bit at bit 0 of view v
  int nview;
};

template <int W, int BS>
constexpr GkTab<W, BS> gk_tab() {
  GkTab<W, BS> t{};
  t.nview = 0;
  int cur = -1;
  for (int k = 0; k < BS; k++) {
    const int bit = k * W, wi = bit / 32, s = bit % 32;
    if (s + W <= 24) {
      t.view[k] = -1;
      t.word[k] = wi;
      t.pos[k] = s;
    } else {
      if (cur < 0 || bit + W - cur > 24) {
        t.view_bit[t.nview++] = bit;
        cur = bit;
      }
      t.view[k] = t.nview - 1;
      t.word[k] = 0;
      t.pos[k] = bit - cur;
    }
  }
  return t;
}

template <int W, int BS>
struct GkScheme {
  static constexpr int NQ = BS / 4;                  // staged quads per block
  static constexpr int CODE_BYTES = BS * W / 8;      // k-bit schemes: whole bytes for BS 32/64
  static constexpr int BB = 4 + CODE_BYTES;          // block bytes
  static constexpr int NW = BB / 4;                  // 32-bit words (header + codes)
  static constexpr int D = (1 << W) - 1;             // levels (Eq. 1)
  static constexpr int NV = gk_tab<W, BS>().nview;
  static constexpr int RMAX = NW <= 9 ? 4 : 2;       // rows per unit (register budget)
};

// compile-time table entries (kept out of device storage: each is a constant)
template <int W, int BS, int K>
struct GkSrc {
  static constexpr GkTab<W, BS> t = gk_tab<W, BS>();
  static constexpr int view = t.view[K], word = t.word[K], pos = t.pos[K];
};
template <int W, int BS, int V>
struct GkViewBit {
  static constexpr int bit = gk_tab<W, BS>().view_bit[V];
};

// view v of a block whose words are w[0] (header), w[1..NW-1] (codes), w[NW] = 0
template <int W, int BS, int V, int NWP>
__device__ __forceinline__ uint32_t gk_view(const uint32_t (&w)[NWP]) {
  constexpr int bit = GkViewBit<W, BS, V>::bit;
  constexpr int wi = 1 + bit / 32, sh = bit % 32;
  if constexpr (sh == 0) {
    return w[wi];
  } else {
    return __funnelshift_r(w[wi], w[wi + 1], sh);
  }
}

// bits of code K masked in its source: the float c_K * 2^(s_K - 149)
template <int W, int BS, int K, int NWP, int NVP>
__device__ __forceinline__ uint32_t gk_code_bits(const uint32_t (&w)[NWP], const uint32_t (&vw)[NVP]) {
  using Src = GkSrc<W, BS, K>;
  constexpr uint32_t mask = ((1u << W) - 1u) << Src::pos;
  if constexpr (Src::view < 0) {
    return w[1 + Src::word] & mask;
  } else {
    return vw[Src::view] & mask;
  }
}

}  // namespace ifb
