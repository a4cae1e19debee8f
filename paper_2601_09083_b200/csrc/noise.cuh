// noise.cuh — the counter-based Gumbel noise of srt_verify (BJ:north_star part 4;
// DESIGN.md readings O11, O12).  Every float op is an explicit round-to-nearest
// intrinsic so nvcc can neither contract nor reorder: the bits are defined by
// the operation sequence in DESIGN.md O12, not by this code.
#pragma once
#include <cstdint>

namespace srt {

// Philox4x32-10 with the cuRAND/Random123 multipliers and Weyl key bumps.
struct Philox4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return Philox4{c0, c1, c2, c3};
}

// Deterministic fp32 natural log for positive normal x (O12):
// x = m 2^e, m in [sqrt(1/2), sqrt(2)], f = m - 1, s = f/(2+f),
// log x = e ln2 + 2s + s^3 P(s^2), P = 2/3 + 2/5 z + 2/7 z^2 + 2/9 z^3 + 2/11 z^4.
__device__ __forceinline__ float log_det(float x) {
  const float C3 = __uint_as_float(0x3f2aaaabu);
  const float C5 = __uint_as_float(0x3ecccccdu);
  const float C7 = __uint_as_float(0x3e924925u);
  const float C9 = __uint_as_float(0x3e638e39u);
  const float C11 = __uint_as_float(0x3e3a2e8cu);
  const float LN2_HI = __uint_as_float(0x3f317200u);
  const float LN2_LO = __uint_as_float(0x35bfbe8eu);
  const uint32_t b = __float_as_uint(x);
  int e = (int)((b >> 23) & 0xFFu) - 127;
  uint32_t mb = (b & 0x007FFFFFu) | 0x3F800000u;
  if (mb > 0x3FB504F3u) {
    mb -= 0x00800000u;
    e += 1;
  }
  const float m = __uint_as_float(mb);
  const float f = __fsub_rn(m, 1.0f);
  const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
  const float z = __fmul_rn(s, s);
  float p = __fmaf_rn(z, C11, C9);
  p = __fmaf_rn(z, p, C7);
  p = __fmaf_rn(z, p, C5);
  p = __fmaf_rn(z, p, C3);
  const float r = __fmaf_rn(__fmul_rn(s, z), p, __fmul_rn(2.0f, s));
  const float ef = (float)e;  // exact
  return __fmaf_rn(ef, LN2_HI, __fmaf_rn(ef, LN2_LO, r));
}

// g(r) for the 23-bit noise input r = w >> 9.
__device__ __forceinline__ float gumbel_of_r(uint32_t r) {
  const float u = __fmul_rn((float)(2u * r + 1u), __uint_as_float(0x33800000u));  // (2r+1) 2^-24, exact
  return -log_det(-log_det(u));
}

// ---- the top-down Gumbel construction of the sampler (O11) ------
// Blocks of NOISE_BLK = 64 tokens; block b's maximum noise is drawn first from
// one Philox call shared by blocks 2m and 2m+1, the others are truncated below.
constexpr int NOISE_BLK = 64;

// tokens in block b of a V-token row (0 past the end)
__device__ __forceinline__ int block_len(int64_t V, int64_t b) {
  const int64_t rem = V - b * NOISE_BLK;
  return rem <= 0 ? 0 : (rem < NOISE_BLK ? (int)rem : NOISE_BLK);
}

__device__ __forceinline__ float uniform_of_word(uint32_t w) {
  return __fmul_rn((float)(2u * (w >> 9) + 1u), __uint_as_float(0x33800000u));  // exact
}

// Philox words (wa, wb) of block b
__device__ __forceinline__ void block_words(uint32_t b, uint32_t pos, uint32_t s_lo, uint32_t s_hi,
                                            uint32_t k0, uint32_t k1, uint32_t& wa,
                                            uint32_t& wb) {
  const Philox4 w = philox4x32_10(0x80000000u | (b >> 1), pos, s_lo, s_hi, k0, k1);
  wa = (b & 1) ? w.z : w.x;
  wb = (b & 1) ? w.w : w.y;
}

struct BlockNoise {
  float E;     // e^{-G}: the block's first "arrival" ~ Exp(n)/1
  float G;     // the block's maximum noise
  uint32_t p;  // its position in the block
};

__device__ __forceinline__ BlockNoise block_noise(uint32_t wa, uint32_t wb, uint32_t n) {
  const float a = -log_det(uniform_of_word(wa));
  const float E = __fdiv_rn(a, (float)n);
  const float G = -log_det(E);
  const uint32_t p = __umulhi(wb, n);
  return BlockNoise{E, G, p};
}

// g_v for element v at offset j of its block (j != bn.p):
// min(G, -log_det(RN(E + A_v))), A_v = -log_det(u(word (v&3) of Philox(v>>2, ...)))
__device__ __forceinline__ float element_noise_from_word(uint32_t w, const BlockNoise& bn) {
  const float A = -log_det(uniform_of_word(w));
  const float g = -log_det(__fadd_rn(bn.E, A));
  return g > bn.G ? bn.G : g;
}

// z = RN(RN(x / T) + g); T == 1 skips the division (O11).
__device__ __forceinline__ float perturbed(float x, float g, float temperature, bool unit_t) {
  const float xs = unit_t ? x : __fdiv_rn(x, temperature);
  return __fadd_rn(xs, g);
}

// (z, v) candidate order: larger z first, then smaller index (first maximum).
__device__ __forceinline__ bool cand_better(float z, int32_t v, float bz, int32_t bv) {
  return z > bz || (z == bz && v < bv);
}

}  // namespace srt
