// Device RNG: the reference's seed tree and numpy's Generator(PCG64) streams.
//
//  * child_seed  -- src/rng.py:15-19: first 8 bytes (LE) of SHA-256 over
//                   "{parent}:{label}..." (single 64-byte block, messages < 56 B)
//  * SeedSequence + PCG64 seeding -- numpy/random/bit_generator.pyx,
//                   pcg64.c pcg_setseq_128_srandom_r
//  * next64 / next32 (persistent half buffer) / random / uniform /
//    integers (Lemire 32/64) / interval (masked rejection) -- numpy
//    distributions.c; restated in oracle/rng.py:PCG64Emu and checked
//    against the reference's numpy draws in tests/golden/rng_kat.npz.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace cw {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- SHA-256
__device__ __constant__ uint32_t kSha256K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

CW_DEV uint32_t rotr32(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

// SHA-256 of msg[0..len) (len <= 55), returns the first 8 digest bytes as LE u64.
CW_DEV uint64_t sha256_first8_le(const uint8_t* msg, int len) {
  uint32_t w[64];
  for (int i = 0; i < 16; ++i) w[i] = 0;
  for (int i = 0; i < len; ++i) w[i >> 2] |= (uint32_t)msg[i] << (24 - 8 * (i & 3));
  w[len >> 2] |= 0x80u << (24 - 8 * (len & 3));
  w[15] = (uint32_t)len * 8u;
  for (int i = 16; i < 64; ++i) {
    uint32_t s0 = rotr32(w[i - 15], 7) ^ rotr32(w[i - 15], 18) ^ (w[i - 15] >> 3);
    uint32_t s1 = rotr32(w[i - 2], 17) ^ rotr32(w[i - 2], 19) ^ (w[i - 2] >> 10);
    w[i] = w[i - 16] + s0 + w[i - 7] + s1;
  }
  uint32_t a = 0x6a09e667, b = 0xbb67ae85, c = 0x3c6ef372, d = 0xa54ff53a;
  uint32_t e = 0x510e527f, f = 0x9b05688c, g = 0x1f83d9ab, h = 0x5be0cd19;
  for (int i = 0; i < 64; ++i) {
    uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
    uint32_t ch = (e & f) ^ (~e & g);
    uint32_t t1 = h + S1 + ch + kSha256K[i] + w[i];
    uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
    uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
    uint32_t t2 = S0 + mj;
    h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  uint32_t h0 = 0x6a09e667 + a, h1 = 0xbb67ae85 + b;
  // digest bytes are big-endian words; take bytes 0..7 little-endian
  uint64_t out = 0;
  uint32_t hw[2] = {h0, h1};
  for (int i = 0; i < 8; ++i) {
    uint64_t byte = (hw[i >> 2] >> (24 - 8 * (i & 3))) & 0xff;
    out |= byte << (8 * i);
  }
  return out;
}

CW_DEV int fmt_u64(uint8_t* dst, uint64_t v) {
  uint8_t tmp[20];
  int n = 0;
  do { tmp[n++] = (uint8_t)('0' + v % 10); v /= 10; } while (v);
  for (int i = 0; i < n; ++i) dst[i] = tmp[n - 1 - i];
  return n;
}

CW_DEV int fmt_str(uint8_t* dst, const char* s) {
  int n = 0;
  while (s[n]) { dst[n] = (uint8_t)s[n]; ++n; }
  return n;
}

// child_seed(parent, label) and child_seed(parent, label, k)
CW_DEV uint64_t child_seed(uint64_t parent, const char* label) {
  uint8_t m[64];
  int n = fmt_u64(m, parent);
  m[n++] = ':';
  n += fmt_str(m + n, label);
  return sha256_first8_le(m, n);
}
CW_DEV uint64_t child_seed(uint64_t parent, const char* label, uint64_t k) {
  uint8_t m[64];
  int n = fmt_u64(m, parent);
  m[n++] = ':';
  n += fmt_str(m + n, label);
  m[n++] = ':';
  n += fmt_u64(m + n, k);
  return sha256_first8_le(m, n);
}

// ---------------------------------------------------------------- PCG64
struct Pcg64 {
  u128 state;
  u128 inc;
  uint32_t buf32;
  uint32_t has32;
};

// Plain-old-data mirror used in global memory (u128 is 16-B aligned anyway).
struct Pcg64Raw {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint32_t buf32, has32;
  uint32_t pad[2];
};

CW_DEV Pcg64 pcg_load(const Pcg64Raw& r) {
  Pcg64 p;
  p.state = ((u128)r.s_hi << 64) | r.s_lo;
  p.inc = ((u128)r.i_hi << 64) | r.i_lo;
  p.buf32 = r.buf32;
  p.has32 = r.has32;
  return p;
}
CW_DEV void pcg_store(Pcg64Raw& r, const Pcg64& p) {
  r.s_hi = (uint64_t)(p.state >> 64);
  r.s_lo = (uint64_t)p.state;
  r.i_hi = (uint64_t)(p.inc >> 64);
  r.i_lo = (uint64_t)p.inc;
  r.buf32 = p.buf32;
  r.has32 = p.has32;
}

CW_DEV u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// numpy SeedSequence(entropy).generate_state(4, uint64) + pcg64_set_seed.
CW_DEV Pcg64 pcg_seed(uint64_t entropy) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t ent[2] = {(uint32_t)entropy, (uint32_t)(entropy >> 32)};
  int n_ent = (entropy >> 32) ? 2 : 1;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [&](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  uint32_t st[8];
  uint32_t h = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ h;
    h *= MULT_B;
    v *= h;
    st[i] = v ^ (v >> 16);
  }
  uint64_t v0 = st[0] | ((uint64_t)st[1] << 32), v1 = st[2] | ((uint64_t)st[3] << 32);
  uint64_t v2 = st[4] | ((uint64_t)st[5] << 32), v3 = st[6] | ((uint64_t)st[7] << 32);
  u128 initstate = ((u128)v0 << 64) | v1;
  u128 initseq = ((u128)v2 << 64) | v3;
  Pcg64 p;
  p.inc = (initseq << 1) | 1;
  p.state = 0;
  p.state = p.state * pcg_mult() + p.inc;
  p.state += initstate;
  p.state = p.state * pcg_mult() + p.inc;
  p.buf32 = 0;
  p.has32 = 0;
  return p;
}

// make_rng(seed, label) (src/rng.py:22-26)
CW_DEV Pcg64 make_rng(uint64_t seed, const char* label) { return pcg_seed(child_seed(seed, label)); }

// LCG jump-ahead by `delta` steps (numpy pcg64 advance: Brown's algorithm).
CW_DEV void pcg_jump_coeffs(u128 delta, u128& mult, u128& plus, u128 inc) {
  u128 acc_m = 1, acc_p = 0, cur_m = pcg_mult(), cur_p = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  mult = acc_m;
  plus = acc_p;
}

CW_DEV uint64_t xsl_rr(u128 state) {
  uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

CW_DEV uint64_t next64(Pcg64& p) {
  p.state = p.state * pcg_mult() + p.inc;
  uint64_t hi = (uint64_t)(p.state >> 64), lo = (uint64_t)p.state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

CW_DEV uint32_t next32(Pcg64& p) {
  if (p.has32) { p.has32 = 0; return p.buf32; }
  uint64_t v = next64(p);
  p.has32 = 1;
  p.buf32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

CW_DEV double next_double(Pcg64& p) { return (double)(next64(p) >> 11) * (1.0 / 9007199254740992.0); }

// Generator.uniform(lo, hi) = lo + (hi - lo) * random()
CW_DEV double uniform(Pcg64& p, double lo, double hi) {
  double span = hi - lo;
  return lo + span * next_double(p);
}

// Generator.integers(0, n) for 1 <= n <= 2^32 (Lemire on next32)
CW_DEV uint32_t integers32(Pcg64& p, uint64_t n) {
  uint64_t rng = n - 1;
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFull) return next32(p);
  uint32_t excl = (uint32_t)(rng + 1);
  uint64_t m = (uint64_t)next32(p) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    uint32_t thr = (uint32_t)((0xFFFFFFFFu - (uint32_t)rng) % excl);
    while (left < thr) {
      m = (uint64_t)next32(p) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// Generator.integers(2**63) == next64 >> 1 (Lemire-64 with a power-of-two range)
CW_DEV uint64_t integers_2p63(Pcg64& p) { return next64(p) >> 1; }

// numpy random_interval(bitgen, max) for max < 2^32 (Fisher-Yates draw)
CW_DEV uint32_t interval32(Pcg64& p, uint32_t mx) {
  if (mx == 0) return 0;
  uint32_t mask = mx;
  mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
  uint32_t v;
  do { v = next32(p) & mask; } while (v > mx);
  return v;
}

}  // namespace cw
