// Counter-indexed port of numpy's SeedSequence + PCG64 (XSL-RR 128/64), the
// RNG every seeded quantity on the TAR+RHT path comes from:
//   * derive_seed            hadamard.py:31-34   SeedSequence([job, bucket, gen])
//   * Rademacher signs       hadamard.py:49-51   PCG64(SeedSequence(seed)).integers(0,2)
//   * datagram drop coin     datagram.py:70-72,122  PCG64(SeedSequence([seed, rank])).random()
//
// Everything is usable from host and device.  "Counter-indexed" means the
// k-th output is computed directly with an LCG jump-ahead instead of by
// replaying k draws, so any GPU thread can produce any packet's coin or any
// entry's sign independently.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define OPTR_HD __host__ __device__ __forceinline__
#else
#define OPTR_HD inline
#endif

namespace optr {

typedef unsigned __int128 u128;

// PCG64 default multiplier (numpy pcg64.h PCG_DEFAULT_MULTIPLIER_128).
OPTR_HD u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

// ---------------------------------------------------------------- SeedSequence
// numpy/random/bit_generator.pyx: hashmix / mix / mix_entropy / generate_state.
struct SeedSeq {
  uint32_t pool[4];
};

OPTR_HD uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= 0x931e8875u;
  v *= *hc;
  v ^= v >> 16;
  return v;
}

OPTR_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}

// entropy: a list of non-negative integers given as u64 values; each becomes
// its little-endian u32 words ([0] for 0) and the lists are concatenated
// (bit_generator.pyx _coerce_to_uint32_array / _int_to_uint32_array).
OPTR_HD SeedSeq seedseq_from_u64(const uint64_t* ent, int n_ent) {
  uint32_t words[64];
  int nw = 0;
  for (int i = 0; i < n_ent && nw < 62; ++i) {
    uint64_t v = ent[i];
    if (v == 0) {
      words[nw++] = 0;
    } else {
      while (v) {
        words[nw++] = (uint32_t)(v & 0xffffffffu);
        v >>= 32;
      }
    }
  }
  SeedSeq s;
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) s.pool[i] = ss_hashmix(i < nw ? words[i] : 0u, &hc);
  for (int src = 0; src < 4; ++src)
    for (int dst = 0; dst < 4; ++dst)
      if (src != dst) s.pool[dst] = ss_mix(s.pool[dst], ss_hashmix(s.pool[src], &hc));
  for (int src = 4; src < nw; ++src)
    for (int dst = 0; dst < 4; ++dst) s.pool[dst] = ss_mix(s.pool[dst], ss_hashmix(words[src], &hc));
  return s;
}

// generate_state(n, uint64): 2n u32 words, paired little-endian.
OPTR_HD void seedseq_generate_u64(const SeedSeq& s, uint64_t* out, int n) {
  uint32_t hc = 0x8b51f9ddu;
  for (int i = 0; i < n; ++i) {
    uint32_t w[2];
    for (int h = 0; h < 2; ++h) {
      uint32_t v = s.pool[(2 * i + h) & 3];
      v ^= hc;
      hc *= 0x58f38dedu;
      v *= hc;
      v ^= v >> 16;
      w[h] = v;
    }
    out[i] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  }
}

// ---------------------------------------------------------------------- PCG64
struct Pcg {
  u128 state;  // seeded state (before the first output step)
  u128 inc;    // odd increment
};

// _pcg64.pyx _reset_state_variables/seed: generate_state(4, uint64) then
// pcg64_srandom_r: state=0; step; state+=initstate; step.
OPTR_HD Pcg pcg_from_seedseq(const SeedSeq& ss) {
  uint64_t v[4];
  seedseq_generate_u64(ss, v, 4);
  u128 init = ((u128)v[0] << 64) | v[1];
  u128 seq = ((u128)v[2] << 64) | v[3];
  Pcg p;
  p.inc = (seq << 1) | 1u;
  p.state = 0;
  p.state = p.state * pcg_mult() + p.inc;
  p.state += init;
  p.state = p.state * pcg_mult() + p.inc;
  return p;
}

OPTR_HD Pcg pcg_from_u64s(const uint64_t* ent, int n_ent) {
  return pcg_from_seedseq(seedseq_from_u64(ent, n_ent));
}

OPTR_HD uint64_t pcg_xsl_rr(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

OPTR_HD u128 pcg_step(u128 s, u128 inc) { return s * pcg_mult() + inc; }

// State after `k` LCG steps from `s` (Brown's jump-ahead, O(log k)).
OPTR_HD u128 pcg_advance(u128 s, u128 inc, uint64_t k) {
  u128 acc_mult = 1, acc_plus = 0;
  u128 cur_mult = pcg_mult(), cur_plus = inc;
  while (k) {
    if (k & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    k >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// k-th (0-based) 64-bit output of the generator.
OPTR_HD uint64_t pcg_output_at(const Pcg& p, uint64_t k) {
  return pcg_xsl_rr(pcg_advance(p.state, p.inc, k + 1));
}

// Generator.random(): (next_uint64 >> 11) * 2^-53 (distributions.c
// next_double).  Returns true iff the datagram coin DROPS the packet
// (datagram.py:122: rng.random() < drop_prob).
OPTR_HD bool coin_drops(uint64_t out, double p) {
  return (double)(out >> 11) * (1.0 / 9007199254740992.0) < p;
}

// Rademacher sign of entry k: integers(0, 2) draws buffered u32 halves of
// each u64 (low half first) through Lemire's bounded method with range 2,
// which returns the top bit of the u32.  +1 iff that bit is set.
OPTR_HD int sign_bit_from_output(uint64_t out, int odd) {
  return (int)((out >> (odd ? 63 : 31)) & 1u);
}

// derive_seed(job, bucket, gen) (hadamard.py:31-34).
OPTR_HD uint64_t derive_seed(uint64_t job, uint64_t bucket, uint64_t gen) {
  uint64_t e[3] = {job, bucket, gen};
  SeedSeq s = seedseq_from_u64(e, 3);
  uint64_t out;
  seedseq_generate_u64(s, &out, 1);
  return out;
}

}  // namespace optr
