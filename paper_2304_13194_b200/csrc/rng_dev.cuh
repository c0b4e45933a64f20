// rng_dev.cuh — device restatement of numpy's SeedSequence + PCG64 stream
// (see rng.h for the host twin and the algorithm references). PCG64 is an
// LCG, so the j-th output can be computed directly with an O(log j) jump
// ahead: the weak-rebalance draws of a pass are generated in parallel, one
// thread per 32-bit word, and only a Lemire rejection (probability < k/2^32
// per draw) forces a sequential redo.
#pragma once
#include <cstdint>

namespace jet {

typedef unsigned __int128 du128;

struct DevPcg {
  du128 state, inc;
};

__device__ __forceinline__ du128 pcg_mult() {
  return ((du128)0x2360ED051FC65DA4ULL << 64) | (du128)0x4385DF649FCCF645ULL;
}

// default_rng([a, b, c]) / default_rng([a, b]) for non-negative ints
__device__ inline DevPcg dev_seed(const uint64_t* seeds, int ns) {
  uint32_t ent[8];
  int ne = 0;
  for (int i = 0; i < ns; ++i) {
    uint64_t x = seeds[i];
    if (!x) ent[ne++] = 0;
    while (x) {
      ent[ne++] = (uint32_t)x;
      x >>= 32;
    }
  }
  uint32_t hc = 0x43b0d7e5u, pool[4];
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
  };
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = 0x8b51f9ddu, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  uint64_t val[4];
  for (int i = 0; i < 4; ++i) val[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  DevPcg g;
  g.inc = ((((du128)val[2] << 64) | val[3]) << 1) | 1;
  g.state = g.inc;  // 0 * mult + inc
  g.state += ((du128)val[0] << 64) | val[1];
  g.state = g.state * pcg_mult() + g.inc;
  return g;
}

// state after `delta` further steps
__device__ inline du128 pcg_advance(du128 state, du128 inc, uint64_t delta) {
  du128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  return am * state + ap;
}

__device__ __forceinline__ uint64_t pcg_out(du128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// j-th 32-bit word of a fresh generator (has_uint32 = 0): low half of the
// (j/2)-th 64-bit output first, then its high half.
__device__ __forceinline__ uint32_t pcg_word(const DevPcg& g, uint64_t j) {
  const uint64_t o = pcg_out(pcg_advance(g.state, g.inc, (j >> 1) + 1));
  return (j & 1) ? (uint32_t)(o >> 32) : (uint32_t)o;
}

// sequential reference draw (rejection fix-up path)
struct DevPcgSeq {
  DevPcg g;
  bool has = false;
  uint32_t buf = 0;
  __device__ uint32_t next32() {
    if (has) {
      has = false;
      return buf;
    }
    g.state = g.state * pcg_mult() + g.inc;
    const uint64_t o = pcg_out(g.state);
    has = true;
    buf = (uint32_t)(o >> 32);
    return (uint32_t)o;
  }
  __device__ uint32_t below(uint32_t n) {  // Generator.integers(0, n), n >= 2
    const uint32_t excl = n, r = n - 1;
    uint64_t m = (uint64_t)next32() * excl;
    if ((uint32_t)m < excl) {
      const uint32_t t = (0xffffffffu - r) % excl;
      while ((uint32_t)m < t) m = (uint64_t)next32() * excl;
    }
    return (uint32_t)(m >> 32);
  }
};

}  // namespace jet
