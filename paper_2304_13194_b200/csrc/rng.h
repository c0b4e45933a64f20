// rng.h — host restatement of the numpy random streams the reference draws.
//
// The reference seeds `np.random.default_rng([seed, level, pass_index])` for
// every rebalancing pass (refine.py:245) and `default_rng([seed, restart])`
// for every initial-partition restart (initpart.py:89), then calls
// `Generator.integers(0, n, size=c)` (rebalance.py:174-175, initpart.py:34).
// Bit-exact parity needs the same stream, so this header restates numpy's
// published algorithms (numpy 2.x, `bit_generator.pyx` SeedSequence,
// `pcg64.h` PCG64 XSL-RR 128/64, `distributions.c` bounded Lemire draws).
// The stream is checked against numpy itself in tests/test_rng.py.
#pragma once
#include <cstdint>
#include <vector>

namespace jet {

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state = 0, inc = 0;
  bool has_uint32 = false;
  uint32_t uinteger = 0;

  static constexpr u128 mult() {
    return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
  }
  void step() { state = state * mult() + inc; }
  uint64_t next64() {
    step();
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  uint32_t next32() {
    if (has_uint32) {
      has_uint32 = false;
      return uinteger;
    }
    uint64_t v = next64();
    has_uint32 = true;
    uinteger = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffu);
  }
  // Generator.integers(0, high) for one int64 value (high >= 1).
  uint64_t bounded(uint64_t high) {
    uint64_t rng = high - 1;
    if (rng == 0) return 0;  // numpy returns `low` without drawing
    if (rng <= 0xffffffffULL) {
      if (rng == 0xffffffffULL) return next32();
      uint32_t r = (uint32_t)rng, excl = r + 1u;
      uint64_t m = (uint64_t)next32() * excl;
      uint32_t left = (uint32_t)m;
      if (left < excl) {
        uint32_t thr = (uint32_t)(0xffffffffu - r) % excl;
        while (left < thr) {
          m = (uint64_t)next32() * excl;
          left = (uint32_t)m;
        }
      }
      return m >> 32;
    }
    if (rng == ~0ULL) return next64();
    uint64_t excl = rng + 1;
    u128 m = (u128)next64() * excl;
    uint64_t left = (uint64_t)m;
    if (left < excl) {
      uint64_t thr = (~0ULL - rng) % excl;
      while (left < thr) {
        m = (u128)next64() * excl;
        left = (uint64_t)m;
      }
    }
    return (uint64_t)(m >> 64);
  }
};

// numpy SeedSequence(entropy).generate_state(4, uint64) -> PCG64 seeding.
inline Pcg64 seed_pcg64(const std::vector<uint32_t>& entropy) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  const int POOL = 4;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[POOL];
  for (int i = 0; i < POOL; ++i)
    pool[i] = hashmix(i < (int)entropy.size() ? entropy[i] : 0u);
  for (int s = 0; s < POOL; ++s)
    for (int d = 0; d < POOL; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (size_t s = POOL; s < entropy.size(); ++s)
    for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(entropy[s]));
  uint32_t words[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % POOL];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    words[i] = v;
  }
  uint64_t val[4];
  for (int i = 0; i < 4; ++i)
    val[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
  u128 s = ((u128)val[0] << 64) | val[1];
  u128 q = ((u128)val[2] << 64) | val[3];
  Pcg64 g;
  g.state = 0;
  g.inc = (q << 1) | 1u;
  g.step();
  g.state += s;
  g.step();
  return g;
}

// _coerce_to_uint32_array of a list of non-negative Python ints.
inline void append_words(std::vector<uint32_t>& out, uint64_t x) {
  if (x == 0) {
    out.push_back(0);
    return;
  }
  while (x) {
    out.push_back((uint32_t)(x & 0xffffffffu));
    x >>= 32;
  }
}

inline Pcg64 default_rng(std::initializer_list<uint64_t> seeds) {
  std::vector<uint32_t> w;
  for (uint64_t s : seeds) append_words(w, s);
  return seed_pcg64(w);
}

}  // namespace jet
