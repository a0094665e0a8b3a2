// synth_host.cpp -- host-side replay of numpy's Generator.choice(c, size=k,
// replace=False) for the synthetic-scene generator (synth_metrics.py:92-94),
// so that 2M-point scenes are generated in seconds with bit-identical camera
// selections. Only used for input generation, never by the solver.
//
// Replays numpy >= 1.17 Generator internals on the PCG64 (XSL-RR 128/64) bit
// generator: Floyd's sampling with random_bounded_uint64 -> Lemire's bounded
// uint32, then the Fisher-Yates shuffle of the k picks (random_interval with
// masked next_uint32), consuming exactly the same stream. Valid for the Floyd
// branch (population <= 10000 or k <= population / 50), which the callers
// check. The caller passes the bit generator state in and gets it back.
#include <stdint.h>
#include <algorithm>

namespace {

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state, inc;
  int has_uint32;
  uint32_t uinteger;

  uint64_t next64() {
    const u128 mult = ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((-rot) & 63));
  }
  uint32_t next32() {
    if (has_uint32) {
      has_uint32 = 0;
      return uinteger;
    }
    const uint64_t n = next64();
    has_uint32 = 1;
    uinteger = (uint32_t)(n >> 32);
    return (uint32_t)(n & 0xffffffffu);
  }
  // buffered_bounded_lemire_uint32: uniform in [0, rng]
  uint32_t lemire(uint32_t rng) {
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (uint32_t)(UINT32_MAX - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    uint64_t v;
    while ((v = (next32() & mask)) > max) {
    }
    return v;
  }
};

}  // namespace

extern "C" int ssfm_synth_choose_sorted(uint64_t* st /* [state_hi, state_lo, inc_hi, inc_lo,
                                                        has_uint32, uinteger] in/out */,
                                        int64_t npoints, int32_t pop, int32_t k, int32_t* out) {
  if (k < 0 || k > pop || pop <= 0) return 1;
  Pcg64 g;
  g.state = ((u128)st[0] << 64) | st[1];
  g.inc = ((u128)st[2] << 64) | st[3];
  g.has_uint32 = (int)st[4];
  g.uinteger = (uint32_t)st[5];
  int64_t pick[64];
  if (k > 64) return 2;
  for (int64_t p = 0; p < npoints; ++p) {
    // Floyd: j in [pop-k, pop): val ~ U[0, j]; take val if new else j
    int n = 0;
    for (int64_t j = pop - k; j < pop; ++j) {
      const int64_t val = (j == 0) ? 0 : (int64_t)g.lemire((uint32_t)j);
      bool seen = false;
      for (int t = 0; t < n; ++t) seen |= (pick[t] == val);
      pick[n++] = seen ? j : val;
    }
    // _shuffle_int (numpy 2.x: random_bounded_uint64 per swap) consumes the
    // stream; the order itself is irrelevant after sorting
    for (int64_t i = k - 1; i >= 1; --i) {
      const int64_t jj = (int64_t)g.lemire((uint32_t)i);
      std::swap(pick[i], pick[jj]);
    }
    std::sort(pick, pick + k);
    for (int t = 0; t < k; ++t) out[p * k + t] = (int32_t)pick[t];
  }
  st[0] = (uint64_t)(g.state >> 64);
  st[1] = (uint64_t)g.state;
  st[2] = (uint64_t)(g.inc >> 64);
  st[3] = (uint64_t)g.inc;
  st[4] = (uint64_t)g.has_uint32;
  st[5] = (uint64_t)g.uinteger;
  return 0;
}
