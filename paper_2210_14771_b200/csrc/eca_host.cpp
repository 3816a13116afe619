// Host-side helpers of libeca_b200.so: strip placement, the seeded RANSAC
// triplet table (numpy PCG64 stream, bit-exact) and the FP32-prefilter bound.
//
// numpy's default_rng(seed) = SeedSequence(seed) -> PCG64 (XSL-RR 128/64);
// random() = (next_u64 >> 11) * 2^-53.  The reference draws all triplet keys
// as default_rng(seed).random((attempts, n)) (fitting.py:147-156), so the
// table for each n comes from a fresh stream.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/eca_b200.h"

namespace {

typedef unsigned __int128 u128;

// ---- numpy SeedSequence (pool size 4, 32-bit words) ------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

struct Hasher {
  uint32_t h = kInitA;
  uint32_t operator()(uint32_t v) {
    v ^= h;
    h *= kMultA;
    v *= h;
    return v ^ (v >> 16);
  }
};

inline uint32_t mix32(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

void seed_words64(uint64_t seed, uint64_t out[4]) {
  uint32_t ent[2];
  int n_ent = 0;
  if (seed == 0) {
    ent[n_ent++] = 0;
  } else {
    while (seed) {
      ent[n_ent++] = static_cast<uint32_t>(seed & 0xffffffffu);
      seed >>= 32;
    }
  }
  uint32_t pool[4];
  Hasher hm;
  for (int i = 0; i < 4; ++i) pool[i] = hm(i < n_ent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix32(pool[d], hm(pool[s]));
  // (n_ent <= 2 < pool size: no trailing entropy words to fold in)
  uint32_t h = kInitB;
  uint32_t w32[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ h;
    h *= kMultB;
    v *= h;
    w32[i] = v ^ (v >> 16);
  }
  for (int k = 0; k < 4; ++k) out[k] = uint64_t(w32[2 * k]) | (uint64_t(w32[2 * k + 1]) << 32);
}

// ---- PCG64 ------------------------------------------------------------------
struct Pcg64 {
  u128 state, inc;
  static constexpr u128 kMult = (u128(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
  explicit Pcg64(uint64_t seed) {
    uint64_t w[4];
    seed_words64(seed, w);
    const u128 s = (u128(w[0]) << 64) | w[1];
    const u128 i = (u128(w[2]) << 64) | w[3];
    inc = (i << 1) | 1u;
    state = 0;
    state = state * kMult + inc;
    state += s;
    state = state * kMult + inc;
  }
  uint64_t next() {
    state = state * kMult + inc;
    const uint64_t x = uint64_t(state >> 64) ^ uint64_t(state);
    const unsigned rot = unsigned(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  double uniform() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
};

}  // namespace

extern "C" int eca_pcg64_doubles(uint64_t seed, int64_t count, double* out) {
  if (count < 0 || (count > 0 && !out)) return ECA_ERR_ARG;
  Pcg64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.uniform();
  return ECA_OK;
}

extern "C" int eca_triplet_table(uint64_t seed, int attempts, int max_n, int16_t* out) {
  if (attempts < 1 || attempts > ECA_MAX_ATTEMPTS || max_n < 3 || max_n > 2 * ECA_MAX_STRIPS || !out)
    return ECA_ERR_ARG;
  for (int n = 3; n <= max_n; ++n) {
    Pcg64 g(seed);
    int16_t* t = out + size_t(n - 3) * attempts * 3;
    for (int a = 0; a < attempts; ++a) {
      // three smallest keys of the attempt's row, ascending by key; numpy's
      // argpartition(kth=3)[:, :3] holds the same 3-subset (fitting.py:156)
      double k0 = 2.0, k1 = 2.0, k2 = 2.0;
      int i0 = -1, i1 = -1, i2 = -1;
      for (int i = 0; i < n; ++i) {
        const double k = g.uniform();
        if (k < k0) {
          k2 = k1; i2 = i1; k1 = k0; i1 = i0; k0 = k; i0 = i;
        } else if (k < k1) {
          k2 = k1; i2 = i1; k1 = k; i1 = i;
        } else if (k < k2) {
          k2 = k; i2 = i;
        }
      }
      t[a * 3 + 0] = int16_t(i0);
      t[a * 3 + 1] = int16_t(i1);
      t[a * 3 + 2] = int16_t(i2);
    }
  }
  return ECA_OK;
}

extern "C" int eca_strip_rows(int height, int count, double weighting, int32_t* out_rows) {
  // strips.py:30-60; expression order kept: -(w/count) * (i - (count-1)/2.0)
  if (height < 14 || count < 2 || !(weighting > 0) || !out_rows) return ECA_ERR_ARG;
  const double slope = -(weighting / count);
  const double mid = (count - 1) / 2.0;
  int n = 0;
  for (int i = 0; i < count; ++i) {
    const double raw = height / (1.0 + std::exp(slope * (double(i) - mid)));
    long long r = (long long)std::floor(raw + 0.5);
    if (r < 3) r = 3;
    if (r > height - 4) r = height - 4;
    if (n == 0 || out_rows[n - 1] != r) out_rows[n++] = int32_t(r);
  }
  return n;
}

// Relative error bound of the FP32 prefilter bounds against the exact FP64
// score, per factor (x = the factor's natural-log exponent):
//   tanh term (bounds kernel: 2^(kt*sqrt.approx(q)) by ex2.approx, then
//     (1-e)*rcp(1+e); fused kernel: tanhf):  the cancellation in (1-e)
//     amplifies the ex2 error by 1/x, x >= 2 u_min = 2/(3 t_g):
//     eps_t = 2 * 2^-22 * (1 + 1/(2 u_min))
//   darkness term 2/(1+e^x), x = 2(p/3)/t_i <= 2*255/t_i (ex2.approx / expf
//     error plus the argument's roundings, |dx| <= x * 2^-22):
//     eps_d = 2^-21 + x_max * 2^-22
//   angle term (bounds kernel: FP64 host table, fused kernel: FP32 atan2f +
//     expf at the bin edges), x = 2 * angle_scale * theta <= 2*zero_grad_angle:
//     eps_a = 2 angle_scale * 1.2e-6 (theta error) + x_max * 3 * 2^-24 + 2^-22 + 2^-24
//   products, rcp.approx, the pads' own rounding: 10 * 2^-23
// Each bound is padded by 4x the sum (the pad is applied per factor, so every
// factor is covered with margin); tests/test_gpu_parity.py measures the real
// per-term FP32 error against FP64 on the GPU (eca_prefilter_selftest).
// Returns 1 (always the exhaustive FP64 path) when FP32 range or conditioning
// cannot carry the config: a factor's exponent >= 80 (e^80 < FLT_MAX, and
// every factor's minimum stays a normal float) or a bound >= 1e-2.  A
// PRODUCT of factors may still flush to zero: such a column's true score is
// < 1e-37, below any LB >= tau, and halves with LB < tau are scored
// exhaustively, so a flushed bound never drops a possible argmax.
extern "C" int eca_prefilter_bound(const EcaParams* p, double* out_rel_bound) {
  if (!p || !out_rel_bound) return ECA_ERR_ARG;
  const double tg = p->gradient_threshold, ti = p->intensity_threshold;
  const double u_min = 1.0 / (3.0 * tg);
  const double max_exp_a = 2.0 * p->zero_grad_angle;  // natural-log exponent at 180 deg
  const double max_exp_d = 2.0 * 255.0 / ti;
  const double eps_t = 2.0 * std::ldexp(1.0, -22) * (1.0 + 1.0 / (2.0 * u_min));
  const double eps_d = std::ldexp(1.0, -21) + max_exp_d * std::ldexp(1.0, -22);
  const double eps_a = 2.0 * p->angle_scale * 1.2e-6 + max_exp_a * 3.0 * std::ldexp(1.0, -24) +
                       std::ldexp(1.0, -22) + std::ldexp(1.0, -24);
  const double eps = eps_t + eps_d + eps_a + 10.0 * std::ldexp(1.0, -23);
  *out_rel_bound = 4.0 * eps;
  const bool ok = std::isfinite(*out_rel_bound) && max_exp_a < 80.0 && max_exp_d < 80.0 &&
                  *out_rel_bound < 1e-2;
  return ok ? 0 : 1;
}
