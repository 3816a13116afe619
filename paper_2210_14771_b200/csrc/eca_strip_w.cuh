// Warp-per-half-row helpers shared by the K1 bounds kernel (eca_points.cuh):
// per-warp shared-memory layout, the half-row TMA issue, and the FP32 bound
// terms (handcrafted.py:148-205).
//
// Work item = one HALF of one strip row of one frame: the left half's argmax
// depends only on columns [0, split) (prefix max from the left border) and the
// right half's only on [split, W) (suffix max from the right border), so each
// half-row is independent.  Each WARP owns a ring of 1-D TMA bulk copies
// (3 rows x half width + 1 neighbour column) and its mbarriers.
// The tanh and darkness terms are evaluated with MUFU ex2/rcp/sqrt and padded
// by StripJob::pad (eca_prefilter_bound: >= 4x their modelled FP32 error for
// the config; tests/test_gpu_parity.py measures the real error of every term
// against FP64 with eca_prefilter_selftest); the angle term comes from a small
// per-CTA table (A over a pseudo-angle).
#pragma once

#include "eca_strip.cuh"

namespace eca {

constexpr int kWChunk = 256;       // columns per chunk (32 lanes x kPx)
constexpr int kWMaxChunks = 8;     // half width <= 2048
constexpr int kWListCap = 64;      // per-warp survivor list (flushed to FP64 when full)


// Per-warp region: [stages][list][ulist][bars][ut][exs][sel]
//   list  survivor entries (x | pre << 16), flushed to FP64 when full
//   ulist their upper bounds (float)
//   bars  NS mbarriers (16 reserved)
//   ut    pass-1 upper bound of every lane-chunk      half    [kWMaxChunks][32]
//   exs   preceding sum before every lane-chunk      uint16  [kWMaxChunks][32]
//   sel   compacted lane-chunk list (k << 5 | lane)  uint16  [kWMaxChunks * 32]
struct WarpLayout {
  size_t atab, warp0, per_warp, stage, list, ulist, bars, ut, exs, sel, total;
};

// min_stage: bytes a stage must hold at least (besides the rows)
__host__ __device__ inline WarpLayout warp_layout(int nstage, int rowcap_h, int warps,
                                                  int min_stage = 0) {
  WarpLayout L;
  size_t o = 0;
  L.atab = o;
  o += ((kABins + 2) * 8 + 127) & ~size_t(127);
  L.stage = size_t(3) * rowcap_h;
  if (L.stage < size_t(min_stage)) L.stage = size_t(min_stage);
  L.stage = (L.stage + 127) & ~size_t(127);
  L.list = size_t(nstage) * L.stage;
  L.ulist = L.list + kWListCap * 4;
  L.bars = L.ulist + kWListCap * 4;
  L.ut = L.bars + 16 * 8;
  L.exs = L.ut + kWMaxChunks * 32 * 2;
  L.sel = L.exs + kWMaxChunks * 32 * 2;
  L.per_warp = (L.sel + kWMaxChunks * 32 * 2 + 127) & ~size_t(127);
  L.warp0 = o;
  o += size_t(warps) * L.per_warp;
  L.total = o;
  return L;
}

ECA_DEV float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
ECA_DEV float sqrtf_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// identical left/right sums per row and identical top/bottom rows make numpy's
// gx and gy exactly 0.0 (no rounding residue): such a column scores exactly 0
ECA_DEV bool flat_column(const uint8_t* st, const int rb[3], int x) {
  const int l0 = px_sum(st, rb[0] + 3 * (x - 1)), r0 = px_sum(st, rb[0] + 3 * (x + 1));
  const int l1 = px_sum(st, rb[1] + 3 * (x - 1)), r1 = px_sum(st, rb[1] + 3 * (x + 1));
  const int l2 = px_sum(st, rb[2] + 3 * (x - 1)), r2 = px_sum(st, rb[2] + 3 * (x + 1));
  const int m0 = px_sum(st, rb[0] + 3 * x), m2 = px_sum(st, rb[2] + 3 * x);
  return l0 == r0 && l1 == r1 && l2 == r2 && l0 == l2 && m0 == m2 && r0 == r2;
}

struct TermK {
  float kt;   // -2*log2(e)/(3 t_g): e_t = 2^(kt*sqrt(q)) = exp(-2u), u = |g|/t_g
  float kd;   // 2*log2(e)/(3 t_i):  e_d = 2^(kd*p)      = exp(2 * (p/3) / t_i)
};

// tanh(|g|/t_g) for q = (3gx)^2 + (3gy)^2 > 0, relative error < 1e-5
ECA_DEV float t_term(int q, const TermK& k) {
  const float e = ex2f(k.kt * sqrtf_approx(float(q)));
  return (1.0f - e) * rcpf(1.0f + e);
}
// 2 / (1 + exp(2 (p/3) / t_i)) for the integer preceding sum p
ECA_DEV float d_term(int p, const TermK& k) { return 2.0f * rcpf(1.0f + ex2f(k.kd * float(p))); }

// issue the three row copies of one half strip row into `stage` (lane 0)
ECA_DEV void issue_half(const StripJob& J, int half, int frame, int strip, uint8_t* stage,
                        uint64_t* bar, uint64_t pol, int split) {
  const int W = J.p.width;
  const int xs = half ? split - 1 : 0;          // first staged column
  const int xe = half ? W : min(split + 1, W);  // one past the last staged column
  const uint8_t* row0 = J.frames + int64_t(frame) * J.frame_stride +
                        int64_t(J.band[strip]) * J.row_stride + 3 * xs;
  uint32_t sizes[3];
  uintptr_t starts[3];
  uint32_t total = 0;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + r * J.row_stride);
    starts[r] = a & ~uintptr_t(15);
    sizes[r] = uint32_t((a - starts[r]) + 3 * (xe - xs) + 15) & ~15u;
    total += sizes[r];
  }
  mbar_arrive_expect_tx(bar, total);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    bulk_g2s(stage + r * J.rowcap, reinterpret_cast<const void*>(starts[r]), sizes[r], bar, pol);
}

// Zero-copy mode: issue only scan-order chunk k (kWChunk columns plus one
// neighbour column on each side, 3 rows) of a half strip row into the same
// stage positions issue_half would fill (lane 0).  Returns the bytes copied.
ECA_DEV uint32_t issue_chunk(const StripJob& J, int half, int frame, int strip, int k,
                             uint8_t* stage, uint64_t* bar, uint64_t pol, int split) {
  const int W = J.p.width;
  const int xs = half ? split - 1 : 0;          // first staged column
  const int xe = half ? W : min(split + 1, W);  // one past the last staged column
  int x_lo, x_hi;                               // inclusive column range of the chunk
  if (half) {
    x_hi = W - 1 - kWChunk * k + 1;
    x_lo = W - 1 - kWChunk * k - kWChunk;
  } else {
    x_lo = kWChunk * k - 1;
    x_hi = kWChunk * k + kWChunk;
  }
  x_lo = max(x_lo, xs);
  x_hi = min(x_hi, xe - 1);
  const uint8_t* row0 = J.frames + int64_t(frame) * J.frame_stride +
                        int64_t(J.band[strip]) * J.row_stride + 3 * xs;
  uintptr_t src[3];
  uint32_t dst[3], sizes[3], total = 0;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + r * J.row_stride);
    const uintptr_t base = a & ~uintptr_t(15);   // = issue_half's copy start of this row
    const uintptr_t lo = (a + 3 * (x_lo - xs)) & ~uintptr_t(15);
    const uintptr_t hi = (a + 3 * (x_hi - xs) + 3 + 15) & ~uintptr_t(15);
    src[r] = lo;
    dst[r] = uint32_t(r * J.rowcap + (lo - base));
    sizes[r] = uint32_t(hi - lo);
    total += sizes[r];
  }
  mbar_arrive_expect_tx(bar, total);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    bulk_g2s(stage + dst[r], reinterpret_cast<const void*>(src[r]), sizes[r], bar, pol);
  return total;
}

}  // namespace eca
