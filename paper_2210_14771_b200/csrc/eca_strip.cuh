// K1: fused handcrafted strip scoring + half-row candidate selection.
//
// One work item = one strip (rows h-1, h, h+1) of one frame.  Persistent,
// warp-specialised CTAs walk the items:
//   * a TMA ring (cp.async.bulk + mbarrier, NSTAGE deep) streams the rows of
//     upcoming items into shared memory;
//   * PIXEL warps (8 columns per thread) score every column of the item;
//   * two FP64 warps (even / odd items) rescore the few surviving columns of
//     the previous item in FP64, pick the winners, write the candidates, run
//     the fused RANSAC fit when a frame completes and refill the TMA stage.
// Pixel and FP64 warps meet only at named barriers over double-buffered
// survivor lists, so the FP64 latency chain never stalls the pixel warps.
//
// Per item (handcrafted.py:148-205):
//   1. RGB sums of each thread's 8 columns in the 3 rows (exact, dp4a);
//      c = s0 + 2 s1 + s2 and e = s2 - s0 per column, neighbours by shuffle
//   2. preceding max of the centre row: block prefix scan (left half) and
//      suffix scan (right half), exclusive of the column (handcrafted.py:184-191)
//   3. every column: exact integer Sobel (3gx = c[x+1]-c[x-1],
//      3gy = e[x-1]+2e[x]+e[x+1]) and RIGOROUS FP32 bounds L <= score <= U from
//      three monotone tables (tanh term over log-binned |3g|^2, angle term over
//      a pseudo-angle, darkness term over the preceding sum; entries padded
//      outward); block max LB of L per half
//   4. survivors: columns with U >= LB (nothing else can be the argmax), or
//      every non-flat column of a half whose LB is ~0 (flat rows: there numpy
//      sees rounding residues of ~1e-14 and those decide the argmax)
//   5. (FP64 warp) survivors scored in FP64 in the reference's exact
//      evaluation order; argmax with the reference's outermost tie-break.
// The winner is the reference's winner up to ulp-level differences of the FP64
// transcendental libraries (no approximation error can change the outcome).
#pragma once

#include "eca_common.cuh"
#include "eca_fit.cuh"

namespace eca {

constexpr int kPx = 8;        // pixels per thread
constexpr int kTBins = 800;   // tanh-term bins: float(|3g|^2) exponent (25) x 5 mantissa bits
#ifndef ECA_ABINS
#define ECA_ABINS 128
#endif
constexpr int kABins = ECA_ABINS;   // angle-term bins over pseudo-angle [0, 2]
constexpr int kDBins = 768;   // darkness-term table over preceding sums 0..765
// Relative outward pad of every FP32 bound: not a constant but the modelled
// error bound of the config (StripJob::pad = eca_prefilter_bound, >= 4x the
// summed per-factor FP32 error), so every accepted config is covered.
constexpr int kFpWarps = 2;   // FP64 warps per CTA (item parity)

// named barriers (0 is __syncthreads)
constexpr int kBarPix = 1;       // pixel warps only
constexpr int kBarReady = 2;     // + parity: list ready   (pixel arrive, FP64 sync)
constexpr int kBarFree = 4;      // + parity: list drained (FP64 arrive, pixel sync)

struct StripJob {
  const uint8_t* frames;
  int64_t frame_stride, row_stride;
  int batch, n_strips, nthreads, rowcap, contiguous;
  float tau;          // halves whose LB < tau are scored fully in FP64
  float pad;          // relative pad of the FP32 bounds (eca_prefilter_bound)
  int exhaustive;
  EcaParams p;
  int16_t rows[ECA_MAX_STRIPS];  // geometric centre row y of each strip
  int16_t band[ECA_MAX_STRIPS];  // memory row (within a frame buffer) holding row y-1
  int32_t* out_x;
  int32_t* out_y;
  double* out_score;
  double* out_rows;        // kRows only
  const int16_t* triplets; // kFused only
  int32_t* counters;
  EcaFitRecord* out_fit;
};

struct StripRed {
  int wtot[32];
  float wlb[32][2];
  int cnt[2];
};

ECA_DEV void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
ECA_DEV void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

ECA_DEV float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// v / 3.0 correctly rounded for an RGB sum v in [0, 765]: q0 = v * RN(1/3)
// plus one FMA correction equals the IEEE quotient for every such v
// (exhaustive check: tools/div3_check.c, tests/test_host_lib.py), three
// instructions instead of a full FP64 division.
ECA_DEV double div3(int v) {
  const double third = 1.0 / 3.0;
  const double q0 = __dmul_rn(double(v), third);
  return __fma_rn(__fma_rn(-q0, 3.0, double(v)), third, q0);
}

// handcrafted.py:164-200 for one interior column in numpy's evaluation order.
// l/m/r: integer RGB sums at x-1, x, x+1 of rows h-1, h, h+1.
ECA_DEV double exact_score(const int l[3], const int m[3], const int r[3], int pre_sum, int x,
                           int y, double cx, double cy, const EcaParams& p) {
  double gl[3], gm[3], gr[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ECA_CHECK(l[k] >= 0 && l[k] <= 765 && m[k] >= 0 && m[k] <= 765 && r[k] >= 0 && r[k] <= 765);
    gl[k] = div3(l[k]);
    gm[k] = div3(m[k]);
    gr[k] = div3(r[k]);
  }
  const double gx =
      add_rn(add_rn(sub_rn(gr[0], gl[0]), mul_rn(2.0, sub_rn(gr[1], gl[1]))), sub_rn(gr[2], gl[2]));
  const double gy = sub_rn(add_rn(add_rn(gl[2], gr[2]), mul_rn(2.0, gm[2])),
                           add_rn(add_rn(gl[0], gr[0]), mul_rn(2.0, gm[0])));
  const double tox = sub_rn(cx, double(x));
  const double toy = sub_rn(cy, double(y));
  const double dot = add_rn(mul_rn(gx, tox), mul_rn(gy, toy));
  const double crs = sub_rn(mul_rn(gx, toy), mul_rn(gy, tox));
  const double ang = (gx == 0.0 && gy == 0.0) ? p.zero_grad_angle
                                              : mul_rn(atan2(fabs(crs), dot), p.angle_scale);
  const double t =
      tanh(div_rn(__dsqrt_rn(add_rn(mul_rn(gx, gx), mul_rn(gy, gy))), p.gradient_threshold));
  const double a = div_rn(2.0, add_rn(1.0, exp(mul_rn(2.0, ang))));
  const double pre = div3(pre_sum);
  const double d = div_rn(2.0, add_rn(1.0, exp(div_rn(mul_rn(2.0, pre), p.intensity_threshold))));
  return mul_rn(mul_rn(t, a), d);
}

// 8 RGB pixel sums from 6 little-endian words (24 bytes)
ECA_DEV void sums8(const uint32_t w[6], int s[8]) {
  s[0] = __dp4a(w[0], 0x00010101u, 0u);
  s[1] = __dp4a(w[1], 0x00000101u, __dp4a(w[0], 0x01000000u, 0u));
  s[2] = __dp4a(w[2], 0x00000001u, __dp4a(w[1], 0x01010000u, 0u));
  s[3] = __dp4a(w[2], 0x01010100u, 0u);
  s[4] = __dp4a(w[3], 0x00010101u, 0u);
  s[5] = __dp4a(w[4], 0x00000101u, __dp4a(w[3], 0x01000000u, 0u));
  s[6] = __dp4a(w[5], 0x00000001u, __dp4a(w[4], 0x01010000u, 0u));
  s[7] = __dp4a(w[5], 0x01010100u, 0u);
}

// Read 24 bytes starting at smem byte offset `off` (aligned fast path when off % 8 == 0).
ECA_DEV void load24(const uint8_t* base, int off, uint32_t w[6]) {
  if ((off & 7) == 0) {
    const uint2* p = reinterpret_cast<const uint2*>(base + off);
    const uint2 a = p[0], b = p[1], c = p[2];
    w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y; w[4] = c.x; w[5] = c.y;
    return;
  }
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(base + (off & ~3));
  const int sh = (off & 3) * 8;
  uint32_t v[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) v[k] = wp[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) w[k] = __funnelshift_r(v[k], v[k + 1], sh);
}

ECA_DEV int px_sum(const uint8_t* base, int off) {
  return int(base[off]) + int(base[off + 1]) + int(base[off + 2]);
}

ECA_DEV const uint8_t* item_row0(const StripJob& J, int item) {
  const int frame = item / J.n_strips;
  const int strip = item - frame * J.n_strips;
  return J.frames + int64_t(frame) * J.frame_stride + int64_t(J.band[strip]) * J.row_stride;
}

// smem byte offsets (within a stage) of the first byte of rows 0..2 of an item
ECA_DEV void row_bases(const StripJob& J, const uint8_t* row0, int rb[3]) {
  if (J.contiguous) {
    const int off = int(reinterpret_cast<uintptr_t>(row0) & 15);
    rb[0] = off;
    rb[1] = off + 3 * J.p.width;
    rb[2] = off + 6 * J.p.width;
  } else {
#pragma unroll
    for (int r = 0; r < 3; ++r)
      rb[r] = r * J.rowcap + int(reinterpret_cast<uintptr_t>(row0 + r * J.row_stride) & 15);
  }
}

// one thread: start the TMA copy of an item's three rows into `stage`
ECA_DEV void issue_item(const StripJob& J, int item, uint8_t* stage, uint64_t* bar, uint64_t pol) {
  const uint8_t* row0 = item_row0(J, item);
  const int w3 = 3 * J.p.width;
  if (J.contiguous) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(row0);
    const uintptr_t a0 = a & ~uintptr_t(15);
    const uint32_t bytes = uint32_t((a - a0) + 3 * w3 + 15) & ~15u;
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(stage, reinterpret_cast<const void*>(a0), bytes, bar, pol);
  } else {
    uint32_t sizes[3];
    uintptr_t starts[3];
    uint32_t total = 0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + r * J.row_stride);
      starts[r] = a & ~uintptr_t(15);
      sizes[r] = uint32_t((a - starts[r]) + w3 + 15) & ~15u;
      total += sizes[r];
    }
    mbar_arrive_expect_tx(bar, total);
#pragma unroll
    for (int r = 0; r < 3; ++r)
      bulk_g2s(stage + r * J.rowcap, reinterpret_cast<const void*>(starts[r]), sizes[r], bar, pol);
  }
}

// Shared-memory layout (bytes); host and device agree through this helper.
struct StripLayout {
  size_t raw, stage, ttab, atab, dtab, list, list_cap, red, total;
};

__host__ __device__ inline StripLayout strip_layout(int nstage, int rowcap, int nthreads) {
  StripLayout L;
  size_t o = 128;  // mbarriers
  L.raw = o;
  L.stage = size_t(3) * rowcap;
  if (L.stage < sizeof(FitScratchW)) L.stage = (sizeof(FitScratchW) + 127) & ~size_t(127);
  o += size_t(nstage) * L.stage;
  L.ttab = o;
  o += kTBins * 8;
  L.atab = o;
  o += (kABins + 2) * 8;
  L.dtab = o;
  o += kDBins * 8;
  L.list = o;
  L.list_cap = size_t(nthreads) * kPx;   // every column can survive: no overflow
  o += 2 * L.list_cap * 4;               // double-buffered by item parity
  L.red = o;
  o += (sizeof(StripRed) + 15) & ~size_t(15);
  L.total = (o + 127) & ~size_t(127);
  return L;
}

// A(theta) = 2 / (1 + exp(2 * angle_scale * theta)), FP32 accurate expf
ECA_DEV float angle_term(float theta, float ascale) {
  return 2.0f / (1.0f + expf(2.0f * ascale * theta));
}
// theta of pseudo-angle ps in [0, 2] (ps = |c|/(|d|+|c|), mirrored for d < 0)
ECA_DEV float theta_of(float ps) {
  ps = fminf(fmaxf(ps, 0.0f), 2.0f);
  return ps <= 1.0f ? atan2f(ps, 1.0f - ps) : 3.14159265358979f - atan2f(2.0f - ps, ps - 1.0f);
}

// Bound tables (per CTA, from the config): float2 (lower, upper) per bin.
ECA_DEV void build_tables(const EcaParams& p, float pad, float2* tt, float2* at, float2* dt) {
  const float lo_f = 1.0f - pad, hi_f = 1.0f + pad;
  const float c = float(1.0 / (3.0 * p.gradient_threshold));
  for (int b = threadIdx.x; b < kTBins; b += blockDim.x) {
    const int e = b >> 5, m = b & 31;
    const float q_lo = ldexpf(1.0f + m / 32.0f, e), q_hi = ldexpf(1.0f + (m + 1) / 32.0f, e);
    tt[b] = make_float2(tanhf(sqrtf(q_lo) * c) * lo_f, fminf(tanhf(sqrtf(q_hi) * c) * hi_f, 1.0f));
  }
  const float asc = float(p.angle_scale);
  for (int k = threadIdx.x; k < kABins; k += blockDim.x) {
    const float w = 2.0f / kABins;
    const float th_lo = theta_of(k * w - 1e-5f), th_hi = theta_of((k + 1) * w + 1e-5f);
    at[k] = make_float2(angle_term(th_hi, asc) * lo_f, fminf(angle_term(th_lo, asc) * hi_f, 1.0f));
  }
  if (threadIdx.x == 0)  // dot == cross == 0 (frame-centre pixel): theta is 0 or pi
    at[kABins] = make_float2(angle_term(3.14159265358979f, asc) * lo_f, 1.0f);
  const float ti = float(p.intensity_threshold);
  for (int s = threadIdx.x; s < kDBins; s += blockDim.x) {
    const float d = 2.0f / (1.0f + expf(2.0f * (float(s < 766 ? s : 765) / 3.0f) / ti));
    dt[s] = make_float2(d * lo_f, fminf(d * hi_f, 1.0f));
  }
}

// FP64 score of list entry (x | pre << 16) read from the item's raw rows
ECA_DEV double score_entry(uint32_t v, const uint8_t* st, const int rb[3], int y, double cxf,
                           double cyf, const EcaParams& p, int& x) {
  x = int(v & 0xffffu);
  const int ps = int(v >> 16);
  int l[3], m[3], r[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    l[k] = px_sum(st, rb[k] + 3 * (x - 1));
    m[k] = px_sum(st, rb[k] + 3 * x);
    r[k] = px_sum(st, rb[k] + 3 * (x + 1));
  }
  return exact_score(l, m, r, ps, x, y, cxf, cyf, p);
}

// ----------------------------------------------------- pixel warps: one item
template <bool kRows>
ECA_DEV void pixel_item(const StripJob& J, const uint8_t* st, const int rb[3], int y, int frame,
                        int strip, int par, const float2* ttab, const float2* atab,
                        const float2* dtab, uint32_t* list, StripRed* red, int npx) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, n_warps = npx >> 5;
  const int W = J.p.width, H = J.p.height;
  const int split = (W + 1) / 2;
  const int x0 = tid * kPx;
  const bool interior = x0 >= 1 && x0 + kPx - 1 <= W - 2;  // all 8 columns scoreable
  const bool live = x0 < W;

  // ---- 1. RGB sums; c = s0 + 2 s1 + s2, e = s2 - s0 ----
  int c[kPx + 2], e[kPx + 2], ctr[kPx];
  {
    int s0[kPx], s1[kPx], s2[kPx];
    uint32_t w[6];
    load24(st, rb[0] + 3 * x0, w);
    sums8(w, s0);
    load24(st, rb[1] + 3 * x0, w);
    sums8(w, s1);
    load24(st, rb[2] + 3 * x0, w);
    sums8(w, s2);
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      if (!interior && x0 + i >= W) s0[i] = s1[i] = s2[i] = 0;
      c[i + 1] = s0[i] + 2 * s1[i] + s2[i];
      e[i + 1] = s2[i] - s0[i];
      ctr[i] = s1[i];
    }
  }
  c[0] = __shfl_up_sync(kFull, c[kPx], 1);
  e[0] = __shfl_up_sync(kFull, e[kPx], 1);
  c[kPx + 1] = __shfl_down_sync(kFull, c[1], 1);
  e[kPx + 1] = __shfl_down_sync(kFull, e[1], 1);
  if (lane == 0 && x0 >= 1 && live) {   // warp edges: neighbour column from smem
    const int a0 = px_sum(st, rb[0] + 3 * (x0 - 1)), a1 = px_sum(st, rb[1] + 3 * (x0 - 1)),
              a2 = px_sum(st, rb[2] + 3 * (x0 - 1));
    c[0] = a0 + 2 * a1 + a2;
    e[0] = a2 - a0;
  }
  if (lane == 31 && x0 + kPx < W) {
    const int a0 = px_sum(st, rb[0] + 3 * (x0 + kPx)), a1 = px_sum(st, rb[1] + 3 * (x0 + kPx)),
              a2 = px_sum(st, rb[2] + 3 * (x0 + kPx));
    c[kPx + 1] = a0 + 2 * a1 + a2;
    e[kPx + 1] = a2 - a0;
  }

  // ---- 2. preceding max: warp scans of thread maxima + block combine ----
  int tmax = 0;
#pragma unroll
  for (int i = 0; i < kPx; ++i) tmax = max(tmax, ctr[i]);
  int up = tmax, dn = tmax;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(kFull, up, d);
    const int v = __shfl_down_sync(kFull, dn, d);
    if (lane >= d) up = max(up, u);
    if (lane + d < 32) dn = max(dn, v);
  }
  int ex_up = __shfl_up_sync(kFull, up, 1);
  int ex_dn = __shfl_down_sync(kFull, dn, 1);
  if (lane == 0) ex_up = 0;
  if (lane == 31) ex_dn = 0;
  if (lane == 31) red->wtot[warp] = up;
  bar_sync(kBarPix, npx);  // (A)
  for (int w = 0; w < warp; ++w) ex_up = max(ex_up, red->wtot[w]);
  for (int w = warp + 1; w < n_warps; ++w) ex_dn = max(ex_dn, red->wtot[w]);
  int pre[kPx];
  {
    int run = ex_up;
#pragma unroll
    for (int i = 0; i < kPx; ++i) {   // left: max over columns < x
      pre[i] = run;
      run = max(run, ctr[i]);
    }
    run = ex_dn;
#pragma unroll
    for (int i = kPx - 1; i >= 0; --i) {  // right: max over columns > x
      if (x0 + i >= split) pre[i] = run;
      run = max(run, ctr[i]);
    }
  }
  const int d2y = (H - 1) - 2 * y;

  // ---- 3. bounds.  V = T*D >= score (A <= 1) for every column (cheap);
  //         the angle term only for each thread's best-V column per half,
  //         whose L = T_lo*A_lo*D_lo gives the half's max lower bound LB ----
  // vu[i] = 0 for border / zero-gradient columns; with LB >= tau > 0 they
  // never survive outside full halves (and full halves test flatness instead)
  float vu[kPx];
  float vb0 = 0.0f, vb1 = 0.0f, tdb0 = 0.0f, tdb1 = 0.0f;   // best V per half and its T_lo*D_lo
  uint32_t gb0 = 0, gb1 = 0;                                 // packed (3gx, 3gy, i) of that column
#pragma unroll
  for (int i = 0; i < kPx; ++i) {
    const int x = x0 + i;
    const int gx3 = c[i + 2] - c[i];
    const int gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
    const bool ok = interior || (x >= 1 && x <= W - 2);
    const int q = gx3 * gx3 + gy3 * gy3;
    const int key = max(int(__float_as_uint(float(q)) >> 18) - (127 << 5), 0);
    const float2 tb = ttab[key];
    const float2 db = dtab[pre[i]];
    const float v = (ok && q != 0) ? tb.y * db.y : 0.0f;
    vu[i] = v;
    const uint32_t packed =
        (uint32_t(gx3 + 4096) << 19) | (uint32_t(gy3 + 4096) << 6) | uint32_t(i);
    if (x < split) {
      if (v > vb0) { vb0 = v; tdb0 = tb.x * db.x; gb0 = packed; }
    } else {
      if (v > vb1) { vb1 = v; tdb1 = tb.x * db.x; gb1 = packed; }
    }
  }
  // angle-term bin of a column from its integer gradient
  auto abin = [&](int gx3, int gy3, int x) -> int {
    const int d2x = (W - 1) - 2 * x;
    const int dot = gx3 * d2x + gy3 * d2y;
    const int crs = abs(gx3 * d2y - gy3 * d2x);
    const float fd = float(abs(dot)), fc = float(crs);
    const float ps = fc * rcpf(fd + fc);
    const int k = min(int((dot >= 0 ? ps : 2.0f - ps) * (kABins / 2)), kABins - 1);
    return (dot == 0 && crs == 0) ? kABins : k;
  };
  auto lower = [&](uint32_t packed, float tdb) -> float {
    const int gx3 = int(packed >> 19) - 4096, gy3 = int((packed >> 6) & 0x1fffu) - 4096;
    return tdb * atab[abin(gx3, gy3, x0 + int(packed & 7u))].x;
  };
  float lb0 = vb0 > 0.0f ? lower(gb0, tdb0) : 0.0f;
  float lb1 = vb1 > 0.0f ? lower(gb1, tdb1) : 0.0f;
  lb0 = warp_max(lb0);
  lb1 = warp_max(lb1);
  if (lane == 0) {
    red->wlb[warp][0] = lb0;
    red->wlb[warp][1] = lb1;
  }
  bar_sync(kBarPix, npx);  // (B)
  lb0 = 0.0f;
  lb1 = 0.0f;
  for (int w = 0; w < n_warps; ++w) {
    lb0 = fmaxf(lb0, red->wlb[w][0]);
    lb1 = fmaxf(lb1, red->wlb[w][1]);
  }
  const bool full0 = kRows || !(lb0 >= J.tau);
  const bool full1 = kRows || !(lb1 >= J.tau);

  // ---- 4. survivors: V >= LB, then the angle-refined U = V * A_up >= LB ----
  auto upper = [&](int i) -> float {
    return vu[i] * atab[abin(c[i + 2] - c[i], e[i] + 2 * e[i + 1] + e[i + 2], x0 + i)].y;
  };
  uint32_t surv = 0;
  const bool any_full = (full0 && x0 < split) || (full1 && x0 + kPx - 1 >= split);
  if (!any_full) {
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      const float lb = (x0 + i < split) ? lb0 : lb1;   // >= tau > 0
      if (vu[i] >= lb && upper(i) >= lb) surv |= 1u << i;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      const int x = x0 + i;
      const bool left = x < split;
      bool s;
      if (left ? full0 : full1) {
        // every interior column whose 3x3 neighbourhood is not flat
        s = false;
        if (x >= 1 && x <= W - 2) {
          const int l0 = px_sum(st, rb[0] + 3 * (x - 1)), r0 = px_sum(st, rb[0] + 3 * (x + 1));
          const int l1 = px_sum(st, rb[1] + 3 * (x - 1)), r1 = px_sum(st, rb[1] + 3 * (x + 1));
          const int l2 = px_sum(st, rb[2] + 3 * (x - 1)), r2 = px_sum(st, rb[2] + 3 * (x + 1));
          const int m0 = px_sum(st, rb[0] + 3 * x), m2 = px_sum(st, rb[2] + 3 * x);
          s = !(l0 == r0 && l1 == r1 && l2 == r2 && l0 == l2 && m0 == m2 && r0 == r2);
        }
        if (kRows && !s && x < W) J.out_rows[(size_t(frame) * J.n_strips + strip) * W + x] = 0.0;
      } else {
        const float lb = left ? lb0 : lb1;
        s = vu[i] >= lb && upper(i) >= lb;
      }
      if (s) surv |= 1u << i;
    }
  }
  // the FP64 warp of this parity must have drained its previous list
  bar_sync(kBarFree + par, npx + 32);
  {
    const int cnt = __popc(surv);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += v;
    }
    int base = 0;
    if (lane == 31 && incl > 0) base = atomicAdd(&red->cnt[par], incl);
    base = __shfl_sync(kFull, base, 31) + incl - cnt;
#pragma unroll
    for (int i = 0; i < kPx; ++i)
      if ((surv >> i) & 1u) list[base++] = uint32_t(x0 + i) | (uint32_t(pre[i]) << 16);
  }
  bar_arrive(kBarReady + par, npx + 32);
}

// ------------------------------------------------------------------ kernel
// blockDim.x = npx (pixel threads, = J.nthreads) + 32 * kFpWarps.
template <int NSTAGE, int MAXT, int MINB, bool kRows, bool kFused>
__global__ void __launch_bounds__(MAXT, MINB) strip_kernel(const __grid_constant__ StripJob J) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int npx = J.nthreads;
  const int W = J.p.width, H = J.p.height;
  const int S = J.n_strips;
  const int n_items = J.batch * S;
  const int split = (W + 1) / 2;

  const StripLayout SL = strip_layout(NSTAGE, J.rowcap, npx);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* raw = smem + SL.raw;
  float2* ttab = reinterpret_cast<float2*>(smem + SL.ttab);
  float2* atab = reinterpret_cast<float2*>(smem + SL.atab);
  float2* dtab = reinterpret_cast<float2*>(smem + SL.dtab);
  uint32_t* lists = reinterpret_cast<uint32_t*>(smem + SL.list);
  StripRed* red = reinterpret_cast<StripRed*>(smem + SL.red);

  uint64_t pol = 0;
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    red->cnt[0] = red->cnt[1] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    pol = l2_evict_first();
    for (int s = 0; s < NSTAGE; ++s) {
      const int item = blockIdx.x + s * gridDim.x;
      if (item < n_items) issue_item(J, item, raw + s * SL.stage, &bars[s], pol);
    }
  }
  build_tables(J.p, J.pad, ttab, atab, dtab);
  __syncthreads();

  if (tid < npx) {
    // =========================== pixel warps ===========================
    // frame / strip / stage / parity advance incrementally (no divisions)
    const int fstep = gridDim.x / S, sstep = gridDim.x - (gridDim.x / S) * S;
    int frame = blockIdx.x / S, strip = blockIdx.x - (blockIdx.x / S) * S;
    int stage = 0, par = 0;
    uint32_t phase = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const uint8_t* st = raw + stage * SL.stage;
      int rb[3];
      row_bases(J, J.frames + int64_t(frame) * J.frame_stride +
                       int64_t(J.band[strip]) * J.row_stride, rb);
      mbar_wait(&bars[stage], phase);
      pixel_item<kRows>(J, st, rb, J.rows[strip], frame, strip, par, ttab, atab, dtab,
                        lists + par * SL.list_cap, red, npx);
      par ^= 1;
      if (++stage == NSTAGE) {
        stage = 0;
        phase ^= 1u;
      }
      frame += fstep;
      strip += sstep;
      if (strip >= S) {
        strip -= S;
        ++frame;
      }
    }
  } else {
    // =========================== FP64 warps ============================
    const int par = warp - npx / 32;   // items with (it & 1) == par
    pol = l2_evict_first();
    const double cxf = div_rn(double(W - 1), 2.0);  // geometry.py:44
    const double cyf = div_rn(double(H - 1), 2.0);
    uint32_t* list = lists + par * SL.list_cap;
    if (blockIdx.x + par * gridDim.x < n_items)
      bar_arrive(kBarFree + par, npx + 32);   // the list starts empty
    int it = par;
    for (int item = blockIdx.x + par * gridDim.x; item < n_items; item += 2 * gridDim.x, it += 2) {
      const int stage = it % NSTAGE;
      const int frame = item / S;
      const int strip = item - frame * S;
      const int y = J.rows[strip];
      uint8_t* st = raw + stage * SL.stage;
      int rb[3];
      row_bases(J, item_row0(J, item), rb);
      bar_sync(kBarReady + par, npx + 32);
      const int n_list = red->cnt[par];
      Best b0{0.0, 0}, b1{0.0, W - 1};  // border columns score exactly 0
      for (int k = lane; k < n_list; k += 32) {
        int x;
        const double s = score_entry(list[k], st, rb, y, cxf, cyf, J.p, x);
        if (kRows) J.out_rows[(size_t(frame) * S + strip) * W + x] = s;
        if (x < split) {
          if (better(s, x, b0.s, b0.x, true)) b0 = Best{s, x};
        } else {
          if (better(s, x, b1.s, b1.x, false)) b1 = Best{s, x};
        }
      }
      b0 = warp_best(b0, true);
      b1 = warp_best(b1, false);
      __syncwarp();
      const bool more = item + 2 * gridDim.x < n_items;
      if (lane == 0) red->cnt[par] = 0;
      __syncwarp();
      if (more) bar_arrive(kBarFree + par, npx + 32);   // list may be refilled
      const size_t o = size_t(frame) * 2 * S;
      if (lane == 0) {
        J.out_x[o + strip] = b0.x;
        J.out_y[o + strip] = y;
        J.out_score[o + strip] = b0.s;
        J.out_x[o + S + strip] = b1.x;
        J.out_y[o + S + strip] = y;
        J.out_score[o + S + strip] = b1.s;
      }
      if (kFused) {
        int last = 0;
        if (lane == 0) {
          __threadfence();
          last = atomicAdd(&J.counters[frame], 1) == S - 1;
        }
        if (__shfl_sync(kFull, last, 0)) {
          __threadfence();
          fit_warp(J.out_x + o, J.out_y + o, J.out_score + o, 2 * S, J.p, J.triplets,
                   J.exhaustive, reinterpret_cast<FitScratchW*>(st)->pt,
                   reinterpret_cast<FitScratchW*>(st)->ps, J.out_fit + frame);
          if (lane == 0) J.counters[frame] = 0;
        }
      }
      __syncwarp();
      if (lane == 0) {   // stage drained: refill it with a later item
        const int nxt = item + NSTAGE * gridDim.x;
        if (nxt < n_items) issue_item(J, nxt, st, &bars[stage], pol);
      }
    }
  }
}

}  // namespace eca
