// K1: fused handcrafted strip scoring + half-row candidate selection.
//
// One work item = one strip (rows h-1, h, h+1) of one frame.  Persistent CTAs
// walk the items with an NSTAGE-deep TMA (cp.async.bulk) ring: the rows of
// item i+NSTAGE*grid stream into shared memory while item i is scored.  Per
// item (handcrafted.py:148-205):
//   1. RGB sums R+G+B of the 3 rows (exact ints, dp4a byte sums) -> smem
//   2. preceding max of the centre row: block prefix scan (left half) and
//      suffix scan (right half), exclusive of the column (handcrafted.py:184-191)
//   3. every column: integer Sobel (3*gx, 3*gy exact) and an FP32 score built
//      from MUFU ex2/rcp/sqrt with a proven relative error bound eps
//      (eca_prefilter_bound); per-half block max
//   4. columns within (1-window) of the half max are re-scored in FP64 in the
//      reference's exact evaluation order; the FP64 argmax (outermost on ties)
//      is the candidate.  A half whose FP32 max is ~0 (flat rows, where numpy
//      sees rounding residues of size 1e-14) is scored entirely in FP64.
// The FP64 winner is provably the reference's winner up to ulp-level
// differences of the FP64 transcendental libraries.
#pragma once

#include "eca_common.cuh"
#include "eca_fit.cuh"

namespace eca {

constexpr int kPx = 8;       // pixels per thread
constexpr int kPad = 8;      // u16 left padding of every sum row (16-byte aligned stores)
constexpr int kDTab = 768;   // darkness-term table over preceding sums 0..765

struct StripJob {
  const uint8_t* frames;
  int64_t frame_stride, row_stride;
  int batch, n_strips, nthreads, rowcap, sumcap, contiguous;
  float window;        // 1 - rel window
  float kT, kA;        // ex2 scales of the tanh / angle terms
  float tau;           // below this FP32 half max the half is scored fully in FP64
  int exhaustive;
  EcaParams p;
  int16_t rows[ECA_MAX_STRIPS];  // geometric centre row y of each strip
  int16_t band[ECA_MAX_STRIPS];  // memory row (within a frame buffer) holding row y-1
  float dtab[kDTab];
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
  float wmax[32][2];
  double bs[32][2];
  int bx[32][2];
  int last;
};

// ---------------------------------------------------------------- MUFU
ECA_DEV float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
ECA_DEV float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
ECA_DEV float sqrtf_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// atan(r), r in [0,1]: odd minimax polynomial, |err| <= 3.4e-7 in FP32 Horner
ECA_DEV float atan01(float r) {
  const float r2 = r * r;
  float q = 0.006811779458075762f;
  q = fmaf(q, r2, -0.033604178577661514f);
  q = fmaf(q, r2, 0.07962362468242645f);
  q = fmaf(q, r2, -0.1323333978652954f);
  q = fmaf(q, r2, 0.19807815551757812f);
  q = fmaf(q, r2, -0.3331736922264099f);
  q = fmaf(q, r2, 0.9999961256980896f);
  return q * r;
}

// FP32 prefilter score; caller guarantees q > 0 and (dot, cross) != (0, 0).
// T*A*D = 2 (1-e_t) D / ((1+e_t)(1+e_a)), e_t = exp(-2u), e_a = exp(2 a).
ECA_DEV float approx_score(int gx3, int gy3, int d2x, int d2y, float dval, float kT, float kA) {
  const int q = gx3 * gx3 + gy3 * gy3;
  const int dot = gx3 * d2x + gy3 * d2y;
  const int crs = abs(gx3 * d2y - gy3 * d2x);
  const float et = ex2f(sqrtf_approx(float(q)) * kT);
  const float fx = float(dot), fy = float(crs);
  const float ax = fabsf(fx);
  const float mn = fminf(ax, fy), mx = fmaxf(ax, fy);
  float th = atan01(mn * rcpf(mx));
  if (fy > ax) th = 1.57079632679489662f - th;
  if (fx < 0.0f) th = 3.14159265358979324f - th;
  const float ea = ex2f(th * kA);
  return (2.0f * (1.0f - et) * dval) * rcpf((1.0f + et) * (1.0f + ea));
}

// handcrafted.py:164-200 for one interior column in numpy's evaluation order.
// l/m/r: integer RGB sums at x-1, x, x+1 of rows h-1, h, h+1.
ECA_DEV double exact_score(const int l[3], const int m[3], const int r[3], int pre_sum, int x,
                           int y, double cx, double cy, const EcaParams& p) {
  double gl[3], gm[3], gr[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gl[k] = div_rn(double(l[k]), 3.0);
    gm[k] = div_rn(double(m[k]), 3.0);
    gr[k] = div_rn(double(r[k]), 3.0);
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
  const double t = tanh(div_rn(__dsqrt_rn(add_rn(mul_rn(gx, gx), mul_rn(gy, gy))), p.gradient_threshold));
  const double a = div_rn(2.0, add_rn(1.0, exp(mul_rn(2.0, ang))));
  const double pre = div_rn(double(pre_sum), 3.0);
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

// Read 24 bytes starting at smem byte offset `byte_off` (any alignment).
ECA_DEV void load24(const uint8_t* base, int byte_off, uint32_t w[6]) {
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(base + (byte_off & ~3));
  const int sh = (byte_off & 3) * 8;
  if (sh == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) w[k] = wp[k];
  } else {
    uint32_t v[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) v[k] = wp[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) w[k] = __funnelshift_r(v[k], v[k + 1], sh);
  }
}

// smem byte offset (within a stage) of the first byte of row r of an item
ECA_DEV int row_base(const StripJob& J, const uint8_t* row0, int r) {
  if (J.contiguous) {
    const int off = int(reinterpret_cast<uintptr_t>(row0) & 15);
    return off + r * 3 * J.p.width;
  }
  const int off = int(reinterpret_cast<uintptr_t>(row0 + r * J.row_stride) & 15);
  return r * J.rowcap + off;
}

ECA_DEV const uint8_t* item_row0(const StripJob& J, int item) {
  const int frame = item / J.n_strips;
  const int strip = item - frame * J.n_strips;
  return J.frames + int64_t(frame) * J.frame_stride + int64_t(J.band[strip]) * J.row_stride;
}

// thread 0: start the TMA copy of an item's three rows into `stage`
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

template <int NSTAGE>
__host__ __device__ inline size_t strip_smem_bytes(int rowcap, int sumcap, bool fused) {
  size_t b = 128 + size_t(NSTAGE) * 3 * rowcap + size_t(3) * sumcap * 2 + kDTab * 4 +
             sizeof(StripRed);
  if (fused) b += sizeof(FitScratch) + 16;
  return (b + 127) & ~size_t(127);
}

// ------------------------------------------------------------------ kernel
template <int NSTAGE, bool kRows, bool kFused>
__global__ void __launch_bounds__(512) strip_kernel(const __grid_constant__ StripJob J) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, n_warps = blockDim.x >> 5;
  const int W = J.p.width, H = J.p.height;
  const int S = J.n_strips;
  const int n_items = J.batch * S;
  const int split = (W + 1) / 2;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* raw = smem + 128;
  uint16_t* sums = reinterpret_cast<uint16_t*>(raw + size_t(NSTAGE) * 3 * J.rowcap);
  float* dtab = reinterpret_cast<float*>(sums + 3 * J.sumcap);
  StripRed* red = reinterpret_cast<StripRed*>(dtab + kDTab);
  FitScratch* fs = reinterpret_cast<FitScratch*>(
      (reinterpret_cast<uintptr_t>(red + 1) + 15) & ~uintptr_t(15));
  const int stage_bytes = 3 * J.rowcap;

  uint64_t pol = 0;
  if (tid == 0) {
    pol = l2_evict_first();
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  for (int i = tid; i < kDTab; i += blockDim.x) dtab[i] = J.dtab[i];
  // zero the sum-row padding once (columns -1 and >= W read as 0)
  for (int i = tid; i < 3 * J.sumcap; i += blockDim.x) sums[i] = 0;
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      const int item = blockIdx.x + s * gridDim.x;
      if (item < n_items) issue_item(J, item, raw + s * stage_bytes, &bars[s], pol);
    }
  }
  const double cxf = div_rn(double(W - 1), 2.0);  // geometry.py:44
  const double cyf = div_rn(double(H - 1), 2.0);
  const int x0 = tid * kPx;

  int it = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
    const int stage = it % NSTAGE;
    const uint32_t parity = uint32_t(it / NSTAGE) & 1u;
    const int frame = item / S;
    const int strip = item - frame * S;
    const int y = J.rows[strip];
    const uint8_t* row0 = item_row0(J, item);
    uint8_t* st = raw + stage * stage_bytes;

    mbar_wait(&bars[stage], parity);

    // ---- 1. RGB sums of my 8 pixels in rows h-1, h, h+1 ----
    int a[3][kPx];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      uint32_t w[6];
      load24(st, row_base(J, row0, r) + 3 * x0, w);
      sums8(w, a[r]);
#pragma unroll
      for (int i = 0; i < kPx; ++i)
        if (x0 + i >= W) a[r][i] = 0;
      uint4 pk;
      pk.x = uint32_t(a[r][0]) | (uint32_t(a[r][1]) << 16);
      pk.y = uint32_t(a[r][2]) | (uint32_t(a[r][3]) << 16);
      pk.z = uint32_t(a[r][4]) | (uint32_t(a[r][5]) << 16);
      pk.w = uint32_t(a[r][6]) | (uint32_t(a[r][7]) << 16);
      if (x0 < W) *reinterpret_cast<uint4*>(sums + r * J.sumcap + kPad + x0) = pk;
    }
    // centre-row local scans + warp scans of the thread maxima
    int pre_in[kPx], suf_in[kPx];
    int run = 0;
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      pre_in[i] = run;
      run = max(run, a[1][i]);
    }
    const int tmax = run;
    run = 0;
#pragma unroll
    for (int i = kPx - 1; i >= 0; --i) {
      suf_in[i] = run;
      run = max(run, a[1][i]);
    }
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
    __syncthreads();  // (A) stage consumed, sums + warp totals visible

    if (tid == 0) {
      const int nxt = item + NSTAGE * gridDim.x;
      if (nxt < n_items) issue_item(J, nxt, st, &bars[stage], pol);
    }
    for (int w = 0; w < warp; ++w) ex_up = max(ex_up, red->wtot[w]);
    for (int w = warp + 1; w < n_warps; ++w) ex_dn = max(ex_dn, red->wtot[w]);

    int nl[3], nr[3];  // sums at x0-1 and x0+8
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      nl[r] = sums[r * J.sumcap + kPad + x0 - 1];
      nr[r] = sums[r * J.sumcap + kPad + x0 + kPx];
    }
    int pre[kPx];
#pragma unroll
    for (int i = 0; i < kPx; ++i)
      pre[i] = (x0 + i < split) ? max(ex_up, pre_in[i]) : max(ex_dn, suf_in[i]);

    // neighbour access helpers
    auto at = [&](int r, int i) -> int {  // i in [-1, kPx]
      return i < 0 ? nl[r] : (i >= kPx ? nr[r] : a[r][i]);
    };
    const int d2y = (H - 1) - 2 * y;

    // ---- 3. FP32 prefilter scores + per-half max ----
    float ap[kPx];
    float hm0 = 0.0f, hm1 = 0.0f;
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      const int x = x0 + i;
      float s = 0.0f;
      if (!kRows && x >= 1 && x <= W - 2) {
        const int gx3 = (at(0, i + 1) - at(0, i - 1)) + 2 * (at(1, i + 1) - at(1, i - 1)) +
                        (at(2, i + 1) - at(2, i - 1));
        const int gy3 = (at(2, i - 1) + at(2, i + 1) + 2 * at(2, i)) -
                        (at(0, i - 1) + at(0, i + 1) + 2 * at(0, i));
        if (gx3 != 0 || gy3 != 0) {
          const int d2x = (W - 1) - 2 * x;
          if (d2x == 0 && d2y == 0) {
            // frame-centre pixel: atan2(+-0, +-0) sign cases -> exact value
            const int l[3] = {at(0, i - 1), at(1, i - 1), at(2, i - 1)};
            const int m[3] = {at(0, i), at(1, i), at(2, i)};
            const int rr[3] = {at(0, i + 1), at(1, i + 1), at(2, i + 1)};
            s = float(exact_score(l, m, rr, pre[i], x, y, cxf, cyf, J.p));
          } else {
            s = approx_score(gx3, gy3, d2x, d2y, dtab[pre[i]], J.kT, J.kA);
          }
        }
      }
      ap[i] = s;
      if (x < split) hm0 = fmaxf(hm0, s);
      else hm1 = fmaxf(hm1, s);
    }
    bool full0 = true, full1 = true;
    float thr0 = 0.0f, thr1 = 0.0f;
    if (!kRows) {
      hm0 = warp_max(hm0);
      hm1 = warp_max(hm1);
      if (lane == 0) {
        red->wmax[warp][0] = hm0;
        red->wmax[warp][1] = hm1;
      }
      __syncthreads();  // (B)
      hm0 = 0.0f;
      hm1 = 0.0f;
      for (int w = 0; w < n_warps; ++w) {
        hm0 = fmaxf(hm0, red->wmax[w][0]);
        hm1 = fmaxf(hm1, red->wmax[w][1]);
      }
      full0 = !(hm0 >= J.tau);
      full1 = !(hm1 >= J.tau);
      thr0 = hm0 * J.window;
      thr1 = hm1 * J.window;
    }

    // ---- 4. FP64 re-score of the window (or whole flat halves) ----
    Best b0{-1.0, 0x7fffffff}, b1{-1.0, -1};
#pragma unroll
    for (int i = 0; i < kPx; ++i) {
      const int x = x0 + i;
      if (x >= W) continue;
      const bool left = x < split;
      const bool need = kRows || (left ? (full0 || ap[i] >= thr0) : (full1 || ap[i] >= thr1));
      if (!need) continue;
      double s = 0.0;
      if (x >= 1 && x <= W - 2) {
        const int l[3] = {at(0, i - 1), at(1, i - 1), at(2, i - 1)};
        const int m[3] = {at(0, i), at(1, i), at(2, i)};
        const int rr[3] = {at(0, i + 1), at(1, i + 1), at(2, i + 1)};
        s = exact_score(l, m, rr, pre[i], x, y, cxf, cyf, J.p);
      }
      if (kRows) J.out_rows[(size_t(frame) * S + strip) * W + x] = s;
      if (left) {
        if (better(s, x, b0.s, b0.x, true)) b0 = Best{s, x};
      } else {
        if (better(s, x, b1.s, b1.x, false)) b1 = Best{s, x};
      }
    }
    b0 = warp_best(b0, true);
    b1 = warp_best(b1, false);
    if (lane == 0) {
      red->bs[warp][0] = b0.s;
      red->bx[warp][0] = b0.x;
      red->bs[warp][1] = b1.s;
      red->bx[warp][1] = b1.x;
    }
    __syncthreads();  // (C)
    if (tid == 0) {
      Best L{-1.0, 0x7fffffff}, R{-1.0, -1};
      for (int w = 0; w < n_warps; ++w) {
        if (better(red->bs[w][0], red->bx[w][0], L.s, L.x, true)) L = Best{red->bs[w][0], red->bx[w][0]};
        if (better(red->bs[w][1], red->bx[w][1], R.s, R.x, false)) R = Best{red->bs[w][1], red->bx[w][1]};
      }
      const size_t o = size_t(frame) * 2 * S;
      J.out_x[o + strip] = L.x;
      J.out_y[o + strip] = y;
      J.out_score[o + strip] = L.s;
      J.out_x[o + S + strip] = R.x;
      J.out_y[o + S + strip] = y;
      J.out_score[o + S + strip] = R.s;
      if (kFused) {
        __threadfence();
        const int prev = atomicAdd(&J.counters[frame], 1);
        red->last = (prev == S - 1);
      }
    }
    if (kFused) {
      __syncthreads();
      if (red->last) {
        __threadfence();
        const size_t o = size_t(frame) * 2 * S;
        fit_frame(J.out_x + o, J.out_y + o, J.out_score + o, 2 * S, true, J.p, J.triplets,
                  J.exhaustive, fs, J.out_fit + frame);
        if (tid == 0) J.counters[frame] = 0;
      }
    }
    __syncthreads();  // (D) red / sums reused by the next item
  }
}

}  // namespace eca
