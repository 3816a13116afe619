// K1 (v6): handcrafted candidate extraction as three dense stages
// (handcrafted.py:148-205, 120-138).
//
//  bounds_kernel   warp per HALF strip row, persistent, own TMA ring: exact
//                  integer sums / Sobel / preceding max and rigorous FP32
//                  bounds; writes the columns that can still hold the half's
//                  FP64 argmax ("survivors", ~2 per half on the C2 mix) into
//                  a fixed slot array together with their 3x3 RGB sums.
//  rescore_kernel  one lane per slot, 8 slots per half row: the reference's
//                  FP64 score of each survivor in numpy's evaluation order,
//                  then the half-row argmax (outermost tie-break) by shuffles.
//  (fit_kernel)    eca_fit.cuh, one warp per frame.
//
// Splitting the FP64 work out keeps its long latency chains off the pixel
// warps and runs it at full lane occupancy.  A half row with more than kSlots
// survivors (adversarial / near-flat rows) is resolved inside bounds_kernel
// with the same FP64 code.
#pragma once

#include "eca_strip.cuh"
#include "eca_strip_w.cuh"

namespace eca {

constexpr int kSlots = 8;

// one survivor: column, preceding sum and the 9 neighbourhood sums (rows h-1..h+1)
struct SurvSlot {
  uint16_t x, pre;
  uint16_t l[3], m[3], r[3];
  uint16_t pad;
};
static_assert(sizeof(SurvSlot) == 24, "slot layout");

struct PointsJob {
  StripJob J;          // geometry, params, candidate outputs
  SurvSlot* slots;     // [n_halfrows][kSlots]
  int32_t* counts;     // [n_halfrows]: survivors, or -1 when resolved in bounds_kernel
};

template <int NS>
__global__ void __launch_bounds__(256, 2) bounds_kernel(const __grid_constant__ PointsJob PJ) {
  const StripJob& J = PJ.J;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const int W = J.p.width, H = J.p.height;
  const int S = J.n_strips;
  const int n_items = J.batch * S * 2;
  const int split = (W + 1) / 2;
  const WarpLayout WL = warp_layout(NS, J.rowcap, warps);
  float2* atab = reinterpret_cast<float2*>(smem + WL.atab);
  uint8_t* mine = smem + WL.warp0 + size_t(wib) * WL.per_warp;
  uint32_t* list = reinterpret_cast<uint32_t*>(mine + WL.list);
  uint64_t* bars = reinterpret_cast<uint64_t*>(mine + WL.list + kWListCap * 4);

  {
    const float lo_f = 1.0f - kPadRel, hi_f = 1.0f + kPadRel;
    const float asc = float(J.p.angle_scale);
    for (int k = threadIdx.x; k < kABins; k += blockDim.x) {
      const float w = 2.0f / kABins;
      const float th_lo = theta_of(k * w - 1e-5f), th_hi = theta_of((k + 1) * w + 1e-5f);
      atab[k] = make_float2(angle_term(th_hi, asc) * lo_f, fminf(angle_term(th_lo, asc) * hi_f, 1.0f));
    }
    if (threadIdx.x == 0)
      atab[kABins] = make_float2(angle_term(3.14159265358979f, asc) * lo_f, 1.0f);
  }
  const int gw = blockIdx.x * warps + wib, nw = gridDim.x * warps;
  uint64_t pol = 0;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    pol = l2_evict_first();
    for (int s = 0; s < NS; ++s) {
      const int it = gw + s * nw;
      if (it < n_items) issue_half(J, it, mine + s * WL.stage, &bars[s], pol, split);
    }
  }
  __syncthreads();

  const double log2e = 1.4426950408889634;
  const TermK tk{float(-2.0 * log2e / (3.0 * J.p.gradient_threshold)),
                 float(2.0 * log2e / (3.0 * J.p.intensity_threshold))};
  const float lo_f = 1.0f - kPadRel, hi_f = 1.0f + kPadRel;

  int stage = 0;
  uint32_t phase = 0;
  for (int item = gw; item < n_items; item += nw) {
    const int half = item & 1;
    const int fs = item >> 1;
    const int frame = fs / S;
    const int strip = fs - frame * S;
    const int y = J.rows[strip];
    const int d2y = (H - 1) - 2 * y;
    const int xa = half ? split : 0, xb = half ? W : split;
    const int xs = half ? split - 1 : 0;
    const int xe = half ? W : min(split + 1, W);
    uint8_t* st = mine + stage * WL.stage;
    int rb[3];
    {
      const uint8_t* row0 = J.frames + int64_t(frame) * J.frame_stride +
                            int64_t(J.band[strip]) * J.row_stride + 3 * xs;
#pragma unroll
      for (int r = 0; r < 3; ++r)
        rb[r] = r * J.rowcap + int(reinterpret_cast<uintptr_t>(row0 + r * J.row_stride) & 15) -
                3 * xs;
    }
    mbar_wait(&bars[stage], phase);

    const int nch = (xb - xa + kWChunk - 1) / kWChunk;
    auto chunk_x0 = [&](int k) -> int {
      return half ? (xa + (nch - 1 - k) * kWChunk) : (xa + k * kWChunk);
    };
    auto abin = [&](int gx3, int gy3, int x) -> int {
      const int d2x = (W - 1) - 2 * x;
      const int dot = gx3 * d2x + gy3 * d2y;
      const int crs = abs(gx3 * d2y - gy3 * d2x);
      const float fd = float(abs(dot)), fc = float(crs);
      const float ps = fc * rcpf(fd + fc);
      const int k = min(int((dot >= 0 ? ps : 2.0f - ps) * (kABins / 2)), kABins - 1);
      return (dot == 0 && crs == 0) ? kABins : k;
    };
    auto col_sum = [&](int r, int x) -> int { return px_sum(st, rb[r] + 3 * x); };
    auto load_chunk = [&](int x0, int c[kPx + 2], int e[kPx + 2], int ctr[kPx]) {
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
        c[i + 1] = s0[i] + 2 * s1[i] + s2[i];
        e[i + 1] = s2[i] - s0[i];
        ctr[i] = (x0 + i >= xa && x0 + i < xb) ? s1[i] : 0;
      }
      c[0] = __shfl_up_sync(kFull, c[kPx], 1);
      e[0] = __shfl_up_sync(kFull, e[kPx], 1);
      c[kPx + 1] = __shfl_down_sync(kFull, c[1], 1);
      e[kPx + 1] = __shfl_down_sync(kFull, e[1], 1);
      if (lane == 0 && x0 - 1 >= xs) {
        const int a0 = col_sum(0, x0 - 1), a1 = col_sum(1, x0 - 1), a2 = col_sum(2, x0 - 1);
        c[0] = a0 + 2 * a1 + a2;
        e[0] = a2 - a0;
      }
      if (lane == 31 && x0 + kPx < xe) {
        const int a0 = col_sum(0, x0 + kPx), a1 = col_sum(1, x0 + kPx), a2 = col_sum(2, x0 + kPx);
        c[kPx + 1] = a0 + 2 * a1 + a2;
        e[kPx + 1] = a2 - a0;
      }
    };

    // ---- pass 1: lane-chunk bounds (U over its columns, L of its best column)
    float ut[kWMaxChunks];
    int exk[kWMaxChunks];
    float lb = 0.0f;
    int carry = 0;
#pragma unroll 1
    for (int k = 0; k < nch; ++k) {
      const int x0 = chunk_x0(k) + kPx * lane;
      int c[kPx + 2], e[kPx + 2], ctr[kPx];
      load_chunk(x0, c, e, ctr);
      int tmax = 0;
#pragma unroll
      for (int i = 0; i < kPx; ++i) tmax = max(tmax, ctr[i]);
      int sc = tmax;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = half ? __shfl_down_sync(kFull, sc, d) : __shfl_up_sync(kFull, sc, d);
        if (half ? (lane + d < 32) : (lane >= d)) sc = max(sc, v);
      }
      int ex = half ? __shfl_down_sync(kFull, sc, 1) : __shfl_up_sync(kFull, sc, 1);
      if (half ? lane == 31 : lane == 0) ex = 0;
      ex = max(ex, carry);
      carry = max(carry, __shfl_sync(kFull, sc, half ? 0 : 31));
      exk[k] = ex;
      // per column: V = T_up * D_up needs the column's own preceding sum; the
      // lane bound uses the head (smallest preceding) and the best column
      float u = 0.0f, l = 0.0f;
      int qmax = 0, bgx = 0, bgy = 0, bi = 0;
#pragma unroll
      for (int i = 0; i < kPx; ++i) {
        const int x = x0 + i;
        const int gx3 = c[i + 2] - c[i], gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
        const int q = (x >= xa && x < xb && x >= 1 && x <= W - 2) ? gx3 * gx3 + gy3 * gy3 : 0;
        if (q > qmax) {
          qmax = q;
          bgx = gx3;
          bgy = gy3;
          bi = i;
        }
      }
      if (qmax > 0) {
        int pbi = ex;
#pragma unroll
        for (int i = 0; i < kPx; ++i)
          if (half ? (i > bi) : (i < bi)) pbi = max(pbi, ctr[i]);
        const float t = t_term(qmax, tk);
        u = fminf(t * hi_f, 1.0f) * fminf(d_term(ex, tk) * hi_f, 1.0f);
        l = t * lo_f * d_term(pbi, tk) * lo_f * atab[abin(bgx, bgy, x0 + bi)].x;
      }
      ut[k] = u;
      lb = fmaxf(lb, l);
    }
    lb = warp_max(lb);
    const bool full = !(lb >= J.tau);

    // ---- pass 2: survivors of chunks whose bound reaches LB
    int n_list = 0;
    bool flushed = false;
    Best best = half ? Best{0.0, W - 1} : Best{0.0, 0};   // border columns score 0
    const double cxf = div_rn(double(W - 1), 2.0);
    const double cyf = div_rn(double(H - 1), 2.0);
    auto flush = [&]() {   // rare: score the pending survivors here
      for (int k = lane; k < n_list; k += 32) {
        int x;
        const double s = score_entry(list[k], st, rb, y, cxf, cyf, J.p, x);
        if (better(s, x, best.s, best.x, !half)) best = Best{s, x};
      }
      n_list = 0;
      flushed = true;
      __syncwarp();
    };
#pragma unroll 1
    for (int k = 0; k < nch; ++k) {
      const bool look = full || (ut[k] > 0.0f && ut[k] >= lb);
      if (!__any_sync(kFull, look)) continue;
      const int x0 = chunk_x0(k) + kPx * lane;
      int c[kPx + 2], e[kPx + 2], ctr[kPx];
      load_chunk(x0, c, e, ctr);
      int pre[kPx];
      {
        int run = exk[k];
        if (half) {
#pragma unroll
          for (int i = kPx - 1; i >= 0; --i) {
            pre[i] = run;
            run = max(run, ctr[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < kPx; ++i) {
            pre[i] = run;
            run = max(run, ctr[i]);
          }
        }
      }
      uint32_t surv = 0;
      if (look) {
#pragma unroll
        for (int i = 0; i < kPx; ++i) {
          const int x = x0 + i;
          if (x < xa || x >= xb || x < 1 || x > W - 2) continue;
          bool s;
          if (full) {
            s = !flat_column(st, rb, x);
          } else {
            const int gx3 = c[i + 2] - c[i], gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
            const int q = gx3 * gx3 + gy3 * gy3;
            s = false;
            if (q > 0) {
              const float v = fminf(t_term(q, tk) * hi_f, 1.0f) *
                              fminf(d_term(pre[i], tk) * hi_f, 1.0f);
              s = v >= lb && v * atab[abin(gx3, gy3, x)].y >= lb;
            }
          }
          if (s) surv |= 1u << i;
        }
      }
      const int cnt = __popc(surv);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += v;
      }
      const int tot = __shfl_sync(kFull, incl, 31);
      if (n_list + tot > kWListCap) flush();
      int base = n_list + incl - cnt;
#pragma unroll
      for (int i = 0; i < kPx; ++i)
        if ((surv >> i) & 1u) list[base++] = uint32_t(x0 + i) | (uint32_t(pre[i]) << 16);
      n_list += tot;
      __syncwarp();
    }

    // ---- hand the survivors to the rescore stage (or resolve here if many)
    const int hrow = item;
    SurvSlot* out = PJ.slots + size_t(hrow) * kSlots;
    if (!flushed && n_list <= kSlots) {
      if (lane < n_list) {
        const uint32_t v = list[lane];
        const int x = int(v & 0xffffu);
        SurvSlot s;
        s.x = uint16_t(x);
        s.pre = uint16_t(v >> 16);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          s.l[r] = uint16_t(col_sum(r, x - 1));
          s.m[r] = uint16_t(col_sum(r, x));
          s.r[r] = uint16_t(col_sum(r, x + 1));
        }
        s.pad = 0;
        out[lane] = s;
      }
      if (lane == 0) PJ.counts[hrow] = n_list;
    } else {
      // rare: more survivors than slots -> score them in this warp
      flush();
      best = warp_best(best, !half);
      if (lane == 0) {
        const size_t slot = size_t(frame) * 2 * S + (half ? S : 0) + strip;
        J.out_x[slot] = best.x;
        J.out_y[slot] = y;
        J.out_score[slot] = best.s;
        PJ.counts[hrow] = -1;
      }
    }
    __syncwarp();
    if (lane == 0) {
      const int nxt = item + NS * nw;
      if (nxt < n_items) issue_half(J, nxt, st, &bars[stage], pol, split);
    }
    if (++stage == NS) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

// One lane per slot, 4 half rows per warp: FP64 rescoring + half-row argmax.
__global__ void __launch_bounds__(128) rescore_kernel(const __grid_constant__ PointsJob PJ) {
  const StripJob& J = PJ.J;
  const int lane = threadIdx.x & 31;
  const int S = J.n_strips, W = J.p.width, H = J.p.height;
  const int n_hr = J.batch * S * 2;
  const int hrow = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  const int k = lane & 7;
  if (hrow - (lane >> 3) >= n_hr) return;   // whole warp past the end
  const bool valid_hr = hrow < n_hr;
  const int cnt = valid_hr ? __ldg(PJ.counts + hrow) : -1;
  const int half = hrow & 1;
  const int fs = hrow >> 1;
  const int frame = fs / S, strip = fs - (fs / S) * S;
  const int y = valid_hr ? J.rows[strip] : 0;
  Best b = half ? Best{0.0, W - 1} : Best{0.0, 0};
  if (valid_hr && k < cnt) {
    const SurvSlot s = PJ.slots[size_t(hrow) * kSlots + k];
    const int l[3] = {s.l[0], s.l[1], s.l[2]}, m[3] = {s.m[0], s.m[1], s.m[2]},
              r[3] = {s.r[0], s.r[1], s.r[2]};
    const double cxf = div_rn(double(W - 1), 2.0);
    const double cyf = div_rn(double(H - 1), 2.0);
    b = Best{exact_score(l, m, r, s.pre, s.x, y, cxf, cyf, J.p), int(s.x)};
  }
  // argmax inside each 8-lane group (half rows never mix)
#pragma unroll
  for (int d = 4; d; d >>= 1) {
    const double os = __shfl_xor_sync(kFull, b.s, d);
    const int ox = __shfl_xor_sync(kFull, b.x, d);
    if (better(os, ox, b.s, b.x, !half)) {
      b.s = os;
      b.x = ox;
    }
  }
  if (valid_hr && k == 0 && cnt >= 0) {
    const size_t slot = size_t(frame) * 2 * S + (half ? S : 0) + strip;
    J.out_x[slot] = b.x;
    J.out_y[slot] = y;
    J.out_score[slot] = b.s;
  }
}

}  // namespace eca
