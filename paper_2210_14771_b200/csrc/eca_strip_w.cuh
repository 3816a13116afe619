// K1 v5: warp-per-half-row strip scoring (handcrafted.py:148-205, 120-138).
//
// Work item = one HALF of one strip row of one frame: the left half's argmax
// depends only on columns [0, split) (prefix max from the left border) and the
// right half's only on [split, W) (suffix max from the right border), so each
// half-row is independent.  Each WARP owns its items end to end:
//   * its own NSTAGE-deep ring of 1-D TMA bulk copies (3 rows x half width + 1
//     neighbour column) and mbarriers; no CTA barrier after the prologue;
//   * chunks of 256 columns (8 per lane) in scan order (left half left-to-right,
//     right half right-to-left), carrying the preceding max across chunks;
//   * per lane and chunk, rigorous bounds: U_t = T_up(max q) * D_up(first
//     preceding) >= every column's score, L_t = T_lo * A_lo * D_lo of the
//     max-|g| column; LB = warp max of L_t;
//   * only chunks with some U_t >= LB are revisited column by column
//     (V = T_up*D_up, U = V*A_up >= LB); survivors are scored in FP64 in the
//     reference's evaluation order, lane-parallel, argmax with the
//     reference's outermost tie-break.
// The tanh and darkness terms are evaluated with MUFU ex2/rcp/sqrt and padded
// by kPadRel (their FP32 error is < 1e-5 for every config eca_prefilter_bound
// accepts); the angle term comes from a small per-CTA table (A over a
// pseudo-angle).  Flat rows fall back to exhaustive FP64 over non-flat columns.
#pragma once

#include "eca_strip.cuh"

namespace eca {

constexpr int kWChunk = 256;       // columns per chunk (32 lanes x kPx)
constexpr int kWMaxChunks = 8;     // half width <= 2048
constexpr int kWListCap = 256;     // per-warp survivor list (flushed to FP64 when full)

#ifdef ECA_STATS
// diagnostic counters: [0] half-rows, [1] full halves, [2] chunks, [3] revisited
// chunks, [4] survivors, [5] uniform lane-chunks, [6] lanes with u >= lb
__device__ unsigned long long g_warp_stats[8];
#define ECA_WSTAT(k, v) atomicAdd(&g_warp_stats[k], (unsigned long long)(v))
#else
#define ECA_WSTAT(k, v)
#endif

struct WarpLayout {
  size_t atab, warp0, per_warp, stage, list, total;
};

__host__ __device__ inline WarpLayout warp_layout(int nstage, int rowcap_h, int warps) {
  WarpLayout L;
  size_t o = 0;
  L.atab = o;
  o += ((kABins + 2) * 8 + 127) & ~size_t(127);
  L.stage = size_t(3) * rowcap_h;
  if (L.stage < sizeof(FitScratchW)) L.stage = sizeof(FitScratchW);
  L.stage = (L.stage + 127) & ~size_t(127);
  L.list = size_t(nstage) * L.stage;
  L.per_warp = L.list + ((kWListCap * 4 + 16 * 8 + 127) & ~size_t(127));  // list + mbarriers
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

// issue the three row copies of half-row item into `stage` (lane 0)
ECA_DEV void issue_half(const StripJob& J, int item, uint8_t* stage, uint64_t* bar, uint64_t pol,
                        int split) {
  const int half = item & 1;
  const int fs = item >> 1;
  const int frame = fs / J.n_strips;
  const int strip = fs - frame * J.n_strips;
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

template <int NSTAGE, bool kFused>
#ifndef ECA_WMINB
#define ECA_WMINB 2
#endif
__global__ void __launch_bounds__(256, ECA_WMINB) strip_warp_kernel(const __grid_constant__ StripJob J) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const int W = J.p.width, H = J.p.height;
  const int S = J.n_strips;
  const int n_items = J.batch * S * 2;
  const int split = (W + 1) / 2;
  const WarpLayout WL = warp_layout(NSTAGE, J.rowcap, warps);
  float2* atab = reinterpret_cast<float2*>(smem + WL.atab);
  uint8_t* mine = smem + WL.warp0 + size_t(wib) * WL.per_warp;
  uint32_t* list = reinterpret_cast<uint32_t*>(mine + WL.list);
  uint64_t* bars = reinterpret_cast<uint64_t*>(mine + WL.list + kWListCap * 4);

  // ---- prologue: angle table (whole CTA), per-warp barriers + first copies
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
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    pol = l2_evict_first();
    for (int s = 0; s < NSTAGE; ++s) {
      const int it = gw + s * nw;
      if (it < n_items) issue_half(J, it, mine + s * WL.stage, &bars[s], pol, split);
    }
  }
  __syncthreads();   // the only CTA barrier: atab + barrier init visible

  const double log2e = 1.4426950408889634;
  const TermK tk{float(-2.0 * log2e / (3.0 * J.p.gradient_threshold)),
                 float(2.0 * log2e / (3.0 * J.p.intensity_threshold))};
  const float lo_f = 1.0f - kPadRel, hi_f = 1.0f + kPadRel;
  const double cxf = div_rn(double(W - 1), 2.0);
  const double cyf = div_rn(double(H - 1), 2.0);

  int stage = 0;
  uint32_t phase = 0;
  for (int item = gw; item < n_items; item += nw) {
    const int half = item & 1;
    const int fs = item >> 1;
    const int frame = fs / S;
    const int strip = fs - frame * S;
    const int y = J.rows[strip];
    const int d2y = (H - 1) - 2 * y;
    const int xa = half ? split : 0, xb = half ? W : split;   // the half [xa, xb)
    const int xs = half ? split - 1 : 0;                     // first staged column
    uint8_t* st = mine + stage * WL.stage;
    int rb[3];
    {
      const uint8_t* row0 = J.frames + int64_t(frame) * J.frame_stride +
                            int64_t(J.band[strip]) * J.row_stride + 3 * xs;
#pragma unroll
      for (int r = 0; r < 3; ++r)
        rb[r] = r * J.rowcap + int(reinterpret_cast<uintptr_t>(row0 + r * J.row_stride) & 15) -
                3 * xs;   // smem byte of column x in row r = rb[r] + 3x
    }
    mbar_wait(&bars[stage], phase);

    const int hw = xb - xa;
    const int nch = (hw + kWChunk - 1) / kWChunk;
    auto chunk_x0 = [&](int k) -> int {   // first column of lane 0 in chunk k
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

    // load one chunk: c/e (with neighbours) and centre sums of my 8 columns
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
        const bool in = x0 + i >= xa && x0 + i < xb;
        c[i + 1] = s0[i] + 2 * s1[i] + s2[i];
        e[i + 1] = s2[i] - s0[i];
        ctr[i] = in ? s1[i] : 0;
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
      if (lane == 31 && x0 + kPx < min(xb + 1, W)) {
        const int a0 = col_sum(0, x0 + kPx), a1 = col_sum(1, x0 + kPx), a2 = col_sum(2, x0 + kPx);
        c[kPx + 1] = a0 + 2 * a1 + a2;
        e[kPx + 1] = a2 - a0;
      }
    };

    // ---- pass 1: per chunk, lane bounds + preceding-max carry ----
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
      int sc = tmax;   // inclusive scan in scan order
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
      const bool uniform = x0 >= max(xa, 1) && x0 + kPx - 1 <= min(xb, W - 1) - 1;
      float u = 0.0f, l = 0.0f;
      if (uniform) {
        int qmax = 0, bgx = 0, bgy = 0, bi = 0;
#pragma unroll
        for (int i = 0; i < kPx; ++i) {
          const int gx3 = c[i + 2] - c[i], gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
          const int q = gx3 * gx3 + gy3 * gy3;
          if (q > qmax) {
            qmax = q;
            bgx = gx3;
            bgy = gy3;
            bi = i;
          }
        }
        if (qmax > 0) {
          int pbi = ex;   // preceding sum of the max-|g| column
#pragma unroll
          for (int i = 0; i < kPx; ++i)
            if (half ? (i > bi) : (i < bi)) pbi = max(pbi, ctr[i]);
          const float t = t_term(qmax, tk);
          u = fminf(t * hi_f, 1.0f) * fminf(d_term(ex, tk) * hi_f, 1.0f);
          l = t * lo_f * d_term(pbi, tk) * lo_f * atab[abin(bgx, bgy, x0 + bi)].x;
        }
      } else {
        u = INFINITY;   // edge lanes are always revisited
#pragma unroll
        for (int i = 0; i < kPx; ++i) {
          const int x = x0 + i;
          const int gx3 = c[i + 2] - c[i], gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
          const int q = gx3 * gx3 + gy3 * gy3;
          if (x >= xa && x < xb && x >= 1 && x <= W - 2 && q > 0) {
            int p = ex;
#pragma unroll
            for (int k2 = 0; k2 < kPx; ++k2)
              if (half ? (k2 > i) : (k2 < i)) p = max(p, ctr[k2]);
            l = fmaxf(l, t_term(q, tk) * lo_f * d_term(p, tk) * lo_f *
                             atab[abin(gx3, gy3, x)].x);
          }
        }
      }
      ut[k] = u;
      lb = fmaxf(lb, l);
    }
    lb = warp_max(lb);
    const bool full = !(lb >= J.tau);
#ifdef ECA_STATS
    if (lane == 0) {
      ECA_WSTAT(0, 1);
      ECA_WSTAT(1, full ? 1 : 0);
      ECA_WSTAT(2, nch);
    }
    for (int k = 0; k < nch; ++k) {
      const bool anyk = __any_sync(kFull, full || ut[k] >= lb);
      if (lane == 0 && anyk) ECA_WSTAT(3, 1);
      if (ut[k] >= lb && ut[k] < INFINITY) ECA_WSTAT(6, 1);
      if (ut[k] < INFINITY) ECA_WSTAT(5, 1);
    }
#endif

    // ---- pass 2: revisit chunks that can hold the argmax; FP64 survivors ----
    Best best = half ? Best{0.0, W - 1} : Best{0.0, 0};   // border columns score 0
    int n_list = 0;
    auto flush = [&]() {
      for (int k = lane; k < n_list; k += 32) {
        int x;
        const double s = score_entry(list[k], st, rb, y, cxf, cyf, J.p, x);
        if (better(s, x, best.s, best.x, !half)) best = Best{s, x};
      }
      n_list = 0;
      __syncwarp();
    };
#pragma unroll 1
    for (int k = 0; k < nch; ++k) {
      const bool look = full || ut[k] >= lb;
      if (!__any_sync(kFull, look)) continue;
      const int x0 = chunk_x0(k) + kPx * lane;
      int c[kPx + 2], e[kPx + 2], ctr[kPx];
      load_chunk(x0, c, e, ctr);
      uint32_t surv = 0;
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
              const float v = fminf(t_term(q, tk) * hi_f, 1.0f) * fminf(d_term(pre[i], tk) * hi_f, 1.0f);
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
#ifdef ECA_STATS
    if (lane == 0) ECA_WSTAT(4, n_list);
#endif
    flush();
    best = warp_best(best, !half);

    // ---- outputs (+ fused fit when this half-row completes its frame) ----
    const size_t o = size_t(frame) * 2 * S;
    if (lane == 0) {
      const size_t slot = o + (half ? S : 0) + strip;
      J.out_x[slot] = best.x;
      J.out_y[slot] = y;
      J.out_score[slot] = best.s;
    }
    if (kFused) {
      int last = 0;
      if (lane == 0) {
        __threadfence();
        last = atomicAdd(&J.counters[frame], 1) == 2 * S - 1;
      }
      if (__shfl_sync(kFull, last, 0)) {
        __threadfence();
        fit_warp(J.out_x + o, J.out_y + o, J.out_score + o, 2 * S, J.p, J.triplets, J.exhaustive,
                 reinterpret_cast<FitScratchW*>(st), J.out_fit + frame);
        if (lane == 0) J.counters[frame] = 0;
      }
    }
    __syncwarp();
    if (lane == 0) {   // this stage is drained: refill it
      const int nxt = item + NSTAGE * nw;
      if (nxt < n_items) issue_half(J, nxt, st, &bars[stage], pol, split);
    }
    if (++stage == NSTAGE) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

}  // namespace eca
