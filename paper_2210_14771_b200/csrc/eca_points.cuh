// K1 (v7): handcrafted candidate extraction as two dense stages
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
// bounds_kernel, per half row:
//  pass 1   chunks of 256 columns in scan order (left half: x ascending from
//           the border, right half: x descending from the border), 8 columns
//           per lane ("lane-chunk").  Each lane loads its 8 columns plus both
//           neighbours straight from shared memory, so lanes exchange no
//           pixels.  Per lane-chunk only the upper bound
//           U = T_up(max |g|^2) * D_up(preceding sum before the lane-chunk)
//           is kept; it bounds every column's score because T rises with |g|,
//           D falls with the preceding sum and A <= 1.
//  step A/B the 4 lane-chunks of highest U are evaluated column by column
//           (one lane per column): L = T_lo*A_lo*D_lo is a lower bound of the
//           half's max score, so LB = max L.
//  step C   every other lane-chunk with U >= LB is compacted and evaluated
//           the same way; columns with U_col = T_up*D_up*A_up >= LB survive.
// A half whose LB is below the FP32 resolution (tau) keeps every non-flat
// column instead (flat-row residues, see eca_prefilter_bound).  A half row
// with more than kSlots survivors is resolved in this kernel with the same
// FP64 code.  Splitting the FP64 work out keeps its long latency chains off
// the pixel warps and runs it at full lane occupancy.
#pragma once

#include <cuda_fp16.h>

#include "eca_strip.cuh"
#include "eca_strip_w.cuh"

namespace eca {

constexpr int kSlots = 8;
#ifndef ECA_STATIC_ROUNDS
#define ECA_STATIC_ROUNDS 1
#endif
constexpr int kStaticRounds = ECA_STATIC_ROUNDS;   // items per warp assigned before tickets
// Scheduling knobs (the results do not depend on them: they decide when the
// exact bound tests run, not what they conclude); r02 sweep, tools/time_pipe.py
// + tools/prof_zc.py: early LB at D_up 0.05 / 0.1 / 0.2 / 0.35 / 0.6 / 1.01 ->
// 28.1 / 27.6 / 27.3 / 27.3 / 27.3 / 42.3 us per step; refine above 4 / 8 / 16
// -> 27.8 / 27.6 / 27.5; 0.35 + 16: 27.2 us and 3 % fewer zero-copy bytes.
#ifndef ECA_REFINE_MIN
#define ECA_REFINE_MIN 16
#endif
#ifndef ECA_EARLY_D
#define ECA_EARLY_D 0.35f
#endif
constexpr int kRefineMin = ECA_REFINE_MIN;   // step C: refine lane-chunk bounds above this many
constexpr float kEarlyD = ECA_EARLY_D;       // D_up(carry) level that triggers the early LB (gray ~28)

// one survivor: column, preceding sum and the 9 neighbourhood sums (rows h-1..h+1)
struct SurvSlot {
  uint16_t x, pre;
  uint16_t l[3], m[3], r[3];
  uint16_t pad;
};
static_assert(sizeof(SurvSlot) == 24, "slot layout");

#ifdef ECA_TIMELINE   // diagnostic builds: per-CTA start / end (tools/timeline.py)
__device__ unsigned long long g_tl[2][64][1024][2];   // [bounds|fit][launch][cta][start|end]
ECA_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL_STAMP(kind, seq, which)                                                   \
  do {                                                                               \
    if (threadIdx.x == 0 && blockIdx.x < 1024)                                       \
      g_tl[kind][(seq) & 63][blockIdx.x][which] = gtime();                           \
  } while (0)
#else
#define TL_STAMP(kind, seq, which) \
  do {                             \
  } while (0)
#endif
#ifdef ECA_WARP_TIMES   // diagnostic builds: per-warp timeline (tools/warp_times.py)
__device__ uint64_t g_warp_times[3 * 8192];
#endif

struct PointsJob {
  StripJob J;          // geometry, params, candidate outputs
  SurvSlot* slots;     // [n_halfrows][kSlots]
  int32_t* counts;     // [n_halfrows]: survivors, or -1 when resolved in bounds_kernel
  int32_t* ticket;     // [0] next item, [1] warps done (zero between launches);
                       // [2] 16-byte units fetched in zero-copy mode (diagnostic);
                       // [4..5] u64 claim word (high: uses of this workspace,
                       //     low: CTAs of the current use that claimed it),
                       // [6] launches finished on it (set-reuse guard)
  int chunked;         // zero-copy mode: fetch scan chunks on demand (NS == 1)
  int wait_prev;       // griddepcontrol.wait before the first frame load
  int guard;           // set-reuse guard: a launch's CTAs wait until every
                       // earlier launch on this workspace finished
  int dbg_seq;         // launch number (ECA_TIMELINE diagnostic builds)
  // host-computed constants (launch_points_t): no FP64 division, atan2f or
  // integer division in the kernel prologue / item decode
  float2 atab[kABins + 1];   // A bounds per pseudo-angle bin (see eca_strip.cuh)
  float kt, kd;              // TermK
  double cxf, cyf;           // (W-1)/2, (H-1)/2
  uint32_t s_magic;          // ceil(2^32 / n_strips) when batch*n_strips < 2^25, else 0
};

// item -> (frame, strip): multiply-high division when the host provided it
ECA_DEV void decode_item(const PointsJob& PJ, int fs, int& frame, int& strip) {
  const int S = PJ.J.n_strips;
  frame = PJ.s_magic ? int(__umulhi(uint32_t(fs), PJ.s_magic)) : fs / S;
  strip = fs - frame * S;
}

// first TMA copies of a half-row item (lane 0): the whole half, or in
// zero-copy mode its first scan chunk
template <bool kChunked>
ECA_DEV void issue_item_half(const PointsJob& PJ, int item, uint8_t* stage, uint64_t* bar,
                             uint64_t pol, int split) {
  int frame, strip;
  decode_item(PJ, item >> 1, frame, strip);
  if (kChunked) {
    const uint32_t b = issue_chunk(PJ.J, item & 1, frame, strip, 0, stage, bar, pol, split);
    atomicAdd(PJ.ticket + 2, int(b >> 4));
  } else {
    issue_half(PJ.J, item & 1, frame, strip, stage, bar, pol, split);
  }
}

#ifndef ECA_COLD_FLUSH
#define ECA_COLD_FLUSH 1
#endif
// the FP64 score of a list entry outside the kernel body (the overflow path
// runs on a few percent of half rows; inlined, its ~700 FP64 instructions sit
// between the hot blocks)
__device__ __noinline__ double score_entry_cold(uint32_t v, const uint8_t* st, const int* rb, int y, double cxf,
                                                double cyf, const EcaParams& p, int& x) {
  return score_entry(v, st, rb, y, cxf, cyf, p, x);
}

// RGB sums of the 10 pixels x0-1 .. x0+8 of one staged row; B = smem byte of
// pixel x0.  `al`: B % 8 == 0 (warp-uniform), else funnel-shifted word loads.
ECA_DEV void load10(const uint8_t* st, int B, bool al, int s[10]) {
  uint32_t w[8];   // w[0]: bytes B-4..B-1, w[1..6]: B..B+23, w[7]: B+24..B+27
  if (al) {
    const uint2* p = reinterpret_cast<const uint2*>(st + B);
    const uint2 a = p[0], b = p[1], c = p[2];
    w[0] = *reinterpret_cast<const uint32_t*>(st + B - 4);
    w[1] = a.x; w[2] = a.y; w[3] = b.x; w[4] = b.y; w[5] = c.x; w[6] = c.y;
    w[7] = *reinterpret_cast<const uint32_t*>(st + B + 24);
  } else {
    const int a0 = (B - 4) & ~3;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(st + a0);
    const int sh = ((B - 4) - a0) * 8;
    uint32_t v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = wp[k];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = __funnelshift_r(v[k], v[k + 1], sh);
  }
  s[0] = __dp4a(w[0], 0x01010100u, 0u);
  sums8(w + 1, s + 1);
  s[9] = __dp4a(w[7], 0x00010101u, 0u);
}

// One column evaluated by one lane (steps A-C).
struct ColEval {
  int x, pre;
  int l[3], m[3], r[3];
  float U, L;
  bool ok;     // scoreable column of this half (x in [slo, shi])
  bool flat;   // numpy's gx and gy are exactly 0.0 (score exactly 0)
};

// Set-reuse guard (pipelines with programmatic dependent launch, where a
// launch may start before earlier launches on the same workspace finished).
// ticket block: [1] CTAs / warps done, [4..5] u64 claim word (high: uses so
// far, low: CTAs of the current use that claimed), [6] uses finished.  Every
// CTA claims before it triggers its dependents, so all CTAs of use u claim
// before any CTA of use u+1; the last claimer of a use advances the use index.
// Returns the use index u of this launch (thread 0 of a CTA).
ECA_DEV int guard_claim(int32_t* ticket) {
  unsigned long long* claim = reinterpret_cast<unsigned long long*>(ticket + 4);
  const unsigned long long old = atomicAdd(claim, 1ull);
  if (uint32_t(old) + 1u == gridDim.x) atomicAdd(claim, (1ull << 32) - gridDim.x);
  return int(old >> 32);
}
// wait until the u earlier uses of the workspace have finished
ECA_DEV void guard_wait(const int32_t* ticket, int u) {
  int done;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(done) : "l"(ticket + 6) : "memory");
    if (done >= u) break;
    __nanosleep(128);
  }
}
// the last unit out (counter ticket[1] reaching `units`) re-arms the item
// tickets and publishes the end of this use; callers fence their writes first
ECA_DEV bool guard_release(int32_t* ticket, int units) {
  if (atomicAdd(ticket + 1, 1) != units - 1) return false;
  ticket[0] = 0;
  ticket[1] = 0;
  __threadfence();
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ticket + 6) : "memory");
  return true;
}

#ifndef ECA_BOUNDS_MAXREG   // 96: 5 warps per SM sub-partition (120 would allow 4)
#define ECA_BOUNDS_MAXREG 96
#endif
#ifndef ECA_LOAD_ONLY
#define ECA_LOAD_ONLY 0
#endif
#ifndef ECA_EARLY_EXIT
#define ECA_EARLY_EXIT 1
#endif
// kChunked: zero-copy mode (ECA_BOUNDS_ZERO_COPY), a separate instantiation so
// the device-resident kernel carries none of its code
// kInWarp (small batches, the latency path): each warp also rescoring its
// half row's survivors in FP64 and writing the candidate (no survivor slots)
template <int NS, bool kChunked, bool kInWarp = false>
__global__ void __maxnreg__(ECA_BOUNDS_MAXREG) bounds_kernel(const __grid_constant__ PointsJob PJ) {
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
  uint64_t* bars = reinterpret_cast<uint64_t*>(mine + WL.bars);
  __half* ut_s = reinterpret_cast<__half*>(mine + WL.ut);   // rounded up: still a bound
  uint16_t* ex_s = reinterpret_cast<uint16_t*>(mine + WL.exs);
  uint16_t* sel_s = reinterpret_cast<uint16_t*>(mine + WL.sel);

  for (int k = threadIdx.x; k <= kABins; k += blockDim.x) atab[k] = PJ.atab[k];
  const int gw = blockIdx.x * warps + wib, nw = gridDim.x * warps;
  // Items: the first kStaticRounds per warp are fixed (gw, gw + nw, ...), the
  // rest come from a ticket counter (item costs vary ~5x with the early exit
  // and row content; static assignment alone left a long tail, tickets alone
  // cost an atomic round trip per item).  qitem[s] = item in flight in stage s.
  int* qitem = reinterpret_cast<int*>(bars + 8);
  int assigned = 0;   // items handed to this warp so far (lane 0)
  auto next_item = [&]() -> int {
    const int r = assigned++;
    return r < kStaticRounds ? gw + r * nw : kStaticRounds * nw + atomicAdd(PJ.ticket, 1);
  };
  uint64_t pol = 0;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    pol = l2_evict_first();
    // the kernel before this one in the stream may have produced the frames:
    // with programmatic dependent launch, wait for it (and its memory) unless
    // the caller vouched that the frames were complete before that launch
    if (PJ.wait_prev) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int s = 0; s < NS; ++s) {
      const int it = next_item();
      qitem[s] = it;
      if (it < n_items) issue_item_half<kChunked>(PJ, it, mine + s * WL.stage, &bars[s], pol, split);
    }
  }
  if (PJ.guard && threadIdx.x == 0) guard_wait(PJ.ticket, guard_claim(PJ.ticket));
  TL_STAMP(0, PJ.dbg_seq, 0);
  __syncthreads();
  // a dependent launch (the next batch, ECA_BOUNDS_OVERLAP_PREVIOUS) may start
  // filling SMs as this grid's CTAs drain; triggered after the prologue (its
  // first frame loads are in flight), measured 1 us faster per launch than
  // triggering at entry
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef ECA_WARP_TIMES
  if (lane == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_warp_times[3 * (blockIdx.x * warps + wib)] = t;
  }
#endif

  const TermK tk{PJ.kt, PJ.kd};
  const float lo_f = 1.0f - J.pad, hi_f = 1.0f + J.pad;
  const double cxf = PJ.cxf, cyf = PJ.cyf;
  // configs outside the FP32 envelope (tau = inf: every half is scored in
  // FP64) never stop the scan on a bound
  const bool trusted = J.tau < 1.0f;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int gi = lane & 7;   // column within an evaluated lane-chunk

  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    const int item = qitem[stage];   // tickets rise: the first past the end ends the warp
    if (item >= n_items) break;
#ifdef ECA_WARP_TIMES
    uint64_t t_item;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_item));
    int dbg_groups = 0;
#endif
    const int half = item & 1;
    const int fs = item >> 1;
    int frame, strip;
    decode_item(PJ, fs, frame, strip);
    const int y = J.rows[strip];
    const int d2y = (H - 1) - 2 * y;
    const int hw = half ? W - split : split;        // columns in this half
    const int xs = half ? split - 1 : 0;            // first staged column
    const int lo = half ? split : 0, hi = half ? W - 1 : split - 1;   // the half, inclusive
    const int slo = max(lo, 1), shi = min(hi, W - 2);                 // scoreable columns
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
    // first column (x order) of lane-chunk (k, l)
    auto xa_of = [&](int k, int l) -> int {
      return half ? W - kPx - kWChunk * k - kPx * l : kWChunk * k + kPx * l;
    };
    const int xa0 = xa_of(0, 0);
    const bool al = (((rb[0] + 3 * xa0) | (rb[1] + 3 * xa0) | (rb[2] + 3 * xa0)) & 7) == 0;
    const int nch = (hw + kWChunk - 1) / kWChunk;
    mbar_wait(&bars[stage], phase);
    uint32_t cpar = phase ^ 1u;   // zero-copy mode: parity of the next chunk's copy
    // take the next item and start its TMA into this stage (once per item,
    // as soon as the stage's bytes are no longer needed)
    bool advanced = false;
    auto advance = [&]() {
      if (kChunked) phase = cpar ^ 1u;   // (flipped back to cpar below, NS == 1)
      __syncwarp();
      if (lane == 0) {
        // the ticket is taken only now: a warp never holds work it cannot start
        // (prefetching it measured 30% slower from the end-of-kernel imbalance)
        const int nxt = next_item();
        qitem[stage] = nxt;
        if (nxt < n_items) issue_item_half<kChunked>(PJ, nxt, st, &bars[stage], pol, split);
      }
      __syncwarp();
      advanced = true;
    };
#if ECA_LOAD_ONLY   // diagnostic: the TMA ring alone
    if (lane == 0) PJ.counts[item] = 0;
#else

    // ---- one lane per column of lane-chunk entry e = (k << 5 | l)
    auto eval = [&](bool valid, int e) -> ColEval {
      ColEval ce;
      const int k = e >> 5, l = e & 31;
      ce.x = xa_of(k, l) + gi;
      const bool in_half = valid && ce.x >= lo && ce.x <= hi;
      ce.ok = in_half && ce.x >= slo && ce.x <= shi;
      const int xc = in_half ? ce.x : lo;   // keep the reads inside the staged rows
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        ce.l[r] = px_sum(st, rb[r] + 3 * (xc - 1));
        ce.m[r] = px_sum(st, rb[r] + 3 * xc);
        ce.r[r] = px_sum(st, rb[r] + 3 * (xc + 1));
      }
      // preceding sum: lane-chunk prefix + exclusive max over the earlier
      // columns of the lane-chunk in scan order (x ascending left, descending right)
      int v = in_half ? ce.m[1] : 0;
#pragma unroll
      for (int d = 1; d < kPx; d <<= 1) {
        const int o = half ? __shfl_down_sync(kFull, v, d, kPx) : __shfl_up_sync(kFull, v, d, kPx);
        if (half ? gi + d < kPx : gi >= d) v = max(v, o);
      }
      int pre = half ? __shfl_down_sync(kFull, v, 1, kPx) : __shfl_up_sync(kFull, v, 1, kPx);
      if (half ? gi == kPx - 1 : gi == 0) pre = 0;
      ce.pre = max(pre, valid ? int(ex_s[e]) : 0);
      const int cl = ce.l[0] + 2 * ce.l[1] + ce.l[2], cr = ce.r[0] + 2 * ce.r[1] + ce.r[2];
      const int gx3 = cr - cl;
      const int gy3 = (ce.l[2] - ce.l[0]) + 2 * (ce.m[2] - ce.m[0]) + (ce.r[2] - ce.r[0]);
      const int q = gx3 * gx3 + gy3 * gy3;
      ce.U = 0.0f;
      ce.L = 0.0f;
      if (ce.ok && q > 0) {
        const int d2x = (W - 1) - 2 * ce.x;
        const int dot = gx3 * d2x + gy3 * d2y;
        const int crs = abs(gx3 * d2y - gy3 * d2x);
        const float fd = float(abs(dot)), fc = float(crs);
        const float ps = fc * rcpf(fd + fc);
        int ab = min(int((dot >= 0 ? ps : 2.0f - ps) * (kABins / 2)), kABins - 1);
        if (dot == 0 && crs == 0) ab = kABins;
        const float2 a = atab[ab];
        const float t = t_term(q, tk), dd = d_term(ce.pre, tk);
        ce.U = fminf(t * hi_f, 1.0f) * fminf(dd * hi_f, 1.0f) * a.y;
        ce.L = t * lo_f * dd * lo_f * a.x;
      }
      ce.flat = ce.l[0] == ce.r[0] && ce.l[1] == ce.r[1] && ce.l[2] == ce.r[2] &&
                ce.l[0] == ce.l[2] && ce.m[0] == ce.m[2] && ce.r[0] == ce.r[2];
      return ce;
    };

    // survivors: list entries (x | pre << 16) with their column bound U
    float* ulist = reinterpret_cast<float*>(mine + WL.ulist);
    int n_list = 0;
    bool flushed = false;
    Best best = half ? Best{0.0, W - 1} : Best{0.0, 0};   // border columns score 0
    auto flush = [&]() {   // rare: score the pending survivors in this warp
      for (int k = lane; k < n_list; k += 32) {
        int x;
#if ECA_COLD_FLUSH
        const double s = score_entry_cold(list[k], st, rb, y, cxf, cyf, J.p, x);
#else
        const double s = score_entry(list[k], st, rb, y, cxf, cyf, J.p, x);
#endif
        if (better(s, x, best.s, best.x, !half)) best = Best{s, x};
      }
      n_list = 0;
      flushed = true;
      __syncwarp();
    };
    auto compact = [&](float thr) {   // drop entries whose bound fell below LB
      int out = 0;
      for (int base = 0; base < n_list; base += 32) {
        const int k = base + lane;
        const uint32_t v = k < n_list ? list[k] : 0u;
        const float u = k < n_list ? ulist[k] : 0.0f;
        const bool keep = k < n_list && u >= thr;
        const unsigned bm = __ballot_sync(kFull, keep);
        __syncwarp();
        if (keep) {
          const int pos = out + __popc(bm & lt_mask);
          ECA_CHECK(pos < kWListCap);
          list[pos] = v;
          ulist[pos] = u;
        }
        out += __popc(bm);
        __syncwarp();
      }
      n_list = out;
    };
    float lb = 0.0f;
    bool full = false;
    auto emit = [&](bool valid, const ColEval& ce) {
      const bool surv = valid && ce.ok && (full ? !ce.flat : ce.U >= lb);
      const unsigned bm = __ballot_sync(kFull, surv);
      const int tot = __popc(bm);
      if (tot == 0) return;
      if (n_list + tot > kWListCap && lb >= J.tau) compact(lb);
      if (n_list + tot > kWListCap) flush();
      if (surv) {
        const int pos = n_list + __popc(bm & lt_mask);
        ECA_CHECK(pos < kWListCap && ce.x >= lo && ce.x <= hi);
        list[pos] = uint32_t(ce.x) | (uint32_t(ce.pre) << 16);
        ulist[pos] = ce.U;
      }
      n_list += tot;
      __syncwarp();
    };

    // ---- steps A + B over the first nk chunks
    bool ab_done = false;
    auto step_ab = [&](int nk) {
    // A: the (up to) 4 lane-chunks of highest U, from distinct lanes
    float bu = 0.0f;   // lane-chunks with U == 0 (or marked -1) never qualify
    int bk = 0;
    for (int k = 0; k < nk; ++k) {
      const float v = __half2float(ut_s[k * 32 + lane]);
      if (v > bu) {
        bu = v;
        bk = k;
      }
    }
    int my_e = 0;   // entry this lane's 8-lane group evaluates in step B
    int n_a = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float m = warp_max_nonneg(bu);
      if (!(m > 0.0f)) break;
      const int wl = __ffs(__ballot_sync(kFull, bu == m)) - 1;
      const int wk = __shfl_sync(kFull, bk, wl);
      if ((lane >> 3) == g) my_e = (wk << 5) | wl;
      if (lane == wl) bu = 0.0f;
      n_a = g + 1;
    }
    // B: evaluate them -> LB, then their survivors
    const bool va = (lane >> 3) < n_a;
    {
      const ColEval ca = eval(va, my_e);
      lb = warp_max_nonneg(ca.L);
      full = !(lb >= J.tau);
      emit(va, ca);
    }
    if (va && gi == 0) ut_s[(my_e >> 5) * 32 + (my_e & 31)] = __float2half(-1.0f);   // evaluated
    __syncwarp();
    ab_done = true;
    };

    // ---- pass 1: U of every lane-chunk (stops early, see below)
    int carry = 0;
    int nch_eff = nch;
#pragma unroll 1
    for (int k = 0; k < nch; ++k) {
      if (kChunked && k > 0) {   // zero-copy: fetch this chunk only now
        if (lane == 0) {
          const uint32_t b = issue_chunk(J, half, frame, strip, k, st, &bars[stage], pol, split);
          atomicAdd(PJ.ticket + 2, int(b >> 4));
        }
        mbar_wait(&bars[stage], cpar);
        cpar ^= 1u;
      }
      const int xa = xa_of(k, lane);
      int s0[10], s1[10], s2[10];
      load10(st, rb[0] + 3 * xa, al, s0);
      load10(st, rb[1] + 3 * xa, al, s1);
      load10(st, rb[2] + 3 * xa, al, s2);
      int c[10], e[10];
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        c[i] = s0[i] + 2 * s1[i] + s2[i];
        e[i] = s2[i] - s0[i];
      }
      int tmax = 0, qmax = 0;
#pragma unroll
      for (int i = 1; i <= kPx; ++i) tmax = max(tmax, s1[i]);
      if (k == 0 || k == nch - 1) {   // border / tail chunk: only scoreable columns
#pragma unroll
        for (int i = 0; i < kPx; ++i) {
          const int gx3 = c[i + 2] - c[i], gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
          const int q = gx3 * gx3 + gy3 * gy3;
          const bool in = unsigned(xa + i - slo) <= unsigned(shi - slo);
          qmax = max(qmax, in ? q : 0);
        }
      } else {
#pragma unroll
        for (int i = 0; i < kPx; ++i) {
          const int gx3 = c[i + 2] - c[i], gy3 = e[i] + 2 * e[i + 1] + e[i + 2];
          qmax = max(qmax, gx3 * gx3 + gy3 * gy3);
        }
      }
      int sc = tmax;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(kFull, sc, d);
        if (lane >= d) sc = max(sc, v);
      }
      int ex = __shfl_up_sync(kFull, sc, 1);
      ex = max(lane == 0 ? 0 : ex, carry);
      carry = max(carry, __shfl_sync(kFull, sc, 31));
      float u = 0.0f;
      if (qmax > 0)
        u = fminf(t_term(qmax, tk) * hi_f, 1.0f) * fminf(d_term(ex, tk) * hi_f, 1.0f);
      ECA_CHECK(k < kWMaxChunks);
      ut_s[k * 32 + lane] = __float2half_ru(u);
      ex_s[k * 32 + lane] = uint16_t(ex);
      // every later column has preceding sum >= carry, so its score is below
      // D_up(carry) (T, A <= 1).  Once that is small, get LB from the chunks
      // so far and stop the scan if no later column can reach it.  (Steps A+B
      // have this one call site: the last chunk always triggers them.)
      if (!ab_done) {
        const bool last = k + 1 == nch;
        const float dc = last ? 0.0f : d_term(carry, tk) * hi_f;
        if (last || (ECA_EARLY_EXIT && dc < kEarlyD)) {
          __syncwarp();
          step_ab(k + 1);
          if (!last && lb > dc && trusted) {
            nch_eff = k + 1;
            break;
          }
        }
      }
    }
    __syncwarp();

    // ---- step C: the other lane-chunks whose U reaches LB; LB tightens (and
    // a "full" row can become a normal one) with every evaluated group.
    // Phase 0: lane-chunks with U >= LB (every U > 0 one while full).
    // Phase 1, only if still full: lane-chunks of U == 0 holding a non-flat
    // scoreable column (their scores are FP64 rounding residues).  Flat columns
    // (identical left/right sums per row, identical top and bottom rows) score
    // exactly 0; flat rows (black borders) would otherwise evaluate every column.
    for (int phase1 = 0; phase1 < 2; ++phase1) {
      if (phase1 && !full) break;
      int n_sel = 0;
      for (int k = 0; k < nch_eff; ++k) {
        const float v = __half2float(ut_s[k * 32 + lane]);   // < 0: evaluated in step B
        bool s;
        if (!phase1) {
          s = v > 0.0f && (full || v >= lb);
        } else {
          s = false;
          if (v == 0.0f) {
            const int xa = xa_of(k, lane);
            int s0[10], s1[10], s2[10];
            load10(st, rb[0] + 3 * xa, al, s0);
            load10(st, rb[1] + 3 * xa, al, s1);
            load10(st, rb[2] + 3 * xa, al, s2);
#pragma unroll
            for (int i = 0; i < kPx; ++i) {
              const bool flat = s0[i] == s0[i + 2] && s1[i] == s1[i + 2] && s0[i] == s2[i] &&
                                s0[i + 1] == s2[i + 1] && s0[i + 2] == s2[i + 2];
              s |= !flat && unsigned(xa + i - slo) <= unsigned(shi - slo);
            }
          }
        }
        const unsigned bm = __ballot_sync(kFull, s);
        ECA_CHECK(n_sel + __popc(bm) <= kWMaxChunks * 32);
        if (s) sel_s[n_sel + __popc(bm & lt_mask)] = uint16_t((k << 5) | lane);
        n_sel += __popc(bm);
      }
      __syncwarp();
      if (!phase1 && !full && n_sel > kRefineMin) {
        // refine: one lane per selected lane-chunk, its 8 columns' exact bounds
        // (branch-free, so the columns overlap): U2 = max U_col replaces U,
        // LB takes max L_col; then only lane-chunks with U2 >= LB stay
        for (int p0 = 0; p0 < n_sel; p0 += 32) {
          const int p = p0 + lane;
          const bool valid = p < n_sel;
          const int e = valid ? int(sel_s[p]) : 0;
          const int xa = xa_of(e >> 5, e & 31);
          int s0[10], s1[10], s2[10];
          load10(st, rb[0] + 3 * xa, al, s0);
          load10(st, rb[1] + 3 * xa, al, s1);
          load10(st, rb[2] + 3 * xa, al, s2);
          int pre[kPx];
          int run = int(ex_s[e]);
          if (half) {
#pragma unroll
            for (int i = kPx - 1; i >= 0; --i) {
              pre[i] = run;
              run = max(run, s1[i + 1]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < kPx; ++i) {
              pre[i] = run;
              run = max(run, s1[i + 1]);
            }
          }
          float umax = 0.0f, lmax = 0.0f;
#pragma unroll
          for (int i = 0; i < kPx; ++i) {
            const int x = xa + i;
            const int cl = s0[i] + 2 * s1[i] + s2[i], cr = s0[i + 2] + 2 * s1[i + 2] + s2[i + 2];
            const int gx3 = cr - cl;
            const int gy3 = (s2[i] - s0[i]) + 2 * (s2[i + 1] - s0[i + 1]) + (s2[i + 2] - s0[i + 2]);
            const int q = gx3 * gx3 + gy3 * gy3;
            const int d2x = (W - 1) - 2 * x;
            const int dot = gx3 * d2x + gy3 * d2y;
            const int crs = abs(gx3 * d2y - gy3 * d2x);
            const float fd = float(abs(dot)), fc = float(crs);
            const float ps = fc * rcpf(fmaxf(fd + fc, 1.0f));
            int ab = min(int((dot >= 0 ? ps : 2.0f - ps) * (kABins / 2)), kABins - 1);
            if (dot == 0 && crs == 0) ab = kABins;
            const float2 at = atab[ab];
            const float t = t_term(q, tk), dd = d_term(pre[i], tk);
            const bool in = unsigned(x - slo) <= unsigned(shi - slo) && q > 0;
            umax = fmaxf(umax, in ? fminf(t * hi_f, 1.0f) * fminf(dd * hi_f, 1.0f) * at.y : 0.0f);
            lmax = fmaxf(lmax, in ? t * lo_f * dd * lo_f * at.x : 0.0f);
          }
          if (valid) ut_s[(e >> 5) * 32 + (e & 31)] = __float2half_ru(umax);
          lb = fmaxf(lb, warp_max_nonneg(valid ? lmax : 0.0f));
        }
        full = !(lb >= J.tau);
        __syncwarp();
        int n2 = 0;   // keep the lane-chunks whose refined bound reaches LB
        for (int p0 = 0; p0 < n_sel; p0 += 32) {
          const int p = p0 + lane;
          const int e = p < n_sel ? int(sel_s[p]) : 0;
          const bool keep = p < n_sel && __half2float(ut_s[(e >> 5) * 32 + (e & 31)]) >= lb;
          const unsigned bm = __ballot_sync(kFull, keep);
          __syncwarp();
          if (keep) sel_s[n2 + __popc(bm & lt_mask)] = uint16_t(e);
          n2 += __popc(bm);
          __syncwarp();
        }
        n_sel = n2;
      }
      for (int g0 = 0; g0 < n_sel; g0 += 4) {
        const int p = g0 + (lane >> 3);
        const bool vc = p < n_sel;
        const int e = vc ? int(sel_s[p]) : 0;
        if (!full && !__any_sync(kFull, vc && __half2float(ut_s[(e >> 5) * 32 + (e & 31)]) >= lb))
          continue;
        const ColEval cc = eval(vc, e);
#ifdef ECA_WARP_TIMES
        ++dbg_groups;
#endif
        lb = fmaxf(lb, warp_max_nonneg(cc.L));
        full = !(lb >= J.tau);
        emit(vc, cc);
      }
    }
    if (lb >= J.tau) compact(lb);   // final LB: full rows keep every non-flat column

    // ---- hand the survivors to the FP64 rescore (rescore_kernel, or the fit
    // kernel's rescore stage); resolve the half row here if it has more than
    // kSlots.  The next item's TMA starts as soon as the stage is read.
    const int hrow = item;
    if (kInWarp && !flushed && n_list <= kSlots) {
      // one lane per survivor: the 3x3 sums to registers, refill the stage,
      // then the FP64 score under the next item's TMA
      int sx = 0, spre = 0, sl[3] = {0, 0, 0}, sm[3] = {0, 0, 0}, sr[3] = {0, 0, 0};
      if (lane < n_list) {
        const uint32_t v = list[lane];
        sx = int(v & 0xffffu);
        spre = int(v >> 16);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          sl[r] = px_sum(st, rb[r] + 3 * (sx - 1));
          sm[r] = px_sum(st, rb[r] + 3 * sx);
          sr[r] = px_sum(st, rb[r] + 3 * (sx + 1));
        }
      }
      advance();
      if (lane < n_list) {
        const double sc = exact_score(sl, sm, sr, spre, sx, y, cxf, cyf, J.p);
        if (better(sc, sx, best.s, best.x, !half)) best = Best{sc, sx};
      }
      best = warp_best(best, !half);
      if (lane == 0) {
        const size_t slot = size_t(frame) * 2 * S + (half ? S : 0) + strip;
        J.out_x[slot] = best.x;
        J.out_y[slot] = y;
        J.out_score[slot] = best.s;
      }
    } else if (!flushed && n_list <= kSlots) {
      if (lane < n_list) {
        const uint32_t v = list[lane];
        const int x = int(v & 0xffffu);
        SurvSlot sl;
        sl.x = uint16_t(x);
        sl.pre = uint16_t(v >> 16);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          sl.l[r] = uint16_t(px_sum(st, rb[r] + 3 * (x - 1)));
          sl.m[r] = uint16_t(px_sum(st, rb[r] + 3 * x));
          sl.r[r] = uint16_t(px_sum(st, rb[r] + 3 * (x + 1)));
        }
        sl.pad = 0;
        ECA_CHECK(hrow < n_items && lane < kSlots && x >= slo && x <= shi);
        PJ.slots[size_t(hrow) * kSlots + lane] = sl;
      }
      if (lane == 0) PJ.counts[hrow] = n_list;
      advance();
    } else {
      flush();
      advance();
      best = warp_best(best, !half);
      if (lane == 0) {
        const size_t slot = size_t(frame) * 2 * S + (half ? S : 0) + strip;
        J.out_x[slot] = best.x;
        J.out_y[slot] = y;
        J.out_score[slot] = best.s;
        if (!kInWarp) PJ.counts[hrow] = -1;
      }
    }
#endif
#ifdef ECA_WARP_TIMES
    if (lane == 0) {   // slowest item: (duration/32ns, full, step-C groups, item)
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      const uint64_t rec = (((t - t_item) / 32) << 40) | (uint64_t(full) << 39) |
                           (uint64_t(min(dbg_groups, 127)) << 32) | uint64_t(item);
      const int gw = blockIdx.x * warps + wib;
      if (rec > g_warp_times[3 * gw + 2]) g_warp_times[3 * gw + 2] = rec;
    }
#endif
    if (!advanced) advance();
    if (++stage == NS) {
      stage = 0;
      phase ^= 1u;
    }
  }
#ifdef ECA_WARP_TIMES
  if (lane == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_warp_times[3 * (blockIdx.x * warps + wib) + 1] = t;
  }
#endif
  __syncwarp();
  if (lane == 0) {   // CTA end: the last warp of the CTA to get here stamps
#ifdef ECA_TIMELINE
    if (blockIdx.x < 1024) g_tl[0][PJ.dbg_seq & 63][blockIdx.x][1] = gtime();
#endif
  }
  // the last warp out re-arms the tickets for the next launch on this workspace
  if (lane == 0) {
    if (PJ.guard) {
      __threadfence();   // this warp's outputs before the release
      guard_release(PJ.ticket, nw);
    } else if (atomicAdd(PJ.ticket + 1, 1) == nw - 1) {
      PJ.ticket[0] = 0;
      PJ.ticket[1] = 0;
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
  int frame, strip;
  decode_item(PJ, fs, frame, strip);
  const int y = valid_hr ? J.rows[strip] : 0;
  Best b = half ? Best{0.0, W - 1} : Best{0.0, 0};
  if (valid_hr && k < cnt) {
    const SurvSlot s = PJ.slots[size_t(hrow) * kSlots + k];
    const int l[3] = {s.l[0], s.l[1], s.l[2]}, m[3] = {s.m[0], s.m[1], s.m[2]},
              r[3] = {s.r[0], s.r[1], s.r[2]};
    b = Best{exact_score(l, m, r, s.pre, s.x, y, PJ.cxf, PJ.cyf, J.p), int(s.x)};
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
