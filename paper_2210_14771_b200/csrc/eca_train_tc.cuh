// §8f-4 on the tensor cores: EdgeNet training convolutions (edgenet.py:100-130
// forward, :277-344 backward) as tcgen05 3xTF32 GEMMs with FP32 accumulators
// in TMEM -- the operand layout, split and MMA helpers of the inference CNN
// (eca_umma.cuh, cnn_kernel_tc).
//
//  tc_conv_fwd    y = relu(conv3(x, w) + b): per tile (sample, output row, 128
//                 input columns) three row operands (ky) of 128 positions x K
//                 input channels; the kx shift moves to the output as in
//                 cnn_kernel_tc: B stacks the three kx weight blocks as N rows,
//                 D[kx][m] = sum_ky,c x[row+ky][m][c] w[ky][kx][c], and
//                 y[m] = D0[m] + D1[m+1] + D2[m+2] (126 outputs per tile; the
//                 neighbours come through shared memory).  The last layer also
//                 computes the 1x1 head's logit from its 32 channels.
//  tc_conv_dgrad  dx = (full correlation of dy with w) * (x_in > 0): the same
//                 shape with K = output channels, dy rows y - ky, positions
//                 shifted by -2, dx[j] = D2[j] + D1[j+1] + D0[j+2].
//  tc_conv_wgrad  dW[o][c][ky][kx] = sum over positions of dy[o][p] x[c][p+(ky,kx)]:
//                 M = the (c, ky, kx) rows (+ a row of ones: the bias
//                 gradient), N = output channels, K = positions, 32 per unit;
//                 a fixed number of CTAs each accumulates a fixed contiguous
//                 range of units in TMEM (two smem stages, the next unit built
//                 under the current unit's MMAs) and writes one partial;
//                 tc_wgrad_reduce sums the partials in CTA order
//                 (deterministic, no float atomics).
// Products are hi*hi + hi*lo + lo*hi of TF32 halves.  The tensor core's FP32
// accumulation truncates at every MMA, relative to the running sum, so long
// chains in one TMEM accumulator lose bits (measured: 8e-7 relative logit
// error with one accumulator per output, tools/train_err.py); every kernel
// therefore keeps chains short -- an accumulator per ky (forward, N = 96) or
// per ky pair (N = 48), two alternating over the K steps (dgrad), one per K
// step of each 32-position unit (wgrad) -- and sums those in FP32 registers
// with round-to-nearest.  The reference's sgemm also
// reassociates, so results agree to FP32 rounding level, not bitwise
// (tolerances in tests/test_gpu_train.py).
#pragma once

#include "eca_umma.cuh"

namespace eca {
namespace ttc {

constexpr int kT = 128;          // MMA positions (M) per tile
constexpr int kTOut = kT - 2;    // outputs per tile (the kx shift)
constexpr int kThreads = 128;    // 4 warps: one per TMEM lane quarter
constexpr int kXb = kT + 4;      // row stride of the neighbour exchange
constexpr int kWgK = 32;         // positions per weight-gradient unit
constexpr int kWgCtas = 1024;    // most weight-gradient CTAs (partials) per layer

// FP32 operands as kP TF32 pieces (v = p0 + p1 (+ p2), each the TF32 rounding
// of the remainder) and the products of the pieces summed up to order kP - 1.
// (ECA_TC_PIECES=3 / ECA_TC_LOLO=1: experiment builds; measured no more
// accurate than the default -- the accumulation, not the split, sets the
// error; K7.)
#ifndef ECA_TC_PIECES
#define ECA_TC_PIECES 2
#endif
#ifndef ECA_TC_LOLO
#define ECA_TC_LOLO 0
#endif
constexpr int kP = ECA_TC_PIECES;
static_assert(kP == 2 || kP == 3, "2 or 3 pieces");

ECA_DEV void st_pieces(uint8_t* base, int pstride, int off, float4 v) {
  float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    float p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      p[q] = tf32_rna(r[q]);
      r[q] = r[q] - p[q];   // exact
    }
    *reinterpret_cast<float4*>(base + i * pstride + off) = make_float4(p[0], p[1], p[2], p[3]);
  }
}
ECA_DEV void st_pieces1(uint8_t* base, int pstride, int off, float v) {
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    const float p = tf32_rna(v);
    *reinterpret_cast<float*>(base + i * pstride + off) = p;
    v = v - p;
  }
}
// sum over the terms (i, j) of piece_i(A) x piece_j(B), largest terms last
ECA_DEV void mma_terms(uint32_t tmem, uint32_t a, int astride, int sboa, uint32_t b, int bstride, int sbob,
                       uint32_t idesc, bool first) {
  constexpr int ti[6] = {1, 0, 2, 0, 1, 0}, tj[6] = {1, 2, 0, 1, 0, 0};   // (1,1) (0,2) (2,0) (0,1) (1,0) (0,0)
  constexpr int t0 = kP == 3 ? 0 : (ECA_TC_LOLO ? 0 : 3);
  constexpr int skip_lo = kP == 3 ? 0 : 2;   // (0,2), (2,0) need a third piece
#pragma unroll
  for (int t = t0; t < 6; ++t) {
    if (skip_lo && (t == 1 || t == 2)) continue;
    mma_tf32(tmem, umma_desc(a + ti[t] * astride, sboa), umma_desc(b + tj[t] * bstride, sbob), idesc,
             (first && t == t0) ? 0u : 1u);
  }
}

constexpr int up8(int c) { return (c + 7) / 8 * 8; }
constexpr int up16(int c) { return (c + 15) / 16 * 16; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
#ifndef ECA_TMEM_ALL   // diagnostics: every kernel takes all 512 columns (one CTA per SM's TMEM)
#define ECA_TMEM_ALL 0
#endif
constexpr int tmem_cols(int n) {
  return ECA_TMEM_ALL ? 512 : n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}

ECA_DEV void tmem_alloc(uint32_t* slot, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(slot)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
ECA_DEV void tmem_free(uint32_t tmem, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}
ECA_DEV void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
ECA_DEV void mma_wait(uint32_t bar, uint32_t parity) {
  bar_wait(bar, parity);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
ECA_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// all TMEM reads done -> warp 0 may free it
ECA_DEV void tmem_release(uint32_t tmem, int cols) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) tmem_free(tmem, cols);
}

// 16-byte copy of `bytes` (a multiple of 16) by the CTA's threads
ECA_DEV void copy16(uint8_t* dst, const uint8_t* src, int bytes) {
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
}

// ------------------------------------------------------------------ forward --
template <int CI, int CO>
struct FwdCfg {
  static constexpr int KP = up8(CI);             // K: input channels, zero-padded
  static constexpr int NB = up16(CO);            // rows of one kx block of B
  static constexpr int N = 3 * NB;
  static constexpr int SBO = KP / 4 * 128;       // 8-row group stride of every operand
  static constexpr int A_BYTES = kT * KP * 4;    // one row operand, hi or lo
  static constexpr int B_BYTES = N * KP * 4;
  static constexpr int A_REGION = cmax(3 * kP * A_BYTES, 2 * CO * kXb * 4);   // + exchange after the MMAs
  static constexpr int SMEM = A_REGION + 3 * kP * B_BYTES;
  static constexpr int BIMG = 3 * kP * B_BYTES;  // the packed B operands (pack_b_fwd / pack_slice)
  // accumulators: one per ky (N = 96), or ky 0-1 and ky 2 (N = 48: 128 TMEM
  // columns, so four CTAs fit an SM's TMEM)
  static constexpr int NACC = N > 48 ? 3 : 2;
  static constexpr int COLS = tmem_cols(NACC * N);
  static constexpr int acc(int ky) { return NACC == 3 ? ky : (ky < 2 ? 0 : 1); }
};

template <int CI, int CO>
struct DgCfg {
  static constexpr int KP = CO;                  // K: output channels (16 or 32)
  static_assert(CO % 8 == 0, "K steps of 8");
  static constexpr int NB = up16(CI);
  static constexpr int N = 3 * NB;
  static constexpr int SBO = KP / 4 * 128;
  static constexpr int A_BYTES = kT * KP * 4;
  static constexpr int B_BYTES = N * KP * 4;
  static constexpr int XB = 2 * CI * kXb * 4;
  static constexpr int NACC = KP / 8 < 2 ? KP / 8 : 2;   // K steps alternate between two accumulators
  static constexpr int COLS = tmem_cols(NACC * N);
  // ky rows of dy that exist for some output row: min(3, ho) A slots
  static constexpr int BIMG = 3 * kP * B_BYTES;  // the packed B operands (pack_b_fwd / pack_slice)
  static int a_region(int ho) { return cmax((ho < 3 ? ho : 3) * kP * A_BYTES, XB); }
  static int smem(int ho) { return a_region(ho) + 3 * kP * B_BYTES; }
};

// ------------------------------------------------------- packed B operands --
// The conv kernels' B operands (weights as K-major TF32 pieces) are built once
// per forward (by the layer-0 forward's CTAs, pack_slice) into the workspace,
// in their shared-memory layout, and copied by every CTA of the later kernels
// (instead of each CTA rebuilding them).
// forward: B[ky][piece] row n = kx * NB + o, K = c; dgrad: row n = kx * NB + c, K = o.
template <int CI, int CO>
ECA_DEV void pack_b_fwd(uint8_t* dst, const float* __restrict__ wk, int i) {
  using C = FwdCfg<CI, CO>;
  if (i >= 3 * C::N * C::KP) return;
  const int c = i % C::KP, n = (i / C::KP) % C::N, ky = i / (C::KP * C::N);
  const int kx = n / C::NB, o = n % C::NB;
  const float v = (o < CO && c < CI) ? wk[((o * CI + c) * 3 + ky) * 3 + kx] : 0.f;
  st_pieces1(dst + ky * kP * C::B_BYTES, C::B_BYTES, kmaj_off(n, c, C::SBO), v);
}
template <int CI, int CO>
ECA_DEV void pack_b_dgrad(uint8_t* dst, const float* __restrict__ wk, int i) {
  using C = DgCfg<CI, CO>;
  if (i >= 3 * C::N * C::KP) return;
  const int o = i % C::KP, n = (i / C::KP) % C::N, ky = i / (C::KP * C::N);
  const int kx = n / C::NB, c = n % C::NB;
  const float v = c < CI ? wk[((o * CI + c) * 3 + ky) * 3 + kx] : 0.f;
  st_pieces1(dst + ky * kP * C::B_BYTES, C::B_BYTES, kmaj_off(n, o, C::SBO), v);
}
struct PackJob {
  const float *w0, *w1, *w2;   // OIHW kernels of the three 3x3 layers
  uint8_t *f0, *f1, *f2, *d2, *d1;
};
// the forward-1/2 and dgrad-2/1 images: slice `part` of `parts` of their
// elements (the layer-0 forward kernel's CTAs write them between them, so no
// separate packing launch is needed; stream order makes them visible to the
// later kernels)
ECA_DEV void pack_slice(const PackJob& J, int part, int parts) {
  constexpr int e1 = 3 * FwdCfg<8, 16>::N * FwdCfg<8, 16>::KP, e2 = 3 * FwdCfg<16, 32>::N * FwdCfg<16, 32>::KP;
  constexpr int e3 = 3 * DgCfg<16, 32>::N * DgCfg<16, 32>::KP, e4 = 3 * DgCfg<8, 16>::N * DgCfg<8, 16>::KP;
  constexpr int total = e1 + e2 + e3 + e4;
  const int lo = int(int64_t(total) * part / parts), hi = int(int64_t(total) * (part + 1) / parts);
  for (int g = lo + int(threadIdx.x); g < hi; g += blockDim.x) {
    if (g < e1) pack_b_fwd<8, 16>(J.f1, J.w1, g);
    else if (g < e1 + e2) pack_b_fwd<16, 32>(J.f2, J.w2, g - e1);
    else if (g < e1 + e2 + e3) pack_b_dgrad<16, 32>(J.d2, J.w2, g - e1 - e2);
    else pack_b_dgrad<8, 16>(J.d1, J.w1, g - e1 - e2 - e3);
  }
}


// x: [*][CI][hi][wi] (sample idx[b] when idx) -> y: [m][CO][hi-2][wi-2].
// Persistent CTAs (B, the biases and TMEM set up once) loop over tiles (b, oy,
// 126 output columns).  kHead (CO == 32): also logit = sum_c w3[c] y[c] + b3
// (head = w3[0..31], b3), summed in channel order.
template <int CI, int CO, bool kHead>
__global__ void __launch_bounds__(kThreads) tc_conv_fwd(const float* __restrict__ x,
                                                        const int32_t* __restrict__ idx, int m_, int hi,
                                                        int wi, const uint8_t* __restrict__ bimg,
                                                        const float* __restrict__ bias,
                                                        const float* __restrict__ head, float* __restrict__ y,
                                                        float* __restrict__ logit, const PackJob pack,
                                                        int do_pack) {
  using C = FwdCfg<CI, CO>;
  static_assert(!kHead || CO == 32, "head after the 32-channel layer");
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ float sbias[CO], sw3[32], sb3;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* const A = sm;                  // [ky][piece][A_BYTES]
  uint8_t* const B = sm + C::A_REGION;    // [ky][piece][B_BYTES]
  float* const xb = reinterpret_cast<float*>(sm);   // after the MMAs: D1, D2 [2][CO][kXb]
  const int tid = threadIdx.x, warp = tid >> 5, m = tid;
  const int ho = hi - 2, wo = wi - 2, ntx = (wo + kTOut - 1) / kTOut;
  const int ntiles = m_ * ho * ntx;
  if (warp == 0) tmem_alloc(&tslot, C::COLS);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (do_pack) {   // layer 0: its own B from the weights, and a slice of the other images
    for (int i = tid; i < 3 * C::N * C::KP; i += kThreads) pack_b_fwd<CI, CO>(B, pack.w0, i);
    pack_slice(pack, blockIdx.x, gridDim.x);
  } else {
    copy16(B, bimg, C::BIMG);   // B[ky]: row n = kx * NB + o, K = c (pack_b_fwd)
  }
  if (tid < CO) sbias[tid] = bias[tid];
  if (kHead) {
    if (tid < 32) sw3[tid] = head[tid];
    if (tid == 0) sb3 = head[32];
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot, bar_s = smem_addr(&bar);
  const uint32_t lrow = tmem + (uint32_t(32 * warp) << 16);
  const int plane = ho * wo, iplane = hi * wi;   // < 2^31 (check_dims)
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx = tile % ntx, oy = (tile / ntx) % ho, b = tile / (ntx * ho);
    const int x0 = tx * kTOut;
    const int s = idx ? idx[b] : b;
    {   // A[ky]: input row oy + ky, positions x0 + m (zero past the row), K = channels
      const bool in = x0 + m < wi;
      const float* xs = x + int64_t(s) * CI * iplane + oy * wi + x0 + m;
      float v[3][C::KP];
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int c = 0; c < C::KP; ++c) v[ky][c] = (in && c < CI) ? xs[c * iplane + ky * wi] : 0.f;
      ECA_CHECK(s >= 0 && oy + 2 < hi && x0 < wi);
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int c4 = 0; c4 < C::KP; c4 += 4)
          st_pieces(A + ky * kP * C::A_BYTES, C::A_BYTES, kmaj_off(m, c4, C::SBO),
                    make_float4(v[ky][c4], v[ky][c4 + 1], v[ky][c4 + 2], v[ky][c4 + 3]));
    }
    publish_operands();   // also: the previous tile's TMEM / exchange reads are done
    if (tid == 0) {
      const uint32_t a0 = smem_addr(A), b0 = smem_addr(B);
      constexpr uint32_t idesc = idesc_tf32(C::N);
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int ks = 0; ks < C::KP / 8; ++ks) {
          const uint32_t a = a0 + ky * kP * C::A_BYTES + ks * 256, bb = b0 + ky * kP * C::B_BYTES + ks * 256;
          mma_terms(tmem + C::acc(ky) * C::N, a, C::A_BYTES, C::SBO, bb, C::B_BYTES, C::SBO, idesc,
                    ks == 0 && (C::NACC == 3 || ky != 1));
        }
      mma_commit(bar_s);
    }
    mma_wait(bar_s, phase);
    phase ^= 1u;
    // epilogue: thread m = TMEM lane m.  The accumulators are summed in FP32
    // with round-to-nearest; D0 stays in registers, D1 / D2 go to the
    // exchange (the A operands are dead: the MMAs completed)
    float d0[CO];
#pragma unroll
    for (int o4 = 0; o4 < CO; o4 += 4) {
      float v[C::NACC][3][4];   // [accumulator][kx][o]
#pragma unroll
      for (int a = 0; a < C::NACC; ++a)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) tmem_ld<4>(lrow + a * C::N + kx * C::NB + o4, v[a][kx]);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float s0 = v[0][0][j], s1 = v[0][1][j], s2 = v[0][2][j];
#pragma unroll
        for (int a = 1; a < C::NACC; ++a) {
          s0 += v[a][0][j];
          s1 += v[a][1][j];
          s2 += v[a][2][j];
        }
        d0[o4 + j] = s0;
        xb[(o4 + j) * kXb + m] = s1;
        xb[(CO + o4 + j) * kXb + m] = s2;
      }
    }
    __syncthreads();
    const int ox = x0 + m;
    if (m < kTOut && ox < wo) {
      ECA_CHECK(b < m_ && oy < ho);
      float* yo = y + int64_t(b) * CO * plane + oy * wo + ox;
      float z = 0.f;
#pragma unroll
      for (int o = 0; o < CO; ++o) {
        float v = ((d0[o] + xb[o * kXb + m + 1]) + xb[(CO + o) * kXb + m + 2]) + sbias[o];
        v = v * float(v > 0.f);   // y * (y > 0): -inf and NaN give NaN, as numpy
        yo[o * plane] = v;
        if (kHead) z = fmaf(sw3[o], v, z);
      }
      if (kHead) logit[int64_t(b) * plane + oy * wo + ox] = z + sb3;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();   // exchange reads done before the next tile's A (same bytes)
  }
  tmem_release(tmem, C::COLS);
}

// -------------------------------------------------------------------- dgrad --

// dx: [m][CI][hi][wi] = (sum_{o,ky,kx} dy[o][y-ky][x-kx] w[o][c][ky][kx]) * (xin > 0);
// dy: [m][CO][hi-2][wi-2]; persistent CTAs loop over tiles (b, y, 126 columns)
template <int CI, int CO>
__global__ void __launch_bounds__(kThreads) tc_conv_dgrad(const float* __restrict__ dy,
                                                          const float* __restrict__ xin, int m_, int hi,
                                                          int wi, const uint8_t* __restrict__ bimg,
                                                          int a_region, float* __restrict__ dx) {
  using C = DgCfg<CI, CO>;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* const A = sm;                 // [slot][piece][A_BYTES]
  uint8_t* const B = sm + a_region;      // [ky][piece][B_BYTES]
  float* const xb = reinterpret_cast<float*>(sm);   // after the MMAs: D1, D0 [2][CI][kXb]
  const int tid = threadIdx.x, warp = tid >> 5, m = tid;
  const int ho = hi - 2, wo = wi - 2, ntx = (wi + kTOut - 1) / kTOut;
  const int ntiles = m_ * hi * ntx;
  if (warp == 0) tmem_alloc(&tslot, C::COLS);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  copy16(B, bimg, C::BIMG);   // B[ky]: row n = kx * NB + c, K = o (pack_b_dgrad)
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot, bar_s = smem_addr(&bar);
  const uint32_t lrow = tmem + (uint32_t(32 * warp) << 16);
  const int plane = hi * wi, dplane = ho * wo;   // < 2^31 (check_dims)
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx = tile % ntx, yr = (tile / ntx) % hi, b = tile / (ntx * hi);
    const int x0 = tx * kTOut;
    const int ky0 = yr - ho + 1 > 0 ? yr - ho + 1 : 0, ky1 = yr < 2 ? yr : 2;   // 0 <= yr - ky < ho
    // the slots used fit the A region sized for min(3, ho) rows
    ECA_CHECK(ky1 >= ky0 && (ky1 - ky0 + 1) * kP * C::A_BYTES <= a_region && b < m_);
    {   // A[slot]: dy row yr - ky, positions x0 - 2 + m (zero outside the row)
      const int p = x0 - 2 + m;
      const bool in = p >= 0 && p < wo;
      for (int ky = ky0; ky <= ky1; ++ky) {
        const float* ds = dy + int64_t(b) * CO * dplane + (yr - ky) * wo + p;
        uint8_t* ak = A + (ky - ky0) * kP * C::A_BYTES;
        float v[CO];
#pragma unroll
        for (int o = 0; o < CO; ++o) v[o] = in ? ds[o * dplane] : 0.f;
#pragma unroll
        for (int o4 = 0; o4 < CO; o4 += 4)
          st_pieces(ak, C::A_BYTES, kmaj_off(m, o4, C::SBO), make_float4(v[o4], v[o4 + 1], v[o4 + 2], v[o4 + 3]));
      }
    }
    publish_operands();   // also: the previous tile's TMEM / exchange reads are done
    if (tid == 0) {
      const uint32_t a0 = smem_addr(A), b0 = smem_addr(B);
      constexpr uint32_t idesc = idesc_tf32(C::N);
      for (int ky = ky0; ky <= ky1; ++ky)
#pragma unroll
        for (int ks = 0; ks < C::KP / 8; ++ks) {
          const uint32_t a = a0 + (ky - ky0) * kP * C::A_BYTES + ks * 256;
          const uint32_t bb = b0 + ky * kP * C::B_BYTES + ks * 256;
          mma_terms(tmem + (ks % C::NACC) * C::N, a, C::A_BYTES, C::SBO, bb, C::B_BYTES, C::SBO, idesc,
                    ky == ky0 && ks < C::NACC);
        }
      mma_commit(bar_s);
    }
    mma_wait(bar_s, phase);
    phase ^= 1u;
    // the accumulators summed in FP32 (round-to-nearest)
    float d2[CI];
#pragma unroll
    for (int c4 = 0; c4 < CI; c4 += 4) {
      float v[C::NACC][3][4];   // [accumulator][kx][c]
#pragma unroll
      for (int ks = 0; ks < C::NACC; ++ks)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) tmem_ld<4>(lrow + ks * C::N + kx * C::NB + c4, v[ks][kx]);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float s0 = v[0][0][j], s1 = v[0][1][j], s2 = v[0][2][j];
#pragma unroll
        for (int ks = 1; ks < C::NACC; ++ks) {
          s0 += v[ks][0][j];
          s1 += v[ks][1][j];
          s2 += v[ks][2][j];
        }
        d2[c4 + j] = s2;
        xb[(c4 + j) * kXb + m] = s1;
        xb[(CI + c4 + j) * kXb + m] = s0;
      }
    }
    __syncthreads();
    const int xo = x0 + m;
    if (m < kTOut && xo < wi) {
      const int64_t q0 = int64_t(b) * CI * plane + yr * wi + xo;
#pragma unroll
      for (int c = 0; c < CI; ++c) {
        const float v = (d2[c] + xb[c * kXb + m + 1]) + xb[(CI + c) * kXb + m + 2];
        dx[q0 + c * plane] = v * float(xin[q0 + c * plane] > 0.f);   // dx * mask (inf * 0 = NaN, as numpy)
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();   // exchange reads done before the next tile's A (same bytes)
  }
  tmem_release(tmem, C::COLS);
}

// -------------------------------------------------------------------- wgrad --
template <int CI, int CO, int KS>
struct WgCfg {
  static constexpr int R = CI * KS * KS + 1;     // (c, ky, kx) rows + the bias row of ones
  static constexpr int MT = (R + kT - 1) / kT;   // M tiles
  static constexpr int NB = up16(CO);
  static constexpr int NKS = kWgK / 8;           // K steps per unit
  static constexpr int SBO = kWgK / 4 * 128;     // K = 32 positions
  static constexpr int A_BYTES = kT * kWgK * 4;  // one M tile per CTA (blockIdx.y)
  static constexpr int B_BYTES = NB * kWgK * 4;
  static constexpr int STAGE = kP * A_BYTES + kP * B_BYTES;
  static constexpr int XW = kWgK + KS - 1;       // raw x columns of a unit
  static constexpr int XR = CI * KS * XW;        // raw x values of a unit: rows (c, ky)
  static constexpr int NX = (XR + kThreads - 1) / kThreads;                  // per thread
  static constexpr int NDC = (NB + 15) / 16;    // dy chunk rows per thread
  static constexpr int SMEM = 2 * STAGE + XR * 4;
  static constexpr int ACC = NKS * NB;           // TMEM columns of one unit: an accumulator per K step
  static constexpr int COLS = tmem_cols(2 * ACC);
  static_assert(2 * ACC <= 512, "TMEM");
};

// partial[g][o][r] = sum over CTA g's units of x_row(r) . dy_row(o); a unit is
// (b, oy, 32 output columns); dy: [m][CO][hi-KS+1][wi-KS+1], x: [*][CI][hi][wi].
// Per unit: the raw x rows (c, oy + ky) and the dy chunks were prefetched into
// registers during the previous unit (coalesced); x goes through shared memory
// once and is expanded into the (c, ky, kx) rows of A there.  Unit k's products
// go to fresh TMEM accumulators (one per K step, buffer k & 1); before unit
// k + 2 reuses the buffer the threads add them into FP32 registers (row = TMEM
// lane), in unit order.  Thread t owns the 16-byte chunks (row (t & 7) +
// 8 (t >> 6) + 16 q, positions 4 ((t >> 3) & 7) ..): a warp's chunk stores
// cover 512 contiguous bytes (no bank conflicts); all offsets are computed once.
template <int CI, int CO, int KS>
__global__ void __launch_bounds__(kThreads) tc_conv_wgrad(const float* __restrict__ dy,
                                                          const float* __restrict__ x,
                                                          const int32_t* __restrict__ idx, int m_,
                                                          int hi, int wi, float* __restrict__ part) {
  using C = WgCfg<CI, CO, KS>;
  const int mt = blockIdx.y, row0 = mt * kT;   // this CTA's M tile: rows row0 ..
  constexpr int NA = (C::R < kT ? C::R + 15 : kT) / 16;   // A chunk rows per thread
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tslot;
  float* const xr = reinterpret_cast<float*>(sm + 2 * C::STAGE);   // [c * KS + ky][XW]
  const int tid = threadIdx.x, warp = tid >> 5;
  const int ho = hi - KS + 1, wo = wi - KS + 1, nxc = (wo + kWgK - 1) / kWgK;
  const int units = m_ * ho * nxc;
  const int u0 = int(int64_t(units) * blockIdx.x / gridDim.x);
  const int nu = int(int64_t(units) * (blockIdx.x + 1) / gridDim.x) - u0;
  if (warp == 0) tmem_alloc(&tslot, C::COLS);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  // per-thread offsets, the same for every unit
  const int j4 = 4 * ((tid >> 3) & 7), rbase = (tid & 7) + 8 * (tid >> 6);
  int xoff[C::NX], xcol[C::NX];   // raw x value q: offset from the unit's (c=0, ky=0, x0), column
#pragma unroll
  for (int q = 0; q < C::NX; ++q) {
    const int i = tid + q * kThreads, row = i / C::XW, col = i % C::XW;
    xoff[q] = ((row / KS) * hi + row % KS) * wi + col;
    xcol[q] = i < C::XR ? col : (1 << 30);   // past the end: never loaded
  }
  int asrc[NA], adst[NA];   // A chunk: source in xr, destination in the operand
#pragma unroll
  for (int q = 0; q < NA; ++q) {
    const int r = row0 + rbase + 16 * q;
    asrc[q] = r < C::R - 1 ? (r / (KS * KS)) * KS * C::XW + ((r / KS) % KS) * C::XW + r % KS + j4 : -1;
    adst[q] = r < C::R ? kmaj_off(r - row0, j4, C::SBO) : -1;
    ECA_CHECK(asrc[q] + 3 < C::XR && adst[q] + 16 <= C::A_BYTES && (r - row0 < kT || adst[q] < 0));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t lrow = tmem + (uint32_t(32 * warp) << 16);
  float acc[CO];
#pragma unroll
  for (int o = 0; o < CO; ++o) acc[o] = 0.f;
  // unit k's accumulators (buffer k & 1) -> registers, after its MMAs completed
  const auto drain = [&](int k) {
    mma_wait(smem_addr(&bars[k & 1]), uint32_t(k >> 1) & 1u);
    const uint32_t base = lrow + (k & 1) * C::ACC;
#pragma unroll
    for (int o4 = 0; o4 < CO; o4 += 4) {
      float v[C::NKS][4];
#pragma unroll
      for (int ks = 0; ks < C::NKS; ++ks) tmem_ld<4>(base + ks * C::NB + o4, v[ks]);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (o4 + j >= CO) break;
        float s = v[0][j];
#pragma unroll
        for (int ks = 1; ks < C::NKS; ++ks) s += v[ks][j];
        acc[o4 + j] += s;
      }
    }
  };
  // the unit to fetch next, stepped without divisions
  int fxc = u0 % nxc, foy = (u0 / nxc) % ho, fb = u0 / (nxc * ho);
  float px[C::NX], pd[C::NDC][4];
  int fx0 = 0;
  const auto fetch = [&]() {
    const int x0 = fxc * kWgK, s = idx ? idx[fb] : fb;
    ECA_CHECK(fb < m_ && foy < ho && s >= 0);
    const float* xs = x + (int64_t(s) * CI * hi + foy) * wi + x0;
#pragma unroll
    for (int q = 0; q < C::NX; ++q) px[q] = x0 + xcol[q] < wi ? xs[xoff[q]] : 0.f;
    const float* ds = dy + (int64_t(fb) * CO * ho + foy) * wo + x0 + j4;
#pragma unroll
    for (int q = 0; q < C::NDC; ++q) {
      const int o = rbase + 16 * q;
#pragma unroll
      for (int t = 0; t < 4; ++t) pd[q][t] = (o < CO && x0 + j4 + t < wo) ? ds[int64_t(o) * ho * wo + t] : 0.f;
    }
    fx0 = x0;
    if (++fxc == nxc) {
      fxc = 0;
      if (++foy == ho) {
        foy = 0;
        ++fb;
      }
    }
  };
  if (nu > 0) fetch();
  for (int k = 0; k < nu; ++k) {
    const int st = k & 1;
    uint8_t* const A = sm + st * C::STAGE;
    uint8_t* const Bm = A + kP * C::A_BYTES;
    const int x0 = fx0;
    // the raw rows of unit k -> shared (the previous unit's expansion read
    // them before its publish barrier); dy chunks straight into B's stage
    // once the stage is free
#pragma unroll
    for (int q = 0; q < C::NX; ++q)
      if (tid + q * kThreads < C::XR) xr[tid + q * kThreads] = px[q];
    if (k >= 2) drain(k - 2);   // frees stage st and TMEM buffer st
#pragma unroll
    for (int q = 0; q < C::NDC; ++q)
      if (rbase + 16 * q < C::NB)
        st_pieces(Bm, C::B_BYTES, kmaj_off(rbase + 16 * q, j4, C::SBO),
                  make_float4(pd[q][0], pd[q][1], pd[q][2], pd[q][3]));
    if (k + 1 < nu) fetch();   // in flight during the expansion and the MMAs
    __syncthreads();
    // A: row r = (c*KS + ky)*KS + kx -> x[c][oy+ky][x0 + j + kx] at valid
    // positions (x0 + j < wo); row R-1: ones
    bool valid[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) valid[t] = x0 + j4 + t < wo;
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      if (adst[q] < 0) continue;
      float v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) v[t] = valid[t] ? (asrc[q] >= 0 ? xr[asrc[q] + t] : 1.f) : 0.f;
      st_pieces(A, C::A_BYTES, adst[q], make_float4(v[0], v[1], v[2], v[3]));
    }
    publish_operands();
    if (tid == 0) {
      const uint32_t a0 = smem_addr(A), b0 = smem_addr(Bm);
      constexpr uint32_t idesc = idesc_tf32(C::NB);
#pragma unroll
      for (int ks = 0; ks < C::NKS; ++ks)
        mma_terms(tmem + st * C::ACC + ks * C::NB, a0 + ks * 256, C::A_BYTES, C::SBO, b0 + ks * 256, C::B_BYTES,
                  C::SBO, idesc, true);
      mma_commit(smem_addr(&bars[st]));
    }
  }
  if (nu >= 2) drain(nu - 2);
  if (nu >= 1) drain(nu - 1);
  const int lane_row = 32 * warp + (tid & 31);
  float* pg = part + int64_t(blockIdx.x) * C::R * CO;   // [G][CO][R]: a warp's stores are contiguous
  const int r = row0 + lane_row;
  ECA_CHECK(int(blockIdx.x) < kWgCtas);
  if (r < C::R)
#pragma unroll
    for (int o = 0; o < CO; ++o) pg[o * C::R + r] = acc[o];
  tmem_release(tmem, C::COLS);
}

// gradients from the per-CTA partials of all layers ([G][CO][R]; the head's
// are the loss kernel's per-block sums), summed in a fixed order: layer
// blockIdx.y, 32 outputs per block (OIHW order then the biases); group
// threadIdx.y sums partials g = y, y + 32, ... (4 independent chains), then
// the 32 group sums are added in group order
struct WgLayer {
  const float* part;
  int R, CO, G;
  float *gw, *gb;
};
struct WgReduceJob {
  WgLayer l[4];
  // blockIdx.y == 4: the mean loss from the loss kernel's block partials, as
  // loss_final does (same order), and the non-finite flag
  const double* lpart;
  int nlblk;
  int64_t n;
  double* out_loss;
  int32_t* flag;
};
constexpr int kRedG = 32;
__global__ void __launch_bounds__(32 * kRedG) tc_wgrad_reduce(const __grid_constant__ WgReduceJob J) {
  __shared__ float red[kRedG][32];
  if (blockIdx.y == 4) {   // the loss (one block; loss_final's 256-thread order)
    if (blockIdx.x != 0) return;
    __shared__ double lred[256];
    const int t = threadIdx.y * 32 + threadIdx.x;
    if (t < 256) {
      double v = 0.0;
      for (int i = t; i < J.nlblk; i += 256) v += J.lpart[i];
      lred[t] = v;
    }
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
      if (t < o) lred[t] += lred[t + o];
      __syncthreads();
    }
    if (t == 0) {
      const double loss = lred[0] / double(J.n);
      *J.out_loss = loss;
      if (!isfinite(loss) && J.flag) *J.flag = 1;
    }
    return;
  }
  const WgLayer& L = J.l[blockIdx.y];
  const int n = L.R * L.CO, i = blockIdx.x * 32 + threadIdx.x, g0 = threadIdx.y;
  if (blockIdx.x * 32 >= n) return;
  const int nw = L.CO * (L.R - 1);
  const int o = i < nw ? i / (L.R - 1) : i - nw, r = i < nw ? i % (L.R - 1) : L.R - 1;
  const int64_t stride = int64_t(L.R) * L.CO;
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  if (i < n) {
    const float* p = L.part + o * L.R + r;
    int g = g0;
    for (; g + 3 * kRedG < L.G; g += 4 * kRedG)
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] += p[(g + q * kRedG) * stride];
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (g + q * kRedG < L.G) s4[q] += p[(g + q * kRedG) * stride];
  }
  red[g0][threadIdx.x] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  __syncthreads();
  if (g0 == 0 && i < n) {
    float v = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < kRedG; ++k) v += red[k][threadIdx.x];
    if (i < nw) L.gw[i] = v;
    else L.gb[o] = v;
  }
}

}  // namespace ttc
}  // namespace eca
