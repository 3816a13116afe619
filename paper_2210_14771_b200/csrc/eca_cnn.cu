// K3: learned strip scorer (edgenet.py) — fused RGBXY build + 3x(valid 3x3
// conv + ReLU) + 1x1 head + sigmoid per strip, FP32 like the reference.
//
// Persistent CTAs (2 per SM): the transposed weights, the exact per-byte
// normalisation table and the biases are loaded once per CTA, which then loops
// over tiles of kTX output columns of one strip of one frame.  The 7-row input
// window is built straight from the uint8 frame (no full-frame make_rgbxy,
// edgenet.py:67-83: values computed in FP64 then rounded to FP32 exactly as
// numpy does; the per-byte table holds those exact values).  The conv layers
// run out of shared memory, weights as warp-broadcast float4 reads; the
// 32-channel layer is split over all 256 threads (two threads per column, 16
// channels each; the head's channel sum continues in order through shared
// memory).  A second small kernel selects the half-row winners
// (handcrafted.py:120-138 rules).
// Accumulation is sequential FMA over (c, ky, kx); the reference's sgemm
// reassociates, so probabilities agree to ~1e-7, not bitwise.
#include <mutex>

#include "eca_common.cuh"
#include "eca_umma.cuh"

using namespace eca;

namespace {

constexpr int kTX = 128;                 // output columns per tile
constexpr int kW0 = 360, kB0 = 8, kW1 = 1152, kB1 = 16, kW2 = 4608, kB2 = 32, kW3 = 32;
constexpr int kOffB0 = kW0, kOffW1 = kOffB0 + kB0, kOffB1 = kOffW1 + kW1, kOffW2 = kOffB1 + kB1;
constexpr int kOffB2 = kOffW2 + kW2, kOffW3 = kOffB2 + kB2, kOffB3 = kOffW3 + kW3;
constexpr int kNetFloats = kOffB3 + 1;
static_assert(kNetFloats == ECA_NET_FLOATS, "weight layout");

struct CnnJob {
  const uint8_t* frames;
  int64_t fstride, rstride;
  int batch, S, H, W;
  int16_t rows[ECA_MAX_STRIPS];
  int16_t band[ECA_MAX_STRIPS];  // memory row of y-3
  double mean[3], stdv[3];
  const float* weights;
  float* probs;
};

struct CnnSmem {
  // weights transposed to [in][ky][kx][out] so one position reads out-vectors
  float4 w0[5 * 9 * 2];
  float4 w1[8 * 9 * 4];
  float4 w2[16 * 9 * 8];
  float b0[8], b1[16], b2[32], w3[32], b3;
  float in[5][7][kTX + 8];
  float o1[8][5][kTX + 4];
  float o2[16][3][kTX + 2];
  float lut[3][256];             // float((v - mean_c) / std_c), computed in FP64
  float zpart[kTX];              // head partial sum over channels 0..15
};

__global__ void __launch_bounds__(256, 2) cnn_kernel(const __grid_constant__ CnnJob J) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CnnSmem& s = *reinterpret_cast<CnnSmem*>(smem_raw);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int W = J.W, H = J.H;
  const float* wg = J.weights;

  // ---- weights -> smem (transposed) ----
  float* w0f = reinterpret_cast<float*>(s.w0);
  float* w1f = reinterpret_cast<float*>(s.w1);
  float* w2f = reinterpret_cast<float*>(s.w2);
  for (int i = tid; i < kW0; i += nt) {  // i = ((o*5 + c)*3 + ky)*3 + kx
    const int o = i / 45, r = i % 45;
    w0f[r * 8 + o] = wg[i];
  }
  for (int i = tid; i < kW1; i += nt) {
    const int o = i / 72, r = i % 72;
    w1f[r * 16 + o] = wg[kOffW1 + i];
  }
  for (int i = tid; i < kW2; i += nt) {
    const int o = i / 144, r = i % 144;
    w2f[r * 32 + o] = wg[kOffW2 + i];
  }
  if (tid < 8) s.b0[tid] = wg[kOffB0 + tid];
  if (tid < 16) s.b1[tid] = wg[kOffB1 + tid];
  if (tid < 32) {
    s.b2[tid] = wg[kOffB2 + tid];
    s.w3[tid] = wg[kOffW3 + tid];
  }
  if (tid == 0) s.b3 = wg[kOffB3];
  for (int i = tid; i < 3 * 256; i += nt) {
    const int ch = i >> 8, v = i & 255;
    s.lut[ch][v] = float(div_rn(sub_rn(double(v), J.mean[ch]), J.stdv[ch]));
  }
  const double xden = double(W - 1 > 1 ? W - 1 : 1), yden = double(H - 1 > 1 ? H - 1 : 1);
  const double xc = div_rn(double(W - 1), 2.0), yc = div_rn(double(H - 1), 2.0);
  const int tiles_x = (W - 6 + kTX - 1) / kTX;
  const int n_tiles = tiles_x * J.S * J.batch;

  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
  const int tx = t % tiles_x, fs = t / tiles_x;
  const int strip = fs % J.S, b = fs / J.S;
  const int j0 = tx * kTX;               // first output column (frame x = j0 + 3)
  __syncthreads();                       // previous tile's buffers are free; tables ready

  // ---- RGBXY window (edgenet.py:75-82), rows h-3..h+3, columns j0..j0+kTX+5 ----
  const int h = J.rows[strip];
  const int band = J.band[strip];
  const uint8_t* fb = J.frames + int64_t(b) * J.fstride;
  for (int c = tid; c < kTX + 6; c += nt) {   // X channel: one FP64 division per column
    const int x = j0 + c;
    const float fx = x < W ? float(div_rn(sub_rn(double(x), xc), xden)) : 0.f;
#pragma unroll
    for (int r = 0; r < 7; ++r) s.in[3][r][c] = fx;
  }
  if (tid < 7) {
    const float fy = float(div_rn(sub_rn(double(h - 3 + tid), yc), yden));
    for (int c = 0; c < kTX + 6; ++c) s.in[4][tid][c] = j0 + c < W ? fy : 0.f;
  }
  for (int i = tid; i < 7 * (kTX + 6); i += nt) {
    const int r = i / (kTX + 6), c = i % (kTX + 6);
    const int x = j0 + c;
    float f0 = 0.f, f1 = 0.f, f2 = 0.f;
    if (x < W) {
      const uint8_t* px = fb + int64_t(band + r) * J.rstride + 3 * x;
      f0 = s.lut[0][px[0]];
      f1 = s.lut[1][px[1]];
      f2 = s.lut[2][px[2]];
    }
    s.in[0][r][c] = f0;
    s.in[1][r][c] = f1;
    s.in[2][r][c] = f2;
  }
  __syncthreads();

  // ---- layer 0: 5 -> 8, rows 7 -> 5 ----
  for (int i = tid; i < 5 * (kTX + 4); i += nt) {
    const int r = i / (kTX + 4), c = i % (kTX + 4);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int ci = 0; ci < 5; ++ci)
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const float v = s.in[ci][r + k / 3][c + k % 3];
        const float4 wa = s.w0[(ci * 9 + k) * 2], wb = s.w0[(ci * 9 + k) * 2 + 1];
        acc[0] = fmaf(wa.x, v, acc[0]); acc[1] = fmaf(wa.y, v, acc[1]);
        acc[2] = fmaf(wa.z, v, acc[2]); acc[3] = fmaf(wa.w, v, acc[3]);
        acc[4] = fmaf(wb.x, v, acc[4]); acc[5] = fmaf(wb.y, v, acc[5]);
        acc[6] = fmaf(wb.z, v, acc[6]); acc[7] = fmaf(wb.w, v, acc[7]);
      }
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const float y = acc[o] + s.b0[o];
      s.o1[o][r][c] = y > 0.f ? y : 0.f;
    }
  }
  __syncthreads();

  // ---- layer 1: 8 -> 16, rows 5 -> 3 ----
  for (int i = tid; i < 3 * (kTX + 2); i += nt) {
    const int r = i / (kTX + 2), c = i % (kTX + 2);
    float acc[16];
#pragma unroll
    for (int o = 0; o < 16; ++o) acc[o] = 0.f;
    for (int ci = 0; ci < 8; ++ci)
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const float v = s.o1[ci][r + k / 3][c + k % 3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 w = s.w1[(ci * 9 + k) * 4 + q];
          acc[4 * q + 0] = fmaf(w.x, v, acc[4 * q + 0]);
          acc[4 * q + 1] = fmaf(w.y, v, acc[4 * q + 1]);
          acc[4 * q + 2] = fmaf(w.z, v, acc[4 * q + 2]);
          acc[4 * q + 3] = fmaf(w.w, v, acc[4 * q + 3]);
        }
      }
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const float y = acc[o] + s.b1[o];
      s.o2[o][r][c] = y > 0.f ? y : 0.f;
    }
  }
  __syncthreads();

  // ---- layer 2: 16 -> 32 (one row), two threads per column (channels
  // 16*hh .. 16*hh+15), then the 1x1 head + sigmoid ----
  const int c = tid & (kTX - 1), hh = tid / kTX;   // hh is warp-uniform
  float acc[16];
#pragma unroll
  for (int o = 0; o < 16; ++o) acc[o] = 0.f;
  for (int ci = 0; ci < 16; ++ci)
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float v = s.o2[ci][k / 3][c + k % 3];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 w = s.w2[(ci * 9 + k) * 8 + 4 * hh + q];
        acc[4 * q + 0] = fmaf(w.x, v, acc[4 * q + 0]);
        acc[4 * q + 1] = fmaf(w.y, v, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(w.z, v, acc[4 * q + 2]);
        acc[4 * q + 3] = fmaf(w.w, v, acc[4 * q + 3]);
      }
    }
  // head: z = sum over channels 0..31 in order, so the second half continues
  // the first half's partial sum
  float z = 0.f;
  if (hh == 0) {
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const float y = acc[o] + s.b2[o];
      z = fmaf(s.w3[o], y > 0.f ? y : 0.f, z);
    }
    s.zpart[c] = z;
  }
  __syncthreads();
  if (hh == 1) {
    z = s.zpart[c];
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const float y = acc[o] + s.b2[16 + o];
      z = fmaf(s.w3[16 + o], y > 0.f ? y : 0.f, z);
    }
    z += s.b3;
    const int j = j0 + c;
    if (j < W - 6) {
      float p;
      if (z >= 0.f) {
        p = 1.0f / (1.0f + expf(-z));
      } else {
        const float e = expf(z);
        p = e / (1.0f + e);
      }
      J.probs[(size_t(b) * J.S + strip) * (W - 6) + j] = p;
    }
  }
  }
}


// ---------------------------------------------------------------------------
// Tensor-core variant (ECA_LEARNED_TCGEN05): the three 3x3 layers on tcgen05
// (layer 0 with its 5 input / 8 output channels zero-padded to 8 / 16), the
// epilogues, 1x1 head and sigmoid on the CUDA cores; one 512-thread CTA per
// SM, one tile of kTP = 128 positions of one strip at a time.
//
// No im2col.  A 3x3 valid conv is 9 shifted GEMMs; the vertical shift (ky)
// selects an input ROW (each row is its own K-major operand), and the
// horizontal shift (kx) is moved to the output: accumulator D[kx][m] =
// sum_ky sum_c in[row + ky][m][c] * W[ky][kx][c] over the UNshifted positions
// m, and out[m] = D[0][m] + D[1][m + 1] + D[2][m + 2], combined in the
// epilogue with warp shuffles (lanes 30/31 take their neighbours from the next
// warp through shared memory).  Each layer input is written once, by the
// previous layer's epilogue, straight into the canonical K-major operand
// layout (8-row x 16-byte core matrices), split hi/lo for 3xTF32
// (hi*hi + hi*lo + lo*hi: FP32-level error, tools/umma_test.cu).  128 MMA
// positions give 122 valid outputs per tile (the 3x3 halo of three layers).
//   layer 0: per output row one N = 32 chain (the three 8-row kx blocks
//            adjacent): 3 ky x 3 split terms, 45 MMAs
//   layer 1: per output row one N = 48 MMA chain (the 3 kx weight blocks
//            stacked as rows of B): 3 ky x 3 split terms, 27 MMAs
//   layer 2: one N = 96 chain: 3 ky x 2 K-steps x 3 terms, 18 MMAs
// TMEM: 256 columns per group, reused by the three layers in turn (layer 0
// [0, 160), layer 1 [0, 144), layer 2 [0, 96)).
constexpr int kTP = 128, kTOut = kTP - 6;   // 3 layers x 2 columns of halo
constexpr int kSbo1 = 2 * 128, kSbo2 = 4 * 128;       // K = 8 / 16 channels
constexpr int kA1 = 16 * kSbo1, kA2 = 16 * kSbo2;     // one row operand (128 positions)
constexpr int kWt1 = 2 * kSbo1, kWt2 = 4 * kSbo2;     // one (ky, kx) weight operand

constexpr int kGroups = 2, kGThreads = 256;          // tiles in flight per CTA, threads per tile
constexpr int kAct = 7 * 2 * kA1;                     // a0 (7 x 2 x 4 KB) >= a2 (3 x 2 x 8 KB) >= a1
static_assert(kAct >= 3 * 2 * kA2 && kAct >= 5 * 2 * kA1, "activation region");

struct CnnGroupTc {               // one tile in flight
  // a0 -> a1 -> a2 in turn: each is dead once the MMAs reading it completed
  alignas(1024) uint8_t act[kAct];
  float xch[768];                 // epilogue neighbour exchange (lanes 0/1 of each warp)
  float zpart[2][kTP];            // head partial sums per channel half
  uint64_t bar[3];                // MMA completion per layer (5 / 3 / 1 issuing threads)
};

struct CnnSmemTc {
  CnnGroupTc grp[kGroups];
  uint8_t b0[2][3][3][kWt1];      // layer-0 weights [hi/lo][ky][kx][out 8 + 8 zero][in 5 + 3 zero]
  uint8_t b1[2][3][3][kWt1];      // layer-1 weights [hi/lo][ky][kx][out 16][in 8]
  uint8_t b2[2][3][3][kWt2];      // layer-2 weights [hi/lo][ky][kx][out 32][in 16]
  float b0v[8], b1v[16], b2v[32], w3[32], b3;
  float lut[3][256];              // float((v - mean_c) / std_c), computed in FP64
  float ytab[ECA_MAX_STRIPS * 7];  // Y channel of rows y-3..y+3 of every strip (edgenet.py:80-82)
  uint32_t tmem;
};

// the same within one tile group (named barrier 1 + group, its 256 threads)
ECA_DEV void group_sync(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kGThreads) : "memory");
}
ECA_DEV void publish_group(int grp) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  group_sync(grp);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__global__ void __launch_bounds__(512, 1) cnn_kernel_tc(const __grid_constant__ CnnJob J) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  CnnSmemTc& s = *reinterpret_cast<CnnSmemTc*>(smem_raw);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int W = J.W, H = J.H;
  const float* wg = J.weights;

  // ---- weights -> smem as K-major hi/lo operands [hi/lo][ky][kx][out][in];
  // layer 0: per ky one 32 x 8 operand, rows kx * 8 + o (the three 8-output
  // kx blocks adjacent, rows 24..31 and input lanes 5..7 zero) ----
  for (int i = tid; i < 2 * 9 * kWt1 / 4; i += nt) reinterpret_cast<float*>(&s.b0[0][0][0][0])[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < kW0; i += nt) {   // i = ((o*5 + c)*3 + ky)*3 + kx
    const int o = i / 45, c = (i / 9) % 5, ky = (i % 9) / 3, kx = i % 3;
    const float v = wg[i], hi = tf32_rna(v);
    *reinterpret_cast<float*>(s.b0[0][ky][0] + kmaj_off(kx * 8 + o, c, kSbo1)) = hi;
    *reinterpret_cast<float*>(s.b0[1][ky][0] + kmaj_off(kx * 8 + o, c, kSbo1)) = tf32_rna(v - hi);
  }
  for (int i = tid; i < kW1; i += nt) {   // i = ((o*8 + c)*3 + ky)*3 + kx
    const int o = i / 72, c = (i / 9) % 8, ky = (i % 9) / 3, kx = i % 3;
    const float v = wg[kOffW1 + i], hi = tf32_rna(v);
    *reinterpret_cast<float*>(s.b1[0][ky][kx] + kmaj_off(o, c, kSbo1)) = hi;
    *reinterpret_cast<float*>(s.b1[1][ky][kx] + kmaj_off(o, c, kSbo1)) = tf32_rna(v - hi);
  }
  for (int i = tid; i < kW2; i += nt) {   // i = ((o*16 + c)*3 + ky)*3 + kx
    const int o = i / 144, c = (i / 9) % 16, ky = (i % 9) / 3, kx = i % 3;
    const float v = wg[kOffW2 + i], hi = tf32_rna(v);
    *reinterpret_cast<float*>(s.b2[0][ky][kx] + kmaj_off(o, c, kSbo2)) = hi;
    *reinterpret_cast<float*>(s.b2[1][ky][kx] + kmaj_off(o, c, kSbo2)) = tf32_rna(v - hi);
  }
  if (tid < 8) s.b0v[tid] = wg[kOffB0 + tid];
  if (tid < 16) s.b1v[tid] = wg[kOffB1 + tid];
  if (tid < 32) {
    s.b2v[tid] = wg[kOffB2 + tid];
    s.w3[tid] = wg[kOffW3 + tid];
  }
  if (tid == 0) s.b3 = wg[kOffB3];
  for (int i = tid; i < 3 * 256; i += nt) {
    const int ch = i >> 8, v = i & 255;
    s.lut[ch][v] = float(div_rn(sub_rn(double(v), J.mean[ch]), J.stdv[ch]));
  }
  {
    const double yden0 = double(H - 1 > 1 ? H - 1 : 1), yc0 = div_rn(double(H - 1), 2.0);
    for (int i = tid; i < J.S * 7; i += nt)
      s.ytab[i] = float(div_rn(sub_rn(double(J.rows[i / 7] - 3 + i % 7), yc0), yden0));
  }
  const int grp = warp >> 3, gtid = tid & (kGThreads - 1);
  CnnGroupTc& G = s.grp[grp];
  // the MMA chains of different output rows are independent: layer 0's five
  // rows are issued by five warps, layer 1's three by three, layer 2's one
  // chain by one thread; each layer's mbarrier counts its issuers' commits
  const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(&G.bar[0]));
  const uint32_t bar1 = bar0 + 8u, bar2 = bar0 + 16u;
  if (gtid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 5;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 3;" ::"r"(bar1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar2));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int gw = (gtid >> 5);   // warp index within the group
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&s.tmem))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  publish_operands();
  const uint32_t tmem = s.tmem + uint32_t(grp * 256);   // this group's 256 TMEM columns
  uint32_t phase = 0;
  const auto saddr = [](const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); };
  const int q = warp & 3, ch = (warp >> 2) & 1;   // TMEM lane quarter, channel half
  const int m = 32 * q + lane;                    // this thread's MMA position
  const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
  uint8_t* act = G.act;
  auto a0 = [&](int r, int part) { return act + (r * 2 + part) * kA1; };
  auto a1 = [&](int r, int part) { return act + (r * 2 + part) * kA1; };
  auto a2 = [&](int r, int part) { return act + (r * 2 + part) * kA2; };

  const double xden = double(W - 1 > 1 ? W - 1 : 1), yden = double(H - 1 > 1 ? H - 1 : 1);
  const double xc = div_rn(double(W - 1), 2.0), yc = div_rn(double(H - 1), 2.0);
  const int tiles_x = (W - 6 + kTOut - 1) / kTOut;
  const int n_tiles = tiles_x * J.S * J.batch;
  const int t_step = kGroups * gridDim.x;

  // the RGB bytes of a tile's window, 4 pixels per thread, loaded one tile
  // ahead (issued under the current tile's tensor-core work)
  constexpr int kWinPx = 7 * kTP;
  constexpr int kPxPer = (kWinPx + kGThreads - 1) / kGThreads;
  uint32_t px_next[kPxPer];
  auto load_window = [&](int t) {
    if (t >= n_tiles) return;
    const int tx = t % tiles_x, fs = t / tiles_x;
    const int strip = fs % J.S, b = fs / J.S;
    const uint8_t* fb = J.frames + int64_t(b) * J.fstride;
#pragma unroll
    for (int k = 0; k < kPxPer; ++k) {
      const int i = gtid + k * kGThreads;
      uint32_t v = 0u;
      if (i < kWinPx) {
        const int r = i / kTP, c = i % kTP, x = tx * kTOut + c;
        if (x < W) {
          const uint8_t* px = fb + int64_t(J.band[strip] + r) * J.rstride + 3 * x;
          v = uint32_t(__ldg(px)) | (uint32_t(__ldg(px + 1)) << 8) | (uint32_t(__ldg(px + 2)) << 16);
        }
      }
      px_next[k] = v;
    }
  };
  load_window(blockIdx.x + grp * gridDim.x);

  // group g runs this CTA's tiles g, g + 2, ...: while one group's MMAs run,
  // the other group's CUDA-core work (window, epilogues) proceeds
  for (int t = blockIdx.x + grp * gridDim.x; t < n_tiles; t += t_step) {
  const int tx = t % tiles_x, fs = t / tiles_x;
  const int strip = fs % J.S, b = fs / J.S;
  const int j0 = tx * kTOut;              // first output column (frame x = j0 + 3)
  group_sync(grp);                        // the previous tile's epilogue is done

  // ---- RGBXY window (edgenet.py:75-82), rows h-3..h+3, positions j0..j0+127,
  // written as the layer-0 operand rows (K lanes: R, G, B, X, Y, 0, 0, 0) ----
  static_assert(kGThreads % kTP == 0, "a thread keeps one window column");
  const int wc = gtid % kTP;   // this thread's column for all its window pixels
  const float fx_c = j0 + wc < W ? float(div_rn(sub_rn(double(j0 + wc), xc), xden)) : 0.f;
#pragma unroll
  for (int k = 0; k < kPxPer; ++k) {
    const int i = gtid + k * kGThreads;
    if (i < kWinPx) {
      const int r = i / kTP, c = wc, x = j0 + c;
      const uint32_t v = px_next[k];
      float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
      float fy = 0.f;
      if (x < W) {
        f.x = s.lut[0][v & 255u];
        f.y = s.lut[1][(v >> 8) & 255u];
        f.z = s.lut[2][(v >> 16) & 255u];
        f.w = fx_c;
        fy = s.ytab[strip * 7 + r];
      }
      st_hilo(a0(r, 0), a0(r, 1), kmaj_off(c, 0, kSbo1), f);
      st_hilo(a0(r, 0), a0(r, 1), kmaj_off(c, 4, kSbo1), make_float4(fy, 0.f, 0.f, 0.f));
    }
  }
  publish_group(grp);

  // ---- layer 0 (tensor cores): D0[r][kx] = sum_ky a0[r + ky] . b0[ky][kx],
  // N = 32 (three adjacent 8-row kx blocks + 8 zero rows) ----
  if (gw < 5 && lane == 0) {   // output row r = gw
    constexpr uint32_t id0 = idesc_tf32(32);
    const int r = gw;
    for (int ky = 0; ky < 3; ++ky)
      mma3(tmem + uint32_t(r * 32), saddr(a0(r + ky, 0)), saddr(a0(r + ky, 1)), kSbo1,
           saddr(s.b0[0][ky][0]), saddr(s.b0[1][ky][0]), kSbo1, id0, ky == 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0)
                 : "memory");
  }
  load_window(t + t_step);   // the next tile's bytes arrive under this tile's MMAs
  bar_wait(bar0, phase);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- layer-0 epilogue: o1[r][m] = D[0][m] + D[1][m+1] + D[2][m+2] + b0, ReLU,
  // as the layer-1 operand rows (over a0: its MMAs completed); warp (q, ch):
  // positions 32q.., channels 4ch.. ----
  {
    float d[5][3][4];
#pragma unroll
    for (int r = 0; r < 5; ++r)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) tmem_ld<4>(lane_base + uint32_t(r * 32 + kx * 8 + 4 * ch), d[r][kx]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float* xch = G.xch;   // [r][q][lane][kx-1][8]
    if (lane < 2) {
#pragma unroll
      for (int r = 0; r < 5; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int c = 0; c < 4; ++c) xch[(((r * 4 + q) * 2 + lane) * 2 + k) * 8 + 4 * ch + c] = d[r][k + 1][c];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    group_sync(grp);   // also: every a0 read of this tile's MMAs is long complete
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      float v1[4], v2[4], y[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v1[c] = __shfl_down_sync(kFull, d[r][1][c], 1);
        v2[c] = __shfl_down_sync(kFull, d[r][2][c], 2);
      }
      if (q < 3 && lane >= 30) {   // two lanes: the next warp's first positions
        const float* nx = xch + ((r * 4 + q + 1) * 2) * 2 * 8 + 4 * ch;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (lane == 31) v1[c] = nx[c];                       // lane 0, kx 1
          v2[c] = nx[((lane - 30) * 2 + 1) * 8 + c];           // lane 0/1, kx 2
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float v = (d[r][0][c] + v1[c]) + v2[c] + s.b0v[4 * ch + c];
        y[c] = v > 0.f ? v : 0.f;
      }
      st_hilo(a1(r, 0), a1(r, 1), kmaj_off(m, 4 * ch, kSbo1), make_float4(y[0], y[1], y[2], y[3]));
    }
  }
  publish_group(grp);

  // ---- layer 1 (tensor cores): D1[r][kx] = sum_ky a1[r + ky] . b1[ky][kx];
  // the three kx weight blocks are adjacent rows of one N = 48 operand ----
  if (gw < 3 && lane == 0) {   // output row r = gw
    constexpr uint32_t id1 = idesc_tf32(48);
    const int r = gw;
    for (int ky = 0; ky < 3; ++ky)
      mma3(tmem + uint32_t(r * 48), saddr(a1(r + ky, 0)), saddr(a1(r + ky, 1)), kSbo1,
           saddr(s.b1[0][ky][0]), saddr(s.b1[1][ky][0]), kSbo1, id1, ky == 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar1)
                 : "memory");
  }
  bar_wait(bar1, phase);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- layer-1 epilogue -> layer-2 operand rows (over a1: its MMAs completed);
  // warp (q, ch): channels 8ch.. ----
  {
    float d[3][3][8];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) tmem_ld<8>(lane_base + uint32_t(r * 48 + kx * 16 + 8 * ch), d[r][kx]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float* xch = G.xch;   // [r][q][lane][kx-1][16]
    if (lane < 2) {
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int c = 0; c < 8; ++c) xch[(((r * 4 + q) * 2 + lane) * 2 + k) * 16 + 8 * ch + c] = d[r][k + 1][c];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    group_sync(grp);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      float v1[8], v2[8], y[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        v1[c] = __shfl_down_sync(kFull, d[r][1][c], 1);
        v2[c] = __shfl_down_sync(kFull, d[r][2][c], 2);
      }
      if (q < 3 && lane >= 30) {   // two lanes: the next warp's first positions
        const float* nx = xch + ((r * 4 + q + 1) * 2) * 2 * 16 + 8 * ch;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (lane == 31) v1[c] = nx[c];
          v2[c] = nx[((lane - 30) * 2 + 1) * 16 + c];
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float v = (d[r][0][c] + v1[c]) + v2[c] + s.b1v[8 * ch + c];
        y[c] = v > 0.f ? v : 0.f;
      }
      st_hilo(a2(r, 0), a2(r, 1), kmaj_off(m, 8 * ch, kSbo2), make_float4(y[0], y[1], y[2], y[3]));
      st_hilo(a2(r, 0), a2(r, 1), kmaj_off(m, 8 * ch + 4, kSbo2), make_float4(y[4], y[5], y[6], y[7]));
    }
  }
  publish_group(grp);

  // ---- layer 2 (tensor cores): D2[kx] = sum_ky a2[ky] . b2[ky][kx], K = 16,
  // the three kx blocks as one N = 96 operand ----
  if (gtid == 0) {
    constexpr uint32_t id2 = idesc_tf32(96);
    for (int ky = 0; ky < 3; ++ky)
      for (int j = 0; j < 2; ++j)   // 8 channels (32 bytes of K) per instruction
        mma3(tmem, saddr(a2(ky, 0)) + 256u * j, saddr(a2(ky, 1)) + 256u * j, kSbo2,
             saddr(s.b2[0][ky][0]) + 256u * j, saddr(s.b2[1][ky][0]) + 256u * j, kSbo2, id2,
             ky == 0 && j == 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar2)
                 : "memory");
  }
  bar_wait(bar2, phase);
  phase ^= 1u;   // each layer's barrier completes once per tile
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- layer-2 epilogue + head: channels 16ch..16ch+15 per warp, partial
  // head sums per channel half, then the sigmoid ----
  {
    float d[3][16];
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) tmem_ld<16>(lane_base + uint32_t(kx * 32 + 16 * ch), d[kx]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float* xch = G.xch;   // [q][lane][kx-1][32]
    if (lane < 2) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int c = 0; c < 16; ++c) xch[((q * 2 + lane) * 2 + k) * 32 + 16 * ch + c] = d[k + 1][c];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    group_sync(grp);
    float v1[16], v2[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      v1[c] = __shfl_down_sync(kFull, d[1][c], 1);
      v2[c] = __shfl_down_sync(kFull, d[2][c], 2);
    }
    if (q < 3 && lane >= 30) {   // two lanes: the next warp's first positions
      const float* nx = xch + ((q + 1) * 2) * 2 * 32 + 16 * ch;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (lane == 31) v1[c] = nx[c];
        v2[c] = nx[((lane - 30) * 2 + 1) * 32 + c];
      }
    }
    float z = 0.f;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float v = (d[0][c] + v1[c]) + v2[c] + s.b2v[16 * ch + c];
      z = fmaf(s.w3[16 * ch + c], v > 0.f ? v : 0.f, z);
    }
    G.zpart[ch][m] = z;
  }
  group_sync(grp);
  if (gtid < kTOut) {
    const float z = (G.zpart[0][gtid] + G.zpart[1][gtid]) + s.b3;
    const int j = j0 + gtid;
    if (j < W - 6) {
      float p;
      if (z >= 0.f) {
        p = 1.0f / (1.0f + expf(-z));
      } else {
        const float e = expf(z);
        p = e / (1.0f + e);
      }
      J.probs[(size_t(b) * J.S + strip) * (W - 6) + j] = p;
    }
  }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s.tmem));
}

// half-row winners of the zero-padded probability row (edgenet.py:363-369)
__global__ void __launch_bounds__(256) select_kernel(const float* probs, int S, int W,
                                                     const int32_t* rows_dev_unused,
                                                     int32_t* out_x, int32_t* out_y,
                                                     double* out_s, CnnJob J) {
  const int strip = blockIdx.x, b = blockIdx.y;
  const int split = (W + 1) / 2;
  const float* pr = probs + (size_t(b) * S + strip) * (W - 6);
  Best L{-1.0, 0x7fffffff}, R{-1.0, -1};
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    const double v = (x >= 3 && x <= W - 4) ? double(pr[x - 3]) : 0.0;
    if (x < split) {
      if (better(v, x, L.s, L.x, true)) L = Best{v, x};
    } else {
      if (better(v, x, R.s, R.x, false)) R = Best{v, x};
    }
  }
  __shared__ double bs[8][2];
  __shared__ int bx[8][2];
  L = warp_best(L, true);
  R = warp_best(R, false);
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    bs[warp][0] = L.s; bx[warp][0] = L.x;
    bs[warp][1] = R.s; bx[warp][1] = R.x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
      if (better(bs[w][0], bx[w][0], L.s, L.x, true)) L = Best{bs[w][0], bx[w][0]};
      if (better(bs[w][1], bx[w][1], R.s, R.x, false)) R = Best{bs[w][1], bx[w][1]};
    }
    const size_t o = size_t(b) * 2 * S;
    const int y = J.rows[strip];
    out_x[o + strip] = L.x; out_y[o + strip] = y; out_s[o + strip] = L.s;
    out_x[o + S + strip] = R.x; out_y[o + S + strip] = y; out_s[o + S + strip] = R.s;
  }
}

}  // namespace

extern "C" int eca_points_learned_ex(const uint8_t* frames, int batch, int64_t frame_stride,
                                     int64_t row_stride, const int32_t* strip_rows,
                                     const int32_t* band_rows, int n_strips, int height, int width,
                                     const float* weights, const double* norm, int flags,
                                     float* out_probs, int32_t* out_x, int32_t* out_y,
                                     double* out_score, void* stream) {
  ECA_RANGE("eca_points_learned_ex");
  if ((flags & ~(ECA_LEARNED_TCGEN05 | ECA_LEARNED_SIMT)) ||
      (flags & (ECA_LEARNED_TCGEN05 | ECA_LEARNED_SIMT)) == (ECA_LEARNED_TCGEN05 | ECA_LEARNED_SIMT))
    return ECA_ERR_ARG;
  if (batch < 0 || !strip_rows || !norm) return ECA_ERR_ARG;
  if (width < 8 || height < 14 || row_stride < 3LL * width) return ECA_ERR_ARG;
  if (height > 32767) return ECA_ERR_UNSUPPORTED;
  if (n_strips < 1 || n_strips > ECA_MAX_STRIPS || batch > 65535) return ECA_ERR_UNSUPPORTED;
  if (batch == 0) return ECA_OK;
  if (!frames || !weights || !out_probs || !out_x || !out_y || !out_score) return ECA_ERR_ARG;
  CnnJob J;
  J.frames = frames;
  J.fstride = frame_stride;
  J.rstride = row_stride;
  J.batch = batch;
  J.S = n_strips;
  J.H = height;
  J.W = width;
  for (int k = 0; k < n_strips; ++k) {
    if (strip_rows[k] < 3 || strip_rows[k] > height - 4) return ECA_ERR_ARG;
    J.rows[k] = int16_t(strip_rows[k]);
    const int band = band_rows ? band_rows[k] : strip_rows[k] - 3;
    if (band < 0 || band > 32767) return ECA_ERR_ARG;
    J.band[k] = int16_t(band);
  }
  for (int c = 0; c < 3; ++c) {
    J.mean[c] = norm[c];
    J.stdv[c] = norm[3 + c];
  }
  J.weights = weights;
  J.probs = out_probs;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const bool tc = (flags & ECA_LEARNED_SIMT) == 0;   // tcgen05 unless the SIMT kernel is asked for
  // per device: shared-memory opt-in and occupancy (checked)
  static std::once_flag once[64];
  static int per_sm_d[64], per_sm_tc_d[64], sms_d[64], tc_smem_d[64];
  static bool ok_d[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return ECA_ERR_CUDA;
  std::call_once(once[dev], [dev] {
    int a = 0, b = 0, c = 0, optin_max = 0;
    // cnn_kernel_tc holds all 512 TMEM columns: its CTA takes the whole
    // shared memory too, so the block scheduler cannot co-locate another
    // TMEM-using CTA with it (the scheduler does not account TMEM)
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, cnn_kernel_tc);
    cudaDeviceGetAttribute(&optin_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    tc_smem_d[dev] = optin_max - int(fa.sharedSizeBytes);
    if (tc_smem_d[dev] < int(sizeof(CnnSmemTc))) tc_smem_d[dev] = int(sizeof(CnnSmemTc));
    ok_d[dev] = cudaFuncSetAttribute(cnn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(CnnSmem))) == cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, cnn_kernel, 256, sizeof(CnnSmem)) ==
                    cudaSuccess &&
                cudaFuncSetAttribute(cnn_kernel_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tc_smem_d[dev]) == cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, cnn_kernel_tc, 512, tc_smem_d[dev]) ==
                    cudaSuccess &&
                cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess;
    per_sm_d[dev] = a > 0 ? a : 1;
    per_sm_tc_d[dev] = b > 0 ? b : 1;
    sms_d[dev] = c > 0 ? c : 148;
  });
  if (!ok_d[dev]) return ECA_ERR_CUDA;
  const int per_sm = per_sm_d[dev], per_sm_tc = per_sm_tc_d[dev], sms = sms_d[dev];
  const int64_t tiles = int64_t((width - 6 + kTX - 1) / kTX) * n_strips * batch;
  const int64_t cap = int64_t(sms) * (tc ? per_sm_tc : per_sm);
  const int grid = int(tiles < cap ? tiles : cap);
  if (tc)
    cnn_kernel_tc<<<grid, 512, tc_smem_d[dev], st>>>(J);
  else
    cnn_kernel<<<grid, 256, sizeof(CnnSmem), st>>>(J);
  select_kernel<<<dim3(n_strips, batch), 256, 0, st>>>(out_probs, n_strips, width, nullptr, out_x,
                                                        out_y, out_score, J);
  return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

extern "C" int eca_points_learned(const uint8_t* frames, int batch, int64_t frame_stride,
                                  int64_t row_stride, const int32_t* strip_rows,
                                  const int32_t* band_rows, int n_strips,
                                  int height, int width, const float* weights, const double* norm,
                                  float* out_probs, int32_t* out_x, int32_t* out_y,
                                  double* out_score, void* stream) {
  ECA_RANGE("eca_points_learned");
  return eca_points_learned_ex(frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                               n_strips, height, width, weights, norm, 0, out_probs, out_x, out_y,
                               out_score, stream);
}
