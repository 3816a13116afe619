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
// Tensor-core variant (ECA_LEARNED_TCGEN05): the same network with layer 2 on
// tcgen05.  Measured on B200, 256 x 1080p: 7.5 ms against 6.2 ms for the SIMT
// kernel above -- building the im2col operand and waiting for the per-piece
// MMAs costs more than layer 2's FMAs, and layers 0-1 stay SIMT at one
// 512-thread CTA per SM.  Kept as a parity-tested option; chaining all three
// layers through TMEM is the step that would make it pay.
// Layer 2 (16 -> 32 channels, K = 16*3*3 = 144) runs on the tensor cores:
// per tile D[128 columns][32 channels] = im2col(o2)[128][144] . W2^T, tcgen05
// kind::tf32 with a 3xTF32 split (hi*hi + hi*lo + lo*hi, FP32-level error
// ~2e-6, tools/umma_test.cu), FP32 accumulators in TMEM.  Operands sit in
// shared memory in the K-major no-swizzle canonical layout: 8-row x 16-byte
// core matrices, LBO = 128 B between K chunks, SBO between 8-row groups.
// The im2col operand is built in K-ninths (16 K each), double-buffered so one
// ninth is written while the tensor core consumes the other, in shared memory
// aliased over the input / layer-0 buffers (dead during layer 2): the CTA stays
// under 113 KB, two CTAs per SM.
#ifndef ECA_CNN_NO_MMA   // diagnostic: skip the MMAs (wrong results), time the rest
#define ECA_CNN_NO_MMA 0
#endif
constexpr int kK2 = 144, kK2p = 16;             // layer-2 K, per built piece
constexpr int kSboA = (kK2p / 4) * 128;         // 512 B
constexpr int kSboB = (kK2 / 4) * 128;          // 4608 B
constexpr int kAPiece = kTX * kK2p * 4;         // 8 KB (hi or lo)

struct CnnSmemTc {
  union {   // 1024-byte aligned (kernel smem base): descriptor addresses are 16-byte units
    struct {                      // layers 0-1
      float in[5][7][kTX + 8];
      float o1[8][5][kTX + 4];
    } l01;
    uint8_t a[2][2][kAPiece];     // layer 2: [buffer][hi, lo] im2col piece
  } u;
  uint8_t b_hi[32 * kK2 * 4];     // layer-2 weights [out][k] (reference order = K-major)
  uint8_t b_lo[32 * kK2 * 4];
  // layers 0-1: weights transposed to [in][ky][kx][out] so one position reads out-vectors
  float4 w0[5 * 9 * 2];
  float4 w1[8 * 9 * 4];
  int koff[kK2];                  // layer-2 k -> offset of o2[ci][ky][kx] (column 0)
  uint64_t bar[2];                // MMA completion per A buffer
  uint32_t tmem;                  // TMEM base address (32 columns)
  float b0[8], b1[16], b2[32], w3[32], b3;
  float o2[16][3][kTX + 2];
  float lut[3][256];             // float((v - mean_c) / std_c), computed in FP64
  float ybuf[32][kTX];           // layer-2 outputs after bias + ReLU
};

ECA_DEV float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// byte offset of (row, k) in a K-major no-swizzle operand with row-group stride sbo
ECA_DEV int kmaj_off(int row, int k, int sbo) {
  return (row >> 3) * sbo + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
}
ECA_DEV uint64_t umma_desc(uint32_t saddr, int sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);   // version 1, no swizzle
}
// kind::tf32, D F32, A/B TF32 K-major, M = 128, N = 32
constexpr uint32_t kIdescL2 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(32 >> 3) << 17) |
                              (uint32_t(128 >> 4) << 24);

// 512 threads, one CTA per SM (the occupancy API grants this kernel one)
__global__ void __launch_bounds__(512, 1) cnn_kernel_tc(const __grid_constant__ CnnJob J) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  CnnSmemTc& s = *reinterpret_cast<CnnSmemTc*>(smem_raw);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int W = J.W, H = J.H;
  const float* wg = J.weights;

  // ---- weights -> smem (transposed) ----
  float* w0f = reinterpret_cast<float*>(s.w0);
  float* w1f = reinterpret_cast<float*>(s.w1);
  for (int i = tid; i < kW0; i += nt) {  // i = ((o*5 + c)*3 + ky)*3 + kx
    const int o = i / 45, r = i % 45;
    w0f[r * 8 + o] = wg[i];
  }
  for (int i = tid; i < kW1; i += nt) {
    const int o = i / 72, r = i % 72;
    w1f[r * 16 + o] = wg[kOffW1 + i];
  }
  for (int i = tid; i < kW2; i += nt) {   // i = o*144 + k: already K-major
    const int o = i / kK2, k = i % kK2;
    const float v = wg[kOffW2 + i], hi = tf32_rna(v);
    *reinterpret_cast<float*>(s.b_hi + kmaj_off(o, k, kSboB)) = hi;
    *reinterpret_cast<float*>(s.b_lo + kmaj_off(o, k, kSboB)) = tf32_rna(v - hi);
  }
  for (int k = tid; k < kK2; k += nt) {
    const int ci = k / 9, ky = (k % 9) / 3, kx = k % 3;
    s.koff[k] = (ci * 3 + ky) * (kTX + 2) + kx;
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int q = 0; q < 2; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&s.bar[q]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&s.tmem))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s.tmem;
  const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(&s.bar[0]));
  uint32_t mma_phase = 0;   // bit q: parity of buffer q's next completion
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
    for (int r = 0; r < 7; ++r) s.u.l01.in[3][r][c] = fx;
  }
  if (tid < 7) {
    const float fy = float(div_rn(sub_rn(double(h - 3 + tid), yc), yden));
    for (int c = 0; c < kTX + 6; ++c) s.u.l01.in[4][tid][c] = j0 + c < W ? fy : 0.f;
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
    s.u.l01.in[0][r][c] = f0;
    s.u.l01.in[1][r][c] = f1;
    s.u.l01.in[2][r][c] = f2;
  }
  __syncthreads();

  // ---- layer 0: 5 -> 8, rows 7 -> 5 ----
  for (int i = tid; i < 5 * (kTX + 4); i += nt) {
    const int r = i / (kTX + 4), c = i % (kTX + 4);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int ci = 0; ci < 5; ++ci)
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const float v = s.u.l01.in[ci][r + k / 3][c + k % 3];
        const float4 wa = s.w0[(ci * 9 + k) * 2], wb = s.w0[(ci * 9 + k) * 2 + 1];
        acc[0] = fmaf(wa.x, v, acc[0]); acc[1] = fmaf(wa.y, v, acc[1]);
        acc[2] = fmaf(wa.z, v, acc[2]); acc[3] = fmaf(wa.w, v, acc[3]);
        acc[4] = fmaf(wb.x, v, acc[4]); acc[5] = fmaf(wb.y, v, acc[5]);
        acc[6] = fmaf(wb.z, v, acc[6]); acc[7] = fmaf(wb.w, v, acc[7]);
      }
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const float y = acc[o] + s.b0[o];
      s.u.l01.o1[o][r][c] = y > 0.f ? y : 0.f;
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
        const float v = s.u.l01.o1[ci][r + k / 3][c + k % 3];
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

  // ---- layer 2 on the tensor cores: 9 pieces of im2col(o2), 6 MMAs each ----
  auto wait_buf = [&](int q) {
    asm volatile(
        "{\n.reg .pred P1;\nECA_MW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra ECA_MW;\n}\n" ::"r"(bar0 + 8u * uint32_t(q)),
        "r"((mma_phase >> q) & 1u)
        : "memory");
    mma_phase ^= 1u << q;
  };
  for (int piece = 0; piece < kK2 / kK2p; ++piece) {
    const int q = piece & 1;
    if (piece >= 2) wait_buf(q);         // the MMAs of piece - 2 have read this buffer
    // one warp per 8x4 core matrix: lane = (row & 7) * 4 + (k & 3), so a warp
    // writes 128 contiguous bytes
    const int r8 = lane >> 2, c4 = lane & 3;
    uint8_t* ahi = s.u.a[q][0];
    uint8_t* alo = s.u.a[q][1];
    for (int cm = warp; cm < (kTX / 8) * (kK2p / 4); cm += nt >> 5) {
      const int mi = cm / (kK2p / 4), kc = cm % (kK2p / 4);
      const int m = mi * 8 + r8, kk = kc * 4 + c4;
      const float v = (&s.o2[0][0][0])[s.koff[piece * kK2p + kk] + m];
      const float hi = tf32_rna(v);
      const int off = mi * kSboA + kc * 128 + lane * 4;
      *reinterpret_cast<float*>(ahi + off) = hi;
      *reinterpret_cast<float*>(alo + off) = tf32_rna(v - hi);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // st.shared -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
      const uint32_t ah = static_cast<uint32_t>(__cvta_generic_to_shared(ahi));
      const uint32_t al = static_cast<uint32_t>(__cvta_generic_to_shared(alo));
      const uint32_t bh = static_cast<uint32_t>(__cvta_generic_to_shared(s.b_hi));
      const uint32_t bl = static_cast<uint32_t>(__cvta_generic_to_shared(s.b_lo));
#pragma unroll
      for (int j = 0; j < kK2p / 8; ++j) {   // 8 tf32 (32 bytes) of K per instruction
        const uint32_t oa = uint32_t(j) * 256u;
        const uint32_t ob = uint32_t(piece * (kK2p / 8) + j) * 256u;
        const uint64_t da[3] = {umma_desc(ah + oa, kSboA), umma_desc(ah + oa, kSboA),
                                umma_desc(al + oa, kSboA)};
        const uint64_t db[3] = {umma_desc(bh + ob, kSboB), umma_desc(bl + ob, kSboB),
                                umma_desc(bh + ob, kSboB)};
#pragma unroll
        for (int t3 = 0; t3 < (ECA_CNN_NO_MMA ? 0 : 3); ++t3) {
          const uint32_t accum = (piece > 0 || j > 0 || t3 > 0) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da[t3]), "l"(db[t3]), "r"(kIdescL2), "r"(accum));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       bar0 + 8u * uint32_t(q))
                   : "memory");
    }
  }
  // the last two pieces (buffers 1 and 0) have completed: accumulators final,
  // the aliased input buffers free again
  wait_buf(1);
  wait_buf(0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // accumulators -> registers: warp w reads TMEM lanes 32*(w%4).. (output
  // columns) and channels 8*(w/4) .. 8*(w/4)+7; bias + ReLU into ybuf, then the
  // 1x1 head sums the 32 channels in order
  {
    const int g = warp >> 2, c = (warp & 3) * 32 + lane;
    uint32_t v[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7])
        : "r"(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(8 * g)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const float y = __uint_as_float(v[o]) + s.b2[8 * g + o];
      s.ybuf[8 * g + o][c] = y > 0.f ? y : 0.f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < kTX) {
    float z = 0.f;
#pragma unroll
    for (int o = 0; o < 32; ++o) z = fmaf(s.w3[o], s.ybuf[o][tid], z);
    z += s.b3;
    const int j = j0 + tid;
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
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
  if (flags & ~ECA_LEARNED_TCGEN05) return ECA_ERR_ARG;
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
  const bool tc = (flags & ECA_LEARNED_TCGEN05) != 0;
  static std::once_flag once;
  static int per_sm = 1, per_sm_tc = 1, sms = 148;
  std::call_once(once, [] {
    cudaFuncSetAttribute(cnn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(CnnSmem)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cnn_kernel, 256, sizeof(CnnSmem));
    cudaFuncSetAttribute(cnn_kernel_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(CnnSmemTc)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_tc, cnn_kernel_tc, 512, sizeof(CnnSmemTc));
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
    if (per_sm_tc < 1) per_sm_tc = 1;
  });
  const int64_t tiles = int64_t((width - 6 + kTX - 1) / kTX) * n_strips * batch;
  const int64_t cap = int64_t(sms) * (tc ? per_sm_tc : per_sm);
  const int grid = int(tiles < cap ? tiles : cap);
  if (tc)
    cnn_kernel_tc<<<grid, 512, sizeof(CnnSmemTc), st>>>(J);
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
  return eca_points_learned_ex(frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                               n_strips, height, width, weights, norm, 0, out_probs, out_x, out_y,
                               out_score, stream);
}
