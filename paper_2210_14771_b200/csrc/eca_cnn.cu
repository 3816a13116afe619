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

extern "C" int eca_points_learned(const uint8_t* frames, int batch, int64_t frame_stride,
                                  int64_t row_stride, const int32_t* strip_rows,
                                  const int32_t* band_rows, int n_strips,
                                  int height, int width, const float* weights, const double* norm,
                                  float* out_probs, int32_t* out_x, int32_t* out_y,
                                  double* out_score, void* stream) {
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
  static bool attr = false;
  static int per_sm = 1, sms = 148;
  if (!attr) {
    cudaFuncSetAttribute(cnn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(CnnSmem)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cnn_kernel, 256, sizeof(CnnSmem));
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
    attr = true;
  }
  const int64_t tiles = int64_t((width - 6 + kTX - 1) / kTX) * n_strips * batch;
  const int grid = int(tiles < int64_t(sms) * per_sm ? tiles : int64_t(sms) * per_sm);
  cnn_kernel<<<grid, 256, sizeof(CnnSmem), st>>>(J);
  select_kernel<<<dim3(n_strips, batch), 256, 0, st>>>(out_probs, n_strips, width, nullptr, out_x,
                                                        out_y, out_score, J);
  return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}
