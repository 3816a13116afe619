// §8f-4: EdgeNet training on the GPU (edgenet.py:100-130, 213-344), FP32 like
// the reference.
//
// Inputs are the reference's training tensors: x [*][5][h][W] (NCHW float32,
// RGBXY rows), targets [*][1][h-6][W-6]; a batch is a list of sample indices
// into them (the epoch permutation), gathered inside the first kernels.
//
// Default: the convolutions on the tensor cores (eca_train_tc.cuh, tcgen05
// 3xTF32; 10 launches per SGD step):
//  forward    tc_conv_fwd x3 (3x3 valid conv + bias + ReLU; the first also
//             packs the later kernels' weight operands, the last computes the
//             1x1 head's logits); activations stay in the workspace (the
//             reference's caches; ReLU masks are y > 0).
//  backward   loss_head_kernel: stable BCE terms in FP64 (edgenet.py:236-241),
//             dlogits = (sigmoid(z) - t) / N in FP32 (:315), the head's input
//             gradient and block partials of its weight gradient; per 3x3
//             layer tc_conv_wgrad (partials per CTA) and tc_conv_dgrad (x the
//             previous layer's ReLU mask; not for layer 0); tc_wgrad_reduce
//             sums all partials in a fixed order (deterministic, no float
//             atomics) and the loss (loss_final's order).
//  sgd        w = w - fl32(lr) * g without contraction (:327-328), skipped
//             once a non-finite loss was seen (the reference raises before
//             that update), so an epoch runs without host round trips.
// ECA_TRAIN_SIMT=1: the CUDA-core kernels below (conv3_fwd / head_fwd,
// loss_kernel, head_dgrad, conv3_dgrad, conv_wgrad + wgrad_reduce; sequential
// FMA, per-row-segment weight-gradient partials); kept for comparison.
// The reference's sgemm reassociates, so logits / gradients agree to FP32
// rounding, not bitwise.
#include <math.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "eca_common.cuh"
#include "eca_train_tc.cuh"

using namespace eca;

namespace {

constexpr int kOffW0 = 0, kOffB0 = 360, kOffW1 = 368, kOffB1 = 1520, kOffW2 = 1536, kOffB2 = 6144,
              kOffW3 = 6176, kOffB3 = 6208, kNetN = 6209;
static_assert(kNetN == ECA_NET_FLOATS, "weight layout");
constexpr int kSeg = 128;   // output columns per weight-gradient segment

// tensor-core weight-gradient partials: [kWgCtas][R][CO] per layer
constexpr size_t kTcPart0 = size_t(ttc::kWgCtas) * ttc::WgCfg<5, 8, 3>::R * 8;
constexpr size_t kTcPart1 = size_t(ttc::kWgCtas) * ttc::WgCfg<8, 16, 3>::R * 16;
constexpr size_t kTcPart2 = size_t(ttc::kWgCtas) * ttc::WgCfg<16, 32, 3>::R * 32;

struct TrainWs {   // workspace layout (floats unless noted)
  size_t a1, a2, a3, logit, d3, d2, d1, dlog, wpart, lpart, tcpart, hpart, bimg[5], total;
  int nseg3, nseg2, nseg1, nseg0, nlblk;
};

size_t up256(size_t v) { return (v + 255) & ~size_t(255); }

constexpr int kLossThreads = 256;

TrainWs train_ws(int m, int h, int w) {
  TrainWs L;
  const size_t p1 = size_t(m) * (h - 2) * (w - 2), p2 = size_t(m) * (h - 4) * (w - 4),
               p3 = size_t(m) * (h - 6) * (w - 6);
  size_t o = 0;
  L.a1 = o;    o = up256(o + 4 * 8 * p1);
  L.a2 = o;    o = up256(o + 4 * 16 * p2);
  L.a3 = o;    o = up256(o + 4 * 32 * p3);
  L.logit = o; o = up256(o + 4 * p3);
  L.d3 = o;    o = up256(o + 4 * 32 * p3);
  L.d2 = o;    o = up256(o + 4 * 16 * p2);
  L.d1 = o;    o = up256(o + 4 * 8 * p1);
  L.dlog = o;  o = up256(o + 4 * p3);
  // weight-gradient segments: (sample, output row, kSeg columns) per layer
  L.nseg3 = int(size_t(m) * (h - 6) * ((w - 6 + kSeg - 1) / kSeg));
  L.nseg2 = L.nseg3;   // layer 2's output grid is the head's
  L.nseg1 = int(size_t(m) * (h - 4) * ((w - 4 + kSeg - 1) / kSeg));
  L.nseg0 = int(size_t(m) * (h - 2) * ((w - 2 + kSeg - 1) / kSeg));
  const size_t parts = size_t(L.nseg3) * (32 + 1) + size_t(L.nseg2) * (4608 + 32) +
                       size_t(L.nseg1) * (1152 + 16) + size_t(L.nseg0) * (360 + 8);
  L.wpart = o; o = up256(o + 4 * parts);
  L.nlblk = int((p3 + kLossThreads - 1) / kLossThreads);
  L.lpart = o; o = up256(o + 8 * size_t(L.nlblk));
  L.tcpart = o; o = up256(o + 4 * (kTcPart0 + kTcPart1 + kTcPart2));
  L.hpart = o; o = up256(o + 4 * 33 * size_t(L.nlblk));
  const size_t img[5] = {ttc::FwdCfg<5, 8>::BIMG, ttc::FwdCfg<8, 16>::BIMG, ttc::FwdCfg<16, 32>::BIMG,
                         ttc::DgCfg<16, 32>::BIMG, ttc::DgCfg<8, 16>::BIMG};
  for (int k = 0; k < 5; ++k) {
    L.bimg[k] = o;
    o = up256(o + img[k]);
  }
  L.total = o;
  return L;
}

// ---------------------------------------------------------------- forward ---
// x: [*][CI][hi][wi] (sample idx[b] when idx, else b) -> y: [m][CO][hi-2][wi-2];
// blockIdx.y picks a group of CO / OG output channels (more threads per layer)
template <int CI, int CO, int OG>
__global__ void __launch_bounds__(128) conv3_fwd(const float* x, const int32_t* idx, int m, int hi,
                                                 int wi, const float* wk, const float* bias, float* y) {
  constexpr int CPG = CO / OG;
  // weights transposed to [in][ky][kx][out]: a position's output-channel
  // vector is contiguous (16-byte shared loads)
  __shared__ __align__(16) float sw[CO * CI * 9];
  __shared__ float sb[CO];
  for (int j = threadIdx.x; j < CO * CI * 9; j += blockDim.x)   // contiguous shared stores
    sw[j] = wk[(j % CO) * CI * 9 + j / CO];
  for (int i = threadIdx.x; i < CO; i += blockDim.x) sb[i] = bias[i];
  __syncthreads();
  const int ho = hi - 2, wo = wi - 2, o0 = blockIdx.y * CPG;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= int64_t(m) * ho * wo) return;
  const int ox = int(p % wo), oy = int((p / wo) % ho), b = int(p / (int64_t(wo) * ho));
  const int s = idx ? idx[b] : b;
  const float* xs = x + int64_t(s) * CI * hi * wi;
  float acc[CPG];
#pragma unroll
  for (int o = 0; o < CPG; ++o) acc[o] = 0.f;
  for (int c = 0; c < CI; ++c)
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float v = xs[(int64_t(c) * hi + oy + k / 3) * wi + ox + k % 3];
#pragma unroll
      for (int o = 0; o < CPG; ++o) acc[o] = fmaf(sw[(c * 9 + k) * CO + o0 + o], v, acc[o]);
    }
  float* ys = y + int64_t(b) * CO * ho * wo + int64_t(oy) * wo + ox;
#pragma unroll
  for (int o = 0; o < CPG; ++o) {
    const float v = acc[o] + sb[o0 + o];
    ys[int64_t(o0 + o) * ho * wo] = v * float(v > 0.f);   // y * (y > 0): -inf and NaN give NaN, as numpy
  }
}

// 1x1 head: logit = sum_c w3[c] * a3[c] + b3
__global__ void __launch_bounds__(128) head_fwd(const float* a3, int64_t plane, int m,
                                                const float* net, float* logit) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= int64_t(m) * plane) return;
  const int64_t b = p / plane, q = p % plane;
  const float* a = a3 + b * 32 * plane + q;
  float z = 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) z = fmaf(net[kOffW3 + c], a[c * plane], z);
  logit[p] = z + net[kOffB3];
}

// --------------------------------------------------------------- backward ---
// stable BCE terms (FP64) + dlogits (FP32); block partial sums of the terms
__global__ void __launch_bounds__(kLossThreads) loss_kernel(const float* logit, const float* tgt,
                                                            const int32_t* idx, int m, int64_t plane,
                                                            float* dlog, double* lpart) {
  const int64_t n = int64_t(m) * plane;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double term = 0.0;
  if (p < n) {
    const int64_t b = p / plane, q = p % plane;
    const float t = tgt[(idx ? int64_t(idx[b]) : b) * plane + q];
    const float z = logit[p];
    const double zd = double(z), td = double(t);
    term = add_rn(sub_rn(fmax(zd, 0.0), mul_rn(zd, td)), log1p(exp(-fabs(zd))));
    float sg;   // _sigmoid (edgenet.py:227-233), FP32
    if (z >= 0.f) {
      sg = 1.0f / (1.0f + expf(-z));
    } else {
      const float e = expf(z);
      sg = e / (1.0f + e);
    }
    dlog[p] = __fdiv_rn(__fsub_rn(sg, t), float(n));
  }
  __shared__ double red[kLossThreads];
  red[threadIdx.x] = term;
  __syncthreads();
  for (int o = kLossThreads / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) lpart[blockIdx.x] = red[0];
}

// mean loss (fixed order over blocks); flags a non-finite loss
__global__ void loss_final(const double* lpart, int nblk, int64_t n, double* out_loss, int32_t* flag) {
  __shared__ double red[256];
  double v = 0.0;
  for (int i = threadIdx.x; i < nblk; i += 256) v += lpart[i];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double loss = red[0] / double(n);
    *out_loss = loss;
    if (!isfinite(loss) && flag) *flag = 1;
  }
}

// the loss kernel fused with the 1x1 head's backward (tensor-core path): per
// position the BCE term, dlogit g, the head's input gradient
// d3[c] = g * w3[c] * (a3[c] > 0), and per block the partial head gradients
// sum g * a3[c] (r = c) and sum g (r = 32), summed in a fixed order (xor tree
// within each warp, then the warps in order); hpart[block][33] is reduced by
// tc_wgrad_reduce like the conv layers' partials
__global__ void __launch_bounds__(kLossThreads) loss_head_kernel(
    const float* __restrict__ logit, const float* __restrict__ tgt, const int32_t* __restrict__ idx, int m,
    int64_t plane, const float* __restrict__ a3, const float* __restrict__ net, float* __restrict__ dlog,
    float* __restrict__ d3, double* __restrict__ lpart, float* __restrict__ hpart) {
  const int64_t n = int64_t(m) * plane;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double term = 0.0;
  float g = 0.f, av[32];
  if (p < n) {
    const int64_t b = p / plane, q = p % plane;
    const float t = tgt[(idx ? int64_t(idx[b]) : b) * plane + q];
    const float z = logit[p];
    const float* a = a3 + b * 32 * plane + q;
#pragma unroll
    for (int c = 0; c < 32; ++c) av[c] = a[c * plane];
    const double zd = double(z), td = double(t);
    term = add_rn(sub_rn(fmax(zd, 0.0), mul_rn(zd, td)), log1p(exp(-fabs(zd))));
    float sg;   // _sigmoid (edgenet.py:227-233), FP32
    if (z >= 0.f) {
      sg = 1.0f / (1.0f + expf(-z));
    } else {
      const float e = expf(z);
      sg = e / (1.0f + e);
    }
    g = __fdiv_rn(__fsub_rn(sg, t), float(n));
    dlog[p] = g;
    float* d = d3 + b * 32 * plane + q;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      d[c * plane] = (g * net[kOffW3 + c]) * float(av[c] > 0.f);   // dx * mask (inf * 0 = NaN, as numpy)
  } else {
#pragma unroll
    for (int c = 0; c < 32; ++c) av[c] = 0.f;
  }
  __shared__ double red[kLossThreads];
  __shared__ float hred[kLossThreads / 32][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 33; ++c) {
    float v = c < 32 ? g * av[c] : g;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) hred[wid][c] = v;
  }
  red[threadIdx.x] = term;
  __syncthreads();
  for (int o = kLossThreads / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) lpart[blockIdx.x] = red[0];
  if (threadIdx.x < 33) {
    float v = hred[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < kLossThreads / 32; ++w) v += hred[w][threadIdx.x];
    hpart[int64_t(blockIdx.x) * 33 + threadIdx.x] = v;
  }
}

// head backward: da3 = g * w3 * (a3 > 0), one thread per (position, channel)
__global__ void __launch_bounds__(256) head_dgrad(const float* dlog, const float* a3, int64_t plane,
                                                  int m, const float* net, float* d3) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= int64_t(m) * 32 * plane) return;
  const int64_t q = t % plane, bc = t / plane;   // bc = b * 32 + c
  const int c = int(bc % 32);
  const float g = dlog[(bc / 32) * plane + q];
  d3[t] = (g * net[kOffW3 + c]) * float(a3[t] > 0.f);   // dx * mask (inf * 0 = NaN, as numpy)
}

// Weight / bias gradient partials of one segment (sample, output row, kSeg
// output columns) for a KxK valid correlation: part[seg][(o*CI + c)*K*K + k]
// and part[seg][CO*CI*K*K + o].  x: the layer input (sample idx[b] when idx).
template <int CI, int CO, int K>
__global__ void __launch_bounds__(256) conv_wgrad(const float* dy, const float* x, const int32_t* idx,
                                                  int m, int hi, int wi, float* part) {
  constexpr int NW = CO * CI * K * K;
  const int ho = hi - K + 1, wo = wi - K + 1;
  const int segs_x = (wo + kSeg - 1) / kSeg;
  const int seg = blockIdx.x;
  const int sx = seg % segs_x, oy = (seg / segs_x) % ho, b = seg / (segs_x * ho);
  const int x0 = sx * kSeg, len = min(kSeg, wo - x0);
  __shared__ float sdy[CO][kSeg];
  __shared__ float sx_[CI][K][kSeg + K - 1];
  const int s = idx ? idx[b] : b;
  for (int i = threadIdx.x; i < CO * kSeg; i += blockDim.x) {
    const int o = i / kSeg, j = i % kSeg;
    sdy[o][j] = j < len ? dy[((int64_t(b) * CO + o) * ho + oy) * wo + x0 + j] : 0.f;
  }
  for (int i = threadIdx.x; i < CI * K * (kSeg + K - 1); i += blockDim.x) {
    const int c = i / (K * (kSeg + K - 1)), r = (i / (kSeg + K - 1)) % K, j = i % (kSeg + K - 1);
    sx_[c][r][j] = j < len + K - 1 ? x[((int64_t(s) * CI + c) * hi + oy + r) * wi + x0 + j] : 0.f;
  }
  __syncthreads();
  float* out = part + size_t(seg) * (NW + CO);
  const int per = (NW + CO + gridDim.y - 1) / gridDim.y;   // this block's share of the weights
  const int w0 = blockIdx.y * per, w1 = min(NW + CO, w0 + per);
  for (int wi_ = w0 + threadIdx.x; wi_ < w1; wi_ += blockDim.x) {
    float acc = 0.f;
    if (wi_ < NW) {
      const int o = wi_ / (CI * K * K), c = (wi_ / (K * K)) % CI, k = wi_ % (K * K);
      const int ky = k / K, kx = k % K;
      for (int j = 0; j < len; ++j) acc = fmaf(sdy[o][j], sx_[c][ky][j + kx], acc);
    } else {
      const int o = wi_ - NW;
      for (int j = 0; j < len; ++j) acc += sdy[o][j];
    }
    out[wi_] = acc;
  }
}

// grads[i] = sum over segments of part[seg][i] in a fixed order: 8 groups of
// consecutive segments summed in parallel (threadIdx.y), then the 8 partial
// sums in group order -- deterministic, and 8x shorter dependent chains
constexpr int kRedGroups = 8;
__global__ void __launch_bounds__(32 * kRedGroups) wgrad_reduce(const float* part, int nseg, int nw,
                                                                float* gw, float* gb, int nb) {
  __shared__ float red[kRedGroups][32];
  const int i = blockIdx.x * 32 + threadIdx.x, g = threadIdx.y;
  const int per = (nseg + kRedGroups - 1) / kRedGroups;
  const int s0 = g * per, s1 = min(nseg, s0 + per);
  float acc = 0.f;
  if (i < nw + nb)
    for (int s = s0; s < s1; ++s) acc += part[size_t(s) * (nw + nb) + i];
  red[g][threadIdx.x] = acc;
  __syncthreads();
  if (g == 0 && i < nw + nb) {
    float v = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < kRedGroups; ++k) v += red[k][threadIdx.x];
    if (i < nw) gw[i] = v;
    else gb[i - nw] = v;
  }
}

void reduce_grads(const float* part, int nseg, int nw, float* gw, float* gb, int nb, cudaStream_t st) {
  wgrad_reduce<<<(nw + nb + 31) / 32, dim3(32, kRedGroups), 0, st>>>(part, nseg, nw, gw, gb, nb);
}

// dx[c][y][x] = sum_{o,ky,kx} dy[o][y-ky][x-kx] * w[o][c][ky][kx], times the
// ReLU mask of the input (x_in > 0); blockIdx.y picks a group of CI / IG input
// channels
template <int CI, int CO, int IG>
__global__ void __launch_bounds__(128) conv3_dgrad(const float* dy, const float* xin, int m, int hi,
                                                   int wi, const float* wk, float* dx) {
  constexpr int CPG = CI / IG;
  // weights as [out][ky][kx][in]: the input-channel vector of (o, ky, kx) is contiguous
  __shared__ __align__(16) float sw[CO * CI * 9];
  for (int j = threadIdx.x; j < CO * CI * 9; j += blockDim.x) {   // contiguous shared stores
    const int o = j / (9 * CI), k = (j / CI) % 9, c = j % CI;
    sw[j] = wk[(o * CI + c) * 9 + k];
  }
  __syncthreads();
  const int ho = hi - 2, wo = wi - 2, c0 = blockIdx.y * CPG;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= int64_t(m) * hi * wi) return;
  const int x = int(p % wi), y = int((p / wi) % hi), b = int(p / (int64_t(wi) * hi));
  float acc[CPG];
#pragma unroll
  for (int c = 0; c < CPG; ++c) acc[c] = 0.f;
  for (int o = 0; o < CO; ++o)
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int yy = y - k / 3, xx = x - k % 3;
      if (yy < 0 || yy >= ho || xx < 0 || xx >= wo) continue;
      const float g = dy[((int64_t(b) * CO + o) * ho + yy) * wo + xx];
#pragma unroll
      for (int c = 0; c < CPG; ++c) acc[c] = fmaf(g, sw[(o * 9 + k) * CI + c0 + c], acc[c]);
    }
#pragma unroll
  for (int c = 0; c < CPG; ++c) {
    const int64_t q = ((int64_t(b) * CI + c0 + c) * hi + y) * wi + x;
    dx[q] = acc[c] * float(xin[q] > 0.f);
  }
}

__global__ void sgd_kernel(float* w, const float* g, int n, float lr, const int32_t* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (flag && *flag)) return;
  w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
}

unsigned blocks(int64_t n, int t) { return unsigned((n + t - 1) / t); }

int check_dims(int m, int h, int w) {
  if (m < 1 || h < 7 || w < 7) return ECA_ERR_ARG;
  if (int64_t(m) * h * w > (int64_t(1) << 31) / 32) return ECA_ERR_UNSUPPORTED;
  return ECA_OK;
}

// the SIMT kernels above instead of the tensor-core ones (comparison runs)
bool train_simt() {
  static const bool v = [] {
    const char* e = std::getenv("ECA_TRAIN_SIMT");
    return e && *e && *e != '0';
  }();
  return v;
}

// Launch plan of a tensor-core training kernel on the current device: the
// dynamic shared memory to request and the CTAs one wave holds.  The block
// scheduler does not account TMEM: CTAs it co-locates -- of one kernel, or of
// kernels on concurrent streams -- must not ask for more than the SM's 512
// columns together (oversubscribing faults; measured).  So every kernel's
// shared memory is padded until its share of the SM's shared memory is at
// least its share of the TMEM columns: any set of CTAs that fits the shared
// memory then fits the TMEM.
struct TcPlan {
  int dyn, slots;
};
TcPlan tc_plan(const void* kern, int need, int cols) {
  struct Entry {
    const void* kern;
    int dev, need;
    TcPlan plan;
  };
  static std::mutex mu;
  static std::vector<Entry> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return {0, 0};
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.kern == kern && d.dev == dev && d.need == need) return d.plan;
  TcPlan p{0, 0};
  cudaFuncAttributes fa{};
  int sm_smem = 0, reserved = 0, optin_max = 0, sms = 0, per_sm = 0;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess &&
      cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&optin_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) {
    const int64_t share = (int64_t(cols) * sm_smem + 511) / 512;   // per-CTA footprint for `cols`
    int dyn = int(share - int64_t(fa.sharedSizeBytes) - reserved);
    if (dyn < need) dyn = need;
    if (dyn > optin_max - int(fa.sharedSizeBytes)) dyn = optin_max - int(fa.sharedSizeBytes);
    // CTAs per SM from the shared memory, registers and threads (the
    // occupancy API answered 1 for these kernels where ncu shows 2-3
    // resident; only the grid size depends on this, the TMEM bound comes
    // from the padding above)
    const int foot = dyn + int(fa.sharedSizeBytes) + reserved;
    const int regs = (fa.numRegs + 7) / 8 * 8 * ttc::kThreads;
    per_sm = sm_smem / foot;
    if (regs > 0 && 65536 / regs < per_sm) per_sm = 65536 / regs;
    if (2048 / ttc::kThreads < per_sm) per_sm = 2048 / ttc::kThreads;
    if (dyn >= need &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) == cudaSuccess &&
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess &&
        per_sm >= 1 && per_sm * cols <= 512)
      p = {dyn, per_sm * sms};
  }
  if (std::getenv("ECA_TRAIN_PLAN_LOG"))
    std::fprintf(stderr, "tc_plan %p need %d cols %d: static %zu dyn %d per_sm %d slots %d\n", kern, need, cols,
                 size_t(fa.sharedSizeBytes), p.dyn, per_sm, p.slots);
  done.push_back({kern, dev, need, p});
  return p;
}

template <int CI, int CO, bool kHead>
bool launch_fwd_tc(const float* x, const int32_t* idx, int m, int hi, int wi, const float* net,
                   const uint8_t* bimg, int ob, float* y, float* logit, cudaStream_t st,
                   const ttc::PackJob* pack = nullptr) {
  using C = ttc::FwdCfg<CI, CO>;
  auto k = ttc::tc_conv_fwd<CI, CO, kHead>;
  const TcPlan p = tc_plan(reinterpret_cast<const void*>(k), C::SMEM, C::COLS);
  if (!p.slots) return false;
  const int64_t tiles = int64_t(m) * (hi - 2) * ((wi - 2 + ttc::kTOut - 1) / ttc::kTOut);
  k<<<unsigned(tiles < p.slots ? tiles : p.slots), ttc::kThreads, p.dyn, st>>>(
      x, idx, m, hi, wi, bimg, net + ob, kHead ? net + kOffW3 : nullptr, y, logit,
      pack ? *pack : ttc::PackJob{}, pack ? 1 : 0);
  return true;
}

template <int CI, int CO>
bool launch_dgrad_tc(const float* dy, const float* xin, int m, int hi, int wi, const uint8_t* bimg,
                     float* dx, cudaStream_t st) {
  using C = ttc::DgCfg<CI, CO>;
  auto k = ttc::tc_conv_dgrad<CI, CO>;
  const TcPlan p = tc_plan(reinterpret_cast<const void*>(k), C::smem(hi - 2), C::COLS);
  if (!p.slots) return false;
  const int64_t cap = p.slots;
  const int64_t tiles = int64_t(m) * hi * ((wi + ttc::kTOut - 1) / ttc::kTOut);
  k<<<unsigned(tiles < cap ? tiles : cap), ttc::kThreads, p.dyn, st>>>(dy, xin, m, hi, wi, bimg,
                                                                     C::a_region(hi - 2), dx);
  return true;
}

// returns the number of partials (CTAs), 0 on failure
template <int CI, int CO, int KS>
int launch_wgrad_tc(const float* dy, const float* x, const int32_t* idx, int m, int hi, int wi, float* part,
                    cudaStream_t st) {
  using C = ttc::WgCfg<CI, CO, KS>;
  auto k = ttc::tc_conv_wgrad<CI, CO, KS>;
  const TcPlan p = tc_plan(reinterpret_cast<const void*>(k), C::SMEM, C::COLS);
  if (!p.slots) return 0;
  const int wo = wi - KS + 1;
  const int64_t units = int64_t(m) * (hi - KS + 1) * ((wo + ttc::kWgK - 1) / ttc::kWgK);
  int per_tile = p.slots / C::MT;   // one wave of (unit range, M tile) CTAs
  static const int force_g = [] {   // diagnostics: ECA_WG_CTAS=<weight-gradient CTAs per M tile>
    const char* e = std::getenv("ECA_WG_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  if (force_g > 0 && force_g < per_tile) per_tile = force_g;
  const int cap = per_tile < ttc::kWgCtas ? per_tile : ttc::kWgCtas;
  const int g = int(units < cap ? units : cap);
  k<<<dim3(g, C::MT), ttc::kThreads, p.dyn, st>>>(dy, x, idx, m, hi, wi, part);
  return g;
}

}  // namespace

extern "C" {

int eca_train_workspace_bytes(int m, int h, int w, int64_t* bytes) {
  if (!bytes) return ECA_ERR_ARG;
  if (const int rc = check_dims(m, h, w)) return rc;
  *bytes = int64_t(train_ws(m, h, w).total);
  return ECA_OK;
}

int eca_edgenet_forward(const float* x, const int32_t* index, int m, int h, int w, const float* net,
                        void* workspace, int64_t workspace_bytes, float* out_logits, void* stream) {
  if (const int rc = check_dims(m, h, w)) return rc;
  if (!x || !net || !workspace) return ECA_ERR_ARG;
  const TrainWs L = train_ws(m, h, w);
  if (workspace_bytes < int64_t(L.total)) return ECA_ERR_ARG;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  float* a1 = reinterpret_cast<float*>(ws + L.a1);
  float* a2 = reinterpret_cast<float*>(ws + L.a2);
  float* a3 = reinterpret_cast<float*>(ws + L.a3);
  float* logit = reinterpret_cast<float*>(ws + L.logit);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t plane = int64_t(h - 6) * (w - 6);
  if (!train_simt()) {   // tcgen05: three conv launches, the head fused into the last
    const ttc::PackJob P{net + kOffW0, net + kOffW1, net + kOffW2, ws + L.bimg[0], ws + L.bimg[1],
                         ws + L.bimg[2], ws + L.bimg[3], ws + L.bimg[4]};
    // layer 0 builds its own weight operand and packs the other four images
    if (!launch_fwd_tc<5, 8, false>(x, index, m, h, w, net, ws + L.bimg[0], kOffB0, a1, nullptr, st, &P) ||
        !launch_fwd_tc<8, 16, false>(a1, nullptr, m, h - 2, w - 2, net, ws + L.bimg[1], kOffB1, a2, nullptr,
                                     st) ||
        !launch_fwd_tc<16, 32, true>(a2, nullptr, m, h - 4, w - 4, net, ws + L.bimg[2], kOffB2, a3, logit, st))
      return ECA_ERR_CUDA;
  } else {
    conv3_fwd<5, 8, 1><<<dim3(blocks(int64_t(m) * (h - 2) * (w - 2), 128), 1), 128, 0, st>>>(
        x, index, m, h, w, net + kOffW0, net + kOffB0, a1);
    conv3_fwd<8, 16, 2><<<dim3(blocks(int64_t(m) * (h - 4) * (w - 4), 128), 2), 128, 0, st>>>(
        a1, nullptr, m, h - 2, w - 2, net + kOffW1, net + kOffB1, a2);
    conv3_fwd<16, 32, 4><<<dim3(blocks(int64_t(m) * (h - 6) * (w - 6), 128), 4), 128, 0, st>>>(
        a2, nullptr, m, h - 4, w - 4, net + kOffW2, net + kOffB2, a3);
    head_fwd<<<blocks(m * plane, 128), 128, 0, st>>>(a3, plane, m, net, logit);
  }
  if (out_logits)
    cudaMemcpyAsync(out_logits, logit, sizeof(float) * size_t(m * plane), cudaMemcpyDeviceToDevice, st);
  return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

int eca_edgenet_backward(const float* x, const float* targets, const int32_t* index, int m, int h,
                         int w, const float* net, void* workspace, int64_t workspace_bytes,
                         float* out_grads, double* out_loss, int32_t* diverged, void* stream) {
  if (const int rc = check_dims(m, h, w)) return rc;
  if (!x || !targets || !net || !workspace || !out_loss) return ECA_ERR_ARG;
  const TrainWs L = train_ws(m, h, w);
  if (workspace_bytes < int64_t(L.total)) return ECA_ERR_ARG;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  auto f = [&](size_t o) { return reinterpret_cast<float*>(ws + o); };
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t plane = int64_t(h - 6) * (w - 6), n = int64_t(m) * plane;
  double* lpart = reinterpret_cast<double*>(ws + L.lpart);
  const bool tc = out_grads && !train_simt();
  if (tc)
    loss_head_kernel<<<L.nlblk, kLossThreads, 0, st>>>(f(L.logit), targets, index, m, plane, f(L.a3), net,
                                                       f(L.dlog), f(L.d3), lpart, f(L.hpart));
  else
    loss_kernel<<<L.nlblk, kLossThreads, 0, st>>>(f(L.logit), targets, index, m, plane, f(L.dlog), lpart);
  if (!tc) loss_final<<<1, 256, 0, st>>>(lpart, L.nlblk, n, out_loss, diverged);   // (tc: in the reduction)
  if (!out_grads) return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;   // loss only
  if (tc) {   // tcgen05 weight / input gradients, one fixed-order reduction
    float* tp0 = f(L.tcpart);
    float* tp1 = tp0 + kTcPart0;
    float* tp2 = tp1 + kTcPart1;
    ttc::WgReduceJob R{};
    R.l[3] = {f(L.hpart), 33, 1, L.nlblk, out_grads + kOffW3, out_grads + kOffB3};
    R.l[2] = {tp2, ttc::WgCfg<16, 32, 3>::R, 32,
              launch_wgrad_tc<16, 32, 3>(f(L.d3), f(L.a2), nullptr, m, h - 4, w - 4, tp2, st),
              out_grads + kOffW2, out_grads + kOffB2};
    // the packed B operands of the forward on the same weights (backward
    // always follows its forward in this workspace)
    if (!launch_dgrad_tc<16, 32>(f(L.d3), f(L.a2), m, h - 4, w - 4, ws + L.bimg[3], f(L.d2), st))
      return ECA_ERR_CUDA;
    R.l[1] = {tp1, ttc::WgCfg<8, 16, 3>::R, 16,
              launch_wgrad_tc<8, 16, 3>(f(L.d2), f(L.a1), nullptr, m, h - 2, w - 2, tp1, st),
              out_grads + kOffW1, out_grads + kOffB1};
    if (!launch_dgrad_tc<8, 16>(f(L.d2), f(L.a1), m, h - 2, w - 2, ws + L.bimg[4], f(L.d1), st))
      return ECA_ERR_CUDA;
    R.l[0] = {tp0, ttc::WgCfg<5, 8, 3>::R, 8, launch_wgrad_tc<5, 8, 3>(f(L.d1), x, index, m, h, w, tp0, st),
              out_grads + kOffW0, out_grads + kOffB0};
    for (const auto& l : R.l)
      if (l.G == 0) return ECA_ERR_CUDA;
    R.lpart = lpart;
    R.nlblk = L.nlblk;
    R.n = n;
    R.out_loss = out_loss;
    R.flag = diverged;
    ttc::tc_wgrad_reduce<<<dim3(blocks(ttc::WgCfg<16, 32, 3>::R * 32, 32), 5), dim3(32, ttc::kRedG), 0, st>>>(R);
    return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
  }
  // head (1x1, 32 -> 1)
  float* part = f(L.wpart);
  float* p3 = part;
  float* p2 = p3 + size_t(L.nseg3) * 33;
  float* p1 = p2 + size_t(L.nseg2) * (4608 + 32);
  float* p0 = p1 + size_t(L.nseg1) * (1152 + 16);
  conv_wgrad<32, 1, 1><<<L.nseg3, 256, 0, st>>>(f(L.dlog), f(L.a3), nullptr, m, h - 6, w - 6, p3);
  reduce_grads(p3, L.nseg3, 32, out_grads + kOffW3, out_grads + kOffB3, 1, st);
  head_dgrad<<<blocks(n * 32, 256), 256, 0, st>>>(f(L.dlog), f(L.a3), plane, m, net, f(L.d3));
  // layer 2 (16 -> 32)
  conv_wgrad<16, 32, 3><<<dim3(L.nseg2, 4), 256, 0, st>>>(f(L.d3), f(L.a2), nullptr, m, h - 4, w - 4, p2);
  reduce_grads(p2, L.nseg2, 4608, out_grads + kOffW2, out_grads + kOffB2, 32, st);
  conv3_dgrad<16, 32, 4><<<dim3(blocks(int64_t(m) * (h - 4) * (w - 4), 128), 4), 128, 0, st>>>(
      f(L.d3), f(L.a2), m, h - 4, w - 4, net + kOffW2, f(L.d2));
  // layer 1 (8 -> 16)
  conv_wgrad<8, 16, 3><<<dim3(L.nseg1, 2), 256, 0, st>>>(f(L.d2), f(L.a1), nullptr, m, h - 2, w - 2, p1);
  reduce_grads(p1, L.nseg1, 1152, out_grads + kOffW1, out_grads + kOffB1, 16, st);
  conv3_dgrad<8, 16, 2><<<dim3(blocks(int64_t(m) * (h - 2) * (w - 2), 128), 2), 128, 0, st>>>(
      f(L.d2), f(L.a1), m, h - 2, w - 2, net + kOffW1, f(L.d1));
  // layer 0 (5 -> 8): weights only (the input gradient is not needed)
  conv_wgrad<5, 8, 3><<<L.nseg0, 256, 0, st>>>(f(L.d1), x, index, m, h, w, p0);
  reduce_grads(p0, L.nseg0, 360, out_grads + kOffW0, out_grads + kOffB0, 8, st);
  return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

int eca_sgd_step(float* net, const float* grads, float lr, const int32_t* diverged, void* stream) {
  if (!net || !grads) return ECA_ERR_ARG;
  sgd_kernel<<<blocks(kNetN, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(net, grads, kNetN, lr,
                                                                              diverged);
  return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

}  // extern "C"
