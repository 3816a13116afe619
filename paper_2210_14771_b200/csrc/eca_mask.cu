// K4 draw_mask and K5 crop: bandwidth-bound writers.
//
// Mask: closed-disk test of geometry.py:30-34 at every pixel centre,
// dx*dx + dy*dy <= r*r in FP64 without contraction.  The predicate is
// monotone in |fl(x - cx)|, so each row's inside set is one interval; a warp
// finds its exact FP64 end points (sqrt estimate + exact +-1 fix-up) and then
// streams the row as 16-byte stores.  FP64 work is O(rows), not O(pixels).
//
// Crop: crop_augment's rectangle (dataset.py:151-187) evaluated in FP64 on the
// device, then a coalesced row copy into a packed HWC buffer.
#include <cstdlib>

#include "eca_common.cuh"

using namespace eca;

#ifndef ECA_MASK_CS   // tuning knob: streaming (evict-first) stores for the mask body
#define ECA_MASK_CS 0
#endif
#ifndef ECA_MASK_BPS  // tuning knob: resident-CTA cap per SM of the mask grid
#define ECA_MASK_BPS 16
#endif

namespace {

ECA_DEV bool inside(double x, double cx, double dy2, double r2) {
  const double dx = sub_rn(x, cx);
  return add_rn(mul_rn(dx, dx), dy2) <= r2;
}

// exact [lo, hi] of inside columns of one row (lo > hi: empty)
ECA_DEV void row_interval(double cx, double dy2, double r2, int W, int& lo, int& hi) {
  const double rem = sub_rn(r2, dy2);
  const double hw = rem > 0.0 ? __dsqrt_rn(rem) : 0.0;
  double flo = ceil(sub_rn(cx, hw)), fhi = floor(add_rn(cx, hw));
  lo = flo < 0.0 ? 0 : (flo > double(W) ? W : int(flo));
  hi = fhi > double(W - 1) ? W - 1 : (fhi < -1.0 ? -1 : int(fhi));
  while (lo - 1 >= 0 && inside(double(lo - 1), cx, dy2, r2)) --lo;
  while (lo < W && lo <= hi && !inside(double(lo), cx, dy2, r2)) ++lo;
  while (hi + 1 <= W - 1 && inside(double(hi + 1), cx, dy2, r2)) ++hi;
  while (hi >= 0 && hi >= lo && !inside(double(hi), cx, dy2, r2)) --hi;
  if (lo > hi) {  // estimate missed a tiny interval: probe the columns next to cx
    const double c0 = floor(cx);
    for (int k = 0; k < 2; ++k) {
      const double xc = c0 + k;
      if (xc >= 0.0 && xc <= double(W - 1) && inside(xc, cx, dy2, r2)) {
        lo = hi = int(xc);
        while (lo - 1 >= 0 && inside(double(lo - 1), cx, dy2, r2)) --lo;
        while (hi + 1 <= W - 1 && inside(double(hi + 1), cx, dy2, r2)) ++hi;
        break;
      }
    }
  }
}

// 16 mask bytes of columns xb..xb+15 for the inside interval [lo, hi]
ECA_DEV uint4 mask16(int xb, int lo, int hi) {
  if (xb >= lo && xb + 15 <= hi) return make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  if (xb + 15 < lo || xb > hi) return make_uint4(0u, 0u, 0u, 0u);
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t word = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int x = xb + q * 4 + k;
      word |= uint32_t(x >= lo && x <= hi) << (8 * k);
    }
    w[q] = word;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// A warp takes 32 rows at a time: lane i finds row i's interval (the FP64
// chains run in parallel across lanes), then the warp streams the 32 rows as
// 16-byte stores; only the <= 2 chunks per row that straddle an interval end
// are built bytewise.
__global__ void __launch_bounds__(256) mask_kernel(const EcaFitRecord* fits, int batch, int H,
                                                   int W, uint8_t* out, int64_t fstride) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t n_rows = int64_t(batch) * H;
  for (int64_t r0 = warp * 32; r0 < n_rows; r0 += n_warps * 32) {
    int lo = 0, hi = W - 1;
    uintptr_t my_dst = 0;   // this lane's row start
    const int64_t my = r0 + lane;
    if (my < n_rows) {
      const int b = int(my / H);
      const int y = int(my - int64_t(b) * H);
      my_dst = reinterpret_cast<uintptr_t>(out + int64_t(b) * fstride + int64_t(y) * W);
      const EcaFitRecord f = fits[b];
      if (f.status == ECA_ACCEPTED) {
        const double dy = sub_rn(double(y), f.cy);
        row_interval(f.cx, mul_rn(dy, dy), mul_rn(f.r, f.r), W, lo, hi);
      }
    }
    const int nr = int(n_rows - r0 < 32 ? n_rows - r0 : 32);
    for (int i = 0; i < nr; ++i) {
      const int rlo = __shfl_sync(kFull, lo, i), rhi = __shfl_sync(kFull, hi, i);
      uint8_t* dst = reinterpret_cast<uint8_t*>(
          static_cast<uintptr_t>(__shfl_sync(kFull, static_cast<unsigned long long>(my_dst), i)));
      // head bytes up to 16-byte alignment, 16-byte body, tail bytes
      const int head = int((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15);
      const int h = head < W ? head : W;
      if (lane < h) dst[lane] = (lane >= rlo && lane <= rhi) ? 1 : 0;
      const int n16 = (W - h) >> 4;
      uint4* body = reinterpret_cast<uint4*>(dst + h);
#if ECA_MASK_CS
      for (int v = lane; v < n16; v += 32) __stcs(body + v, mask16(h + v * 16, rlo, rhi));
#else
      for (int v = lane; v < n16; v += 32) body[v] = mask16(h + v * 16, rlo, rhi);
#endif
      for (int x = h + n16 * 16 + lane; x < W; x += 32) dst[x] = (x >= rlo && x <= rhi) ? 1 : 0;
    }
  }
}

// Packed masks (frame stride H*W, W % 16 == 0, 16-byte aligned): the rows of
// the batch are one contiguous byte array.  A CTA takes kFlatRows rows at a
// time: one warp finds their intervals (FP64, as mask_kernel) into shared
// memory, then all its threads stream the rows' bytes as one span of 16-byte
// chunks (row of chunk c = c / (W / 16) by a multiply-high with the host's
// magic), so every warp writes long runs and no per-row loop or shuffle remains.
constexpr int kFlatRows = 32;
__global__ void __launch_bounds__(256) mask_kernel_flat(const EcaFitRecord* fits, int batch, int H, int W,
                                                        uint8_t* out, uint32_t cpr_magic) {
  __shared__ int2 ivl[kFlatRows];
  const int cpr = W >> 4;   // 16-byte chunks per row
  const int64_t n_rows = int64_t(batch) * H;
  for (int64_t r0 = int64_t(blockIdx.x) * kFlatRows; r0 < n_rows; r0 += int64_t(gridDim.x) * kFlatRows) {
    const int nr = int(n_rows - r0 < kFlatRows ? n_rows - r0 : kFlatRows);
    if (threadIdx.x < nr) {
      const int64_t my = r0 + threadIdx.x;
      const int b = int(my / H), y = int(my - int64_t(b) * H);
      int lo = 0, hi = W - 1;
      const EcaFitRecord f = fits[b];
      if (f.status == ECA_ACCEPTED) {
        const double dy = sub_rn(double(y), f.cy);
        row_interval(f.cx, mul_rn(dy, dy), mul_rn(f.r, f.r), W, lo, hi);
      }
      ivl[threadIdx.x] = make_int2(lo, hi);
    }
    __syncthreads();
    uint4* base = reinterpret_cast<uint4*>(out + r0 * W);
    const int n16 = nr * cpr;
    for (int c = threadIdx.x; c < n16; c += blockDim.x) {
      const int row = int(__umulhi(uint32_t(c), cpr_magic));   // c / cpr (c < 2^16 here)
      const int2 iv = ivl[row];
      base[c] = mask16((c - row * cpr) << 4, iv.x, iv.y);
    }
    __syncthreads();
  }
}

ECA_DEV bool contains_pt(double x, double y, double cx, double cy, double r) {
  const double dx = sub_rn(x, cx), dy = sub_rn(y, cy);
  return add_rn(mul_rn(dx, dx), mul_rn(dy, dy)) <= mul_rn(r, r);
}

__global__ void crop_bounds_kernel(const EcaFitRecord* fits, int batch, int H, int W,
                                   int32_t* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const EcaFitRecord f = fits[b];
  int4 res = make_int4(-1, -1, -1, -1);
  if (f.status == ECA_ACCEPTED) {
    const double cx = f.cx, cy = f.cy, r = f.r;
    const double xs[2] = {0.0, double(W - 1)}, ys[2] = {0.0, double(H - 1)};
    bool all_in = true;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) all_in = all_in && contains_pt(xs[i], ys[j], cx, cy, r);
    if (!all_in) {
      const double half = div_rn(r, __dsqrt_rn(2.0));
      const double capx = fmin(cx, sub_rn(double(W - 1), cx));
      const double capy = fmin(cy, sub_rn(double(H - 1), cy));
      double wx = fmin(half, capx), wy = fmin(half, capy);
      const double r2 = mul_rn(r, r);
      if (wx < half) {
        wy = fmin(capy, __dsqrt_rn(fmax(sub_rn(r2, mul_rn(wx, wx)), 0.0)));
      } else if (wy < half) {
        wx = fmin(capx, __dsqrt_rn(fmax(sub_rn(r2, mul_rn(wy, wy)), 0.0)));
      }
      double x0 = ceil(sub_rn(cx, wx)), x1 = floor(add_rn(cx, wx));
      double y0 = ceil(sub_rn(cy, wy)), y1 = floor(add_rn(cy, wy));
      x0 = fmax(x0, 0.0);
      y0 = fmax(y0, 0.0);
      x1 = fmin(x1, double(W - 1));
      y1 = fmin(y1, double(H - 1));
      if (!(x1 - x0 + 1.0 < 14.0 || y1 - y0 + 1.0 < 14.0))
        res = make_int4(int(x0), int(y0), int(x1), int(y1));
    }
  }
  reinterpret_cast<int4*>(out)[b] = res;
}

__global__ void __launch_bounds__(256) crop_copy_kernel(const uint8_t* frames, int64_t fstride,
                                                        int64_t rstride, const int32_t* bounds,
                                                        const int64_t* offs, uint8_t* out) {
  const int b = blockIdx.y;
  const int4 bd = reinterpret_cast<const int4*>(bounds)[b];
  if (bd.x < 0) return;
  const int rows = bd.w - bd.y + 1;
  const int rb = 3 * (bd.z - bd.x + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + warp; r < rows; r += gridDim.x * (blockDim.x >> 5)) {
    const uint8_t* src = frames + int64_t(b) * fstride + int64_t(bd.y + r) * rstride + 3 * bd.x;
    uint8_t* dst = out + offs[b] + int64_t(r) * rb;
    // Row = byte head up to a 16-B aligned dst, 16-B stores whose source bytes
    // come from aligned 32-bit loads joined by funnel shifts (the source row
    // starts at any byte: 3·x0), then a byte tail.
    const int head = min(rb, int((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
    if (lane < head) dst[lane] = __ldg(src + lane);
    const uint8_t* s = src + head;
    uint8_t* d = dst + head;
    const int m = rb - head, nv = m >> 4;
    const uintptr_t sa = reinterpret_cast<uintptr_t>(s);
    const unsigned sh = 8u * unsigned(sa & 3);
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sa & ~uintptr_t(3));
    for (int v = lane; v < nv; v += 32) {
      const uint32_t* p = sw + 4 * v;
      const uint32_t w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2), w3 = __ldg(p + 3);
      // p[4] holds needed bytes only when the source is unaligned (never past the row).
      const uint32_t w4 = sh ? __ldg(p + 4) : 0u;
      uint4 o;
      o.x = __funnelshift_r(w0, w1, sh);
      o.y = __funnelshift_r(w1, w2, sh);
      o.z = __funnelshift_r(w2, w3, sh);
      o.w = __funnelshift_r(w3, w4, sh);
      reinterpret_cast<uint4*>(d)[v] = o;
    }
    for (int i = nv * 16 + lane; i < m; i += 32) d[i] = __ldg(s + i);
  }
}

// ECA_MASK_ROWS=1: always the per-row kernel (comparison runs)
bool getenv_mask_rows() {
  static const bool v = [] {
    const char* e = std::getenv("ECA_MASK_ROWS");
    return e && *e == '1';
  }();
  return v;
}

}  // namespace

extern "C" int eca_draw_mask(const EcaFitRecord* fits, int batch, int height, int width,
                             uint8_t* out, int64_t out_frame_stride, void* stream) {
  ECA_RANGE("eca_draw_mask");
  if (batch < 0 || height < 1 || width < 1 || out_frame_stride < int64_t(height) * width)
    return ECA_ERR_ARG;
  if (batch == 0) return ECA_OK;
  if (!fits || !out) return ECA_ERR_ARG;
  const int64_t rows = int64_t(batch) * height;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool flat = !getenv_mask_rows() && width % 16 == 0 && out_frame_stride == int64_t(height) * width &&
                    (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (flat) {   // one contiguous span of rows
    const uint32_t cpr = uint32_t(width >> 4);
    const uint32_t magic = uint32_t((0xFFFFFFFFull + cpr) / cpr);   // ceil(2^32 / cpr): exact for c < 2^16
    const int64_t blocks64 = (rows + kFlatRows - 1) / kFlatRows;
    const int cap = 148 * ECA_MASK_BPS * 2;
    mask_kernel_flat<<<int(blocks64 < cap ? blocks64 : cap), 256, 0, st>>>(fits, batch, height, width, out,
                                                                           magic);
    return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
  }
  const int64_t blocks64 = (rows + 255) / 256;   // 8 warps x 32 rows per CTA pass
  const int blocks = int(blocks64 < 148 * ECA_MASK_BPS ? blocks64 : 148 * ECA_MASK_BPS);
  mask_kernel<<<blocks, 256, 0, st>>>(fits, batch, height, width, out, out_frame_stride);
  return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

extern "C" int eca_crop_bounds(const EcaFitRecord* fits, int batch, int height, int width,
                               int32_t* out_bounds, void* stream) {
  ECA_RANGE("eca_crop_bounds");
  if (batch < 0 || height < 1 || width < 1) return ECA_ERR_ARG;
  if (batch == 0) return ECA_OK;
  if (!fits || !out_bounds) return ECA_ERR_ARG;
  crop_bounds_kernel<<<(batch + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      fits, batch, height, width, out_bounds);
  return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

extern "C" int eca_crop_copy(const uint8_t* frames, int batch, int64_t frame_stride,
                             int64_t row_stride, const int32_t* bounds, const int64_t* out_offsets,
                             uint8_t* out, int max_rows, void* stream) {
  ECA_RANGE("eca_crop_copy");
  if (batch < 0 || max_rows < 0) return ECA_ERR_ARG;
  if (batch == 0 || max_rows == 0) return ECA_OK;
  if (!frames || !bounds || !out_offsets || !out) return ECA_ERR_ARG;
  const int gx = (max_rows + 7) / 8;
  crop_copy_kernel<<<dim3(gx, batch), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      frames, frame_stride, row_stride, bounds, out_offsets, out);
  return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}
