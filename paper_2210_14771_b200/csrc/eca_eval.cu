// §8f-3: normalised-Hausdorff evaluation of content areas on the GPU
// (metrics.py:148-270), the step after the hot path.
//
//  boundary_kernel  one CTA per (sample, side): thread 0 builds the boundary
//                   pieces of disk ∩ [0,W-1]x[0,H-1] in FP64 exactly as
//                   metrics.py does (_arc_intervals :52-88, _edge_segments
//                   :91-118, _rect_corners :121-130), then all threads write
//                   the numpy.linspace samples (_sample_segment :133-138,
//                   _sample_arc :141-146): FP64 points + an FP32 copy.
//  near32_kernel    FP32 brute force, one thread per two points of A, B
//                   staged through shared memory in tiles: per point of A the
//                   tile holding its (approximate) nearest neighbour in B, and
//                   the point of A with the largest approximate distance.
//  seed_kernel      one warp per (sample, direction): that point's exact FP64
//                   nearest distance L, a lower bound of the directed distance.
//  exact_kernel     per point of A, an FP64 scan of B starting at its FP32
//                   nearest tile that stops at the first distance <= L (the
//                   point cannot raise the maximum); points that never get
//                   there are exact minima above L -> atomic max.
//  finish_kernel    hausdorff = max over both directions (metrics.py:193-203).
//
// The result is exact by construction (the FP32 pass only orders the work):
// distances are sqrt(dx*dx + dy*dy) in FP64 without contraction, cKDTree's
// p=2 distance; the minimum over B and the maximum over A are order-free.
#include <math.h>

#include "eca_common.cuh"

using namespace eca;

namespace {

constexpr int kMaxPieces = 12;   // <= 8 arcs (8 crossings) + 4 edge runs
constexpr int kTile = 512;       // B points per shared-memory tile
constexpr int kNearThreads = 256;
constexpr double kTwoPi = 6.283185307179586;   // 2.0 * math.pi
constexpr double kPi = 3.141592653589793;

struct Piece {
  int arc;                     // 1: arc (a = t0, b = t1), 0: segment p0 -> p1
  double a, b, c, d;           // arc: t0, t1; segment: p0x, p0y, p1x, p1y
  int n;                       // linspace intervals (n + 1 samples)
};

struct EvalJob {
  const EcaFitRecord* area[2];   // [0] predictions, [1] truths
  const int32_t* dims;           // [batch][2] width, height (null: W0 x H0)
  int W0, H0;
  int batch, cap;
  double spacing;
  double2* pts;                  // [batch][2][cap]
  float2* pts32;                 // [batch][2][cap] (null: boundary_points only)
  int32_t* count;                // [batch][2]
  uint16_t* near_tile;           // [batch][2][cap]: FP32-nearest tile of B
  unsigned long long* far32;     // [batch][2]: (FP32 distance bits << 32) | point index
  double* seed;                  // [batch][2]: exact nearest distance of that point
  unsigned long long* dmax;      // [batch][2]: exact directed maxima above seed (double bits)
  double* out_hd;                // [batch]
  int32_t* out_status;           // [batch]: bit0 prediction empty, bit1 truth empty, bit2 overflow
};

ECA_DEV double py_mod_2pi(double v) {   // Python float % (2*pi)
  double m = fmod(v, kTwoPi);
  if (m != 0.0) {
    if (m < 0.0) m = add_rn(m, kTwoPi);
  } else {
    m = 0.0;
  }
  return m;
}

ECA_DEV bool arc_inside(double cx, double cy, double r, double t, double xhi, double yhi) {
  const double x = add_rn(cx, mul_rn(r, cos(t)));
  const double y = add_rn(cy, mul_rn(r, sin(t)));
  return 0.0 <= x && x <= xhi && 0.0 <= y && y <= yhi;
}

ECA_DEV int n_samples(double length, double spacing) {   // max(1, ceil(length / spacing))
  const double q = ceil(div_rn(length, spacing));
  return q < 1.0 ? 1 : int(q);
}

// metrics.boundary_points: pieces in the reference's order (arcs, then edge runs)
ECA_DEV int build_pieces(const EcaFitRecord& rec, int W, int H, double spacing, Piece* pc) {
  const double xhi = double(W - 1), yhi = double(H - 1);
  int np = 0;
  auto seg = [&](double x0, double y0, double x1, double y1) {
    Piece& p = pc[np++];
    p.arc = 0;
    p.a = x0; p.b = y0; p.c = x1; p.d = y1;
    p.n = n_samples(hypot(sub_rn(x1, x0), sub_rn(y1, y0)), spacing);
  };
  if (rec.status != ECA_ACCEPTED) {   // as_circle -> None: the rectangle perimeter
    seg(0.0, 0.0, xhi, 0.0);
    seg(xhi, 0.0, xhi, yhi);
    seg(xhi, yhi, 0.0, yhi);
    seg(0.0, yhi, 0.0, 0.0);
    return np;
  }
  const double cx = rec.cx, cy = rec.cy, r = rec.r;
  // _arc_intervals
  double cr[8];
  int nc = 0;
  const double xb[2] = {0.0, xhi}, yb[2] = {0.0, yhi};
  for (int k = 0; k < 2; ++k) {
    const double c = div_rn(sub_rn(xb[k], cx), r);
    if (-1.0 <= c && c <= 1.0) {
      const double t = acos(c);
      cr[nc++] = t;
      cr[nc++] = sub_rn(kTwoPi, t);
    }
  }
  for (int k = 0; k < 2; ++k) {
    const double s = div_rn(sub_rn(yb[k], cy), r);
    if (-1.0 <= s && s <= 1.0) {
      const double t = asin(s);
      cr[nc++] = py_mod_2pi(t);
      cr[nc++] = py_mod_2pi(sub_rn(kPi, t));
    }
  }
  if (nc == 0) {
    if (arc_inside(cx, cy, r, 0.0, xhi, yhi)) {
      Piece& p = pc[np++];
      p.arc = 1;
      p.a = 0.0; p.b = kTwoPi;
      p.n = n_samples(mul_rn(r, kTwoPi), spacing);
    }
  } else {
    // sorted(set(crossings)): insertion sort, then drop exact duplicates
    for (int i = 1; i < nc; ++i)
      for (int j = i; j > 0 && cr[j] < cr[j - 1]; --j) {
        const double t = cr[j]; cr[j] = cr[j - 1]; cr[j - 1] = t;
      }
    int nu = 0;
    for (int i = 0; i < nc; ++i)
      if (nu == 0 || cr[i] != cr[nu - 1]) cr[nu++] = cr[i];
    for (int k = 0; k < nu; ++k) {
      const double t0 = cr[k];
      double t1 = cr[(k + 1) % nu];
      if (k + 1 == nu) t1 = add_rn(t1, kTwoPi);
      if (sub_rn(t1, t0) <= 1e-12) continue;
      if (arc_inside(cx, cy, r, div_rn(add_rn(t0, t1), 2.0), xhi, yhi)) {
        Piece& p = pc[np++];
        p.arc = 1;
        p.a = t0; p.b = t1;
        p.n = n_samples(mul_rn(r, sub_rn(t1, t0)), spacing);
      }
    }
  }
  // _edge_segments: (fixed, lo, hi, horizontal) per rectangle edge
  const double fx[4] = {0.0, yhi, 0.0, xhi}, fh[4] = {xhi, xhi, yhi, yhi};
  for (int e = 0; e < 4; ++e) {
    const bool horiz = e < 2;
    const double off = sub_rn(fx[e], horiz ? cy : cx);
    const double rad2 = sub_rn(mul_rn(r, r), mul_rn(off, off));
    if (rad2 < 0.0) continue;
    const double half = __dsqrt_rn(rad2);
    const double mid = horiz ? cx : cy;
    const double a = fmax(0.0, sub_rn(mid, half)), b = fmin(fh[e], add_rn(mid, half));
    if (b <= a) continue;
    if (horiz) seg(a, fx[e], b, fx[e]);
    else seg(fx[e], a, fx[e], b);
  }
  return np;
}

// np.linspace(start, stop, n + 1)[i]: i * ((stop - start) / n) + start, last = stop
ECA_DEV double linspace_at(double start, double stop, int n, int i) {
  if (i == n) return stop;
  const double step = div_rn(sub_rn(stop, start), double(n));
  if (step == 0.0) return add_rn(mul_rn(div_rn(double(i), double(n)), sub_rn(stop, start)), start);
  return add_rn(mul_rn(double(i), step), start);
}

__global__ void __launch_bounds__(256) boundary_kernel(EvalJob E) {
  const int b = blockIdx.x, side = blockIdx.y;
  __shared__ Piece pc[kMaxPieces];
  __shared__ int start[kMaxPieces + 1];
  __shared__ int np_s;
  const int W = E.dims ? E.dims[2 * b] : E.W0, H = E.dims ? E.dims[2 * b + 1] : E.H0;
  const size_t set = size_t(b) * 2 + side;
  if (threadIdx.x == 0) {
    const int np = build_pieces(E.area[side][b], W, H, E.spacing, pc);
    int tot = 0;
    for (int k = 0; k < np; ++k) {
      start[k] = tot;
      tot += pc[k].n + 1;
    }
    start[np] = tot;
    np_s = np;
    int st = 0;
    if (tot == 0) st = 1 << side;
    if (tot > E.cap) st = 4;
    if (st && E.out_status) atomicOr(E.out_status + b, st);
    E.count[set] = tot;   // > cap: nothing written (boundary_points reports the size)
  }
  __syncthreads();
  const int np = np_s, tot = start[np];
  if (tot > E.cap) return;
  double2* out = E.pts + set * E.cap;
  float2* out32 = E.pts32 ? E.pts32 + set * E.cap : nullptr;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    int k = 0;
    while (k + 1 < np && start[k + 1] <= i) ++k;
    const Piece& p = pc[k];
    const int j = i - start[k];
    double x, y;
    if (p.arc) {
      const double t = linspace_at(p.a, p.b, p.n, j);
      const EcaFitRecord& rec = E.area[side][b];
      x = add_rn(rec.cx, mul_rn(rec.r, cos(t)));
      y = add_rn(rec.cy, mul_rn(rec.r, sin(t)));
    } else {
      const double t = linspace_at(0.0, 1.0, p.n, j);
      x = add_rn(p.a, mul_rn(t, sub_rn(p.c, p.a)));
      y = add_rn(p.b, mul_rn(t, sub_rn(p.d, p.b)));
    }
    out[i] = make_double2(x, y);
    if (out32) out32[i] = make_float2(float(x), float(y));
  }
}

// direction d: A = set d of the sample, B = the other set
__global__ void __launch_bounds__(kNearThreads) near32_kernel(EvalJob E) {
  const int b = blockIdx.z, d = blockIdx.y;
  const size_t sa = size_t(b) * 2 + d, sb = size_t(b) * 2 + (d ^ 1);
  if (E.out_status[b]) return;
  const int na = E.count[sa], nb = E.count[sb];
  const int i0 = blockIdx.x * 2 * kNearThreads + threadIdx.x, i1 = i0 + kNearThreads;
  if (blockIdx.x * 2 * kNearThreads >= na || nb == 0) return;
  __shared__ __align__(16) float2 tile[kTile];
  const float2* A = E.pts32 + sa * E.cap;
  const float2* B = E.pts32 + sb * E.cap;
  const float2 a0 = i0 < na ? A[i0] : make_float2(0.f, 0.f);
  const float2 a1 = i1 < na ? A[i1] : make_float2(0.f, 0.f);
  float m0 = INFINITY, m1 = INFINITY;
  int t0 = 0, t1 = 0;
  for (int base = 0; base < nb; base += kTile) {
    const int n = min(kTile, nb - base);
    __syncthreads();
    for (int k = threadIdx.x; k < kTile; k += blockDim.x)
      tile[k] = k < n ? B[base + k] : B[base];   // pad with a duplicate point
    __syncthreads();
    float p0 = INFINITY, p1 = INFINITY;
    const float4* t4 = reinterpret_cast<const float4*>(tile);
#pragma unroll 8
    for (int k = 0; k < kTile / 2; ++k) {
      const float4 q = t4[k];
      float dx = a0.x - q.x, dy = a0.y - q.y;
      p0 = fminf(p0, fmaf(dy, dy, dx * dx));
      dx = a0.x - q.z; dy = a0.y - q.w;
      p0 = fminf(p0, fmaf(dy, dy, dx * dx));
      dx = a1.x - q.x; dy = a1.y - q.y;
      p1 = fminf(p1, fmaf(dy, dy, dx * dx));
      dx = a1.x - q.z; dy = a1.y - q.w;
      p1 = fminf(p1, fmaf(dy, dy, dx * dx));
    }
    const int tix = base / kTile;
    if (p0 < m0) { m0 = p0; t0 = tix; }
    if (p1 < m1) { m1 = p1; t1 = tix; }
  }
  uint16_t* nt = E.near_tile + sa * E.cap;
  unsigned long long key = 0;
  if (i0 < na) {
    nt[i0] = uint16_t(t0);
    key = (uint64_t(__float_as_uint(m0)) << 32) | uint32_t(i0);
  }
  if (i1 < na) {
    nt[i1] = uint16_t(t1);
    const unsigned long long k1 = (uint64_t(__float_as_uint(m1)) << 32) | uint32_t(i1);
    key = k1 > key ? k1 : key;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(kFull, key, o);
    key = v > key ? v : key;
  }
  if ((threadIdx.x & 31) == 0 && key) atomicMax(E.far32 + sa, key);
}

// hausdorff() on caller point sets: side 0 = a, side 1 = b
__global__ void load_points_kernel(EvalJob E, const double2* a, int na, const double2* b, int nb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    E.count[0] = na;
    E.count[1] = nb;
  }
  if (i < na) {
    E.pts[i] = a[i];
    E.pts32[i] = make_float2(float(a[i].x), float(a[i].y));
  }
  if (i < nb) {
    E.pts[E.cap + i] = b[i];
    E.pts32[E.cap + i] = make_float2(float(b[i].x), float(b[i].y));
  }
}

ECA_DEV double dist2(double2 a, double2 b) {
  const double dx = sub_rn(a.x, b.x), dy = sub_rn(a.y, b.y);
  return add_rn(mul_rn(dx, dx), mul_rn(dy, dy));
}

// one warp per (sample, direction): exact nearest distance of the FP32-farthest point
__global__ void __launch_bounds__(128) seed_kernel(EvalJob E) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= 2 * E.batch || E.out_status[w >> 1]) return;
  const int na = E.count[w], nb = E.count[w ^ 1];
  if (na == 0 || nb == 0) return;
  const int ia = int(uint32_t(E.far32[w] & 0xffffffffull));
  const double2 a = E.pts[size_t(w) * E.cap + ia];
  const double2* B = E.pts + size_t(w ^ 1) * E.cap;
  double m = INFINITY;
  for (int k = lane; k < nb; k += 32) m = fmin(m, dist2(a, B[k]));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(kFull, m, o));
  if (lane == 0) E.seed[w] = __dsqrt_rn(m);
}

__global__ void __launch_bounds__(256) exact_kernel(EvalJob E) {
  const int b = blockIdx.z, d = blockIdx.y;
  const size_t sa = size_t(b) * 2 + d, sb = size_t(b) * 2 + (d ^ 1);
  if (E.out_status[b]) return;
  const int na = E.count[sa], nb = E.count[sb];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na || nb == 0) return;
  const double L = E.seed[sa];
  const double2 a = E.pts[sa * E.cap + i];
  const double2* B = E.pts + sb * E.cap;
  const int first = int(E.near_tile[sa * E.cap + i]) * kTile;
  // m <= fl_down(L*L) <= L^2 implies sqrt_rn(m) <= L: this point cannot raise the maximum
  const double stop2 = __dmul_rd(L, L);
  double m = INFINITY;
  // scan B from the FP32-nearest tile, wrapping, until a distance <= L
  for (int s = 0; s < nb; ++s) {
    int k = first + s;
    if (k >= nb) k -= nb;
    m = fmin(m, dist2(a, B[k]));
    if (m <= stop2) return;
  }
  const double dm = __dsqrt_rn(m);
  if (dm > L) atomicMax(E.dmax + sa, __double_as_longlong(dm));
}

__global__ void finish_kernel(EvalJob E) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= E.batch) return;
  if (E.out_status[b]) {
    E.out_hd[b] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double h = 0.0;
  for (int d = 0; d < 2; ++d) {
    const size_t s = size_t(b) * 2 + d;
    h = fmax(h, fmax(E.seed[s], __longlong_as_double(E.dmax[s])));
  }
  E.out_hd[b] = h;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

struct WsLayout {
  size_t pts, pts32, count, near_tile, far32, seed, dmax, total;
};

WsLayout ws_layout(int batch, int cap) {
  WsLayout L;
  const size_t sets = size_t(batch) * 2;
  size_t o = 0;
  L.pts = o;       o = align256(o + sets * cap * sizeof(double2));
  L.pts32 = o;     o = align256(o + sets * cap * sizeof(float2));
  L.near_tile = o; o = align256(o + sets * cap * sizeof(uint16_t));
  L.count = o;     o = align256(o + sets * sizeof(int32_t));
  L.far32 = o;     o = align256(o + sets * sizeof(unsigned long long));
  L.seed = o;      o = align256(o + sets * sizeof(double));
  L.dmax = o;      o = align256(o + sets * sizeof(unsigned long long));
  L.total = o;
  return L;
}

// metrics.boundary_points sample bound: the boundary of a convex subset of
// the rectangle is no longer than its perimeter; each of <= 12 pieces adds
// <= 2 samples beyond length / spacing
int boundary_cap(int width, int height, double spacing) {
  const double per = 2.0 * (double(width - 1) + double(height - 1));
  const double c = ceil(per / spacing) + 2.0 * kMaxPieces + 64.0;
  return c > 2.0e9 ? -1 : int(c);
}

EvalJob make_job(const EcaFitRecord* pred, const EcaFitRecord* truth, const int32_t* dims,
                 int batch, int cap, double spacing, void* ws, double* out_hd, int32_t* out_status) {
  const WsLayout L = ws_layout(batch, cap);
  uint8_t* w = static_cast<uint8_t*>(ws);
  EvalJob E;
  E.area[0] = pred;
  E.area[1] = truth;
  E.dims = dims;
  E.batch = batch;
  E.cap = cap;
  E.spacing = spacing;
  E.pts = reinterpret_cast<double2*>(w + L.pts);
  E.pts32 = reinterpret_cast<float2*>(w + L.pts32);
  E.count = reinterpret_cast<int32_t*>(w + L.count);
  E.near_tile = reinterpret_cast<uint16_t*>(w + L.near_tile);
  E.far32 = reinterpret_cast<unsigned long long*>(w + L.far32);
  E.seed = reinterpret_cast<double*>(w + L.seed);
  E.dmax = reinterpret_cast<unsigned long long*>(w + L.dmax);
  E.out_hd = out_hd;
  E.out_status = out_status;
  return E;
}

int run_distance(const EvalJob& E, const WsLayout& L, void* ws, cudaStream_t st) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  // far32, seed and dmax are contiguous: one memset clears the reduction state
  cudaMemsetAsync(w + L.far32, 0, L.total - L.far32, st);
  const int blocks_a = (E.cap + 2 * kNearThreads - 1) / (2 * kNearThreads);
  near32_kernel<<<dim3(blocks_a, 2, E.batch), kNearThreads, 0, st>>>(E);
  seed_kernel<<<(2 * E.batch * 32 + 127) / 128, 128, 0, st>>>(E);
  exact_kernel<<<dim3((E.cap + 255) / 256, 2, E.batch), 256, 0, st>>>(E);
  finish_kernel<<<(E.batch + 127) / 128, 128, 0, st>>>(E);
  return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

}  // namespace

extern "C" {

int eca_nh_workspace_bytes(int batch, int max_width, int max_height, double spacing,
                           int64_t* bytes) {
  if (batch < 0 || max_width < 2 || max_height < 2 || !(spacing > 0.0) || !bytes) return ECA_ERR_ARG;
  const int cap = boundary_cap(max_width, max_height, spacing);
  if (cap < 0 || cap > 65535 * kTile) return ECA_ERR_UNSUPPORTED;
  *bytes = int64_t(ws_layout(batch, cap).total);
  return ECA_OK;
}

int eca_area_hausdorff(const EcaFitRecord* pred, const EcaFitRecord* truth, const int32_t* dims,
                       int batch, int max_width, int max_height, double spacing, void* workspace,
                       int64_t workspace_bytes, double* out_hd, int32_t* out_status, void* stream) {
  if (batch < 0 || max_width < 2 || max_height < 2 || !(spacing > 0.0)) return ECA_ERR_ARG;
  if (batch == 0) return ECA_OK;
  if (!pred || !truth || !dims || !workspace || !out_hd || !out_status) return ECA_ERR_ARG;
  const int cap = boundary_cap(max_width, max_height, spacing);
  if (cap < 0 || cap > 65535 * kTile) return ECA_ERR_UNSUPPORTED;
  const WsLayout L = ws_layout(batch, cap);
  if (workspace_bytes < int64_t(L.total)) return ECA_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const EvalJob E = make_job(pred, truth, dims, batch, cap, spacing, workspace, out_hd, out_status);
  cudaMemsetAsync(out_status, 0, size_t(batch) * sizeof(int32_t), st);
  boundary_kernel<<<dim3(batch, 2), 256, 0, st>>>(E);
  return run_distance(E, L, workspace, st);
}

int eca_boundary_points(const EcaFitRecord* area, int width, int height, double spacing,
                        double* out_xy, int cap, int32_t* out_count, void* stream) {
  if (width < 2 || height < 2 || !(spacing > 0.0) || !area || !out_xy || !out_count || cap < 1)
    return ECA_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  EvalJob E{};
  E.area[0] = area;
  E.W0 = width;
  E.H0 = height;
  E.batch = 1;
  E.cap = cap;
  E.spacing = spacing;
  E.pts = reinterpret_cast<double2*>(out_xy);
  E.count = out_count;
  boundary_kernel<<<dim3(1, 1), 256, 0, st>>>(E);
  return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

int eca_hausdorff_workspace_bytes(int max_points, int64_t* bytes) {
  if (max_points < 1 || max_points > 65535 * kTile || !bytes) return ECA_ERR_ARG;
  *bytes = int64_t(ws_layout(1, max_points).total);
  return ECA_OK;
}

int eca_hausdorff_points(const double* a, int na, const double* b, int nb, void* workspace,
                         int64_t workspace_bytes, double* out_hd, int32_t* out_status,
                         void* stream) {
  if (na < 1 || nb < 1 || !a || !b || !workspace || !out_hd || !out_status) return ECA_ERR_ARG;
  const int cap = na > nb ? na : nb;
  if (cap > 65535 * kTile) return ECA_ERR_UNSUPPORTED;
  const WsLayout L = ws_layout(1, cap);
  if (workspace_bytes < int64_t(L.total)) return ECA_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  EvalJob E = make_job(nullptr, nullptr, nullptr, 1, cap, 1.0, workspace, out_hd, out_status);
  cudaMemsetAsync(out_status, 0, sizeof(int32_t), st);
  load_points_kernel<<<(cap + 255) / 256, 256, 0, st>>>(E, reinterpret_cast<const double2*>(a),
                                                         na, reinterpret_cast<const double2*>(b), nb);
  return run_distance(E, L, workspace, st);
}

}  // extern "C"
