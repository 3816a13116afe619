// §8f-3: normalised-Hausdorff evaluation of content areas on the GPU
// (metrics.py:148-270), the step after the hot path.
//
//  boundary_kernel  one CTA per (sample, side): thread 0 builds the boundary
//                   pieces of disk ∩ [0,W-1]x[0,H-1] in FP64 exactly as
//                   metrics.py does (_arc_intervals :52-88, _edge_segments
//                   :91-118, _rect_corners :121-130), then all threads write
//                   the numpy.linspace samples (_sample_segment :133-138,
//                   _sample_arc :141-146): FP64 points + an FP32 copy.
//  box_kernel       bounding boxes of every 32-point tile of each point set
//                   (points in boundary order, so a tile is a short curve
//                   piece) and of every 16-tile supertile, in FP64.
//  nn_kernel        one thread per point of A: exact FP64 nearest distance in
//                   B by branch-and-bound -- nearest supertile / tile first,
//                   then only the (super)tiles whose box distance does not
//                   exceed the best so far -- and a stop as soon as the best
//                   falls to the directed maximum found so far (the point
//                   cannot raise it).  Directed maxima by atomic max.
//  finish_kernel    hausdorff = max over both directions (metrics.py:193-203).
//
// Box distances are FP64 lower bounds of every point distance in the box
// (each rounding step is monotone), so pruning never drops a nearer point:
// the result is exactly max_a min_b sqrt(dx*dx + dy*dy) in FP64 without
// contraction, cKDTree's p=2 distance, in any order.
#include <math.h>

#include "eca_common.cuh"

using namespace eca;

namespace {

constexpr int kMaxPieces = 12;   // <= 8 arcs (8 crossings) + 4 edge runs
constexpr int kTileP = 32;       // points per tile
constexpr int kSuper = 16;       // tiles per supertile
constexpr int kSuperP = kTileP * kSuper;
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
  double4* tbox;                 // [batch][2][cap / 32]: (xmin, ymin, xmax, ymax) per tile
  double4* sbox;                 // [batch][2][cap / 512] per supertile
  int32_t* count;                // [batch][2]
  unsigned long long* dmax;      // [batch][2]: directed maxima (non-negative double bits)
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
  }
}

// hausdorff() on caller point sets: side 0 = a, side 1 = b
__global__ void load_points_kernel(EvalJob E, const double2* a, int na, const double2* b, int nb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    E.count[0] = na;
    E.count[1] = nb;
  }
  if (i < na) E.pts[i] = a[i];
  if (i < nb) E.pts[E.cap + i] = b[i];
}

ECA_DEV double4 box_merge(double4 a, double4 b) {
  return make_double4(fmin(a.x, b.x), fmin(a.y, b.y), fmax(a.z, b.z), fmax(a.w, b.w));
}

// one CTA (16 warps) per supertile of one set: warp = tile, lane = point
__global__ void __launch_bounds__(kSuperP) box_kernel(EvalJob E) {
  const int set = blockIdx.y, st = blockIdx.x;
  if (E.out_status[set >> 1]) return;
  const int n = E.count[set];
  if (st * kSuperP >= n) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = st * kSuperP + threadIdx.x;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double4 bx = make_double4(inf, inf, -inf, -inf);
  if (i < n) {
    const double2 p = E.pts[size_t(set) * E.cap + i];
    bx = make_double4(p.x, p.y, p.x, p.y);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double4 q = make_double4(__shfl_xor_sync(kFull, bx.x, o), __shfl_xor_sync(kFull, bx.y, o),
                                   __shfl_xor_sync(kFull, bx.z, o), __shfl_xor_sync(kFull, bx.w, o));
    bx = box_merge(bx, q);
  }
  __shared__ double4 tb[kSuper];
  const int tiles = E.cap / kTileP;
  if (lane == 0) {
    tb[w] = bx;
    const int t = st * kSuper + w;
    if (t < tiles) E.tbox[size_t(set) * tiles + t] = bx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double4 sb = tb[0];
    for (int k = 1; k < kSuper; ++k) sb = box_merge(sb, tb[k]);
    E.sbox[size_t(set) * (E.cap / kSuperP) + st] = sb;
  }
}

ECA_DEV double dist2(double2 a, double2 b) {
  const double dx = sub_rn(a.x, b.x), dy = sub_rn(a.y, b.y);
  return add_rn(mul_rn(dx, dx), mul_rn(dy, dy));
}

// squared distance from a to the box: <= dist2(a, b) for every b in the box
ECA_DEV double box_d2(double2 a, double4 b) {
  const double dx = fmax(fmax(sub_rn(b.x, a.x), sub_rn(a.x, b.z)), 0.0);
  const double dy = fmax(fmax(sub_rn(b.y, a.y), sub_rn(a.y, b.w)), 0.0);
  return add_rn(mul_rn(dx, dx), mul_rn(dy, dy));
}

ECA_DEV double tile_min(const double2* B, int t, int nb, double2 a, double best) {
  const int k1 = min(nb, (t + 1) * kTileP);
  for (int k = t * kTileP; k < k1; ++k) best = fmin(best, dist2(a, B[k]));
  return best;
}

__global__ void __launch_bounds__(128) nn_kernel(EvalJob E) {
  const int b = blockIdx.z, d = blockIdx.y;
  if (E.out_status[b]) return;
  const size_t sa = size_t(b) * 2 + d, sb = size_t(b) * 2 + (d ^ 1);
  const int na = E.count[sa], nb = E.count[sb];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na || nb == 0) return;
  const double2 a = E.pts[sa * E.cap + i];
  const double2* B = E.pts + sb * E.cap;
  const int tiles = E.cap / kTileP, supers = E.cap / kSuperP;
  const double4* TB = E.tbox + sb * tiles;
  const double4* SB = E.sbox + sb * supers;
  const int nt = (nb + kTileP - 1) / kTileP, ns = (nb + kSuperP - 1) / kSuperP;
  // nearest supertile box, then its nearest tile box: the first upper bound
  int s0 = 0;
  double sd = INFINITY;
  for (int s = 0; s < ns; ++s) {
    const double v = box_d2(a, SB[s]);
    if (v < sd) { sd = v; s0 = s; }
  }
  int t0 = s0 * kSuper;
  double td = INFINITY;
  for (int t = s0 * kSuper; t < min(nt, (s0 + 1) * kSuper); ++t) {
    const double v = box_d2(a, TB[t]);
    if (v < td) { td = v; t0 = t; }
  }
  double best = tile_min(B, t0, nb, a, INFINITY);
  // the directed maximum so far is a lower bound of the result: a point whose
  // nearest distance is already below it cannot change the result
  const double lo = __longlong_as_double(
      static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(E.dmax + sa)));
  const double stop2 = __dmul_rd(lo, lo);
  if (best <= stop2) return;
  for (int s = 0; s < ns && best > stop2; ++s) {
    if (box_d2(a, SB[s]) > best) continue;
    for (int t = s * kSuper; t < min(nt, (s + 1) * kSuper); ++t)
      if (t != t0 && box_d2(a, TB[t]) <= best) best = tile_min(B, t, nb, a, best);
  }
  if (best > stop2) atomicMax(E.dmax + sa, static_cast<unsigned long long>(__double_as_longlong(__dsqrt_rn(best))));
}

__global__ void finish_kernel(EvalJob E) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= E.batch) return;
  if (E.out_status[b]) {
    E.out_hd[b] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  E.out_hd[b] = fmax(__longlong_as_double(static_cast<long long>(E.dmax[2 * b])),
                     __longlong_as_double(static_cast<long long>(E.dmax[2 * b + 1])));
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

struct WsLayout {
  size_t pts, tbox, sbox, count, dmax, total;
};

// cap: a multiple of kSuperP (so tiles and supertiles index without remainders)
WsLayout ws_layout(int batch, int cap) {
  WsLayout L;
  const size_t sets = size_t(batch) * 2;
  size_t o = 0;
  L.pts = o;   o = align256(o + sets * cap * sizeof(double2));
  L.tbox = o;  o = align256(o + sets * (cap / kTileP) * sizeof(double4));
  L.sbox = o;  o = align256(o + sets * (cap / kSuperP) * sizeof(double4));
  L.count = o; o = align256(o + sets * sizeof(int32_t));
  L.dmax = o;  o = align256(o + sets * sizeof(unsigned long long));
  L.total = o;
  return L;
}

int round_cap(int64_t n) {
  const int64_t c = (n + kSuperP - 1) / kSuperP * kSuperP;
  return c > (int64_t(1) << 30) ? -1 : int(c);
}

// metrics.boundary_points sample bound: the boundary of a convex subset of
// the rectangle is no longer than its perimeter; each of <= 12 pieces adds
// <= 2 samples beyond length / spacing
int boundary_cap(int width, int height, double spacing) {
  const double per = 2.0 * (double(width - 1) + double(height - 1));
  const double c = ceil(per / spacing) + 2.0 * kMaxPieces + 64.0;
  return c > 1.0e9 ? -1 : round_cap(int64_t(c));
}

EvalJob make_job(const EcaFitRecord* pred, const EcaFitRecord* truth, const int32_t* dims,
                 int batch, int cap, double spacing, void* ws, double* out_hd, int32_t* out_status) {
  const WsLayout L = ws_layout(batch, cap);
  uint8_t* w = static_cast<uint8_t*>(ws);
  EvalJob E{};
  E.area[0] = pred;
  E.area[1] = truth;
  E.dims = dims;
  E.batch = batch;
  E.cap = cap;
  E.spacing = spacing;
  E.pts = reinterpret_cast<double2*>(w + L.pts);
  E.tbox = reinterpret_cast<double4*>(w + L.tbox);
  E.sbox = reinterpret_cast<double4*>(w + L.sbox);
  E.count = reinterpret_cast<int32_t*>(w + L.count);
  E.dmax = reinterpret_cast<unsigned long long*>(w + L.dmax);
  E.out_hd = out_hd;
  E.out_status = out_status;
  return E;
}

int run_distance(const EvalJob& E, const WsLayout& L, void* ws, cudaStream_t st) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  cudaMemsetAsync(w + L.dmax, 0, L.total - L.dmax, st);
  box_kernel<<<dim3(E.cap / kSuperP, 2 * E.batch), kSuperP, 0, st>>>(E);
  nn_kernel<<<dim3((E.cap + 127) / 128, 2, E.batch), 128, 0, st>>>(E);
  finish_kernel<<<(E.batch + 127) / 128, 128, 0, st>>>(E);
  return cudaPeekAtLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA;
}

}  // namespace

extern "C" {

int eca_nh_workspace_bytes(int batch, int max_width, int max_height, double spacing,
                           int64_t* bytes) {
  if (batch < 0 || max_width < 2 || max_height < 2 || !(spacing > 0.0) || !bytes) return ECA_ERR_ARG;
  const int cap = boundary_cap(max_width, max_height, spacing);
  if (cap < 0) return ECA_ERR_UNSUPPORTED;
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
  if (cap < 0) return ECA_ERR_UNSUPPORTED;
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
  const int cap = round_cap(max_points);
  if (max_points < 1 || cap < 0 || !bytes) return ECA_ERR_ARG;
  *bytes = int64_t(ws_layout(1, cap).total);
  return ECA_OK;
}

int eca_hausdorff_points(const double* a, int na, const double* b, int nb, void* workspace,
                         int64_t workspace_bytes, double* out_hd, int32_t* out_status,
                         void* stream) {
  if (na < 1 || nb < 1 || !a || !b || !workspace || !out_hd || !out_status) return ECA_ERR_ARG;
  const int cap = round_cap(na > nb ? na : nb);
  if (cap < 0) return ECA_ERR_UNSUPPORTED;
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
