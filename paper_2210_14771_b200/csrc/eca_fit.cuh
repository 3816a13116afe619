// K2: candidate filter + seeded RANSAC with iterated FP64 least squares.
//
// Restates fitting.py:39-230 in the reference's evaluation order: every FP64
// expression is written with explicit round-to-nearest intrinsics (no FMA
// contraction) so circumcircles, gates and LSQ systems see numpy's doubles.
// Only the moment sums (numpy: OpenBLAS dgemm) and the 3x3 solve (LAPACK
// gesv) reassociate; the survey measured that headroom at <=2.3e-13 px.
//
// Mapping (fit_warp, one warp per frame): LANE = hypothesis (32 attempts per
// pass), so a hypothesis' circle, inlier tests, moment sums and 3x3 solve live
// in one thread and need no shuffles.  Ties between hypotheses resolve to the
// lowest attempt index (fitting.py:222).
#pragma once

#include "eca_common.cuh"

namespace eca {

constexpr int kMom = 10;   // sx sy sz sxx sxy syy sxz syz count score

struct Circ {
  double cx, cy, r;
  bool alive;
};

// fitting.py:55-75 for one triplet of normalised points.
ECA_DEV Circ circumcircle(double ax, double ay, double bx, double by, double qx, double qy) {
  const double abx = sub_rn(bx, ax), aby = sub_rn(by, ay);
  const double acx = sub_rn(qx, ax), acy = sub_rn(qy, ay);
  const double det = sub_rn(mul_rn(abx, acy), mul_rn(aby, acx));
  const double scale = mul_rn(hypot(abx, aby), hypot(acx, acy));
  const bool valid = (scale > 0.0) && (fabs(det) > mul_rn(1e-9, scale));
  const double safe = valid ? det : 1.0;
  const double b2 = div_rn(add_rn(mul_rn(abx, abx), mul_rn(aby, aby)), 2.0);
  const double c2 = div_rn(add_rn(mul_rn(acx, acx), mul_rn(acy, acy)), 2.0);
  const double ux = div_rn(sub_rn(mul_rn(b2, acy), mul_rn(c2, aby)), safe);
  const double uy = div_rn(sub_rn(mul_rn(c2, abx), mul_rn(b2, acx)), safe);
  const double r = hypot(ux, uy);
  Circ c;
  c.cx = add_rn(ax, ux);
  c.cy = add_rn(ay, uy);
  c.r = r;
  c.alive = valid && isfinite(r) && (r > 0.0);
  return c;
}

// fitting.py:89-124 given the masked moments; returns ok and the new circle.
ECA_DEV bool lsq_solve(const double* mo, int cnt, double& a_out, double& b_out, double& r_out) {
  const double sx = mo[0], sy = mo[1], sz = mo[2], sxx = mo[3], sxy = mo[4], syy = mo[5];
  const double sxz = mo[6], syz = mo[7];
  const double n = double(cnt);
  double m[3][3] = {{mul_rn(4.0, sxx), mul_rn(4.0, sxy), mul_rn(2.0, sx)},
                    {mul_rn(4.0, sxy), mul_rn(4.0, syy), mul_rn(2.0, sy)},
                    {mul_rn(2.0, sx), mul_rn(2.0, sy), n}};
  double v[3] = {mul_rn(2.0, sxz), mul_rn(2.0, syz), sz};
  const double t1 = sub_rn(mul_rn(m[1][1], m[2][2]), mul_rn(m[1][2], m[1][2]));
  const double t2 = sub_rn(mul_rn(m[0][1], m[2][2]), mul_rn(m[1][2], m[0][2]));
  const double t3 = sub_rn(mul_rn(m[0][1], m[1][2]), mul_rn(m[1][1], m[0][2]));
  const double det = add_rn(sub_rn(mul_rn(m[0][0], t1), mul_rn(m[0][1], t2)), mul_rn(m[0][2], t3));
  const double nn = n > 1.0 ? n : 1.0;
  const bool ok = (cnt >= 3) && isfinite(det) &&
                  (fabs(det) > mul_rn(1e-12, mul_rn(mul_rn(nn, nn), nn)));
  if (!ok) return false;
  // LU with partial pivoting (dgetrf2/dgetrs order: reciprocal-scaled
  // multipliers, forward then backward substitution).  Rows are exchanged
  // with register selects (constant indices only: no local-memory array).
  // column 0: pivot = first row of largest |m[i][0]|
  {
    const double a0 = fabs(m[0][0]), a1 = fabs(m[1][0]), a2 = fabs(m[2][0]);
    const bool p1 = a1 > a0;
    const int piv = (a2 > (p1 ? a1 : a0)) ? 2 : (p1 ? 1 : 0);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double r0 = m[0][j], r1 = m[1][j], r2 = m[2][j];
      m[0][j] = piv == 1 ? r1 : (piv == 2 ? r2 : r0);
      m[1][j] = piv == 1 ? r0 : r1;
      m[2][j] = piv == 2 ? r0 : r2;
    }
    const double v0 = v[0], v1 = v[1], v2 = v[2];
    v[0] = piv == 1 ? v1 : (piv == 2 ? v2 : v0);
    v[1] = piv == 1 ? v0 : v1;
    v[2] = piv == 2 ? v0 : v2;
    const double rp = __drcp_rn(m[0][0]);   // = 1.0 / pivot, correctly rounded
#pragma unroll
    for (int i = 1; i < 3; ++i) {
      m[i][0] = mul_rn(m[i][0], rp);
#pragma unroll
      for (int j = 1; j < 3; ++j) m[i][j] = sub_rn(m[i][j], mul_rn(m[i][0], m[0][j]));
    }
  }
  // column 1: rows 1 and 2
  {
    const bool sw = fabs(m[2][1]) > fabs(m[1][1]);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double r1 = m[1][j], r2 = m[2][j];
      m[1][j] = sw ? r2 : r1;
      m[2][j] = sw ? r1 : r2;
    }
    const double v1 = v[1], v2 = v[2];
    v[1] = sw ? v2 : v1;
    v[2] = sw ? v1 : v2;
    const double rp = __drcp_rn(m[1][1]);
    m[2][1] = mul_rn(m[2][1], rp);
    m[2][2] = sub_rn(m[2][2], mul_rn(m[2][1], m[1][2]));
  }
  const double y0 = v[0];
  const double y1 = sub_rn(v[1], mul_rn(m[1][0], y0));
  const double y2 = sub_rn(sub_rn(v[2], mul_rn(m[2][0], y0)), mul_rn(m[2][1], y1));
  const double c = div_rn(y2, m[2][2]);
  const double b = div_rn(sub_rn(y1, mul_rn(m[1][2], c)), m[1][1]);
  const double a = div_rn(sub_rn(sub_rn(y0, mul_rn(m[0][1], b)), mul_rn(m[0][2], c)), m[0][0]);
  const double r2 = add_rn(add_rn(c, mul_rn(a, a)), mul_rn(b, b));
  if (!(isfinite(r2) && r2 > 0.0)) return false;
  a_out = a;
  b_out = b;
  r_out = __dsqrt_rn(r2);
  return true;
}

// lexicographic rank -> 3-combination of range(n) (itertools.combinations order)
ECA_DEV void unrank3(int a, int n, int& i, int& j, int& k) {
  i = 0;
  for (;;) {
    const int c = (n - 1 - i) * (n - 2 - i) / 2;
    if (a < c) break;
    a -= c;
    ++i;
  }
  j = i + 1;
  for (;;) {
    const int c = n - 1 - j;
    if (a < c) break;
    a -= c;
    ++j;
  }
  k = j + 1 + a;
}

// Inlier test of fitting.py:199/206 for one candidate.
ECA_DEV bool is_inlier(double x, double y, const Circ& c, double tol) {
  return fabs(sub_rn(hypot(sub_rn(x, c.cx), sub_rn(y, c.cy)), c.r)) <= tol;
}

// The same decision with a cheap squared-distance screen: points whose d^2 is
// outside a 1e-8 relative band around (r -/+ tol)^2 are decided without the
// hypot (rounding of d^2 and of hypot are ~1e-16 relative, so the screen can
// never disagree with is_inlier); only points in the band take the exact test.
struct Ring {
  double in_lo, in_hi, out_lo, out_hi;
};

ECA_DEV Ring ring_of(const Circ& c, double tol) {
  const double e = 1e-8;
  const double ro = c.r + tol, ri = c.r - tol;
  Ring g;
  g.in_hi = ro * ro * (1.0 - e);
  g.out_hi = ro * ro * (1.0 + e);
  if (ri > 1e-6 * c.r) {          // annulus: both edges screened
    g.in_lo = ri * ri * (1.0 + e);
    g.out_lo = ri * ri * (1.0 - e);
  } else if (ri < -1e-6 * c.r) {  // disk: no inner edge
    g.in_lo = -1.0;
    g.out_lo = -1.0;
  } else {                        // r ~ tol: inner edge ambiguous, test exactly
    g.in_lo = __longlong_as_double(0x7ff0000000000000LL);
    g.out_lo = -1.0;
  }
  return g;
}


// ---------------------------------------------------------------------------
// fit_warp: lane = hypothesis, each lane walks the whole candidate list; no CTA
// barriers.  Used by fit_kernel (one warp per frame) and by the fused strip
// kernel, where the warp that completes a frame fits it while the CTA's other
// warps keep scoring strips.
// Per-candidate moment terms (identical for every hypothesis, so computed
// once per frame in fitting.py's per-point order): x, y, z = x^2+y^2 and the
// products the masked least squares sums.
struct FitPt {
  double x, y, z, xx, xy, yy, xz, yz;
  float xf, yf;   // x, y rounded to FP32 (the inlier screen)
  double pad_;
};

struct FitScratchW {
  FitPt pt[2 * ECA_MAX_STRIPS];
  double ps[2 * ECA_MAX_STRIPS];
};

// The inlier screen in FP32 (the decisions of is_inlier, exactly): d^2 of a
// point to the lane's circle is formed from FP32 copies of the coordinates.
// With B >= every |coordinate| of the points and of the centre, that FP32 d^2
// is within 44 * 2^-24 * B^2 < 2.7e-6 B^2 of the exact d^2 (two roundings of
// the inputs and of each operation), so the FP64 ring thresholds are widened
// by E = 4e-6 B^2 and rounded outward to FP32: "in" / "out" there implies
// "in" / "out" of the FP64 screen (ring_of), the rest takes the exact test.
// FP32 runs at twice the FP64 rate with half the dependency latency.
struct RingF {
  float in_lo, in_hi, out_lo, out_hi, cx, cy;
};

ECA_DEV RingF ring_f(const Ring& g, const Circ& c, double bmax) {
  const double b = fmax(bmax, fmax(fabs(c.cx), fabs(c.cy)));
  const double e = 4e-6 * b * b;
  RingF f;
  f.in_hi = __double2float_rd(g.in_hi - e);
  f.in_lo = __double2float_ru(g.in_lo + e);
  f.out_hi = __double2float_ru(g.out_hi + e);
  f.out_lo = __double2float_rd(g.out_lo - e);
  f.cx = float(c.cx);
  f.cy = float(c.cy);
  return f;
}

ECA_DEV RingF ringf_dead() {   // matches no point
  RingF f;
  f.in_lo = 1.0f;
  f.in_hi = -1.0f;
  f.out_lo = -1.0f;
  f.out_hi = -1.0f;
  f.cx = f.cy = 0.0f;
  return f;
}

// Inlier bits of candidates k0 .. k0+kn-1 (kn <= 32) against the lane's
// circle: the FP32 d^2 screen for every candidate first, with no vote inside
// the loop, so consecutive candidates' chains overlap; the rare candidates in
// the screen's band then take the exact test (the decisions of is_inlier).
ECA_DEV uint32_t inlier_bits(const FitPt* pt, int k0, int kn, const Circ& c, const RingF& g,
                             double tol) {
  uint32_t in_m = 0, amb_m = 0;
#pragma unroll 8
  for (int j = 0; j < kn; ++j) {
    const float dx = pt[k0 + j].xf - g.cx, dy = pt[k0 + j].yf - g.cy;
    const float d2 = fmaf(dx, dx, dy * dy);
    const bool in = d2 <= g.in_hi && d2 >= g.in_lo;
    const bool amb = !in && !(d2 > g.out_hi || d2 < g.out_lo);
    in_m |= uint32_t(in) << j;
    amb_m |= uint32_t(amb) << j;
  }
  while (amb_m) {
    const int j = __ffs(amb_m) - 1;
    amb_m &= amb_m - 1u;
    if (is_inlier(pt[k0 + j].x, pt[k0 + j].y, c, tol)) in_m |= 1u << j;
  }
  return in_m;
}

ECA_DEV Ring ring_dead() {   // matches no point (hypothesis no longer alive)
  return Ring{1.0, -1.0, -1.0, -1.0};
}

#ifdef ECA_FIT_TIMES   // diagnostic builds: per-frame phase clocks (tools/fit_times.py)
__device__ unsigned long long g_fit_times[16 * 4096];
#define FIT_STAMP(k)                                                        \
  do {                                                                      \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 4096)                       \
      g_fit_times[16 * blockIdx.x + (k)] = clock64();                       \
  } while (0)
#else
#define FIT_STAMP(k) \
  do {               \
  } while (0)
#endif

// pt / ps: shared scratch for n_cand points (FitScratchW, or n_cand-sized).
// kCG: the candidates are in global memory, written by other CTAs of the same
// kernel (L2 loads); otherwise any memory this warp wrote (e.g. shared).
// the record store; ordered: every field, a system-scope fence, then the
// status word -- a host polling mapped pinned memory for the status sees the
// complete record (the single-frame latency path)
ECA_DEV void store_record(EcaFitRecord* out, const EcaFitRecord& rec, bool ordered) {
  if (!ordered) {
    *out = rec;
    return;
  }
  volatile EcaFitRecord* v = out;
  v->cx = rec.cx;
  v->cy = rec.cy;
  v->r = rec.r;
  v->score = rec.score;
  v->inliers = rec.inliers;
  __threadfence_system();
  v->status = rec.status;
}

template <bool kCG = true>
ECA_DEV void fit_warp(const int32_t* cand_x, const int32_t* cand_y, const double* cand_s,
                      int n_cand, const EcaParams& p, const int16_t* trip, int exhaustive,
                      FitPt* pt, double* ps, EcaFitRecord* out, bool ordered = false) {
  const int lane = threadIdx.x & 31;
  const int W = p.width, H = p.height;
  FIT_STAMP(0);
  int n = 0;
  double bmax = 0.0;   // largest |coordinate| of the kept points (the FP32 screen's margin)
  for (int base = 0; base < n_cand; base += 32) {   // filter_candidates, order-preserving
    const int i = base + lane;
    bool keep = false;
    int x = 0, y = 0;
    double s = 0.0;
    if (i < n_cand) {
      x = kCG ? __ldcg(cand_x + i) : cand_x[i];
      y = kCG ? __ldcg(cand_y + i) : cand_y[i];
      s = kCG ? __ldcg(cand_s + i) : cand_s[i];
      const int edge = min(min(x, W - 1 - x), min(y, H - 1 - y));
      keep = edge >= p.edge_margin_px && s >= p.min_point_score;
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    if (keep) {
      const int pos = n + __popc(bal & ((1u << lane) - 1u));
      FitPt q;
      q.x = div_rn(sub_rn(double(x), p.center_x), double(W));
      q.y = div_rn(sub_rn(double(y), p.center_y), double(W));
      q.z = add_rn(mul_rn(q.x, q.x), mul_rn(q.y, q.y));
      q.xx = mul_rn(q.x, q.x);
      q.xy = mul_rn(q.x, q.y);
      q.yy = mul_rn(q.y, q.y);
      q.xz = mul_rn(q.x, q.z);
      q.yz = mul_rn(q.y, q.z);
      q.xf = float(q.x);
      q.yf = float(q.y);
      q.pad_ = 0.0;
      bmax = fmax(bmax, fmax(fabs(q.x), fabs(q.y)));
      ECA_CHECK(pos < n_cand);
      pt[pos] = q;
      ps[pos] = s;
    }
    n += __popc(bal);
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) bmax = fmax(bmax, __shfl_xor_sync(kFull, bmax, d));
  __syncwarp();
  FIT_STAMP(1);
  if (n < 3) {
    if (lane == 0) store_record(out, EcaFitRecord{0.0, 0.0, 0.0, 0.0, 0, ECA_NO_CANDIDATES}, ordered);
    __syncwarp();
    return;
  }
  const int attempts = exhaustive ? n * (n - 1) * (n - 2) / 6 : p.ransac_attempts;
  const double tol = p.inlier_tol;
  double best_s = -1.0, bcx = 0.0, bcy = 0.0, br = 0.0;
  int best_inl = 0, any_live = 0, any_gated = 0;
  for (int c0 = 0; c0 < attempts; c0 += 32) {
    const int a = c0 + lane;
    Circ c{0.0, 0.0, 1.0, false};
    if (a < attempts) {
      int i0, i1, i2;
      if (exhaustive) {
        unrank3(a, n, i0, i1, i2);
      } else {
        const int16_t* t = trip + (size_t(n - 3) * p.ransac_attempts + a) * 3;
        i0 = t[0];
        i1 = t[1];
        i2 = t[2];
      }
      ECA_CHECK(i0 >= 0 && i0 < n && i1 >= 0 && i1 < n && i2 >= 0 && i2 < n);
      c = circumcircle(pt[i0].x, pt[i0].y, pt[i1].x, pt[i1].y, pt[i2].x,
                       pt[i2].y);
    }
    FIT_STAMP(2);
    // iterated masked least squares (fitting.py:193-203); every lane runs the
    // loop, dead hypotheses with an empty ring.  Outliers contribute fma(0, v, s)
    // = s + (+-0) = s exactly (the sums start at +0.0, so no -0.0 appears).
    for (int it = 0; it < p.ransac_iterations && __any_sync(kFull, c.alive); ++it) {
      const RingF g = c.alive ? ring_f(ring_of(c, tol), c, bmax) : ringf_dead();
      double mo[kMom - 1] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int k0 = 0; k0 < n; k0 += 32) {
        const int kn = min(32, n - k0);
        const uint32_t in_m = inlier_bits(pt, k0, kn, c, g, tol);
        if (it == 1) FIT_STAMP(8);
#pragma unroll 4
        for (int j = 0; j < kn; ++j) {
          const FitPt& P = pt[k0 + j];
          // w in {0, 1}: fma(1, v, s) == add_rn(s, v) and fma(0, v, s) == s
          const double w = (in_m >> j) & 1u ? 1.0 : 0.0;
          mo[0] = __fma_rn(w, P.x, mo[0]);
          mo[1] = __fma_rn(w, P.y, mo[1]);
          mo[2] = __fma_rn(w, P.z, mo[2]);
          mo[3] = __fma_rn(w, P.xx, mo[3]);
          mo[4] = __fma_rn(w, P.xy, mo[4]);
          mo[5] = __fma_rn(w, P.yy, mo[5]);
          mo[6] = __fma_rn(w, P.xz, mo[6]);
          mo[7] = __fma_rn(w, P.yz, mo[7]);
        }
        mo[8] += double(__popc(in_m));   // the member count: exact integers
      }
      if (it == 1) FIT_STAMP(9);
      double na, nb, nr;
      if (c.alive) {
        if (lsq_solve(mo, int(mo[8]), na, nb, nr)) {
          c.cx = na;
          c.cy = nb;
          c.r = nr;
        } else {
          c.alive = false;
        }
      }
      FIT_STAMP(3 + (it < 2 ? it : 2));
    }
    double score = 0.0;
    int inl = 0;
    {
      const RingF g = c.alive ? ring_f(ring_of(c, tol), c, bmax) : ringf_dead();
      for (int k0 = 0; k0 < n; k0 += 32) {
        const int kn = min(32, n - k0);
        const uint32_t in_m = inlier_bits(pt, k0, kn, c, g, tol);
#pragma unroll 4
        for (int j = 0; j < kn; ++j) score = __fma_rn((in_m >> j) & 1u ? 1.0 : 0.0, ps[k0 + j], score);
        inl += __popc(in_m);
      }
    }
    FIT_STAMP(6);
    const bool gated = (c.r < p.min_radius_frac) || (c.r > p.max_radius_frac) ||
                       (hypot(c.cx, c.cy) > p.max_center_offset_frac);
    const bool surv = c.alive && !gated;
    any_live |= __any_sync(kFull, surv);
    any_gated |= __any_sync(kFull, c.alive && gated);
    double s_l = surv ? score : -1.0;
    int a_l = surv ? a : 0x7fffffff;
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      const double os = __shfl_xor_sync(kFull, s_l, d);
      const int oa = __shfl_xor_sync(kFull, a_l, d);
      if (os > s_l || (os == s_l && oa < a_l)) {
        s_l = os;
        a_l = oa;
      }
    }
    if (a_l != 0x7fffffff && s_l > best_s) {
      const int src = a_l - c0;
      best_s = s_l;
      bcx = __shfl_sync(kFull, c.cx, src);
      bcy = __shfl_sync(kFull, c.cy, src);
      br = __shfl_sync(kFull, c.r, src);
      best_inl = __shfl_sync(kFull, inl, src);
    }
  }
  if (lane == 0) {
    EcaFitRecord rec{0.0, 0.0, 0.0, 0.0, 0, ECA_LOW_SCORE};
    if (!any_live) {
      rec.status = any_gated ? ECA_GEOMETRY_GATE : ECA_LOW_SCORE;
    } else if (!(best_s < p.circle_score_threshold)) {
      rec.status = ECA_ACCEPTED;
      rec.cx = add_rn(p.center_x, mul_rn(bcx, double(W)));
      rec.cy = add_rn(p.center_y, mul_rn(bcy, double(W)));
      rec.r = mul_rn(br, double(W));
      rec.score = best_s;
      rec.inliers = best_inl;
    }
    store_record(out, rec, ordered);
  }
  FIT_STAMP(7);
  __syncwarp();
}

}  // namespace eca
