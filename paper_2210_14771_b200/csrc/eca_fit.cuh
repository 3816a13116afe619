// K2: candidate filter + seeded RANSAC with iterated FP64 least squares, one
// CTA per frame, one WARP per hypothesis (lanes = candidates).
//
// Restates fitting.py:39-230 in the reference's evaluation order: every FP64
// expression is written with explicit round-to-nearest intrinsics (no FMA
// contraction) so circumcircles, gates and LSQ systems see numpy's doubles.
// Only the moment sums (numpy: OpenBLAS dgemm) and the 3x3 solve (LAPACK
// gesv) reassociate; the survey measured that headroom at <=2.3e-13 px.
#pragma once

#include "eca_common.cuh"

namespace eca {

struct FitScratch {
  double px[2 * ECA_MAX_STRIPS];
  double py[2 * ECA_MAX_STRIPS];
  double ps[2 * ECA_MAX_STRIPS];
  double wb_s[32], wb_cx[32], wb_cy[32], wb_r[32];
  int wb_a[32], wb_inl[32], wb_flags[32];
  int n;
};

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
ECA_DEV bool lsq_solve(double sx, double sy, double sz, double sxx, double sxy, double syy,
                       double sxz, double syz, int cnt, double& a_out, double& b_out,
                       double& r_out) {
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
  bool ok = (cnt >= 3) && isfinite(det) && (fabs(det) > mul_rn(1e-12, mul_rn(mul_rn(nn, nn), nn)));
  if (!ok) return false;
  // LU with partial pivoting (dgetrf2/dgetrs order: reciprocal-scaled
  // multipliers, forward then backward substitution)
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int piv = k;
    double best = fabs(m[k][k]);
#pragma unroll
    for (int i = k + 1; i < 3; ++i)
      if (fabs(m[i][k]) > best) {
        best = fabs(m[i][k]);
        piv = i;
      }
    if (piv != k) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double t = m[k][j];
        m[k][j] = m[piv][j];
        m[piv][j] = t;
      }
      const double t = v[k];
      v[k] = v[piv];
      v[piv] = t;
    }
    const double rp = div_rn(1.0, m[k][k]);
#pragma unroll
    for (int i = k + 1; i < 3; ++i) {
      m[i][k] = mul_rn(m[i][k], rp);
#pragma unroll
      for (int j = k + 1; j < 3; ++j) m[i][j] = sub_rn(m[i][j], mul_rn(m[i][k], m[k][j]));
    }
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

// Warp-parallel inlier pass: members of circle (cx,cy,r) among n points.
// Returns the count; accumulates moments when `mom` is set, score sum otherwise.
template <bool kMoments>
ECA_DEV int inlier_pass(const FitScratch* fs, int n, double tol, double cx, double cy, double r,
                        double* mom /* [8] */, double& score_sum) {
  const int lane = threadIdx.x & 31;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double ssum = 0.0;
  int cnt = 0;
  for (int k = lane; k < n; k += 32) {
    const double x = fs->px[k], y = fs->py[k];
    const double d = fabs(sub_rn(hypot(sub_rn(x, cx), sub_rn(y, cy)), r));
    if (d <= tol) {
      ++cnt;
      if (kMoments) {
        const double z = add_rn(mul_rn(x, x), mul_rn(y, y));
        acc[0] += x;
        acc[1] += y;
        acc[2] += z;
        acc[3] += mul_rn(x, x);
        acc[4] += mul_rn(x, y);
        acc[5] += mul_rn(y, y);
        acc[6] += mul_rn(x, z);
        acc[7] += mul_rn(y, z);
      } else {
        ssum += fs->ps[k];
      }
    }
  }
  cnt = warp_sum(cnt);
  if (kMoments) {
#pragma unroll
    for (int q = 0; q < 8; ++q) mom[q] = warp_sum(acc[q]);
  } else {
    score_sum = warp_sum(ssum);
  }
  return cnt;
}

// One frame, whole CTA.  cand_* hold n_cand candidates in estimator.py:69
// order; `volatile_loads` reads them through L2 (written by other CTAs).
ECA_DEV void fit_frame(const int32_t* cand_x, const int32_t* cand_y, const double* cand_s,
                       int n_cand, bool volatile_loads, const EcaParams& p,
                       const int16_t* trip, int exhaustive, FitScratch* fs, EcaFitRecord* out) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n_warps = blockDim.x >> 5;
  const int W = p.width, H = p.height;
  // ---- filter_candidates (fitting.py:39-52), order-preserving compaction
  if (warp == 0) {
    int cnt = 0;
    for (int base = 0; base < n_cand; base += 32) {
      const int i = base + lane;
      bool keep = false;
      int x = 0, y = 0;
      double s = 0.0;
      if (i < n_cand) {
        if (volatile_loads) {
          x = __ldcg(cand_x + i);
          y = __ldcg(cand_y + i);
          s = __ldcg(cand_s + i);
        } else {
          x = cand_x[i];
          y = cand_y[i];
          s = cand_s[i];
        }
        const int edge = min(min(x, W - 1 - x), min(y, H - 1 - y));
        keep = edge >= p.edge_margin_px && s >= p.min_point_score;
      }
      const unsigned bal = __ballot_sync(kFull, keep);
      if (keep) {
        const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
        // (pts - (cx0, cy0)) / width  (fitting.py:187)
        fs->px[pos] = div_rn(sub_rn(double(x), p.center_x), double(W));
        fs->py[pos] = div_rn(sub_rn(double(y), p.center_y), double(W));
        fs->ps[pos] = s;
      }
      cnt += __popc(bal);
    }
    if (lane == 0) fs->n = cnt;
  }
  __syncthreads();
  const int n = fs->n;
  if (n < 3) {
    if (threadIdx.x == 0) *out = EcaFitRecord{0.0, 0.0, 0.0, 0.0, 0, ECA_NO_CANDIDATES};
    __syncthreads();
    return;
  }
  const int attempts = exhaustive ? n * (n - 1) * (n - 2) / 6 : p.ransac_attempts;
  const double tol = p.inlier_tol;
  double best_s = -1.0, bcx = 0.0, bcy = 0.0, br = 0.0;
  int best_a = -1, best_inl = 0, flags = 0;  // bit0: any survivor, bit1: any live gated
  for (int a = warp; a < attempts; a += n_warps) {
    int i0, i1, i2;
    if (exhaustive) {
      unrank3(a, n, i0, i1, i2);
    } else {
      const int16_t* t = trip + (size_t(n - 3) * p.ransac_attempts + a) * 3;
      i0 = t[0];
      i1 = t[1];
      i2 = t[2];
    }
    Circ c = circumcircle(fs->px[i0], fs->py[i0], fs->px[i1], fs->py[i1], fs->px[i2], fs->py[i2]);
    for (int it = 0; it < p.ransac_iterations && c.alive; ++it) {
      double mom[8];
      double unused;
      const int cnt = inlier_pass<true>(fs, n, tol, c.cx, c.cy, c.r, mom, unused);
      double na, nb, nr;
      if (lsq_solve(mom[0], mom[1], mom[2], mom[3], mom[4], mom[5], mom[6], mom[7], cnt, na, nb,
                    nr)) {
        c.cx = na;
        c.cy = nb;
        c.r = nr;
      } else {
        c.alive = false;
      }
    }
    if (!c.alive) continue;   // no members, neither survivor nor gated
    double score;
    const int inl = inlier_pass<false>(fs, n, tol, c.cx, c.cy, c.r, nullptr, score);
    const bool gated = (c.r < p.min_radius_frac) || (c.r > p.max_radius_frac) ||
                       (hypot(c.cx, c.cy) > p.max_center_offset_frac);
    if (gated) {
      flags |= 2;
    } else {
      flags |= 1;
      if (score > best_s) {   // strict: first (lowest) attempt wins ties
        best_s = score;
        best_a = a;
        bcx = c.cx;
        bcy = c.cy;
        br = c.r;
        best_inl = inl;
      }
    }
  }
  if (lane == 0) {
    fs->wb_s[warp] = best_s;
    fs->wb_a[warp] = best_a;
    fs->wb_cx[warp] = bcx;
    fs->wb_cy[warp] = bcy;
    fs->wb_r[warp] = br;
    fs->wb_inl[warp] = best_inl;
    fs->wb_flags[warp] = flags;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int all = 0, bw = -1;
    for (int w = 0; w < n_warps; ++w) {
      all |= fs->wb_flags[w];
      if (fs->wb_a[w] < 0) continue;
      if (bw < 0 || fs->wb_s[w] > fs->wb_s[bw] ||
          (fs->wb_s[w] == fs->wb_s[bw] && fs->wb_a[w] < fs->wb_a[bw]))
        bw = w;
    }
    EcaFitRecord rec{0.0, 0.0, 0.0, 0.0, 0, ECA_LOW_SCORE};
    if (!(all & 1)) {
      rec.status = (all & 2) ? ECA_GEOMETRY_GATE : ECA_LOW_SCORE;
    } else if (!(fs->wb_s[bw] < p.circle_score_threshold)) {
      rec.status = ECA_ACCEPTED;
      rec.cx = add_rn(p.center_x, mul_rn(fs->wb_cx[bw], double(W)));
      rec.cy = add_rn(p.center_y, mul_rn(fs->wb_cy[bw], double(W)));
      rec.r = mul_rn(fs->wb_r[bw], double(W));
      rec.score = fs->wb_s[bw];
      rec.inliers = fs->wb_inl[bw];
    }
    *out = rec;
  }
  __syncthreads();
}

}  // namespace eca
