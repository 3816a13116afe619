// C ABI entry points of libeca_b200.so (declared in include/eca_b200.h):
// argument validation, launch geometry and kernel dispatch.  No entry point
// allocates device memory or synchronises the stream.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "eca_fit.cuh"
#include "eca_strip.cuh"
#include "eca_points.cuh"

using namespace eca;

namespace {

constexpr int kStages = 3;

int sm_count() {
  static int count[64];
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::call_once(once[dev], [dev] {
    int c = 0;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    count[dev] = c > 0 ? c : 148;
  });
  return count[dev];
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Large dynamic shared memory opt-in of kernel `kern` on the CURRENT device,
// once per (kernel, device); false if the attribute could not be set.
bool smem_optin_ptr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, bool>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first.first == kern && d.first.second == dev) return d.second;
  const bool ok =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess;
  done.push_back({{kern, dev}, ok});
  return ok;
}
template <typename K>
bool smem_optin(K kern, int bytes = 227 * 1024) {
  return smem_optin_ptr(reinterpret_cast<const void*>(kern), bytes);
}

int check_launch() { return cudaGetLastError() == cudaSuccess ? ECA_OK : ECA_ERR_CUDA; }

bool getenv_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && std::atoi(v) != 0;
}

bool tracing() {
  static const bool on = std::getenv("ECA_TRACE") != nullptr;
  return on;
}
#define ECA_TRACE(...)                              \
  do {                                              \
    if (tracing()) {                                \
      std::fprintf(stderr, "[eca] " __VA_ARGS__);   \
      std::fflush(stderr);                          \
    }                                               \
  } while (0)

// Fill a StripJob; returns ECA_OK or an error code.
int prepare_strip_job(StripJob& J, const uint8_t* frames, int batch, int64_t frame_stride,
                      int64_t row_stride, const int32_t* strip_rows, const int32_t* band_rows,
                      int n_strips, const EcaParams* params) {
  if (!frames || !strip_rows || !params || batch < 0) return ECA_ERR_ARG;
  const int W = params->width, H = params->height;
  if (W < 8 || H < 14) return ECA_ERR_ARG;
  if (H > 32767 || W > ECA_MAX_WIDTH || n_strips < 1 || n_strips > ECA_MAX_STRIPS)
    return ECA_ERR_UNSUPPORTED;
  if (row_stride < 3LL * W || frame_stride < 0) return ECA_ERR_ARG;
  if (batch > 0 && int64_t(batch) * n_strips > (int64_t(1) << 30)) return ECA_ERR_UNSUPPORTED;
  std::memset(&J, 0, sizeof(J));
  J.frames = frames;
  J.frame_stride = frame_stride;
  J.row_stride = row_stride;
  J.batch = batch;
  J.n_strips = n_strips;
  J.nthreads = ((W + kPx - 1) / kPx + 31) / 32 * 32;
  J.rowcap = (24 * J.nthreads + 48 + 15) / 16 * 16;
  J.contiguous = (row_stride == 3LL * W) ? 1 : 0;
  J.p = *params;
  for (int k = 0; k < n_strips; ++k) {
    if (strip_rows[k] < 3 || strip_rows[k] > H - 4) return ECA_ERR_ARG;
    J.rows[k] = int16_t(strip_rows[k]);
    const int band = band_rows ? band_rows[k] : strip_rows[k] - 1;
    if (band < 0 || band > 32767) return ECA_ERR_ARG;
    J.band[k] = int16_t(band);
  }
  double bound = 0.0;
  const int risky = eca_prefilter_bound(params, &bound);
  // residue scores of flat-but-not-identical neighbourhoods stay below
  // ~5e-14 * 20 / t_g; halves whose best lower bound is under tau are scored
  // exhaustively in FP64.  Risky configs (FP32 range) always are.
  J.tau = risky ? INFINITY : float(1e-11 * 20.0 / params->gradient_threshold);
  // every FP32 bound is padded by the config's own modelled error bound,
  // rounded up to float (accepted configs: bound < 1e-2)
  J.pad = risky ? 1e-2f : std::nextafter(float(bound), INFINITY);
  return ECA_OK;
}

template <int MAXT, int MINB, bool kRows, bool kFused>
int launch_strips_t(const StripJob& J, cudaStream_t stream) {
  auto kern = strip_kernel<kStages, MAXT, MINB, kRows, kFused>;
  const StripLayout L = strip_layout(kStages, J.rowcap, J.nthreads);
  ECA_TRACE("launch_strips: job %zu B, smem %zu, threads %d\n", sizeof(StripJob), L.total,
            J.nthreads);
  if (!smem_optin(kern)) return ECA_ERR_CUDA;
  const int block = J.nthreads + 32 * kFpWarps;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, L.total);
  if (e != cudaSuccess || per_sm < 1) return ECA_ERR_CUDA;
  const int items = J.batch * J.n_strips;
  const int grid = items < sm_count() * per_sm ? items : sm_count() * per_sm;
  ECA_TRACE("per_sm %d grid %d\n", per_sm, grid);
  kern<<<grid, block, L.total, stream>>>(J);
  return check_launch();
}

// ---- points: bounds_kernel (warp per half row) -> survivor slots, FP64
// rescore in rescore_kernel or in the fit kernel's rescore stage
// workspace: [0, 256) tickets + set-reuse guard (zero between launches) |
// survivor slots | counts
int64_t slots_bytes(int64_t n_hr) {
  return (n_hr * kSlots * int64_t(sizeof(SurvSlot)) + 255) & ~int64_t(255);
}
int64_t points_workspace(int batch, int n_strips) {
  const int64_t n_hr = int64_t(batch) * n_strips * 2;
  return 256 + slots_bytes(n_hr) + n_hr * 4;
}

template <int NS, bool kChunked, bool kInWarp = false>
int launch_points_t(PointsJob PJ, cudaStream_t stream, bool overlap, bool share) {
  auto kern = bounds_kernel<NS, kChunked, kInWarp>;
  StripJob& J = PJ.J;
  const int W = J.p.width;
  const int split = (W + 1) / 2;
  const int half_w = split > W - split ? split : W - split;
  // a row holds exactly the staged bytes (<= 15 B misalignment + the half and
  // its neighbour column); lane-chunk reads past either end of a row land in
  // the neighbouring row / per-warp scratch (< 3*257 B) and only feed masked
  // columns
  J.rowcap = (15 + 3 * (half_w + 1) + 15) / 16 * 16;
  if (!smem_optin(kern)) return ECA_ERR_CUDA;
  const int fitb = 0;
  // CTA shape: the smallest CTA reaching the most resident warps per SM.
  // Items are handed out dynamically, so independent small CTAs cost
  // nothing; more resident warps shorten the end-of-kernel tail (B200,
  // 1080p B=256: 4 warps x 5 CTAs 50 us, 2 x 9 52 us, 8 x 2 56 us).
  // (cached per host thread and row capacity: the occupancy queries cost
  // microseconds, which matter at one launch per ~40 us batch)
  thread_local int cached_rowcap = -1, cached_dev = -1, cached_warps = 0, cached_per_sm = 0,
                   cached_fitb = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  int warps = 0, per_sm = 0;
  if (cached_rowcap == J.rowcap && cached_dev == dev && cached_fitb == fitb) {
    warps = cached_warps;
    per_sm = cached_per_sm;
  } else {
    for (int w = 1; w <= 8; ++w) {
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 32 * w,
                                                        warp_layout(NS, J.rowcap, w, fitb).total) !=
          cudaSuccess)
        return ECA_ERR_CUDA;
      ECA_TRACE("bounds kernel: %d warps/CTA -> %d CTAs/SM (smem %zu)\n", w, b,
                warp_layout(NS, J.rowcap, w, fitb).total);
      if (b * w > per_sm * warps) {
        warps = w;
        per_sm = b;
      }
    }
    cached_rowcap = J.rowcap;
    cached_dev = dev;
    cached_fitb = fitb;
    cached_warps = warps;
    cached_per_sm = per_sm;
  }
  static const int force_w = [] {   // tuning hook: ECA_BWARPS=<warps per CTA>
    const char* v = std::getenv("ECA_BWARPS");
    return v ? std::atoi(v) : 0;
  }();
  if (force_w >= 1 && force_w <= 8) {
    warps = force_w;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps,
                                                      warp_layout(NS, J.rowcap, warps, fitb).total) !=
        cudaSuccess)
      return ECA_ERR_CUDA;
  }
  static const int cap_ctas = [] {   // tuning hook: ECA_BCTAS=<max CTAs per SM>
    const char* v = std::getenv("ECA_BCTAS");
    return v ? std::atoi(v) : 0;
  }();
  if (cap_ctas > 0 && per_sm > cap_ctas) per_sm = cap_ctas;
  // share: one CTA slot per SM stays free for kernels of other streams (the
  // pipelined rescore + fit of the previous batch); measured on B200 1080p
  // B=256: pipelined step 43 us vs 50 us with every slot taken
  if (share && per_sm > 1) --per_sm;
  if (per_sm < 1) return ECA_ERR_CUDA;
  const size_t smem = warp_layout(NS, J.rowcap, warps, fitb).total;
  const int64_t n_hr = int64_t(J.batch) * J.n_strips * 2;
  const int64_t need = (n_hr + warps - 1) / warps;
  const int grid = int(need < int64_t(sm_count()) * per_sm ? need : int64_t(sm_count()) * per_sm);
  ECA_TRACE("bounds kernel: NS %d warps %d smem %zu per_sm %d grid %d\n", NS, warps, smem, per_sm,
            grid);
  // overlap: programmatic dependent launch, so this grid's CTAs fill SMs as
  // the previous kernel in the stream drains (bounds_kernel triggers its
  // dependents at entry and reads nothing the previous kernel writes)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(32 * warps));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = overlap ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, PJ) != cudaSuccess) return ECA_ERR_CUDA;
  return check_launch();
}

// A bounds per pseudo-angle bin (as build_tables in eca_strip.cuh), in double
// on the host, padded `pad` outward (StripJob::pad)
void angle_table(double angle_scale, double pad, float2* at) {
  const double pi = 3.14159265358979323846;
  auto theta_of = [&](double ps) {
    ps = std::fmin(std::fmax(ps, 0.0), 2.0);
    return ps <= 1.0 ? std::atan2(ps, 1.0 - ps) : pi - std::atan2(2.0 - ps, ps - 1.0);
  };
  auto term = [&](double th) { return 2.0 / (1.0 + std::exp(2.0 * angle_scale * th)); };
  const double lo_f = 1.0 - pad, hi_f = 1.0 + pad;
  for (int k = 0; k < kABins; ++k) {
    const double w = 2.0 / kABins;
    const double th_lo = theta_of(k * w - 1e-5), th_hi = theta_of((k + 1) * w + 1e-5);
    at[k] = make_float2(float(term(th_hi) * lo_f), float(std::fmin(term(th_lo) * hi_f, 1.0)));
  }
  at[kABins] = make_float2(float(term(pi) * lo_f), 1.0f);   // dot == cross == 0
}

PointsJob points_job(const StripJob& J, void* workspace) {
  const int64_t n_hr = int64_t(J.batch) * J.n_strips * 2;
  PointsJob PJ;
  PJ.J = J;
  PJ.chunked = 0;
  {   // the table depends only on angle_scale and the pad: cached per host thread
    thread_local double cached_scale = -1.0;
    thread_local float cached_pad = -1.0f;
    thread_local float2 cached[kABins + 1];
    if (cached_scale != J.p.angle_scale || cached_pad != J.pad) {
      angle_table(J.p.angle_scale, double(J.pad), cached);
      cached_scale = J.p.angle_scale;
      cached_pad = J.pad;
    }
    std::memcpy(PJ.atab, cached, sizeof(cached));
  }
  const double log2e = 1.4426950408889634;
  PJ.kt = float(-2.0 * log2e / (3.0 * J.p.gradient_threshold));
  PJ.kd = float(2.0 * log2e / (3.0 * J.p.intensity_threshold));
  PJ.cxf = double(J.p.width - 1) / 2.0;   // exact (halving)
  PJ.cyf = double(J.p.height - 1) / 2.0;
  const int64_t nfs = int64_t(J.batch) * J.n_strips;
  PJ.s_magic = nfs < (int64_t(1) << 25)
                   ? uint32_t(((uint64_t(1) << 32) + uint64_t(J.n_strips) - 1) / uint64_t(J.n_strips))
                   : 0u;
  uint8_t* w = reinterpret_cast<uint8_t*>(workspace);
  PJ.ticket = reinterpret_cast<int32_t*>(w);
  PJ.slots = reinterpret_cast<SurvSlot*>(w + 256);
  PJ.counts = reinterpret_cast<int32_t*>(w + 256 + slots_bytes(n_hr));
  PJ.wait_prev = 0;
  PJ.guard = 0;
  PJ.dbg_seq = 0;
  return PJ;
}

int launch_bounds_job(PointsJob PJ, cudaStream_t stream, bool overlap, bool share, bool chunked) {
  if (PJ.J.batch == 0) return ECA_OK;
  static const int ns = [] {
    const char* v = std::getenv("ECA_WSTAGES");
    return v ? std::atoi(v) : 1;
  }();
  PJ.chunked = chunked ? 1 : 0;
  if (chunked) return launch_points_t<1, true>(PJ, stream, overlap, share);   // one stage
  return ns == 2 ? launch_points_t<2, false>(PJ, stream, overlap, share)
                 : launch_points_t<1, false>(PJ, stream, overlap, share);
}

int launch_bounds(const StripJob& J, void* workspace, cudaStream_t stream, bool overlap = false,
                  bool share = false, bool chunked = false) {
  if (J.batch == 0) return ECA_OK;
  PointsJob PJ = points_job(J, workspace);
  return launch_bounds_job(PJ, stream, overlap, share, chunked);
}

// one warp per CTA (4 half rows): small CTAs slot in beside a running
// bounds kernel of the next batch when the host pipelines the two
int launch_rescore(const StripJob& J, void* workspace, cudaStream_t stream) {
  if (J.batch == 0) return ECA_OK;
  const int64_t n_hr = int64_t(J.batch) * J.n_strips * 2;
  rescore_kernel<<<unsigned((n_hr + 3) / 4), 32, 0, stream>>>(points_job(J, workspace));
  return check_launch();
}

int launch_points(const StripJob& J, void* workspace, cudaStream_t stream) {
  const int rc = launch_bounds(J, workspace, stream);
  return rc ? rc : launch_rescore(J, workspace, stream);
}

template <bool kRows, bool kFused>
int launch_strips(const StripJob& J, cudaStream_t stream) {
  if (J.batch == 0) return ECA_OK;
  if (J.nthreads <= 256) return launch_strips_t<256 + 32 * kFpWarps, 2, kRows, kFused>(J, stream);
  return launch_strips_t<512 + 32 * kFpWarps, 1, kRows, kFused>(J, stream);
}

struct FitJob {
  const int32_t* x;
  const int32_t* y;
  const double* s;
  int n_cand, exhaustive;
  EcaParams p;
  const int16_t* trip;
  EcaFitRecord* out;
  EcaFitRecord* host_out;   // optional mapped pinned copy of the records
  int ordered;              // out: status word last, after a system-scope fence
  int32_t* guard;           // set-reuse guard ticket block (pipelines) or null
  int wait_prev;            // griddepcontrol.wait: the inputs come from the
                            // kernel before this one (programmatic launch)
  // rescore stage (counts != null): the bound-and-prune kernel's survivor
  // slots of each frame are scored in FP64 here first (handcrafted.py:148-205
  // evaluation order), their half-row winners become the candidates x / y / s
  // (written out too), then the fit runs on them from shared memory
  int dbg_seq;              // launch number (ECA_TIMELINE diagnostic builds)
  const int32_t* counts;    // [batch][n_strips][2] survivors, -1 = resolved
  const SurvSlot* slots;    // [batch][n_strips][2][kSlots]
  double cxf, cyf;
  int16_t rows[ECA_MAX_STRIPS];
};

// fit_kernel shared memory: the fit's point scratch, then (rescore stage) the
// candidates and the per-survivor scores
struct FitSmem {
  size_t pt, ps, cx, cy, cs, ent, ex, esc, total;
};
__host__ __device__ inline FitSmem fit_smem_layout(int n_cand, bool rescore) {
  FitSmem L;
  size_t o = 0;
  L.pt = o;
  o += size_t(n_cand) * sizeof(FitPt);
  L.ps = o;
  o += size_t(n_cand) * 8;
  L.cs = o;
  o += rescore ? size_t(n_cand) * 8 : 0;
  L.esc = o;
  o += rescore ? size_t(n_cand) * kSlots * 8 : 0;
  L.cx = o;
  o += rescore ? size_t(n_cand) * 4 : 0;
  L.cy = o;
  o += rescore ? size_t(n_cand) * 4 : 0;
  L.ent = o;
  o += rescore ? size_t(n_cand) * kSlots * 2 : 0;
  L.ex = o;
  o += rescore ? size_t(n_cand) * kSlots * 2 : 0;
  L.total = (o + 15) & ~size_t(15);
  return L;
}

// Rescore stage of frame b (one warp): compact the frame's survivors (lane =
// candidate / half row), score them 32 at a time (full lanes), then each
// half row's winner with the reference's outermost tie-break.
ECA_DEV void rescore_frame(const FitJob& J, int b, uint8_t* smem) {
  const int lane = threadIdx.x & 31;
  const int nc = J.n_cand, S = nc / 2, W = J.p.width;
  const FitSmem L = fit_smem_layout(nc, true);
  int32_t* cx = reinterpret_cast<int32_t*>(smem + L.cx);
  int32_t* cy = reinterpret_cast<int32_t*>(smem + L.cy);
  double* cs = reinterpret_cast<double*>(smem + L.cs);
  uint16_t* ent = reinterpret_cast<uint16_t*>(smem + L.ent);
  uint16_t* ex = reinterpret_cast<uint16_t*>(smem + L.ex);
  double* esc = reinterpret_cast<double*>(smem + L.esc);
  auto hrow_of = [&](int hk) {
    const int half = hk >= S ? 1 : 0;
    return (b * S + (hk - half * S)) * 2 + half;
  };
  int base = 0;
  for (int h0 = 0; h0 < nc; h0 += 32) {   // compaction: (candidate << 3 | slot)
    const int hk = h0 + lane;
    const int cnt = hk < nc ? __ldcg(J.counts + hrow_of(hk)) : -1;
    const int n = cnt > 0 ? cnt : 0;
    int incl = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += v;
    }
    const int off = base + incl - n;
    ECA_CHECK(n <= kSlots && off + n <= nc * kSlots);
    for (int k = 0; k < n; ++k) ent[off + k] = uint16_t((hk << 3) | k);
    if (hk < nc) {
      cx[hk] = off;   // parked until the winners are taken
      cy[hk] = cnt;
    }
    base += __shfl_sync(kFull, incl, 31);
  }
  __syncwarp();
  for (int e = lane; e < base; e += 32) {   // FP64 scores, full lanes
    const int hk = ent[e] >> 3, k = ent[e] & 7;
    const int half = hk >= S ? 1 : 0;
    const SurvSlot* sp = J.slots + size_t(hrow_of(hk)) * kSlots + k;
    uint2 w[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) w[q] = __ldcg(reinterpret_cast<const uint2*>(sp) + q);
    SurvSlot sl;
    memcpy(&sl, w, sizeof(sl));
    const int l[3] = {sl.l[0], sl.l[1], sl.l[2]}, m[3] = {sl.m[0], sl.m[1], sl.m[2]},
              r[3] = {sl.r[0], sl.r[1], sl.r[2]};
    esc[e] = exact_score(l, m, r, sl.pre, sl.x, J.rows[hk - half * S], J.cxf, J.cyf, J.p);
    ex[e] = sl.x;
  }
  __syncwarp();
  const size_t o = size_t(b) * nc;
  for (int h0 = 0; h0 < nc; h0 += 32) {   // winners
    const int hk = h0 + lane;
    if (hk >= nc) continue;
    const int half = hk >= S ? 1 : 0;
    const int off = cx[hk], cnt = cy[hk];
    Best bb = half ? Best{0.0, W - 1} : Best{0.0, 0};   // border columns score 0
    if (cnt < 0) {   // resolved by its bounds warp (more than kSlots survivors)
      bb = Best{__ldcg(J.s + o + hk), __ldcg(J.x + o + hk)};
    } else {
      for (int k = 0; k < cnt; ++k)
        if (better(esc[off + k], int(ex[off + k]), bb.s, bb.x, !half))
          bb = Best{esc[off + k], int(ex[off + k])};
    }
    const int y = J.rows[hk - half * S];
    cx[hk] = bb.x;
    cy[hk] = y;
    cs[hk] = bb.s;
    if (cnt >= 0) {   // the API's candidate outputs
      const_cast<int32_t*>(J.x)[o + hk] = bb.x;
      const_cast<int32_t*>(J.y)[o + hk] = y;
      const_cast<double*>(J.s)[o + hk] = bb.s;
    }
  }
  __syncwarp();
}

// One frame per single-warp CTA with n_cand-sized shared scratch (5.4 KB at
// 1080p with the rescore stage), same arithmetic order as the fused path's
// fit_warp.  In a pipeline it is launched programmatically after the batch's
// bounds kernel: its CTAs trigger the next batch's bounds launch at once,
// then wait for their own batch's survivors, and run beside the next batch's
// bounds kernel.
// blockDim.x = 32 * frames per CTA; warp w of CTA c fits frame c * warps + w
__global__ void __launch_bounds__(256) fit_kernel(const __grid_constant__ FitJob J, int batch) {
  extern __shared__ __align__(16) uint8_t fit_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int b = blockIdx.x * (blockDim.x >> 5) + wib;
  const FitSmem L = fit_smem_layout(J.n_cand, J.counts != nullptr);
  uint8_t* mine = fit_smem + size_t(wib) * L.total;
  int u = 0;
  if (J.guard && threadIdx.x == 0) u = guard_claim(J.guard);
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // inputs from the kernel just before: a guarded launch waits for exactly
  // that kernel (its use of the workspace, release / acquire); griddepcontrol
  // .wait would also wait for everything before it in the stream (the
  // previous batch's fits, transitively), serialising the fits
  if (J.guard) {
    if (threadIdx.x == 0) guard_wait(J.guard, u);
    __syncthreads();
  } else if (J.wait_prev) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  TL_STAMP(1, J.dbg_seq, 0);
  if (b < batch) {
    FitPt* pt = reinterpret_cast<FitPt*>(mine + L.pt);
    double* ps = reinterpret_cast<double*>(mine + L.ps);
    if (J.counts) {
      rescore_frame(J, b, mine);
      fit_warp<false>(reinterpret_cast<const int32_t*>(mine + L.cx),
                      reinterpret_cast<const int32_t*>(mine + L.cy),
                      reinterpret_cast<const double*>(mine + L.cs), J.n_cand, J.p, J.trip,
                      J.exhaustive, pt, ps, J.out + b, J.ordered != 0);
    } else {
      const size_t o = size_t(b) * J.n_cand;
      fit_warp(J.x + o, J.y + o, J.s + o, J.n_cand, J.p, J.trip, J.exhaustive, pt, ps, J.out + b,
               J.ordered != 0);
    }
    if (J.host_out && lane == 0) J.host_out[b] = J.out[b];
  }
  TL_STAMP(1, J.dbg_seq, 1);
  if (J.guard) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      guard_release(J.guard, int(gridDim.x));
    }
  }
}

// FitJob whose rescore stage reads the survivors of a points workspace
FitJob rescore_fit_job(const StripJob& J, void* workspace, const int16_t* trip, EcaFitRecord* out,
                       EcaFitRecord* host_out) {
  FitJob F;
  std::memset(&F, 0, sizeof(F));
  F.x = J.out_x;
  F.y = J.out_y;
  F.s = J.out_score;
  F.n_cand = 2 * J.n_strips;
  F.p = J.p;
  F.trip = trip;
  F.out = out;
  F.host_out = host_out;
  const PointsJob PJ = points_job(J, workspace);
  F.counts = PJ.counts;
  F.slots = PJ.slots;
  F.cxf = PJ.cxf;
  F.cyf = PJ.cyf;
  for (int k = 0; k < J.n_strips; ++k) F.rows[k] = J.rows[k];
  return F;
}

int check_fit_params(const EcaParams* params) {
  if (params->ransac_attempts < 1 || params->ransac_attempts > ECA_MAX_ATTEMPTS ||
      params->ransac_iterations < 1)
    return ECA_ERR_ARG;
  return ECA_OK;
}

}  // namespace

extern "C" int eca_points_workspace_bytes(int batch, int n_strips, int64_t* out_bytes) {
  if (batch < 0 || n_strips < 1 || n_strips > ECA_MAX_STRIPS || !out_bytes) return ECA_ERR_ARG;
  *out_bytes = points_workspace(batch, n_strips);
  return ECA_OK;
}

extern "C" int eca_points_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                                      int64_t row_stride, const int32_t* strip_rows,
                                      const int32_t* band_rows, int n_strips,
                                      const EcaParams* params, int32_t* out_x, int32_t* out_y,
                                      double* out_score, void* workspace, void* stream) {
  ECA_RANGE("eca_points_handcrafted");
  StripJob J;
  int rc = prepare_strip_job(J, frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                             n_strips, params);
  if (rc) return rc;
  if (!out_x || !out_y || !out_score) return ECA_ERR_ARG;
  J.out_x = out_x;
  J.out_y = out_y;
  J.out_score = out_score;
  if (!workspace) return launch_strips<false, false>(J, as_stream(stream));  // single-kernel path
  return launch_points(J, workspace, as_stream(stream));
}

extern "C" int eca_bounds_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                                      int64_t row_stride, const int32_t* strip_rows,
                                      const int32_t* band_rows, int n_strips,
                                      const EcaParams* params, int32_t* out_x, int32_t* out_y,
                                      double* out_score, void* workspace, int flags,
                                      void* stream) {
  ECA_RANGE("eca_bounds_handcrafted");
  if (flags & ~(ECA_BOUNDS_OVERLAP_PREVIOUS | ECA_BOUNDS_SHARE_SMS | ECA_BOUNDS_ZERO_COPY))
    return ECA_ERR_ARG;
  StripJob J;
  int rc = prepare_strip_job(J, frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                             n_strips, params);
  if (rc) return rc;
  if (!out_x || !out_y || !out_score || !workspace) return ECA_ERR_ARG;
  J.out_x = out_x;
  J.out_y = out_y;
  J.out_score = out_score;
  return launch_bounds(J, workspace, as_stream(stream), (flags & ECA_BOUNDS_OVERLAP_PREVIOUS) != 0,
                       (flags & ECA_BOUNDS_SHARE_SMS) != 0, (flags & ECA_BOUNDS_ZERO_COPY) != 0);
}

extern "C" int eca_rescore_handcrafted(int batch, const int32_t* strip_rows, int n_strips,
                                       const EcaParams* params, int32_t* out_x, int32_t* out_y,
                                       double* out_score, void* workspace, void* stream) {
  ECA_RANGE("eca_rescore_handcrafted");
  if (!strip_rows || !params || !out_x || !out_y || !out_score || !workspace || batch < 0)
    return ECA_ERR_ARG;
  if (n_strips < 1 || n_strips > ECA_MAX_STRIPS) return ECA_ERR_UNSUPPORTED;
  StripJob J;
  std::memset(&J, 0, sizeof(J));
  J.batch = batch;
  J.n_strips = n_strips;
  J.p = *params;
  for (int k = 0; k < n_strips; ++k) {
    if (strip_rows[k] < 3 || strip_rows[k] > params->height - 4) return ECA_ERR_ARG;
    J.rows[k] = int16_t(strip_rows[k]);
  }
  J.out_x = out_x;
  J.out_y = out_y;
  J.out_score = out_score;
  return launch_rescore(J, workspace, as_stream(stream));
}

extern "C" int eca_score_rows_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                                          int64_t row_stride, const int32_t* strip_rows,
                                          const int32_t* band_rows, int n_strips,
                                          const EcaParams* params, double* out_scores,
                                          int32_t* out_x, int32_t* out_y, double* out_score,
                                          void* stream) {
  ECA_RANGE("eca_score_rows_handcrafted");
  StripJob J;
  int rc = prepare_strip_job(J, frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                             n_strips, params);
  if (rc) return rc;
  if (!out_scores || !out_x || !out_y || !out_score) return ECA_ERR_ARG;
  J.out_rows = out_scores;
  J.out_x = out_x;
  J.out_y = out_y;
  J.out_score = out_score;
  return launch_strips<true, false>(J, as_stream(stream));
}

namespace {
// overlap: programmatic dependent launch (then J.wait_prev must be set when
// the candidates come from the kernel before it in the stream)
// spread: no launch follows that must wait for this one's residency (the last
// step of a stream): one frame per CTA, over every SM
int launch_fit(const FitJob& J, int batch, cudaStream_t stream, bool overlap = false,
               bool spread = false) {
  // frames (warps) per CTA: few, wide CTAs find room in a draining bounds
  // kernel sooner than many small ones (the next programmatic launch waits
  // until every CTA of this one is resident)
  static const int fpb_env = [] {
    const char* v = std::getenv("ECA_FIT_FPB");
    return v ? std::atoi(v) : 0;
  }();
  const size_t per = fit_smem_layout(J.n_cand, J.counts != nullptr).total;
  int fpb = fpb_env > 0 ? fpb_env : (overlap && !spread ? 8 : 1);
  if (fpb > 8) fpb = 8;
  while (fpb > 1 && per * fpb > 96 * 1024) fpb /= 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned((batch + fpb - 1) / fpb));
  cfg.blockDim = dim3(unsigned(32 * fpb));
  cfg.dynamicSmemBytes = per * fpb;
  if (cfg.dynamicSmemBytes > 48 * 1024 && !smem_optin(fit_kernel)) return ECA_ERR_CUDA;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = overlap ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, fit_kernel, J, batch) != cudaSuccess) return ECA_ERR_CUDA;
  return check_launch();
}
}  // namespace

extern "C" int eca_fit(const int32_t* cand_x, const int32_t* cand_y, const double* cand_score,
                       int batch, int n_cand, const EcaParams* params, const int16_t* triplets,
                       int exhaustive, EcaFitRecord* out, void* stream) {
  ECA_RANGE("eca_fit");
  if (batch < 0 || n_cand < 0 || n_cand > 2 * ECA_MAX_STRIPS || !params) return ECA_ERR_ARG;
  if (batch == 0) return ECA_OK;
  if (!cand_x || !cand_y || !cand_score || !out || (!exhaustive && !triplets)) return ECA_ERR_ARG;
  if (check_fit_params(params)) return ECA_ERR_ARG;
  FitJob J;
  std::memset(&J, 0, sizeof(J));
  J.x = cand_x;
  J.y = cand_y;
  J.s = cand_score;
  J.n_cand = n_cand;
  J.exhaustive = exhaustive ? 1 : 0;
  J.p = *params;
  J.trip = triplets;
  J.out = out;
  return launch_fit(J, batch, as_stream(stream));
}

extern "C" int eca_estimate_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                                        int64_t row_stride, const int32_t* strip_rows,
                                        const int32_t* band_rows, int n_strips,
                                        const EcaParams* params, const int16_t* triplets,
                                        int32_t* counters, int32_t* out_x, int32_t* out_y,
                                        double* out_score, EcaFitRecord* out, void* stream) {
  ECA_RANGE("eca_estimate_handcrafted");
  StripJob J;
  int rc = prepare_strip_job(J, frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                             n_strips, params);
  if (rc) return rc;
  if (!triplets || !counters || !out || !out_x || !out_y || !out_score) return ECA_ERR_ARG;
  if (check_fit_params(params)) return ECA_ERR_ARG;
  if (batch == 0) return ECA_OK;
  J.out_x = out_x;
  J.out_y = out_y;
  J.out_score = out_score;
  cudaStream_t st = as_stream(stream);
  if (!getenv_flag("ECA_LATENCY_STRIP")) {
    // warp per half row, survivors rescored in the same warp (candidates
    // out), then the fit kernel as a programmatic dependent launch: its CTAs
    // are resident before the candidates are done.  `counters` is the item
    // ticket block (>= 64 int32, left zeroed).
    PointsJob PJ = points_job(J, counters);
    rc = launch_points_t<1, false, true>(PJ, st, false, false);
    if (rc) return rc;
    FitJob F;
    std::memset(&F, 0, sizeof(F));
    F.x = out_x;
    F.y = out_y;
    F.s = out_score;
    F.n_cand = 2 * n_strips;
    F.p = J.p;
    F.trip = triplets;
    F.out = out;
    F.ordered = 1;   // `out` may be mapped pinned memory the caller polls
    F.wait_prev = 1;
    return launch_fit(F, batch, st, /*overlap=*/true);
  }
  // one launch: the block-per-strip kernel whose last CTA per frame fits it
  // (`counters`: batch int32 zeros)
  J.triplets = triplets;
  J.counters = counters;
  J.out_fit = out;
  return launch_strips<false, true>(J, st);
}

extern "C" int eca_h2d_bands(const uint8_t* host, int batch, int64_t host_frame_stride,
                             int64_t host_row_stride, const int32_t* first_rows, int n_bands,
                             int rows_per_band, int width, uint8_t* dev, void* stream) {
  ECA_RANGE("eca_h2d_bands");
  if (batch < 0 || n_bands < 0 || rows_per_band < 1 || width < 1) return ECA_ERR_ARG;
  if (batch == 0 || n_bands == 0) return ECA_OK;
  if (!host || !first_rows || !dev || host_row_stride < 3LL * width) return ECA_ERR_ARG;
  const size_t row_bytes = size_t(3) * width;
  const size_t band_bytes = row_bytes * rows_per_band;
  const size_t dev_frame = band_bytes * n_bands;
  const bool packed = host_row_stride == int64_t(row_bytes);
  auto st = as_stream(stream);
  for (int k = 0; k < n_bands; ++k) {
    // one strided DMA per band (packed host rows) or per band row, across all frames
    for (int r = 0; r < (packed ? 1 : rows_per_band); ++r) {
      const uint8_t* src = host + int64_t(first_rows[k] + r) * host_row_stride;
      uint8_t* dst = dev + k * band_bytes + r * row_bytes;
      const size_t w = packed ? band_bytes : row_bytes;
      if (cudaMemcpy2DAsync(dst, dev_frame, src, size_t(host_frame_stride), w, size_t(batch),
                            cudaMemcpyHostToDevice, st) != cudaSuccess)
        return ECA_ERR_CUDA;
    }
  }
  return ECA_OK;
}



// ---------------------------------------------------------------- pipeline
// Streamed throughput mode (ContentAreaEngine.run_pipelined), two launches
// per batch on the caller's stream, both programmatic dependent launches:
//   bounds_kernel  bound-and-prune -> survivor slots
//   fit_kernel     per frame (one warp): FP64 rescore of the survivors with
//                  full lanes -> candidates, then filter + RANSAC -> records
// so batch i's bounds CTAs fill the SMs as batch i-1's drain, and batch i's
// fits (latency-bound FP64 chains) run beside batch i+1's bounds kernel.
// kPipeSets buffer sets rotate inside the caller-provided scratch; each launch
// claims its set on the device and waits for the launches that used it
// before (guard_claim / guard_wait).  No side stream, no events between the
// launches.
#ifndef ECA_PIPE_SETS
#define ECA_PIPE_SETS 4
#endif
constexpr int kPipeSets = ECA_PIPE_SETS;
struct EcaPipeline {
  int batch, n_strips;
  StripJob J;                 // template: geometry, params, tau, pad
  const int16_t* trip;
  cudaStream_t last_stream;   // stream of the latest step (fence records there)
  cudaEvent_t ev_fence;
  int step, last;
  uint8_t* ws[kPipeSets];
  int32_t *xs[kPipeSets], *ys[kPipeSets];
  double* sc[kPipeSets];
  EcaFitRecord* rec[kPipeSets];
};

namespace {
struct PipeLayout {
  int64_t ws, xs, ys, sc, rec, set, total;
};
PipeLayout pipe_layout(int batch, int n_strips) {
  auto up = [](int64_t v) { return (v + 255) & ~int64_t(255); };
  PipeLayout L;
  const int64_t nc = int64_t(batch) * 2 * n_strips;
  L.ws = 0;
  L.xs = up(points_workspace(batch, n_strips));
  L.ys = L.xs + up(nc * 4);
  L.sc = L.ys + up(nc * 4);
  L.rec = L.sc + up(nc * 8);
  L.set = L.rec + up(int64_t(batch) * int64_t(sizeof(EcaFitRecord)));
  L.total = kPipeSets * L.set;
  return L;
}
}  // namespace

extern "C" int eca_pipeline_bytes(int batch, int n_strips, int64_t* out_bytes) {
  if (batch < 1 || n_strips < 1 || n_strips > ECA_MAX_STRIPS || !out_bytes) return ECA_ERR_ARG;
  *out_bytes = pipe_layout(batch, n_strips).total;
  return ECA_OK;
}

extern "C" int eca_pipeline_create(int batch, int height, int width, const int32_t* strip_rows,
                                   int n_strips, const EcaParams* params, const int16_t* triplets,
                                   void* scratch, int64_t scratch_bytes, EcaPipeline** out) {
  ECA_RANGE("eca_pipeline_create");
  if (!out || !scratch || !triplets || batch < 1) return ECA_ERR_ARG;
  *out = nullptr;
  if (!params || params->width != width || params->height != height) return ECA_ERR_ARG;
  if (check_fit_params(params)) return ECA_ERR_ARG;
  if (n_strips < 1 || n_strips > ECA_MAX_STRIPS) return ECA_ERR_UNSUPPORTED;
  const PipeLayout L = pipe_layout(batch, n_strips);
  if (scratch_bytes < L.total) return ECA_ERR_ARG;
  static const uint8_t dummy[16] = {};
  EcaPipeline* P = new EcaPipeline();
  int rc = prepare_strip_job(P->J, dummy, batch, 0, 3LL * width, strip_rows, nullptr, n_strips,
                             params);
  if (rc) {
    delete P;
    return rc;
  }
  P->batch = batch;
  P->n_strips = n_strips;
  P->trip = triplets;
  P->step = 0;
  P->last = -1;
  P->last_stream = nullptr;
  uint8_t* base = reinterpret_cast<uint8_t*>(scratch);
  for (int k = 0; k < kPipeSets; ++k) {
    uint8_t* b = base + k * L.set;
    P->ws[k] = b + L.ws;
    P->xs[k] = reinterpret_cast<int32_t*>(b + L.xs);
    P->ys[k] = reinterpret_cast<int32_t*>(b + L.ys);
    P->sc[k] = reinterpret_cast<double*>(b + L.sc);
    P->rec[k] = reinterpret_cast<EcaFitRecord*>(b + L.rec);
  }
  // tickets, frame counters and set sequence numbers start at zero
  if (cudaMemset(scratch, 0, size_t(L.total)) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_fence, cudaEventDisableTiming) != cudaSuccess) {
    delete P;
    return ECA_ERR_CUDA;
  }
  *out = P;
  return ECA_OK;
}

namespace {
int pipeline_step(EcaPipeline* P, const uint8_t* frames, int64_t frame_stride, int64_t row_stride,
                  int flags, EcaFitRecord* host_records, void* stream, EcaFitRecord** out_records,
                  bool last);
}

extern "C" int eca_pipeline_step(EcaPipeline* P, const uint8_t* frames, int64_t frame_stride,
                                 int64_t row_stride, int flags, EcaFitRecord* host_records,
                                 void* stream, EcaFitRecord** out_records) {
  ECA_RANGE("eca_pipeline_step");
  return pipeline_step(P, frames, frame_stride, row_stride, flags, host_records, stream,
                       out_records, false);
}

namespace {
int pipeline_step(EcaPipeline* P, const uint8_t* frames, int64_t frame_stride, int64_t row_stride,
                  int flags, EcaFitRecord* host_records, void* stream, EcaFitRecord** out_records,
                  bool last) {
  if (!P || !frames || !out_records || row_stride < 3LL * P->J.p.width || frame_stride < 0)
    return ECA_ERR_ARG;
  if (flags & ~(ECA_BOUNDS_ZERO_COPY | ECA_PIPE_FRAMES_READY)) return ECA_ERR_ARG;
  const int s = P->step % kPipeSets;
  cudaStream_t st = as_stream(stream);
  StripJob J = P->J;
  J.frames = frames;
  J.frame_stride = frame_stride;
  J.row_stride = row_stride;
  J.contiguous = row_stride == 3LL * J.p.width ? 1 : 0;
  J.out_x = P->xs[s];
  J.out_y = P->ys[s];
  J.out_score = P->sc[s];
  PointsJob PJ = points_job(J, P->ws[s]);
  PJ.guard = 1;
  PJ.dbg_seq = P->step;
  // frames produced by the kernel right before this launch must be waited for
  PJ.wait_prev = (flags & ECA_PIPE_FRAMES_READY) ? 0 : 1;
  // share: one bound-and-prune CTA slot per SM stays free for the previous
  // batch's fit CTAs, so the next bounds launch is fully resident at once
  static const bool share = [] {
    const char* v = std::getenv("ECA_PIPE_SHARE");
    return v ? std::atoi(v) != 0 : true;
  }();
  int rc = launch_bounds_job(PJ, st, /*overlap=*/true, share, (flags & ECA_BOUNDS_ZERO_COPY) != 0);
  if (rc) return rc;
  FitJob F = rescore_fit_job(J, P->ws[s], P->trip, P->rec[s], host_records);
  F.guard = PJ.ticket;
  F.dbg_seq = P->step;
  F.wait_prev = 1;   // its survivors come from the bounds kernel just before
  rc = launch_fit(F, P->batch, st, /*overlap=*/true, /*spread=*/last);
  if (rc) return rc;
  P->last = s;
  P->last_stream = st;
  ++P->step;
  *out_records = P->rec[s];
  return ECA_OK;
}
}  // namespace

extern "C" int eca_pipeline_run(EcaPipeline* P, const uint8_t* pool, int64_t batch_stride,
                                int n_slots, int first_slot, int n_steps, int64_t frame_stride,
                                int64_t row_stride, int flags, void* stream) {
  ECA_RANGE("eca_pipeline_run");
  if (!P || !pool || n_slots < 1 || first_slot < 0 || n_steps < 0 || batch_stride < 0)
    return ECA_ERR_ARG;
  EcaFitRecord* out = nullptr;
  for (int j = 0; j < n_steps; ++j) {
    const int slot = int((int64_t(first_slot) + j) % n_slots);
    // the last step's fits run alone: spread them over every SM
    const int rc = pipeline_step(P, pool + slot * batch_stride, frame_stride, row_stride, flags,
                                 nullptr, stream, &out, j + 1 == n_steps);
    if (rc) return rc;
  }
  return ECA_OK;
}

extern "C" int eca_pipeline_records(EcaPipeline* P, int back, EcaFitRecord** out_records) {
  if (!P || !out_records || back < 0 || back >= kPipeSets || back >= P->step) return ECA_ERR_ARG;
  *out_records = P->rec[(P->step - 1 - back) % kPipeSets];
  return ECA_OK;
}

extern "C" int eca_pipeline_reset(EcaPipeline* P) {
  // the device-side claim / done counters keep counting, so a graph captured
  // after eager steps replays safely
  if (!P) return ECA_ERR_ARG;
  return ECA_OK;
}

extern "C" int eca_pipeline_fence(EcaPipeline* P, void* stream) {
  ECA_RANGE("eca_pipeline_fence");
  if (!P) return ECA_ERR_ARG;
  if (P->last < 0) return ECA_OK;
  cudaStream_t st = as_stream(stream);
  if (st == P->last_stream) return ECA_OK;   // stream order already covers it
  if (cudaEventRecord(P->ev_fence, P->last_stream) != cudaSuccess ||
      cudaStreamWaitEvent(st, P->ev_fence, 0) != cudaSuccess)
    return ECA_ERR_CUDA;
  return ECA_OK;
}

extern "C" int eca_pipeline_side_stream(EcaPipeline* P, void** out_stream) {
  if (!P || !out_stream) return ECA_ERR_ARG;
  *out_stream = reinterpret_cast<void*>(P->last_stream);
  return ECA_OK;
}

extern "C" int eca_pipeline_destroy(EcaPipeline* P) {
  ECA_RANGE("eca_pipeline_destroy");
  if (!P) return ECA_OK;
  if (P->last_stream || P->last >= 0) cudaStreamSynchronize(P->last_stream);
  cudaEventDestroy(P->ev_fence);
  delete P;
  return ECA_OK;
}

extern "C" int eca_estimate_batch_handcrafted(const uint8_t* frames, int batch,
                                              int64_t frame_stride, int64_t row_stride,
                                              const int32_t* strip_rows, const int32_t* band_rows,
                                              int n_strips, const EcaParams* params,
                                              const int16_t* triplets, void* workspace,
                                              int32_t* out_x, int32_t* out_y, double* out_score,
                                              EcaFitRecord* out, EcaFitRecord* host_out,
                                              int flags, void* stream) {
  ECA_RANGE("eca_estimate_batch_handcrafted");
  if (flags & ~(ECA_BOUNDS_ZERO_COPY | ECA_PIPE_FRAMES_READY)) return ECA_ERR_ARG;
  StripJob J;
  int rc = prepare_strip_job(J, frames, batch, frame_stride, row_stride, strip_rows, band_rows,
                             n_strips, params);
  if (rc) return rc;
  if (!triplets || !workspace || !out || !out_x || !out_y || !out_score) return ECA_ERR_ARG;
  if (check_fit_params(params)) return ECA_ERR_ARG;
  J.out_x = out_x;
  J.out_y = out_y;
  J.out_score = out_score;
  rc = launch_bounds(J, workspace, as_stream(stream), false, false,
                     (flags & ECA_BOUNDS_ZERO_COPY) != 0);
  if (rc) return rc;
  if (batch == 0) return ECA_OK;
  return launch_fit(rescore_fit_job(J, workspace, triplets, out, host_out), batch,
                    as_stream(stream));
}

#ifdef ECA_TIMELINE
extern "C" int eca_debug_timeline(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl)) == cudaSuccess ? 0 : -2;
}
#endif
#ifdef ECA_FIT_TIMES
extern "C" int eca_debug_fit_times(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_fit_times, sizeof(unsigned long long) * 16 * n) == cudaSuccess ? 0
                                                                                                : -2;
}
#endif
#ifdef ECA_WARP_TIMES
extern "C" int eca_debug_warp_times(uint64_t* out, int n) {
  return cudaMemcpyFromSymbol(out, g_warp_times, sizeof(uint64_t) * 3 * n) == cudaSuccess ? 0 : -2;
}
#endif

// ------------------------------------------------------- prefilter self-test
// Test hook (tests/test_gpu_parity.py): measures, on the device, the FP32
// bound terms of the handcrafted kernels against FP64 for one config.
//   out[0] max relative error of t_term (bounds kernel) over every q in
//          [1, (3*1020)^2 * 2] (every integer |3g|^2 a frame can produce)
//   out[1] max relative error of d_term over every preceding sum 0..765
//   out[2] number of fused-kernel table entries (tanh / angle / darkness,
//          build_tables with the config's pad) that fail to bound the FP64
//          term over their bin
//   out[3] the pad the kernels use (StripJob::pad)
namespace {
constexpr int kSelfQMax = 2 * 3060 * 3060;

__device__ void atomic_max_pos(double* a, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(a), __double_as_longlong(v));
}

__global__ void selftest_terms(const EcaParams p, const TermK tk, double* out) {
  double mt = 0.0, md = 0.0;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int q = 1 + tid; q <= kSelfQMax; q += nt) {
    const double t64 = tanh(sqrt(double(q)) / 3.0 / p.gradient_threshold);
    mt = fmax(mt, fabs(double(t_term(q, tk)) - t64) / t64);
  }
  for (int s = tid; s < 766; s += nt) {
    const double d64 = 2.0 / (1.0 + exp(2.0 * (double(s) / 3.0) / p.intensity_threshold));
    if (d64 > 1e-300) md = fmax(md, fabs(double(d_term(s, tk)) - d64) / d64);
  }
  for (int d = 16; d; d >>= 1) {
    mt = fmax(mt, __shfl_xor_sync(kFull, mt, d));
    md = fmax(md, __shfl_xor_sync(kFull, md, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos(out, mt);
    atomic_max_pos(out + 1, md);
  }
}

__device__ double theta64(double ps) {
  const double pi = 3.14159265358979323846;
  ps = fmin(fmax(ps, 0.0), 2.0);
  return ps <= 1.0 ? atan2(ps, 1.0 - ps) : pi - atan2(2.0 - ps, ps - 1.0);
}

__global__ void selftest_tables(const EcaParams p, float pad, double* out) {
  __shared__ float2 tt[kTBins], at[kABins + 2], dt[kDBins];
  build_tables(p, pad, tt, at, dt);
  __syncthreads();
  const double pi = 3.14159265358979323846, u = ldexp(1.0, -24);
  auto T = [&](double q) { return tanh(sqrt(q) / 3.0 / p.gradient_threshold); };
  auto A = [&](double th) { return 2.0 / (1.0 + exp(2.0 * p.angle_scale * th)); };
  int bad = 0;
  for (int b = threadIdx.x; b < kTBins; b += blockDim.x) {
    const int e = b >> 5, m = b & 31;
    const double q_lo = b == 0 ? 1.0 : ldexp(1.0 + m / 32.0, e) * (1.0 - u);
    const double q_hi = ldexp(1.0 + (m + 1) / 32.0, e) * (1.0 + u);
    bad += double(tt[b].x) > T(q_lo) || (tt[b].y < 1.0f && double(tt[b].y) < T(q_hi));
  }
  for (int k = threadIdx.x; k < kABins; k += blockDim.x) {
    const double w = 2.0 / kABins;
    bad += double(at[k].x) > A(theta64((k + 1) * w + 2e-6)) ||
           (at[k].y < 1.0f && double(at[k].y) < A(theta64(k * w - 2e-6)));
  }
  if (threadIdx.x == 0) bad += double(at[kABins].x) > A(pi);
  for (int s = threadIdx.x; s < 766; s += blockDim.x) {
    const double d = 2.0 / (1.0 + exp(2.0 * (double(s) / 3.0) / p.intensity_threshold));
    bad += double(dt[s].x) > d || (dt[s].y < 1.0f && double(dt[s].y) < d);
  }
  if (bad) atomicAdd(out + 2, double(bad));
}
}  // namespace

extern "C" int eca_prefilter_selftest(const EcaParams* params, double* dev_out, void* stream) {
  ECA_RANGE("eca_prefilter_selftest");
  if (!params || !dev_out) return ECA_ERR_ARG;
  static const uint8_t dummy[16] = {};
  const int32_t row = 3;
  EcaParams q = *params;
  if (q.width < 8) q.width = 8;
  if (q.height < 14) q.height = 14;
  StripJob J;
  const int rc = prepare_strip_job(J, dummy, 0, 0, 3LL * q.width, &row, nullptr, 1, &q);
  if (rc) return rc;
  const PointsJob PJ = points_job(J, nullptr);
  const TermK tk{PJ.kt, PJ.kd};
  cudaStream_t st = as_stream(stream);
  selftest_terms<<<4 * sm_count(), 256, 0, st>>>(q, tk, dev_out);
  selftest_tables<<<1, 256, 0, st>>>(q, J.pad, dev_out);
  const double pad = J.pad;
  if (cudaMemcpyAsync(dev_out + 3, &pad, sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return ECA_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ECA_ERR_CUDA;
  return check_launch();
}
