/*
 * eca_b200.h — C ABI of the B200-native content-area hot path (libeca_b200.so).
 *
 * The reference (/root/reference/pkg/src/eca) is pure Python/numpy and has no
 * FFI of its own; these entry points are what its Python functions would bind
 * through ctypes.  Each declaration names the reference
 * function it replaces.
 *
 * Conventions
 *   - Frames are HWC uint8 RGB in DEVICE memory: pixel (b, y, x, c) lives at
 *     frames + b*frame_stride + y*row_stride + 3*x + c (bytes).  Any strides
 *     are accepted; contiguous frames use frame_stride = H*W*3, row_stride = W*3.
 *   - Every pointer except `params`, `strip_rows` and the host-helper outputs is
 *     a device pointer owned by the caller.  Device calls are asynchronous on
 *     `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - Return 0 on success or a negative ECA_ERR_* code; nothing throws and no
 *     call allocates device memory.
 *   - Candidate arrays are [batch][2*n_strips] in the reference's flatten
 *     order (estimator.py:69): every strip's left winner, then every right one.
 */
#ifndef ECA_B200_H
#define ECA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECA_OK 0
#define ECA_ERR_ARG (-1)         /* bad shape / size / pointer              */
#define ECA_ERR_CUDA (-2)        /* a CUDA launch or runtime call failed    */
#define ECA_ERR_UNSUPPORTED (-3) /* outside the supported envelope         */

#define ECA_MAX_STRIPS 128       /* 2*128 candidates per frame              */
#define ECA_MAX_WIDTH 4096
#define ECA_MAX_ATTEMPTS 8192

/* RejectionReason (fitting.py:18-36) plus acceptance, as stored in EcaFitRecord.status */
enum EcaStatus {
  ECA_ACCEPTED = 0,
  ECA_NO_CANDIDATES = 1,
  ECA_LOW_SCORE = 2,
  ECA_GEOMETRY_GATE = 3
};

/* POD view of EcaConfig (config.py:14-73) with the derived doubles precomputed
 * in the reference's evaluation order (params.py: EcaConfig.device_params). */
typedef struct EcaParams {
  int32_t width, height;
  int32_t strip_count, edge_margin_px;
  int32_t ransac_attempts, ransac_iterations;
  double gradient_threshold;     /* t_g                                      */
  double intensity_threshold;    /* t_i                                      */
  double angle_scale;            /* 180 / (pi * t_theta)   handcrafted.py:178 */
  double zero_grad_angle;        /* pi * angle_scale       handcrafted.py:182 */
  double min_point_score;        /* fitting.py:51                           */
  double inlier_tol;             /* inlier_distance_px / W fitting.py:189    */
  double circle_score_threshold; /* config.py:69-73                         */
  double min_radius_frac, max_radius_frac, max_center_offset_frac;
  double center_x, center_y;     /* fit reference point (fitting.py:186)     */
} EcaParams;

/* One frame's fit result; 40 bytes; also the NCCL gather record. */
typedef struct EcaFitRecord {
  double cx, cy, r;   /* pixels; 0 unless status == ECA_ACCEPTED */
  double score;       /* inlier score sum                         */
  int32_t inliers;
  int32_t status;     /* enum EcaStatus                           */
} EcaFitRecord;

/* ---------------------------------------------------------------- host ---- */

/* strip_heights (strips.py:41-60).  Writes <= count rows; returns how many
 * (after de-duplication) or ECA_ERR_ARG. */
int eca_strip_rows(int height, int count, double weighting, int32_t* out_rows);

/* _sample_triplets (fitting.py:147-156) for every n in [3, max_n]:
 * out[((n-3)*attempts + a)*3 + j], the three smallest PCG64 keys of attempt a
 * in ascending key order.  numpy default_rng(seed) stream, bit-exact. */
int eca_triplet_table(uint64_t seed, int attempts, int max_n, int16_t* out);

/* First `count` doubles of numpy.random.default_rng(seed).random() (test hook). */
int eca_pcg64_doubles(uint64_t seed, int64_t count, double* out);

/* FP32 prefilter tolerance of the handcrafted kernels for `params`: writes the
 * relative bound (4x the modelled FP32 error; every FP32 bound in the kernels
 * is padded outward by exactly this, rounded up to float) and returns 0, or
 * returns 1 when the config needs the all-FP64 path (FP32 range
 * insufficient, or a bound >= 1e-2).  No reference counterpart: it guards the
 * exactness of score_strips (handcrafted.py:148-205) on the GPU. */
int eca_prefilter_bound(const EcaParams* params, double* out_rel_bound);

/* Test hook: measures the FP32 bound terms against FP64 on the device for one
 * config.  dev_out (device, 4 doubles, zeroed): [0] max relative error of the
 * tanh term over every |3g|^2, [1] of the darkness term over every preceding
 * sum, [2] number of fused-kernel table entries that fail to bound their bin,
 * [3] the pad the kernels use.  Synchronises `stream`. */
int eca_prefilter_selftest(const EcaParams* params, double* dev_out, void* stream);

/* -------------------------------------------------------------- device ---- */

/* Every strip entry point takes `strip_rows` (the strip centre rows y, frame
 * coordinates: geometry) and optional `band_rows`: the memory row, within each
 * frame buffer, that holds row y-1 (handcrafted) / y-3 (learned).  NULL means
 * full frames (band = y-1 / y-3).  Non-NULL lets the kernels read compact
 * strip-row buffers produced by eca_h2d_bands. */

/* Frame ingest: copy rows [first_rows[k], first_rows[k]+rows_per_band) of every
 * HOST frame into dev as [batch][n_bands*rows_per_band][width][3] (packed),
 * one strided cudaMemcpy2DAsync per band (pinned host memory for async). */
int eca_h2d_bands(const uint8_t* host, int batch, int64_t host_frame_stride,
                  int64_t host_row_stride, const int32_t* first_rows, int n_bands,
                  int rows_per_band, int width, uint8_t* dev, void* stream);

/* Bytes of device workspace eca_points_handcrafted needs for (batch, n_strips).
 * Zero it once before first use (the kernels hand out work through a ticket
 * counter at its start and leave it zeroed); one launch at a time per workspace. */
int eca_points_workspace_bytes(int batch, int n_strips, int64_t* out_bytes);

/* score_frame_strips + select_candidates_batch, handcrafted variant
 * (estimator.py:35-52, handcrafted.py:148-205, 120-138).  With a workspace of
 * eca_points_workspace_bytes: bound-and-prune kernel + dense FP64 rescoring
 * kernel (fast); workspace == NULL: the block-per-strip kernel. */
int eca_points_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                           int64_t row_stride, const int32_t* strip_rows,
                           const int32_t* band_rows, int n_strips,
                           const EcaParams* params, int32_t* out_x, int32_t* out_y,
                           double* out_score, void* workspace, void* stream);

/* The two stages of eca_points_handcrafted (workspace required) as separate
 * launches.  eca_bounds_handcrafted writes the workspace (survivor slots) and
 * the candidates of the half rows it resolves itself (more than 8
 * survivors); eca_rescore_handcrafted completes out_*. */
#define ECA_BOUNDS_OVERLAP_PREVIOUS 1  /* flags: programmatic dependent launch - the
   grid may start while the previous kernel in `stream` drains; only when this
   call neither reads what that kernel writes nor writes what it reads (e.g. the
   previous batch's eca_bounds_handcrafted on another workspace/output set) */
#define ECA_BOUNDS_SHARE_SMS 2         /* flags: leave one CTA slot per SM free for
   kernels running concurrently on other streams (e.g. the previous batch's
   eca_rescore_handcrafted + eca_fit) */
#define ECA_BOUNDS_ZERO_COPY 4         /* flags: fetch each half strip row chunk by
   chunk (256 columns), only as far as the scan gets (the exact early exit stops
   most rows well before the centre).  For `frames` in pinned host memory
   (mapped, e.g. cudaHostAlloc / torch pin_memory) this reads the strip rows
   straight over PCIe and only the visited columns cross it; the workspace's
   third int32 (offset 8) accumulates the 16-byte units fetched. */
int eca_bounds_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                           int64_t row_stride, const int32_t* strip_rows,
                           const int32_t* band_rows, int n_strips,
                           const EcaParams* params, int32_t* out_x, int32_t* out_y,
                           double* out_score, void* workspace, int flags, void* stream);
int eca_rescore_handcrafted(int batch, const int32_t* strip_rows, int n_strips,
                            const EcaParams* params, int32_t* out_x, int32_t* out_y,
                            double* out_score, void* workspace, void* stream);

/* Streamed throughput mode, two launches per batch on the caller's stream
 * (what ContentAreaEngine.run_pipelined does; estimator.py:85-111 over a
 * stream of batches): the bound-and-prune kernel (survivor columns) and the
 * fit kernel (a warp per frame: FP64 rescore of the survivors -> candidates,
 * then filter + RANSAC), both programmatic dependent launches: a batch's
 * bounds CTAs start in the previous batch's tail and its fits run beside the
 * next batch's bounds kernel.  4 buffer sets rotate in the caller's device
 * `scratch` (eca_pipeline_bytes; zeroed by create); each launch claims its set
 * on the device and waits for the launches that used it before, so the
 * records of step i stay valid until step i+4.  Same records as
 * eca_points_handcrafted + eca_fit.  One host thread per pipeline. */
typedef struct EcaPipeline EcaPipeline;
#define ECA_PIPE_FRAMES_READY 8   /* flags: the frames were complete before the
   previous operation in `stream` was enqueued (e.g. a pre-filled pool, or
   host frames): skip the kernel's griddepcontrol.wait on the previous kernel,
   which otherwise protects frames written by the kernel just before */
int eca_pipeline_bytes(int batch, int n_strips, int64_t* out_bytes);
int eca_pipeline_create(int batch, int height, int width, const int32_t* strip_rows,
                        int n_strips, const EcaParams* params, const int16_t* triplets,
                        void* scratch, int64_t scratch_bytes, EcaPipeline** out);
/* Enqueue one batch on `stream`; *out_records = this step's device records
 * (batch x 40 B), complete in `stream` order (other streams: eca_pipeline_fence).
 * flags: ECA_BOUNDS_ZERO_COPY (frames in pinned host memory, read over PCIe
 * chunk by chunk; they must stay unchanged until the step completes) and / or
 * ECA_PIPE_FRAMES_READY.  host_records (optional, mapped pinned memory): the
 * final stage also stores each frame's record there. */
int eca_pipeline_step(EcaPipeline* pipeline, const uint8_t* frames, int64_t frame_stride,
                      int64_t row_stride, int flags, EcaFitRecord* host_records, void* stream,
                      EcaFitRecord** out_records);
/* n_steps eca_pipeline_step calls in one native call (a host-light stream
 * loop): step j takes the batch at pool + ((first_slot + j) % n_slots) *
 * batch_stride.  Records: eca_pipeline_records. */
int eca_pipeline_run(EcaPipeline* pipeline, const uint8_t* pool, int64_t batch_stride, int n_slots,
                     int first_slot, int n_steps, int64_t frame_stride, int64_t row_stride,
                     int flags, void* stream);
/* The device records of the step `back` steps before the latest one
 * (0 <= back < 4 and < the steps so far). */
int eca_pipeline_records(EcaPipeline* pipeline, int back, EcaFitRecord** out_records);
/* Kept for API stability: steps carry no host-side history (a no-op). */
int eca_pipeline_reset(EcaPipeline* pipeline);
/* Make `stream` wait for every step enqueued so far. */
int eca_pipeline_fence(EcaPipeline* pipeline, void* stream);
/* The stream of the latest step (where its records complete). */
int eca_pipeline_side_stream(EcaPipeline* pipeline, void** out_stream);
/* Synchronises the latest step's stream, releases the pipeline (not the scratch). */
int eca_pipeline_destroy(EcaPipeline* pipeline);

/* estimate_batch (estimator.py:85-111) for a batch of same-size frames:
 * bound-and-prune + the fit kernel (FP64 rescore stage, filter, RANSAC),
 * plain stream order.  workspace: eca_points_workspace_bytes(batch, n_strips),
 * zeroed once (left re-armed).  host_out: optional mapped pinned records,
 * written by the fit kernel.  flags: 0 or ECA_BOUNDS_ZERO_COPY. */
int eca_estimate_batch_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                                   int64_t row_stride, const int32_t* strip_rows,
                                   const int32_t* band_rows, int n_strips,
                                   const EcaParams* params, const int16_t* triplets,
                                   void* workspace, int32_t* out_x, int32_t* out_y,
                                   double* out_score, EcaFitRecord* out, EcaFitRecord* host_out,
                                   int flags, void* stream);

/* Same, plus every column's FP64 score: out_scores[batch][n_strips][width]
 * (StripScoreRow.scores, handcrafted.py:25-31). */
int eca_score_rows_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                               int64_t row_stride, const int32_t* strip_rows,
                               const int32_t* band_rows, int n_strips,
                               const EcaParams* params, double* out_scores, int32_t* out_x,
                               int32_t* out_y, double* out_score, void* stream);

/* filter_candidates + ransac_fit (fitting.py:39-52, 159-230) per frame.
 * triplets: device copy of eca_triplet_table(seed, attempts, n_cand) (ignored
 * when exhaustive != 0, which enumerates all C(n,3) triplets in order). */
int eca_fit(const int32_t* cand_x, const int32_t* cand_y, const double* cand_score,
            int batch, int n_cand, const EcaParams* params, const int16_t* triplets,
            int exhaustive, EcaFitRecord* out, void* stream);

/* estimate() for a small batch (the latency path; estimator.py:55-74): strip
 * scoring with the survivors rescored in FP64 by the same warp, candidates,
 * then filter + RANSAC in a fit kernel launched programmatically behind it.
 * `counters` = max(batch, 64) int32 zeros (scratch: left zeroed on return).
 * The candidate outputs double as the fitter's input.  `out` may be mapped
 * pinned host memory: each record's status word is written last, after a
 * system-scope fence, so a host that set it to a value outside EcaStatus can
 * poll it instead of synchronising the stream.  (ECA_LATENCY_STRIP=1 in the
 * environment: the older single launch, a block-per-strip kernel whose last
 * CTA per frame fits it; no ordered store.) */
int eca_estimate_handcrafted(const uint8_t* frames, int batch, int64_t frame_stride,
                             int64_t row_stride, const int32_t* strip_rows,
                             const int32_t* band_rows, int n_strips,
                             const EcaParams* params, const int16_t* triplets,
                             int32_t* counters, int32_t* out_x, int32_t* out_y,
                             double* out_score, EcaFitRecord* out, void* stream);

/* ---- learned variant (edgenet.py:67-83, 100-116, 182-233, 347-370) ---- */

/* Packed FP32 weights: k0[8*5*9] b0[8] k1[16*8*9] b1[16] k2[32*16*9] b2[32]
  * k3[32] b3[1] (reference (out,in,kh,kw) order) = 6209 floats; norm = mean[3], std[3]. */
#define ECA_NET_FLOATS 6209
int eca_points_learned(const uint8_t* frames, int batch, int64_t frame_stride,
                       int64_t row_stride, const int32_t* strip_rows,
                       const int32_t* band_rows, int n_strips,
                       int height, int width, const float* weights, const double* norm,
                       float* out_probs /* [batch][n_strips][width-6] */,
                       int32_t* out_x, int32_t* out_y, double* out_score, void* stream);

/* Same with flags.  Default (0) / ECA_LEARNED_TCGEN05: the three 3x3 layers
 * on the tensor cores (tcgen05 kind::tf32, 3xTF32 split: FP32-level error,
 * DESIGN.md K3); ECA_LEARNED_SIMT: the CUDA-core kernel (FP32 FMA). */
#define ECA_LEARNED_TCGEN05 1
#define ECA_LEARNED_SIMT 2
int eca_points_learned_ex(const uint8_t* frames, int batch, int64_t frame_stride,
                          int64_t row_stride, const int32_t* strip_rows,
                          const int32_t* band_rows, int n_strips, int height, int width,
                          const float* weights, const double* norm, int flags,
                          float* out_probs, int32_t* out_x, int32_t* out_y, double* out_score,
                          void* stream);

/* -------------------------------------------------------- mask / crop ---- */

/* Vectorised circle_contains (geometry.py:30-34): out[b][y][x] = 1 inside the
 * closed disk of an ACCEPTED record, all ones otherwise (FullFrame). */
int eca_draw_mask(const EcaFitRecord* fits, int batch, int height, int width,
                  uint8_t* out, int64_t out_frame_stride, void* stream);

/* crop_augment bounds (dataset.py:151-187): out_bounds[b] = {x0, y0, x1, y1}
 * inclusive, or {-1,-1,-1,-1} when the reference returns None / the record is
 * not ACCEPTED. */
int eca_crop_bounds(const EcaFitRecord* fits, int batch, int height, int width,
                    int32_t* out_bounds, void* stream);

/* Copy each frame's rectangle (bounds from eca_crop_bounds) to
 * out + out_offsets[b] as a packed HWC crop; max_rows >= the tallest crop. */
int eca_crop_copy(const uint8_t* frames, int batch, int64_t frame_stride, int64_t row_stride,
                  const int32_t* bounds, const int64_t* out_offsets, uint8_t* out,
                  int max_rows, void* stream);

/* ------------------------------------------------ evaluation */

/* Normalised-Hausdorff evaluation (metrics.py:148-213).  A record with status
 * ECA_ACCEPTED is a circle, anything else the full frame (metrics.as_circle).
 * Per sample b (dims[2b] = width, dims[2b+1] = height, each <= max_*):
 * out_hd[b] = hausdorff(boundary_points(pred[b]), boundary_points(truth[b]))
 * (metrics.py:193-203: exact FP64 distances, no KD-tree), or NaN with
 * out_status[b] != 0: bit 0 / bit 1 = the prediction's / truth's boundary is
 * empty (a circle that misses the frame: the reference raises ValueError).
 * The caller scales by REF_DIAGONAL / hypot(W, H) (metrics.py:206-208). */
int eca_nh_workspace_bytes(int batch, int max_width, int max_height, double spacing,
                           int64_t* bytes);
int eca_area_hausdorff(const EcaFitRecord* pred, const EcaFitRecord* truth, const int32_t* dims,
                       int batch, int max_width, int max_height, double spacing, void* workspace,
                       int64_t workspace_bytes, double* out_hd, int32_t* out_status, void* stream);

/* boundary_points (metrics.py:148-176) of one area: out_xy[2i], out_xy[2i+1];
 * *out_count = the number of samples (nothing is written when it exceeds cap;
 * 0: the circle does not intersect the frame). */
int eca_boundary_points(const EcaFitRecord* area, int width, int height, double spacing,
                        double* out_xy, int cap, int32_t* out_count, void* stream);

/* hausdorff(a, b) (metrics.py:193-203) of two device point sets [n][2] f64. */
int eca_hausdorff_workspace_bytes(int max_points, int64_t* bytes);
int eca_hausdorff_points(const double* a, int na, const double* b, int nb, void* workspace,
                         int64_t workspace_bytes, double* out_hd, int32_t* out_status,
                         void* stream);

/* ------------------------------------------- learned training */

/* EdgeNet training pieces (edgenet.py:100-130, 182-211, 213-225, 236-241,
 * 277-344), FP32.  x: [*][5][h][w] float32 RGBXY samples (NCHW, the
 * reference's training inputs), targets: [*][1][h-6][w-6]; index: the m
 * sample indices of this batch, each < the number of samples in x / targets
 * (device int32; null: samples 0..m-1).  net: ECA_NET_FLOATS
 * packed weights (kernel0, bias0, ..., kernel3, bias3 in reference order).
 * forward keeps the activations (the reference's caches) and the packed
 * tensor-core weight operands in the workspace; backward (after forward on
 * the same batch, weights and workspace) writes the mean stable BCE loss
 * (FP64), the packed gradients (out_grads null: the loss only), and sets
 * *diverged = 1 on a non-finite loss (diverged may be null).  The
 * convolutions run on tcgen05 (3xTF32, eca_train_tc.cuh); ECA_TRAIN_SIMT=1
 * selects the CUDA-core kernels.
 * eca_sgd_step: net -= fl32(lr) * grads, skipped while *diverged != 0. */
int eca_train_workspace_bytes(int m, int h, int w, int64_t* bytes);
int eca_edgenet_forward(const float* x, const int32_t* index, int m, int h, int w, const float* net,
                        void* workspace, int64_t workspace_bytes, float* out_logits, void* stream);
int eca_edgenet_backward(const float* x, const float* targets, const int32_t* index, int m, int h,
                         int w, const float* net, void* workspace, int64_t workspace_bytes,
                         float* out_grads, double* out_loss, int32_t* diverged, void* stream);
int eca_sgd_step(float* net, const float* grads, float lr, const int32_t* diverged, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ECA_B200_H */
