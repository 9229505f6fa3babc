/* pf_b200.h — C ABI of the B200-native pose-parsing hot path.
 *
 * The reference (poseflow, /root/reference/pkg/src/poseflow) is pure
 * Python; it has no FFI of its own.  This ABI replaces, one-for-one, the
 * functions on its hot path:
 *
 *   pf_parse_device / pf_parse_host  <- paf.parse                (paf.py:292-305)
 *                                        incl. nms_peaks           (paf.py:74-109)
 *                                        connect_limbs/score_limb  (paf.py:112-199)
 *                                        assemble_humans           (paf.py:210-289)
 *                                        cell_to_pixel             (types.py:233-235)
 *   pf_params                        <- ParserParams               (paf.py:34-54)
 *   pf_set_topology                  <- SkeletonTopology           (types.py:81-166)
 *   pf_preprocess_device             <- make_preprocess.fn         (operators.py:114-131)
 *                                        + read_ppm u8/255         (formats.py:116-117)
 *                                        + bilinear_resize 3-D     (operators.py:79-107)
 *   pf_resize_device                 <- bilinear_resize 2-D, per channel (operators.py:79-107)
 *
 * Plain pointers and sizes only; no torch types.  The Python host layer
 * (paper_2108_11826_b200.parser / .pipeline_ops) binds this with ctypes and
 * mirrors the reference API; INTEGRATION.md shows the binding a poseflow
 * maintainer would add.
 *
 * Status codes map onto the reference exception hierarchy (errors.py):
 *   PF_ERR_CONFIG   -> ConfigError   (raised before any work, like paf.py:295)
 *   PF_ERR_CONTRACT -> ContractError (types.py:185-205, operators.py:83, :121)
 *   PF_ERR_CAPACITY -> a frame exceeded a capacity; never silently truncated
 *   PF_ERR_CUDA     -> CUDA runtime failure
 * pf_last_error() returns the message of the last failing call.
 *
 * Threading: one pf_ctx per (device, stream).  Distinct contexts may be
 * used concurrently from different threads; one context is not reentrant.
 * Device entry points are asynchronous on the context stream; results are
 * valid after pf_sync()/pf_get_results().
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_ERR_CONFIG 1
#define PF_ERR_CONTRACT 2
#define PF_ERR_CAPACITY 3
#define PF_ERR_CUDA 4

#define PF_MAX_KEYPOINTS 32
#define PF_MAX_LIMBS 64
#define PF_ABI_VERSION 1

typedef struct pf_ctx pf_ctx;

/* ParserParams (paf.py:34-42) plus two B200-path knobs:
 *   upsample   — 1: parse on the feature grid (the reference as-is);
 *                u>1: every map is bilinear-resized x u (operators.py:79-107)
 *                before parsing, coordinates in grid*u space (stride/u).
 *   blur_sigma — 0: off (identity).  >0: separable Gaussian on the part
 *                confidence maps after upsampling (no reference). */
typedef struct pf_params {
    double conf_threshold;        /* [0,1], compared in fp32 (numpy NEP 50) */
    int32_t nms_window;           /* odd, >= 3 */
    int32_t n_samples;            /* >= 2 */
    double sample_dot_threshold;  /* [0,1] */
    double good_fraction_min;     /* [0,1] */
    int32_t min_parts;            /* >= 1 */
    double min_human_score;
    int32_t upsample;             /* >= 1, stride % upsample == 0 */
    double blur_sigma;            /* >= 0 */
} pf_params;

/* Capacities of the context workspaces (0 = default).  Exceeding one sets
 * PF_ERR_CAPACITY for the call with the offending frame index. */
typedef struct pf_caps {
    int32_t max_peaks_per_part;    /* default 128 */
    int32_t max_peaks_per_frame;   /* default 256 (automatic caps grow on demand) */
    int32_t max_candidates;        /* gated candidate pairs per frame, default 4096 */
    int32_t max_humans_per_frame;  /* builders per frame before filtering, default 64 */
    int32_t chunk_frames;          /* frames per internal launch chunk, default 8192 */
    int32_t max_humans_total;      /* output pool per call, default 64 * batch */
} pf_caps;

/* Results of the last parse call, in context-owned pinned host memory,
 * valid until the next parse on the same context.  Humans of frame f are
 * entries frame_first[f] .. frame_first[f] + frame_count[f] - 1, already in
 * the reference output order (score descending, stable, paf.py:288).  The
 * placement of whole frames inside the pool is unspecified (frames reserve
 * their slots concurrently); always address a frame through frame_first. */
typedef struct pf_results {
    int32_t n_frames;
    int32_t n_keypoints;
    int32_t total_humans;
    const int32_t *frame_first;    /* [n_frames] */
    const int32_t *frame_count;    /* [n_frames] */
    const double *human_score;     /* [total] */
    const int32_t *human_n_parts;  /* [total] */
    const double *kp_x;            /* [total * K]  cell_to_pixel x */
    const double *kp_y;            /* [total * K] */
    const float *kp_score;         /* [total * K]  peak value (fp32) */
    const int32_t *kp_peak;        /* [total * K]  per-frame peak id, -1 = absent */
} pf_results;

int pf_abi_version(void);

int pf_create(pf_ctx **out, int device, const pf_caps *caps);
void pf_destroy(pf_ctx *ctx);
const char *pf_last_error(const pf_ctx *ctx);

/* Bind the context to a CUDA stream (cudaStream_t passed as void*; NULL is
 * the legacy default stream, e.g. torch's default stream).  A new context
 * uses its own non-blocking stream; pf_use_own_stream() returns to it. */
int pf_set_stream(pf_ctx *ctx, void *cuda_stream);
int pf_use_own_stream(pf_ctx *ctx);

/* SkeletonTopology (types.py:81-166): limbs and paf_channels are [L][2]. */
int pf_set_topology(pf_ctx *ctx, int n_keypoints, int n_limbs,
                    const int32_t *limbs, const int32_t *paf_channels);

/* ParserParams.validate (paf.py:44-54) + the two extension knobs. */
int pf_validate_params(const pf_params *p);

/* Parse `batch` frames whose maps are resident on the device:
 * conf [batch][K+1][grid_h][grid_w], paf [batch][2L][grid_h][grid_w],
 * contiguous f32 (FeatureMaps layout, types.py:169-205).  Asynchronous.
 * The maps must stay valid until pf_get_results() returns: when the
 * auto-sized output pool (max_humans_total = 0) overflows, the call is
 * replayed once with a pool of the exact size instead of failing. */
int pf_parse_device(pf_ctx *ctx, const float *conf, const float *paf, int batch,
                    int grid_h, int grid_w, int stride, const pf_params *p);

/* Same, from HOST buffers (pinned for full overlap): H2D copies are
 * chunked and overlapped with the kernels; returns after results are on
 * the host (implies pf_get_results). */
int pf_parse_host(pf_ctx *ctx, const float *conf, const float *paf, int batch,
                  int grid_h, int grid_w, int stride, const pf_params *p,
                  pf_results *out);

/* Caller-owned results of pf_parse_batch: device (or
 * mapped pinned) arrays the caller allocates for max_humans slots per frame,
 * humans of frame f in slots [f][0 .. n_humans[f]) in the reference output
 * order (paf.py:288).  kp_xy holds cell_to_pixel (x, y) (types.py:233-235),
 * kp_score the peak value, kp_present 1 where the keypoint exists.
 * status[0]: PF_OK, or PF_ERR_CAPACITY when a frame had more than max_humans
 * humans (n_humans[f] is still its true count, only max_humans slots are
 * written) or an internal capacity overflowed (all n_humans 0); status[1]:
 * the smallest such frame, -1 if none. */
typedef struct pf_out {
    int32_t max_humans;      /* slots per frame (Hmax) */
    int32_t *n_humans;       /* [B] */
    double *human_score;     /* [B][Hmax] */
    int32_t *n_parts;        /* [B][Hmax] */
    double *kp_xy;           /* [B][Hmax][K][2] */
    float *kp_score;         /* [B][Hmax][K] */
    uint8_t *kp_present;     /* [B][Hmax][K] */
    int32_t *status;         /* [2] */
} pf_out;

/* The batch entry point of the §8(b) boundary: parse `batch` device-resident
 * frames (layout as pf_parse_device) into the caller-owned `out`, enqueued on
 * `cuda_stream` (cudaStream_t as void*; NULL = the context's stream) and
 * asynchronous: `out` is valid, and the maps may be released, once that
 * stream reaches this point.  Nothing is replayed (capacity overflows are
 * reported in out->status instead); errors raised before any work are
 * returned, as the reference raises before work (paf.py:295). */
int pf_parse_batch(pf_ctx *ctx, const float *conf, const float *paf, int batch,
                   int grid_h, int grid_w, int stride, const pf_params *p,
                   const pf_out *out, void *cuda_stream);

/* Wait for the last parse and expose its results (D2H of the compact pool). */
int pf_get_results(pf_ctx *ctx, pf_results *out);

/* Caller-owned host results: the same as pf_get_results, with the D2H copies
 * going straight into the caller's arrays (pinned for full speed) instead of
 * the context's buffers, so they outlive the next call.  frame_first /
 * frame_count hold n_frames entries, the human arrays `capacity` humans
 * (kp_* capacity * K).  If the call produced more than `capacity` humans the
 * function returns PF_ERR_CAPACITY with *total_humans set to the need and
 * nothing else written; call again with larger arrays (the parse is not
 * repeated). */
typedef struct pf_host_out {
    int32_t capacity;
    int32_t *frame_first;          /* [n_frames] */
    int32_t *frame_count;          /* [n_frames] */
    double *human_score;           /* [capacity] */
    int32_t *human_n_parts;        /* [capacity] */
    double *kp_x;                  /* [capacity * K] */
    double *kp_y;                  /* [capacity * K] */
    float *kp_score;               /* [capacity * K] */
    int32_t *kp_peak;              /* [capacity * K] */
} pf_host_out;
int pf_get_results_into(pf_ctx *ctx, const pf_host_out *dst, int32_t *n_frames, int32_t *total_humans);

/* Wait for all work on the context stream. */
int pf_sync(pf_ctx *ctx);

/* Stage intermediates of the last parse for per-stage parity checks
 * (requires pf_set_debug(ctx, 1) before the parse).  Peaks in id order:
 * part, row, col, score; connections in connect_limbs order: limb, id_a,
 * id_b, score, good_fraction.  Returns counts through n_*; pass NULL
 * arrays to query counts only. */
int pf_set_debug(pf_ctx *ctx, int enable);

/* Options: PF_OPT_DEBUG (= pf_set_debug), PF_OPT_TIMING (CUDA events around
 * every kernel launch, read with pf_get_kernel_times), PF_OPT_MATERIALISE
 * (force the unfused Mode U path: resize -> [blur] -> NMS over HBM maps). */
#define PF_OPT_DEBUG 1
#define PF_OPT_TIMING 2
#define PF_OPT_MATERIALISE 3
#define PF_OPT_GENERIC_FUSED 4   /* use the shared-memory tile kernel for Mode U */
#define PF_OPT_WIN_VARIANT 5     /* Mode U 3x3 kernel: 4 corner-pruned (default); 1-3: the strip kernel */
#define PF_OPT_NO_CHAIN 6        /* corner kernel: disable the chain pre-filter (A/B parity checks) */
#define PF_OPT_CORNER_SPLIT 9    /* Mode U 3x3: survivors classified by a second kernel;
                                    0 off, 1 auto (batches of >= 32 frames, or planes too large
                                    for the one-kernel form; default), 2 always */
#define PF_OPT_CONF_ZERO_COPY 11 /* pf_parse_host: NMS kernels read a pinned host conf in place (default 0) */
#define PF_OPT_PARSE_SPLIT 10    /* line integral over all frames' pairs in its own kernel;
                                    0 off, 1 auto (batches of >= 32 frames, default), 2 always */
#define PF_OPT_PAF_ZERO_COPY 8   /* pf_parse_host (default 1): a pinned host PAF is read in place by the
                                    parse kernel, so only the sampled cells cross PCIe; 0: copy it whole */
#define PF_OPT_PDL 12             /* bitmask: programmatic dependent launch per split-kernel launch site
                                    (process-wide A/B; default: only the small-batch wide parse, bit 6 --
                                    every edge of the big-batch split path measured slower) */
#define PF_OPT_COUNT_PAF 13       /* instrumented parse: count the 32-byte PAF sectors the line integral
                                    reads (one-kernel parse; read with pf_get_paf_sectors) */
#define PF_OPT_LARGE 15           /* 1: parse through the large-frame kernel (HBM tables, 32-bit ids), the
                                    path the context switches to by itself when a frame outgrows the
                                    shared-memory capacities (more than 32767 peaks, ...); 0: usual path */
#define PF_OPT_HOST_OVERLAP 16    /* pf_parse_host (default 1): the NMS stage of chunk c+1 on the context
                                    stream beside the parse of chunk c on a second stream (the in-place
                                    PAF parse waits on PCIe read requests, the NMS stage on the SMs);
                                    0: one compute stream */
#define PF_OPT_EXACT_LIST 17      /* split Mode U 3x3: the finish hands its candidates to k_corner_exact
                                   * (0 = default: batches of >= 4096 planes; -1 = off: the finish tests them itself;
                                   * N > 0 = at most N list entries, the rest tested in the finish) */
int pf_set_option(pf_ctx *ctx, int option, int value);

/* With PF_OPT_COUNT_PAF on: distinct 32-byte PAF sectors the last parse call
 * sampled, summed over its frames (= the PCIe read bytes / 32 of an in-place
 * pinned PAF, each sector fetched once). */
int pf_get_paf_sectors(pf_ctx *ctx, long long *sectors);

/* Per-kernel device time (ms, CUDA events on the launching stream) and launch
 * counts accumulated since the last reset; ids index pf_kernel_name(). */
#define PF_N_KERNELS 17
const char *pf_kernel_name(int id);
int pf_get_kernel_times(pf_ctx *ctx, double *ms, int64_t *launches, int reset);
int pf_get_peaks(pf_ctx *ctx, int frame, int *n_peaks, int32_t *part, int32_t *row,
                 int32_t *col, float *score);
int pf_get_connections(pf_ctx *ctx, int frame, int *n_conns, int32_t *limb,
                       int32_t *id_a, int32_t *id_b, double *score, double *good);

/* Pre-processing (operators.py:114-131): u8 HWC [batch][h][w][3] (device)
 * -> f32 CHW [batch][3][out_h][out_w] (device).  Same size = layout only. */
int pf_preprocess_device(pf_ctx *ctx, const uint8_t *src, int batch, int h, int w,
                         float *dst, int out_h, int out_w);

/* Same, for already-normalised f32 HWC frames (a reference Frame image,
 * types.py:57-72): layout permutation or fp64 bilinear resize only. */
int pf_preprocess_f32_device(pf_ctx *ctx, const float *src, int batch, int h, int w,
                             float *dst, int out_h, int out_w);

/* bilinear_resize 2-D branch per channel: [n_planes][in_h][in_w] ->
 * [n_planes][out_h][out_w] (device). */
int pf_resize_device(pf_ctx *ctx, const float *src, int n_planes, int in_h, int in_w,
                     float *dst, int out_h, int out_w);

/* The smoothing taps used for blur_sigma > 0: radius
 * r = ceil(3 sigma), w_k = exp(-k^2 / (2 sigma^2)) / sum, k = -r..r.  Writes
 * 2r+1 taps (if cap allows) and returns r, or -1 for an invalid sigma. */
int pf_gaussian_taps(double sigma, double *taps, int cap);

/* Synthetic feature maps on the device (the reference synthetic backend's
 * render_feature_maps, synth.py:93-183): kp_cells [frames][max_humans][K][2]
 * (row, col) keypoint cells, NaN = missing; n_humans [frames]; outputs conf
 * [frames][K+1][grid_h][grid_w] and paf [frames][2L][grid_h][grid_w], all
 * device pointers, on the context's stream.  Input generation for tests and
 * benchmarks (a GPU-resident producer); fp64 exp() may differ from numpy's
 * in the last bit, so maps agree with the host renderer up to fp32 rounding
 * boundaries. */
int pf_render_maps(pf_ctx *ctx, const double *kp_cells, const int32_t *n_humans, int frames, int max_humans,
                   int grid_h, int grid_w, double sigma, double halfwidth, float *conf, float *paf);

/* Overlay rasteriser (the reference's visualize, poseflow/operators.py:173-290).
 * Primitives in draw order per frame (later overwrite earlier): kind 0 = line
 * (x0,y0)-(x1,y1) Bresenham-stamped with discs of radius r (thickness // 2);
 * kind 1 = disc at (x0,y0) of radius r (r = 0: one pixel, for label glyphs).
 * rgb is the colour as stored in the f32 image. */
typedef struct {
    int32_t frame, kind, x0, y0, x1, y1, r;
    float rgb[3];
} pf_overlay_prim;
/* prims / prim_first ([frames + 1], frame f owns prims[prim_first[f] ..
 * prim_first[f+1])) and img ([frames][h][w][3] f32, drawn in place) are
 * device pointers; runs on the context's stream. */
int pf_overlay(pf_ctx *ctx, const pf_overlay_prim *prims, const int32_t *prim_first, int n_prims, int frames,
               int h, int w, float *img);

/* Pinned host allocation helpers for callers without their own allocator. */
void *pf_host_alloc(size_t bytes);
void pf_host_free(void *p);

/* Kernel launches issued by this context since creation (evidence counter). */
int64_t pf_launch_count(const pf_ctx *ctx);

/* poses.jsonl for a batch (replaces a Python loop over
 * poseflow/operators.py:293-310 pose_record): one line per frame, seq ids
 * seq_base + f, byte-identical to json.dumps(..., separators=(",", ":")) with
 * CPython float repr.  Inputs are the pf_results SoA arrays (host) and the K
 * keypoint names.  Writes the lines to out if cap is large enough and returns
 * their byte length (call with out = NULL to size the buffer); -1 on bad
 * arguments.  Host-only: needs no device. */
long long pf_format_records(int n_frames, int n_keypoints, const int32_t *frame_first, const int32_t *frame_count,
                            const double *human_score, const double *kp_x, const double *kp_y,
                            const float *kp_score, const int32_t *kp_peak, const char *const *part_names,
                            long long seq_base, char *out, long long cap);
/* One double formatted as CPython repr() (NUL-terminated); length or -1. */
int pf_format_float(double v, char *out, int cap);

#ifdef __cplusplus
}
#endif
#endif
