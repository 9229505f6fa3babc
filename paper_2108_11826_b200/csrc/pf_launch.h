// pf_launch.h — internal launch interface between the C ABI (pf_capi.cu)
// and the kernel translation units.
#pragma once

#include "pf_common.cuh"

namespace pf {

// Programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl may start while its predecessor on the stream drains; it runs
// its input-independent prologue, then pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible.  pdl_trigger()
// lets the successor be scheduled before this grid exits.  Both are no-ops
// for an ordinary launch.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// PF_OPT_PDL: bit i allows programmatic dependent launch for launch site i
// (process-wide; see kPdl*).  Measured on the C5 step: every edge on costs
// 1.99 ms/step against 1.40 ms with none (the early-resident dependents slow
// the running grid), so the default is 0.
extern int g_pdl_mask;
enum PdlSite { kPdlFinish = 0, kPdlCrowded, kPdlParsePeaks, kPdlPairScan, kPdlScorePairs, kPdlParseFrames,
               kPdlParseWide };

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int site, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (g_pdl_mask >> site) & 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
#endif

// One output coordinate of operators.bilinear_resize packed for a single
// 16-byte load: i0 | i1 << 16, t (1 - t is recomputed: the host's omt is the
// same single rounded subtraction).
struct __align__(16) AxisRec {
    int32_t i01;
    int32_t pad;
    double t;
};
// pf_nms.cu
struct UpArgs {
    const float *conf;
    int C, K, h, w;
    int H, W;
    AxisTab rows, cols;
    float thr;
    int half;
    int band_rows;
    int n_bands;
    int cap;
    int *counts;
    uint2 *peaks;
};
constexpr int kMaxFusedHalf = 16;
struct UpWinArgs {
    const float *conf;   // low-res [B][C][h][w]
    int C, K, h, w;
    int H, W;            // parse grid
    double ry, rx;       // h/H, w/W (operators.py:88-89 ratios)
    float thr;
    int half;            // 1 or 2
    int cap;
    int *counts;
    uint2 *peaks;
    const int32_t *first_out, *last_out;   // [h]: output rows reading source row r
};
size_t nms_up_win_smem(int h, int w, int H, int threads);

// Per band, fp32 copies of the axis weights the corner kernel's classification
// uses (filled in-kernel from the axis tables).
struct BandT {
    float omt_f, t_f, omt_l, t_l;   // (1 - t), t at the band's first and last output
    float s_l, s_f, dt, pad;        // t step into the last output, out of the first; min step
};

// k_nms_up_corner (pf_corner.cu): exact slope-pruned fused upsample + 3x3 NMS,
// persistent, planes streamed by 1-D bulk copies.  Canonical bands only
// (band b reads sources b-1, b: any integer upsample of a >= 2 wide axis).
struct UpCornerArgs {
    const float *conf;   // low-res [B][C][h][w]
    int B, C, K, h, w;
    int H, W;
    float thr;
    int cap;
    int *counts;
    uint2 *peaks;
    AxisTab rows, cols;                  // per output row / column
    const int4 *rband, *cband;           // bands: (first, last, src0, src1)
    const double *rdt, *cdt;             // per band: min t step between adjacent outputs
    int nbr, nbc;                        // band counts (h + 1, w + 1)
    int max_band;                        // widest band (outputs) of either axis
    int nst;                             // plane stages in shared memory
    int bulk;                            // set by the launcher: planes fetched by cp.async.bulk
    int chain;                           // chain pre-filter allowed (output t steps >= 2^-5)
    const AxisRec *rrec, *crec;          // packed per-output axis records
    uint32_t *cand_spill;                // [grid][kCornerSpill] candidate overflow slab (or null)
    uint32_t *surv_out;                  // split mode: [B*K][kCornerSurv] chain survivors (or null)
    int *surv_n;                         // split mode: [B*K] survivor counts, -1 = plane finished,
                                         //   sign bit = crowded (low bits: survivors)
    int *crowd_list, *crowd_n;           // split mode: crowded planes (compact) and their count
    uint2 *exact_list;                   // split mode: (plane, y << 16 | x) candidates for k_corner_exact (or null)
    int *exact_n;                        //   their count (zeroed before the scan)
    int exact_cap;
};
cudaError_t launch_corner_exact(const UpCornerArgs &a, cudaStream_t s);
size_t corner_exact_entries_per_plane();
cudaError_t launch_corner_finish(const UpCornerArgs &a, cudaStream_t s);
cudaError_t launch_corner_crowded(const UpCornerArgs &a, cudaStream_t s);
cudaError_t launch_nms_up_scan(const UpCornerArgs &a, cudaStream_t s);
size_t corner_surv_entries_per_plane();
size_t nms_up_corner_spill_entries(int max_ctas);
size_t nms_up_corner_smem(int h, int w, int nbr, int nbc, int nst);
size_t nms_up_scan_smem(int h, int w, int nst);
size_t nms_up_scan_launch_smem(int h, int w);   // the shared memory launch_nms_up_scan requests
#ifndef PF_CORNER_STAGES
#define PF_CORNER_STAGES 1
#endif
constexpr int kCornerStages = PF_CORNER_STAGES;
cudaError_t launch_nms_up_corner(const UpCornerArgs &a, cudaStream_t s);
cudaError_t configure_corner_kernels(int max_smem);
cudaError_t launch_nms_up_win(const UpWinArgs &a, int B, cudaStream_t s);
cudaError_t launch_nms_plane(const float *conf, int B, int C, int K, int H, int W, float thr,
                             int half, int cap, int *counts, uint2 *peaks, cudaStream_t s);
size_t nms_up_smem(int n_src_max, int w, int half, int band_rows, int W);
cudaError_t launch_nms_up(const UpArgs &a, int B, size_t smem, cudaStream_t s);
cudaError_t configure_nms_kernels(int max_smem);

// pf_parse.cu
struct ParseArgs {
    Topo topo;
    const float *paf;
    int h, w;
    int up;
    AxisTab rows, cols;
    int stride_eff;
    int n_samples;
    double dot_thr, good_min, min_score;
    int min_parts;
    int *counts;
    const uint2 *peaks;
    int cap_part, cap_frame, cap_cands, cap_humans;
    int frame_base;
    int *frame_first, *frame_count;
    double *h_score;
    int *h_nparts;
    double *kp_x, *kp_y;
    float *kp_score;
    int *kp_peak;
    int pool_cap;
    Status *st;
    int debug;
    int *dbg_npeaks;
    int4 *dbg_peaks;
    int *dbg_nconns;
    int *dbg_conn_i;
    double *dbg_conn_d;
    void *cand_spill;    // [frames][cap_cands - kCandSmem] candidate records (crowded frames)
    double ry, rx;       // h / H, w / W: operators.py:88-89 ratios (up > 1)
    const AxisRec *rrec, *crec;   // packed operators.py:86-96 axis records (up > 1)
    int good_need;       // least n_good with fl(n_good / n) >= good_min (n + 1: none)
    // split parse (PF_OPT_PARSE_SPLIT): per-frame HBM staging between the kernels
    int split;
    uint32_t *pk_cell;   // [B][cap_frame] peaks in id order
    float *pk_score;
    int *pk_base;        // [B][K+1] part prefix
    int *pair_pp;        // [B][L+1] pair prefix per limb
    int *n_pairs;                            // [B]
    long long *pair_base, *pair_total;       // [B] exclusive prefix, scalar (64-bit: crowded chunks)
    int2 *ferr;          // [B] capacity error (what, value) from k_parse_peaks
    struct Cand *cand_g; // [B][cap_cands] gated candidates
    int *cand_n;         // [B]
    // PF_OPT_COUNT_PAF: per-frame bitmaps of the 32-byte PAF sectors sampled
    // (global frame index * touch_words), or null
    uint32_t *paf_touch;
    int touch_words;
    // split parse: frames whose candidates exceed kCandSmemSplit, finished by
    // k_parse_crowd ([crowd_cap] list + count at crowd_frames[crowd_cap]), or null
    int *crowd_frames;
    int crowd_cap;
};
#ifndef PF_CAND_SMEM
#define PF_CAND_SMEM 256
#endif
constexpr int kCandSmem = PF_CAND_SMEM;   // gated candidates kept in shared memory per frame
#ifndef PF_CAND_SMEM_SPLIT
#define PF_CAND_SMEM_SPLIT 128
#endif
constexpr int kCandSmemSplit = PF_CAND_SMEM_SPLIT;   // the same for k_parse_frames<true> (<= kCandSmem)
#ifndef PF_PARSE_THREADS
#define PF_PARSE_THREADS 128
#endif
constexpr int kParseThreads = PF_PARSE_THREADS;   // k_parse_frames CTA size
#ifndef PF_PARSE_FIN_THREADS
#define PF_PARSE_FIN_THREADS 64
#endif
constexpr int kParseFinThreads = PF_PARSE_FIN_THREADS;   // k_parse_frames<true> (split finish) CTA size
constexpr int kParseCrowdThreads = 512;                  // k_parse_crowd (crowded frames of the split parse)
#ifndef PF_PARSE_WIDE_THREADS
#define PF_PARSE_WIDE_THREADS 512
#endif
constexpr int kParseWideThreads = PF_PARSE_WIDE_THREADS;  // k_parse_frames_wide (small one-kernel batches)

#ifndef PF_CAND_SMEM_CROWD
#define PF_CAND_SMEM_CROWD 4096
#endif
constexpr int kCandSmemCrowd = PF_CAND_SMEM_CROWD;       // candidates in shared memory per crowded frame
constexpr int kParseMaxThreads = kParseCrowdThreads > kParseThreads ? kParseCrowdThreads : kParseThreads;
static_assert(kParseWideThreads <= kParseMaxThreads, "per-thread tables are sized for kParseMaxThreads");
size_t cand_spill_bytes_per_frame(int cap_cands);
size_t cand_record_bytes();
enum { kCapPart = 1, kCapFrame = 2, kCapCands = 3, kCapHumans = 4, kCapPool = 5 };
size_t parse_smem_bytes(int cap_frame, int cap_part, int cap_cands, int cap_humans, int K, int L, int n_warps,
                        bool split, bool crowd = false);
cudaError_t launch_parse_frames(const ParseArgs &a, int B, int threads, size_t smem, cudaStream_t s);
cudaError_t launch_parse_peaks(const ParseArgs &a, int B, cudaStream_t s);    // k_parse_peaks + k_pair_scan
cudaError_t launch_score_pairs(const ParseArgs &a, int B, cudaStream_t s);
cudaError_t configure_parse_kernels(int max_smem);

// pf_large.cu: frames past the shared-memory capacities of k_parse_frames
// (per-frame HBM workspace, 32-bit indices; see pf_large.cu)
struct LargeWs {
    int cap_peaks, cap_cands, cap_humans;    // per frame
    int part_words, used_words;              // bitmap words per part side / per frame (L * 2 * part_words)
    uint32_t *pk_cell;                       // [B][cap_peaks]
    float *pk_score;
    int *owner;
    void *cand;                              // [B][cap_cands] records of large_cand_bytes()
    uint32_t *used;                          // [B][used_words]
    int *h_parts;                            // [B][cap_humans][K]
    int8_t *h_order;                         // [B][cap_humans][K]
    int8_t *h_n, *h_alive;                   // [B][cap_humans]
    uint32_t *h_mask;
    double *h_score;
    int *h_pos;
};
size_t large_cand_bytes();
cudaError_t launch_parse_large(const ParseArgs &a, const LargeWs &ws, int B, cudaStream_t s);

// pf_render.cu
struct RenderArgs {
    Topo topo;
    const double *kp;        // [F][hmax][K][2] keypoint cells (row, col); NaN = missing
    const int *n_humans;     // [F]
    int F, hmax, gh, gw;
    double sigma, halfwidth;
    float *conf, *paf;       // [F][K+1][gh][gw], [F][2L][gh][gw]
};
cudaError_t launch_render_maps(const RenderArgs &a, int sms, cudaStream_t s);

// pf_overlay.cu
using OverlayPrim = pf_overlay_prim;
cudaError_t launch_overlay(const OverlayPrim *prims, const int *prim_first, int n_prims, int frames, int h, int w,
                           unsigned *owner, float *img, int sms, cudaStream_t s);

// pf_image.cu
constexpr int kMaxBlurRadius = 64;
struct BlurTaps { double w[2 * kMaxBlurRadius + 1]; int r; };

// k_up_blur_nms (pf_blur.cu): x`up` upsample -> separable blur -> 3x3 NMS of
// the K part planes, fused (nothing full-resolution in HBM).
struct UpBlurArgs {
    const float *conf;                   // low-res [B][C][h][w]
    int B, C, K, h, w, H, W;
    const AxisRec *rrec, *crec;          // per output row / column
    BlurTaps taps;
    float thr;
    int cap;
    int *counts;                         // [B*K], accumulated with atomics (zero on entry)
    uint2 *peaks;                        // [B*K][cap]
    int tw, tiles;                       // column tile width / tiles per plane (set by the launcher)
    int up;                              // upsample factor (source rows per tile)
    int th, tiles_y, tiles_x;            // k_up_blur_tile: block rows, blocks per plane (set by the launcher)
};
cudaError_t launch_up_blur_nms(const UpBlurArgs &a, cudaStream_t s);
size_t up_blur_smem(int tw, int r);
int up_blur_tile_width(int W, int r);
cudaError_t configure_blur_kernels(int max_smem);
cudaError_t launch_preprocess(const void *src, int src_is_f32, int B, int h, int w, float *dst,
                              int H, int W, const AxisRec *rrec, const AxisRec *crec, cudaStream_t s);
cudaError_t launch_resize_planes(const float *src, long long src_frame, int K, long long P, int h, int w,
                                 float *dst, int H, int W, const AxisRec *rrec, const AxisRec *crec,
                                 cudaStream_t s);
cudaError_t launch_blur(const float *src, long long src_frame, float *tmp, float *dst,
                        long long dst_frame, int B, int K, int H, int W, const BlurTaps &taps,
                        int sms, cudaStream_t s);

}  // namespace pf
