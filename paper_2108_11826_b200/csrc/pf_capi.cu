// pf_capi.cu — the C ABI (include/pf_b200.h): context, workspaces, the
// chunked launch sequence and the host<->device result path.
//
// Launch sequence per chunk of frames (device-resident maps):
//   Mode R (upsample 1, no blur)   k_nms_plane  -> k_parse_frames
//   Mode U (upsample u, no blur)   k_nms_up     -> k_parse_frames   (fused, default)
//   blur or NMS window > 33        k_resize_planes -> k_blur_rows/cols
//                                  -> k_nms_plane -> k_parse_frames
// k_parse_frames resets the per-slab peak counters it consumed, so the
// steady state needs no memset between chunks; one 32-byte memset clears
// the status/pool counter per call.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "pf_launch.h"

using namespace pf;

namespace pf {
#ifndef PF_PDL_DEFAULT
#define PF_PDL_DEFAULT (1 << kPdlParseWide)   // small batches: the parse launch overlaps the NMS tail
#endif
int g_pdl_mask = PF_PDL_DEFAULT;
}

#ifndef PF_CORNER_SPLIT_DEFAULT
#define PF_CORNER_SPLIT_DEFAULT 1
#endif
#ifndef PF_PARSE_SPLIT_DEFAULT
#define PF_PARSE_SPLIT_DEFAULT 1
#endif
#ifndef PF_WIDE_FRAMES_PER_SM
#define PF_WIDE_FRAMES_PER_SM 1
#endif
// Parse split option 1 (auto): batches with more frames than SMs take the
// split parse; up to one frame per SM, the one-kernel parse with a wide
// (512-thread) CTA per frame runs them in one wave and measured faster
// (C2 64 frames 98.9 -> 80.4 us per call, C4 147k -> 185k frames/s, equal
// just past the SM count; the 128-thread one-kernel form needed the split
// parse from 32 frames).
#ifndef PF_CORNER_SPLIT_MIN_FRAMES
#define PF_CORNER_SPLIT_MIN_FRAMES 256   // measured: one-kernel corner faster up to 128 frames (C2 64: 113 -> 98 us), equal at 256
#endif
constexpr int kCornerSplitMinFrames = PF_CORNER_SPLIT_MIN_FRAMES;   // the same for the Mode U scan + finish split
#ifndef PF_EXACT_SPLIT
#define PF_EXACT_SPLIT 1
#endif
constexpr bool kExactSplit = PF_EXACT_SPLIT;   // the finish hands its exact tests to k_corner_exact
constexpr int kExactMinPlanes = 4096;         // ... on batches of at least this many planes

namespace {

struct AxisCache {
    int in_n = 0, out_n = 0;
    std::vector<int32_t> i0, i1;
    std::vector<double> t, omt;
    std::vector<int32_t> first_out, last_out;   // inverse map: outputs reading input row r
    std::vector<int32_t> gend;                  // last output row with the same source pair
    std::vector<int4> bands;                    // (first, last, src0, src1) per band
    std::vector<double> band_dt;                // min t step inside each band (inf if 1 wide)
    int max_band = 0;
    double min_step = 0.0;                      // min t distance of adjacent outputs off the border bands
    bool canonical = false;                     // band b reads sources (b-1, b) clipped: b = 0..in_n
    int4 *d_bands = nullptr;
    double *d_band_dt = nullptr;
    int32_t *d_i0 = nullptr, *d_i1 = nullptr, *d_first = nullptr, *d_last = nullptr;
    AxisRec *d_rec = nullptr;
    double *d_t = nullptr, *d_omt = nullptr;
    AxisTab dev() const { return AxisTab{d_i0, d_i1, d_t, d_omt}; }
};

// operators.py:86-96, evaluated on the host in fp64 with the reference op
// order (built with -ffp-contract=off: no FMA on the host side either).
void fill_axis(AxisCache &a, int in_n, int out_n)
{
    a.in_n = in_n;
    a.out_n = out_n;
    a.i0.resize(out_n); a.i1.resize(out_n); a.t.resize(out_n); a.omt.resize(out_n);
    const volatile double ratio = (double)in_n / (double)out_n;
    for (int o = 0; o < out_n; ++o) {
        const volatile double prod = ((double)o + 0.5) * ratio;
        const double s = prod - 0.5;
        const long long f = (long long)std::floor(s);
        const double t = s - (double)f;
        a.t[o] = t;
        a.omt[o] = 1.0 - t;
        a.i0[o] = (int32_t)(f < 0 ? 0 : (f > in_n - 1 ? in_n - 1 : f));
        a.i1[o] = (int32_t)(f + 1 < 0 ? 0 : (f + 1 > in_n - 1 ? in_n - 1 : f + 1));
    }
    a.gend.resize(out_n);
    for (int o = out_n - 1; o >= 0; --o)
        a.gend[o] = (o + 1 < out_n && a.i0[o + 1] == a.i0[o] && a.i1[o + 1] == a.i1[o]) ? a.gend[o + 1] : o;
    a.bands.clear();
    a.band_dt.clear();
    a.max_band = 0;
    for (int o = 0; o < out_n; o = a.gend[o] + 1) {
        const int e = a.gend[o];
        a.bands.push_back(make_int4(o, e, a.i0[o], a.i1[o]));
        double dt = 1e300;
        for (int u = o; u < e; ++u) dt = std::min(dt, a.t[u + 1] - a.t[u]);
        a.band_dt.push_back(dt);
        a.max_band = std::max(a.max_band, e - o + 1);
    }
    a.canonical = (int)a.bands.size() == in_n + 1 && in_n >= 2;
    // adjacent outputs o, o+1 in interior bands: t[o+1] - t[o] inside a band,
    // (1 - t[o]) + t[o+1] across a band boundary (k_nms_up_corner chain_pruned)
    a.min_step = 1e300;
    for (size_t b = 1; b + 1 < a.bands.size(); ++b) {
        const int4 B = a.bands[b];
        for (int u = B.x; u < B.y; ++u) a.min_step = std::min(a.min_step, a.t[u + 1] - a.t[u]);
        if (b + 2 < a.bands.size()) a.min_step = std::min(a.min_step, a.omt[B.y] + a.t[B.y + 1]);
    }
    for (int b = 0; a.canonical && b <= in_n; ++b)
        a.canonical = a.bands[b].z == std::max(b - 1, 0) && a.bands[b].w == std::min(b, in_n - 1);
    a.first_out.assign(in_n, 0x3fffffff);
    a.last_out.assign(in_n, -1);
    for (int o = 0; o < out_n; ++o) {
        for (int r : {a.i0[o], a.i1[o]}) {
            if (o < a.first_out[r]) a.first_out[r] = o;
            if (o > a.last_out[r]) a.last_out[r] = o;
        }
    }
}

template <typename T>
cudaError_t dev_alloc(T **p, size_t n)
{
    return cudaMalloc(reinterpret_cast<void **>(p), n * sizeof(T) + 16);
}

template <typename T>
cudaError_t host_alloc(T **p, size_t n)
{
    return cudaHostAlloc(reinterpret_cast<void **>(p), n * sizeof(T) + 16, cudaHostAllocDefault);
}

}  // namespace

#ifndef PF_HOST_SLOTS
#define PF_HOST_SLOTS 2   // 3 measured the same (132.2k vs 131.7k e2e)
#endif
constexpr int kHostSlots = PF_HOST_SLOTS;   // device input slots of pf_parse_host (copy / compute overlap)

// Streams of one run_chunk: the NMS stage (upsample / blur / peaks) on
// `nms`, the parse stage on `parse`, NMS slab set `set`.  Serial: both the
// context stream, set 0.
struct Sched {
    cudaStream_t nms, parse;
    int set;
    bool wide;      // small batches may take the wide one-kernel parse (device-resident PAF)
};

struct pf_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    Topo topo{};
    bool has_topo = false;
    pf_caps caps{};
    std::string err;
    int debug = 0;
    int64_t launches = 0;

    // NMS workspace (chunk-sized)
    // NMS slabs (peak counts + records per plane); a second set while
    // pf_parse_host overlaps the NMS stage of one chunk with the parse of the last
    int *d_counts = nullptr, *d_counts2 = nullptr;
    uint2 *d_peaks = nullptr, *d_peaks2 = nullptr;
    int ws_sets = 0;
    cudaStream_t parse_stream = nullptr;    // pf_parse_host: the parse stage beside the NMS stage
    cudaEvent_t ev_nms[2] = {}, ev_parsed[2] = {}, ev_join = nullptr;
    int host_overlap = 1;                   // PF_OPT_HOST_OVERLAP
    int prio_low = 0, prio_high = 0;
    void *d_spill = nullptr;     // candidate spill slab for crowded frames
    uint32_t *d_corner_spill = nullptr;   // k_nms_up_corner candidate overflow (per resident CTA)
    uint32_t *d_surv = nullptr;           // split corner path: survivors per plane
    int *d_surv_n = nullptr;
    uint2 *d_exact = nullptr;             // split corner path: candidates for k_corner_exact
    int exact_opt = 0;                    // PF_OPT_EXACT_LIST
    int *d_crowd = nullptr;                 // crowded plane list + its counter (last slot)
    size_t surv_planes = 0;
    int corner_split = PF_CORNER_SPLIT_DEFAULT;
    int parse_split = PF_PARSE_SPLIT_DEFAULT;
    uint32_t *d_pk_cell = nullptr;          // split parse staging (ensure_split_ws)
    float *d_pk_score = nullptr;
    int *d_pk_base = nullptr, *d_pair_pp = nullptr, *d_npairs = nullptr, *d_cand_n = nullptr;
    int *d_crowd_frames = nullptr;          // split parse: crowded frame list [split_frames] + its count
    long long *d_pair_base = nullptr;       // [frames + 1]: prefix, then the total
    int2 *d_ferr = nullptr;
    unsigned *d_owner = nullptr;            // overlay: draw-order owner per pixel
    size_t overlay_px = 0;
    size_t split_frames = 0;
    int split_cap_frame = 0;
    size_t ws_frames = 0;
    int ws_K = 0;
    int ws_cap_part = 0, ws_cap_cands = 0;
    int auto_caps = 0;           // bit kCap* set: that capacity grows on demand
    int max_smem = 0;

    // resize tables, keyed by (in, out)
    std::map<std::pair<int, int>, AxisCache> axes;

    // outputs
    int *d_frame_first = nullptr, *d_frame_count = nullptr;
    int *h_frame_first = nullptr, *h_frame_count = nullptr;
    size_t frames_cap = 0;
    double *d_hscore = nullptr, *h_hscore = nullptr;
    int *d_hnparts = nullptr, *h_hnparts = nullptr;
    double *d_kpx = nullptr, *d_kpy = nullptr, *h_kpx = nullptr, *h_kpy = nullptr;
    float *d_kps = nullptr, *h_kps = nullptr;
    int *d_kpp = nullptr, *h_kpp = nullptr;
    size_t pool_cap = 0;
    int pool_K = 0;
    Status *d_status = nullptr, *h_status = nullptr;

    // materialised full-resolution workspace (blur / wide NMS window)
    float *d_full = nullptr, *d_tmp = nullptr;
    size_t full_elems = 0;

    // host-path staging (double buffered)
    float *d_in[kHostSlots] = {};
    size_t in_elems = 0;
    cudaEvent_t ev_copied[kHostSlots] = {}, ev_free[kHostSlots] = {};

    // debug slabs
    int *d_dbg_np = nullptr, *d_dbg_nc = nullptr, *d_dbg_ci = nullptr;
    int4 *d_dbg_peaks = nullptr;
    double *d_dbg_cd = nullptr;
    size_t dbg_frames = 0;
    int dbg_cap_frame = 0, dbg_cap_cands = 0;

    // per-kernel timing (PF_OPT_TIMING)
    int timing = 0;
    int materialise = 0;
    int generic_fused = 0;
    int win_variant = 4;
    int no_chain = 0;
    int paf_zero_copy = 1;
    int count_paf = 0;                      // PF_OPT_COUNT_PAF: instrumented one-kernel parse
    int large = 0;                          // parse through k_parse_large (set when a capacity outgrows
                                            // shared memory, or PF_OPT_LARGE)
    LargeWs lws{};                          // its per-frame workspace
    size_t lws_frames = 0;
    int large_auto = 0;                     // switched by grow_cap (per call: the next call starts on
    pf_caps caps_usual{};                   //   the usual path again, with these caps)
    int replaying = 0;
    uint32_t *d_paf_touch = nullptr;        // [batch][touch_words] sampled-sector bitmaps
    size_t touch_cap = 0, touch_used = 0;
    int conf_zero_copy = 0;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double kernel_ms[PF_N_KERNELS] = {0};
    int64_t kernel_launches[PF_N_KERNELS] = {0};

    int last_batch = 0;
    int last_K = 0;
    bool results_ready = false;
    bool status_ready = false;              // h_status holds the last call's final status

    // the last parse call, replayed once with a larger output pool when the
    // default pool (64 humans/frame) overflows and no fixed cap was requested
    struct {
        int kind = 0;                 // 0 none, 1 device, 2 host
        const float *conf = nullptr, *paf = nullptr;
        int batch = 0, h = 0, w = 0, stride = 1;
        pf_params p{};
    } last;
    long long pool_need = 0;
};

namespace {

thread_local std::string g_create_err;   // pf_create failures (no context yet)

int fail(pf_ctx *c, int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    else g_create_err = buf;
    return code;
}

#define CU(expr)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, PF_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                              \
    } while (0)

enum KernelId { kNmsPlane = 0, kNmsUp, kParseFrames, kResize, kBlurRows, kBlurCols, kPreprocess,
                kNmsUpWin, kNmsUpCorner, kCornerFinish, kCornerCrowded, kNmsUpScan, kParsePeaks, kScorePairs,
                kUpBlur, kParseLarge, kScatterOut };
const char *kKernelNames[PF_N_KERNELS] = {"k_nms_plane", "k_nms_up", "k_parse_frames",
                                          "k_resize_planes", "k_blur_rows", "k_blur_cols",
                                          "k_preprocess", "k_nms_up_win", "k_nms_up_corner",
                                          "k_corner_finish", "k_corner_crowded", "k_nms_up_scan",
                                          "k_parse_peaks", "k_score_pairs", "k_up_blur_nms",
                                          "k_parse_large", "k_scatter_out"};

cudaEvent_t take_event(pf_ctx *ctx)
{
    if (!ctx->ev_pool.empty()) {
        cudaEvent_t e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one kernel launch with timing events when PF_OPT_TIMING is on.
struct KernelTimer {
    pf_ctx *ctx;
    int id;
    int n;
    cudaEvent_t a = nullptr;
    cudaStream_t st;
    KernelTimer(pf_ctx *c, int kid, int launches = 1, cudaStream_t s = nullptr)
        : ctx(c), id(kid), n(launches), st(s ? s : c->stream)
    {
        if (ctx->timing) {
            a = take_event(ctx);
            cudaEventRecord(a, st);
        }
    }
    ~KernelTimer()
    {
        ctx->launches += n;
        ctx->kernel_launches[id] += n;
        if (a) {
            cudaEvent_t b = take_event(ctx);
            cudaEventRecord(b, st);
            ctx->pending.push_back({id, {a, b}});
        }
    }
};

int set_device(pf_ctx *ctx)
{
    CU(cudaSetDevice(ctx->device));
    return PF_OK;
}

int get_axis(pf_ctx *ctx, int in_n, int out_n, AxisCache **out)
{
    auto key = std::make_pair(in_n, out_n);
    auto it = ctx->axes.find(key);
    if (it == ctx->axes.end()) {
        AxisCache a;
        fill_axis(a, in_n, out_n);
        CU(dev_alloc(&a.d_i0, out_n));
        CU(dev_alloc(&a.d_i1, out_n));
        CU(dev_alloc(&a.d_t, out_n));
        CU(dev_alloc(&a.d_omt, out_n));
        CU(cudaMemcpy(a.d_i0, a.i0.data(), out_n * sizeof(int32_t), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(a.d_i1, a.i1.data(), out_n * sizeof(int32_t), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(a.d_t, a.t.data(), out_n * sizeof(double), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(a.d_omt, a.omt.data(), out_n * sizeof(double), cudaMemcpyHostToDevice));
        {
            std::vector<AxisRec> rec(out_n);
            for (int o = 0; o < out_n; ++o) {
                rec[o].i01 = a.i0[o] | (a.i1[o] << 16);
                rec[o].pad = 0;
                rec[o].t = a.t[o];
            }
            CU(dev_alloc(&a.d_rec, out_n));
            CU(cudaMemcpy(a.d_rec, rec.data(), out_n * sizeof(AxisRec), cudaMemcpyHostToDevice));
        }
        CU(dev_alloc(&a.d_bands, a.bands.size()));
        CU(cudaMemcpy(a.d_bands, a.bands.data(), a.bands.size() * sizeof(int4), cudaMemcpyHostToDevice));
        CU(dev_alloc(&a.d_band_dt, a.band_dt.size()));
        CU(cudaMemcpy(a.d_band_dt, a.band_dt.data(), a.band_dt.size() * sizeof(double), cudaMemcpyHostToDevice));
        CU(dev_alloc(&a.d_first, in_n));
        CU(dev_alloc(&a.d_last, in_n));
        CU(cudaMemcpy(a.d_first, a.first_out.data(), in_n * sizeof(int32_t), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(a.d_last, a.last_out.data(), in_n * sizeof(int32_t), cudaMemcpyHostToDevice));
        it = ctx->axes.emplace(key, std::move(a)).first;
    }
    *out = &it->second;
    return PF_OK;
}

int ensure_nms_ws(pf_ctx *ctx, size_t frames, int K, int sets = 1)
{
    if (frames <= ctx->ws_frames && K <= ctx->ws_K && ctx->ws_cap_part == ctx->caps.max_peaks_per_part &&
        ctx->ws_cap_cands == ctx->caps.max_candidates && sets <= ctx->ws_sets)
        return PF_OK;
    CU(cudaDeviceSynchronize());                         // the old slabs may still be in use
    ctx->ws_cap_part = ctx->caps.max_peaks_per_part;
    ctx->ws_cap_cands = ctx->caps.max_candidates;
    cudaFree(ctx->d_counts);
    cudaFree(ctx->d_peaks);
    cudaFree(ctx->d_counts2);
    cudaFree(ctx->d_peaks2);
    cudaFree(ctx->d_spill);
    ctx->d_counts = ctx->d_counts2 = nullptr;
    ctx->d_peaks = ctx->d_peaks2 = nullptr;
    ctx->d_spill = nullptr;
    ctx->ws_sets = 0;
    const size_t f = frames > ctx->ws_frames ? frames : ctx->ws_frames;
    const int k = K > ctx->ws_K ? K : ctx->ws_K;
    const int ns = sets > ctx->ws_sets ? sets : 1;
    CU(dev_alloc(&ctx->d_counts, f * k));
    CU(cudaMemset(ctx->d_counts, 0, f * k * sizeof(int)));
    CU(dev_alloc(&ctx->d_peaks, f * k * (size_t)ctx->caps.max_peaks_per_part));
    if (ns > 1) {
        CU(dev_alloc(&ctx->d_counts2, f * k));
        CU(cudaMemset(ctx->d_counts2, 0, f * k * sizeof(int)));
        CU(dev_alloc(&ctx->d_peaks2, f * k * (size_t)ctx->caps.max_peaks_per_part));
    }
    ctx->ws_sets = ns;
    // [f][cap_cands] records: the one-kernel parse uses it as the spill past the
    // shared candidates, the split parse as the whole per-frame candidate list
    CU(dev_alloc(reinterpret_cast<char **>(&ctx->d_spill),
                 f * (size_t)ctx->caps.max_candidates * cand_record_bytes()));
    ctx->ws_frames = f;
    ctx->ws_K = k;
    return PF_OK;
}

// Split-parse staging ([frames] x per-frame arrays), sized for the current caps.
int ensure_split_ws(pf_ctx *ctx, size_t frames)
{
    if (frames <= ctx->split_frames && ctx->split_cap_frame == ctx->caps.max_peaks_per_frame) return PF_OK;
    const size_t f = frames > ctx->split_frames ? frames : ctx->split_frames;
    void *old[] = {ctx->d_pk_cell, ctx->d_pk_score, ctx->d_pk_base, ctx->d_pair_pp, ctx->d_npairs,
                   ctx->d_pair_base, ctx->d_ferr, ctx->d_cand_n, ctx->d_crowd_frames};
    for (void *q : old) cudaFree(q);
    ctx->d_pk_cell = nullptr; ctx->d_pk_score = nullptr; ctx->d_pk_base = nullptr; ctx->d_pair_pp = nullptr;
    ctx->d_npairs = nullptr; ctx->d_pair_base = nullptr; ctx->d_ferr = nullptr; ctx->d_cand_n = nullptr;
    ctx->d_crowd_frames = nullptr;
    ctx->split_frames = 0;
    const size_t cf = (size_t)ctx->caps.max_peaks_per_frame;
    CU(dev_alloc(&ctx->d_pk_cell, f * cf));
    CU(dev_alloc(&ctx->d_pk_score, f * cf));
    CU(dev_alloc(&ctx->d_pk_base, f * (PF_MAX_KEYPOINTS + 1)));
    CU(dev_alloc(&ctx->d_pair_pp, f * (PF_MAX_LIMBS + 1)));
    CU(dev_alloc(&ctx->d_npairs, f));
    CU(dev_alloc(&ctx->d_pair_base, f + 1));         // + the pair total
    CU(dev_alloc(&ctx->d_ferr, f));
    CU(dev_alloc(&ctx->d_cand_n, f));
    CU(dev_alloc(&ctx->d_crowd_frames, f + 1));
    ctx->split_frames = f;
    ctx->split_cap_frame = ctx->caps.max_peaks_per_frame;
    return PF_OK;
}

// Per-frame HBM workspace of k_parse_large, sized by the current caps.
size_t large_bytes_per_frame(const pf_ctx *ctx)
{
    const pf_caps &c = ctx->caps;
    const size_t K = (size_t)ctx->topo.K, L = (size_t)ctx->topo.L;
    const size_t pw = ((size_t)c.max_peaks_per_part + 31) / 32;
    return (size_t)c.max_peaks_per_frame * 12 + (size_t)c.max_candidates * large_cand_bytes() + L * 2 * pw * 4 +
           (size_t)c.max_humans_per_frame * (K * 5 + 2 + 4 + 8 + 4);
}

int ensure_large_ws(pf_ctx *ctx, size_t frames)
{
    LargeWs &w = ctx->lws;
    const pf_caps &c = ctx->caps;
    const int pw = (c.max_peaks_per_part + 31) / 32;
    if (frames <= ctx->lws_frames && w.cap_peaks == c.max_peaks_per_frame && w.cap_cands == c.max_candidates &&
        w.cap_humans == c.max_humans_per_frame && w.part_words == pw)
        return PF_OK;
    void *old[] = {w.pk_cell, w.pk_score, w.owner, w.cand, w.used, w.h_parts, w.h_order, w.h_n, w.h_alive,
                   w.h_mask, w.h_score, w.h_pos};
    for (void *q : old) cudaFree(q);
    w = LargeWs{};
    ctx->lws_frames = 0;
    const size_t f = frames, K = (size_t)ctx->topo.K;
    w.cap_peaks = c.max_peaks_per_frame;
    w.cap_cands = c.max_candidates;
    w.cap_humans = c.max_humans_per_frame;
    w.part_words = pw;
    w.used_words = ctx->topo.L * 2 * pw;
    CU(dev_alloc(&w.pk_cell, f * w.cap_peaks));
    CU(dev_alloc(&w.pk_score, f * w.cap_peaks));
    CU(dev_alloc(&w.owner, f * w.cap_peaks));
    CU(dev_alloc(reinterpret_cast<char **>(&w.cand), f * w.cap_cands * large_cand_bytes()));
    CU(dev_alloc(&w.used, f * (size_t)w.used_words));
    CU(dev_alloc(&w.h_parts, f * w.cap_humans * K));
    CU(dev_alloc(&w.h_order, f * w.cap_humans * K));
    CU(dev_alloc(&w.h_n, f * w.cap_humans));
    CU(dev_alloc(&w.h_alive, f * w.cap_humans));
    CU(dev_alloc(&w.h_mask, f * w.cap_humans));
    CU(dev_alloc(&w.h_score, f * w.cap_humans));
    CU(dev_alloc(&w.h_pos, f * w.cap_humans));
    ctx->lws_frames = f;
    return PF_OK;
}

int ensure_frames(pf_ctx *ctx, size_t frames)
{
    if (frames <= ctx->frames_cap) return PF_OK;
    cudaFree(ctx->d_frame_first); cudaFree(ctx->d_frame_count);
    cudaFreeHost(ctx->h_frame_first); cudaFreeHost(ctx->h_frame_count);
    CU(dev_alloc(&ctx->d_frame_first, frames));
    CU(dev_alloc(&ctx->d_frame_count, frames));
    CU(host_alloc(&ctx->h_frame_first, frames));
    CU(host_alloc(&ctx->h_frame_count, frames));
    ctx->frames_cap = frames;
    return PF_OK;
}

int ensure_pool(pf_ctx *ctx, size_t humans, int K)
{
    if (humans <= ctx->pool_cap && K <= ctx->pool_K) return PF_OK;
    const size_t n = humans > ctx->pool_cap ? humans : ctx->pool_cap;
    const int k = K > ctx->pool_K ? K : ctx->pool_K;
    cudaFree(ctx->d_hscore); cudaFree(ctx->d_hnparts); cudaFree(ctx->d_kpx);
    cudaFree(ctx->d_kpy); cudaFree(ctx->d_kps); cudaFree(ctx->d_kpp);
    cudaFreeHost(ctx->h_hscore); cudaFreeHost(ctx->h_hnparts); cudaFreeHost(ctx->h_kpx);
    cudaFreeHost(ctx->h_kpy); cudaFreeHost(ctx->h_kps); cudaFreeHost(ctx->h_kpp);
    CU(dev_alloc(&ctx->d_hscore, n));
    CU(dev_alloc(&ctx->d_hnparts, n));
    CU(dev_alloc(&ctx->d_kpx, n * k));
    CU(dev_alloc(&ctx->d_kpy, n * k));
    CU(dev_alloc(&ctx->d_kps, n * k));
    CU(dev_alloc(&ctx->d_kpp, n * k));
    CU(host_alloc(&ctx->h_hscore, n));
    CU(host_alloc(&ctx->h_hnparts, n));
    CU(host_alloc(&ctx->h_kpx, n * k));
    CU(host_alloc(&ctx->h_kpy, n * k));
    CU(host_alloc(&ctx->h_kps, n * k));
    CU(host_alloc(&ctx->h_kpp, n * k));
    ctx->pool_cap = n;
    ctx->pool_K = k;
    return PF_OK;
}

int ensure_debug(pf_ctx *ctx, size_t frames)
{
    if (!ctx->debug || (frames <= ctx->dbg_frames && ctx->dbg_cap_frame == ctx->caps.max_peaks_per_frame &&
                        ctx->dbg_cap_cands == ctx->caps.max_candidates))
        return PF_OK;
    if (frames < ctx->dbg_frames) frames = ctx->dbg_frames;
    ctx->dbg_cap_frame = ctx->caps.max_peaks_per_frame;
    ctx->dbg_cap_cands = ctx->caps.max_candidates;
    cudaFree(ctx->d_dbg_np); cudaFree(ctx->d_dbg_nc); cudaFree(ctx->d_dbg_ci);
    cudaFree(ctx->d_dbg_peaks); cudaFree(ctx->d_dbg_cd);
    CU(dev_alloc(&ctx->d_dbg_np, frames));
    CU(dev_alloc(&ctx->d_dbg_nc, frames));
    CU(dev_alloc(&ctx->d_dbg_peaks, frames * (size_t)ctx->caps.max_peaks_per_frame));
    CU(dev_alloc(&ctx->d_dbg_ci, frames * (size_t)ctx->caps.max_candidates * 3));
    CU(dev_alloc(&ctx->d_dbg_cd, frames * (size_t)ctx->caps.max_candidates * 2));
    ctx->dbg_frames = frames;
    return PF_OK;
}

int ensure_full(pf_ctx *ctx, size_t elems)
{
    if (elems <= ctx->full_elems) return PF_OK;
    cudaFree(ctx->d_full);
    cudaFree(ctx->d_tmp);
    CU(dev_alloc(&ctx->d_full, elems));
    CU(dev_alloc(&ctx->d_tmp, elems));
    ctx->full_elems = elems;
    return PF_OK;
}

int validate_params_impl(pf_ctx *ctx, const pf_params *p)
{
    if (!p) return fail(ctx, PF_ERR_CONFIG, "params is NULL");
    // paf.py:44-54
    if (p->nms_window < 3 || p->nms_window % 2 == 0)
        return fail(ctx, PF_ERR_CONFIG, "nms_window must be odd and >= 3");
    if (p->n_samples < 2) return fail(ctx, PF_ERR_CONFIG, "n_samples must be >= 2");
    const double v[3] = {p->conf_threshold, p->sample_dot_threshold, p->good_fraction_min};
    const char *names[3] = {"conf_threshold", "sample_dot_threshold", "good_fraction_min"};
    for (int k = 0; k < 3; ++k)
        if (!(0.0 <= v[k] && v[k] <= 1.0))
            return fail(ctx, PF_ERR_CONFIG, "%s must be in [0, 1], got %g", names[k], v[k]);
    if (p->min_parts < 1) return fail(ctx, PF_ERR_CONFIG, "min_parts must be >= 1");
    // extension knobs
    if (p->upsample < 1) return fail(ctx, PF_ERR_CONFIG, "upsample must be >= 1");
    if (!(p->blur_sigma >= 0.0) || !std::isfinite(p->blur_sigma))
        return fail(ctx, PF_ERR_CONFIG, "blur_sigma must be finite and >= 0");
    if (p->blur_sigma > 0.0 && (int)std::ceil(3.0 * p->blur_sigma) > kMaxBlurRadius)
        return fail(ctx, PF_ERR_CONFIG, "blur_sigma too large (radius > %d)", kMaxBlurRadius);
    if (p->n_samples > (1 << 24) - 1) return fail(ctx, PF_ERR_CONFIG, "n_samples too large for the GPU path");
    return PF_OK;
}

// radius ceil(3 sigma), taps exp(-k^2 / (2 sigma^2)) normalised
// by their sum accumulated in ascending k.
void make_taps(double sigma, BlurTaps &t)
{
    const int r = (int)std::ceil(3.0 * sigma);
    t.r = r;
    double sum = 0.0;
    for (int k = -r; k <= r; ++k) {
        t.w[k + r] = std::exp(-(double)(k * k) / (2.0 * sigma * sigma));
        sum += t.w[k + r];
    }
    for (int k = 0; k <= 2 * r; ++k) t.w[k] /= sum;
}

// Blur on an upsampled grid with the 3x3 window: the fused k_up_blur_nms
// (upsample -> blur -> NMS without full-resolution maps in HBM).
bool fused_blur(const pf_ctx *ctx, const pf_params *p, int W)
{
    if (!(p->blur_sigma > 0.0) || p->upsample < 2 || p->nms_window != 3 || ctx->materialise) return false;
    const int r = (int)std::ceil(3.0 * p->blur_sigma);
    const int tw = up_blur_tile_width(W, r);
    return tw >= 1 && up_blur_smem(tw, r) + 2048 <= (size_t)ctx->max_smem;   // + the static taps table
}

int run_chunk(pf_ctx *ctx, const float *conf, const float *paf, int n, int frame_base,
              int h, int w, int stride, const pf_params *p, AxisCache *rows, AxisCache *cols,
              int pool_cap, Sched sc)
{
    const int K = ctx->topo.K, L = ctx->topo.L;
    const int C = K + 1;
    const int up = p->upsample;
    const int H = h * up, W = w * up;
    const int half = p->nms_window / 2;
    const float thr = (float)p->conf_threshold;   // numpy NEP 50: fp32 compare
    const bool blur = p->blur_sigma > 0.0;
    const bool two = sc.nms != sc.parse;
    int *const counts = sc.set ? ctx->d_counts2 : ctx->d_counts;
    uint2 *const peaks = sc.set ? ctx->d_peaks2 : ctx->d_peaks;
    cudaStream_t s = sc.nms;                       // the NMS stage
    if (two) CU(cudaStreamWaitEvent(s, ctx->ev_parsed[sc.set], 0));   // this slab set consumed

    if (!blur && up == 1) {
        KernelTimer kt(ctx, kNmsPlane, 1, s);
        CU(launch_nms_plane(conf, n, C, K, h, w, thr, half, ctx->caps.max_peaks_per_part,
                            counts, peaks, s));
    } else if (fused_blur(ctx, p, W)) {
        // fused upsample -> blur -> 3x3 NMS (nothing full-resolution in HBM)
        UpBlurArgs a{};
        a.conf = conf; a.B = n; a.C = C; a.K = K; a.h = h; a.w = w; a.H = H; a.W = W;
        a.rrec = rows->d_rec; a.crec = cols->d_rec;
        a.up = up;
        make_taps(p->blur_sigma, a.taps);
        a.thr = thr; a.cap = ctx->caps.max_peaks_per_part;
        a.counts = counts; a.peaks = peaks;
        KernelTimer kt(ctx, kUpBlur, 1, s);
        CU(launch_up_blur_nms(a, s));
    } else if (!blur && half == 1 && !ctx->materialise && !ctx->generic_fused && ctx->win_variant == 4 &&
               rows->canonical && cols->canonical && h + 1 <= 256 && w + 1 <= 256 &&
               (nms_up_corner_smem(h, w, h + 1, w + 1, kCornerStages) <= 100 * 1024 ||
                (ctx->corner_split != 0 && nms_up_scan_launch_smem(h, w) + 2048 <= (size_t)ctx->max_smem))) {
        // maps too large for the one-kernel form's shared-memory budget
        // (e.g. 135x240) take the split kernels at any batch size
        const bool big = nms_up_corner_smem(h, w, h + 1, w + 1, kCornerStages) > 100 * 1024;
        UpCornerArgs a{};
        a.conf = conf; a.B = n; a.C = C; a.K = K; a.h = h; a.w = w; a.H = H; a.W = W;
        a.thr = thr; a.cap = ctx->caps.max_peaks_per_part;
        a.counts = counts; a.peaks = peaks;
        a.rows = rows->dev(); a.cols = cols->dev();
        a.rband = rows->d_bands; a.cband = cols->d_bands;
        a.rdt = rows->d_band_dt; a.cdt = cols->d_band_dt;
        a.nbr = (int)rows->bands.size(); a.nbc = (int)cols->bands.size();
        a.max_band = std::max(rows->max_band, cols->max_band);
        a.nst = kCornerStages;
        a.chain = rows->min_step >= 0.03125 && cols->min_step >= 0.03125 && !ctx->no_chain;
        a.rrec = rows->d_rec; a.crec = cols->d_rec;
        if (!ctx->d_corner_spill)   // persistent grid <= 16 resident CTAs per SM
            CU(dev_alloc(&ctx->d_corner_spill, nms_up_corner_spill_entries(ctx->sms * 16)));
        a.cand_spill = ctx->d_corner_spill;
        // split kernels pay off on batches; a few frames take the one-kernel path (fewer launches)
        const bool csplit = ctx->corner_split == 2 || (ctx->corner_split == 1 && (n >= kCornerSplitMinFrames || big || two));
        // (beside the parse stream the split kernels measured 1 % faster on 128-frame chunks)
        if (csplit) {
            const size_t planes = (size_t)n * K;
            if (planes > ctx->surv_planes) {
                cudaFree(ctx->d_surv);
                cudaFree(ctx->d_surv_n);
                cudaFree(ctx->d_crowd);
                cudaFree(ctx->d_exact);
                ctx->d_surv = nullptr; ctx->d_surv_n = nullptr; ctx->d_crowd = nullptr; ctx->d_exact = nullptr;
                ctx->surv_planes = 0;
                CU(dev_alloc(&ctx->d_surv, planes * corner_surv_entries_per_plane()));
                CU(dev_alloc(&ctx->d_surv_n, planes));
                CU(dev_alloc(&ctx->d_crowd, planes + 3));   // + count + hand-out counter + exact count
                if (kExactSplit) CU(dev_alloc(&ctx->d_exact, planes * corner_exact_entries_per_plane()));
                ctx->surv_planes = planes;
            }
            a.surv_out = ctx->d_surv;
            a.surv_n = ctx->d_surv_n;
            a.crowd_list = ctx->d_crowd;
            a.crowd_n = ctx->d_crowd + ctx->surv_planes;
            // the hand-over pays on large batches; below kExactMinPlanes the extra
            // launch costs more (C4, 576 planes: 0.160 -> 0.167 ms; host-path chunks)
            a.exact_list = (ctx->exact_opt < 0 || (ctx->exact_opt == 0 && (size_t)n * K < (size_t)kExactMinPlanes))
                               ? nullptr : ctx->d_exact;
            a.exact_n = ctx->d_crowd + ctx->surv_planes + 2;
            a.exact_cap = (int)std::min<size_t>(ctx->surv_planes * corner_exact_entries_per_plane(), 0x7fffffff);
            if (ctx->exact_opt > 0) a.exact_cap = std::min(a.exact_cap, ctx->exact_opt);
            CU(cudaMemsetAsync(a.crowd_n, 0, 3 * sizeof(int), s));
        }
        if (csplit) {
            KernelTimer kt(ctx, kNmsUpScan, 1, s);                          // streaming half
            CU(launch_nms_up_scan(a, s));
        } else {
            KernelTimer kt(ctx, kNmsUpCorner, 1, s);                        // one-kernel path
            CU(launch_nms_up_corner(a, s));
        }
        if (csplit) {
            {
                KernelTimer kt(ctx, kCornerFinish, 1, s);   // classification + the exact tests handed over
                CU(launch_corner_finish(a, s));
                if (a.exact_list) {
                    CU(launch_corner_exact(a, s));
                    ctx->launches += 1;
                }
            }
            KernelTimer kt(ctx, kCornerCrowded, 1, s);
            CU(launch_corner_crowded(a, s));
        }
    } else if (!blur && (half == 1 || half == 2) && !ctx->materialise && !ctx->generic_fused &&
               nms_up_win_smem(h, w, H, 128) <= 96 * 1024) {
        UpWinArgs a{};
        a.conf = conf; a.C = C; a.K = K; a.h = h; a.w = w; a.H = H; a.W = W;
        a.ry = (double)h / (double)H;
        a.rx = (double)w / (double)W;
        a.thr = thr; a.half = half; a.cap = ctx->caps.max_peaks_per_part;
        a.counts = counts; a.peaks = peaks;
        a.first_out = rows->d_first; a.last_out = rows->d_last;
        KernelTimer kt(ctx, kNmsUpWin, 1, s);
        CU(launch_nms_up_win(a, n, s));
    } else if (!blur && half <= kMaxFusedHalf && !ctx->materialise) {
        UpArgs a{};
        a.conf = conf; a.C = C; a.K = K; a.h = h; a.w = w; a.H = H; a.W = W;
        a.rows = rows->dev(); a.cols = cols->dev();
        a.thr = thr; a.half = half; a.cap = ctx->caps.max_peaks_per_part;
        a.counts = counts; a.peaks = peaks;
        // band height: keep the fp64 staging of the source rows <= 48 KB
        int band = H;
        auto src_rows = [&](int b0, int b1) {
            const int lo = b0 - half < 0 ? 0 : b0 - half;
            const int hi = b1 + half > H ? H : b1 + half;
            return rows->i1[hi - 1] - rows->i0[lo] + 1;
        };
        while (band > 8 && (size_t)src_rows(0, band) * w * sizeof(double) > 48 * 1024) band = (band + 1) / 2;
        band = ((band + 7) / 8) * 8;
        if (band > H) band = H;
        a.band_rows = band;
        a.n_bands = (H + band - 1) / band;
        int max_src = 0;
        for (int bi = 0; bi < a.n_bands; ++bi) {
            const int b0 = bi * band, b1 = b0 + band < H ? b0 + band : H;
            const int ns = src_rows(b0, b1);
            if (ns > max_src) max_src = ns;
        }
        const size_t smem = nms_up_smem(max_src, w, half, band, W);
        KernelTimer kt(ctx, kNmsUp, 1, s);
        CU(launch_nms_up(a, n, smem, s));
    } else {
        // materialised: resize (if up > 1) -> blur (if sigma > 0) -> NMS
        // materialised maps hold the K part channels only ([n][K][H][W]);
        // the background channel is never read (paf.py:300)
        const size_t frame_full = (size_t)K * H * W;
        int rc = ensure_full(ctx, (size_t)n * frame_full);
        if (rc) return rc;
        const float *nms_src = conf;
        int nms_C = C;
        long long src_frame = (long long)C * h * w;
        if (up > 1) {
            KernelTimer kt(ctx, kResize, 1, s);
            CU(launch_resize_planes(conf, (long long)C * h * w, K, (long long)n * K, h, w, ctx->d_full, H, W,
                                    rows->d_rec, cols->d_rec, s));
            nms_src = ctx->d_full;
            nms_C = K;
            src_frame = (long long)frame_full;
        }
        if (blur) {
            BlurTaps taps;
            make_taps(p->blur_sigma, taps);
            KernelTimer kt(ctx, kBlurRows, 2, s);   // rows + cols pass, timed together
            CU(launch_blur(nms_src, src_frame, ctx->d_tmp, ctx->d_full, (long long)frame_full, n, K,
                           H, W, taps, ctx->sms, s));
            nms_src = ctx->d_full;
            nms_C = K;
        }
        KernelTimer kt(ctx, kNmsPlane, 1, s);
        CU(launch_nms_plane(nms_src, n, nms_C, K, H, W, thr, half, ctx->caps.max_peaks_per_part,
                            counts, peaks, s));
    }

    if (two) {                                      // the parse stage on its own stream
        CU(cudaEventRecord(ctx->ev_nms[sc.set], sc.nms));
        CU(cudaStreamWaitEvent(sc.parse, ctx->ev_nms[sc.set], 0));
    }
    s = sc.parse;
    ParseArgs a{};
    a.topo = ctx->topo;
    a.paf = paf; a.h = h; a.w = w; a.up = up;
    if (up > 1) {
        a.rows = rows->dev(); a.cols = cols->dev();
        a.ry = (double)h / (double)H;
        a.rx = (double)w / (double)W;
        a.rrec = rows->d_rec; a.crec = cols->d_rec;
    }
    a.stride_eff = stride / up;
    a.n_samples = p->n_samples;
    a.dot_thr = p->sample_dot_threshold;
    a.good_min = p->good_fraction_min;
    {
        // paf.py:160-162 gate good >= good_min with good = n_good / n (IEEE
        // double division, the same on host and device): the least passing
        // n_good lets the kernel drop a pair as soon as it cannot pass
        const volatile double nd = (double)p->n_samples;
        a.good_need = p->n_samples + 1;
        for (int g = 0; g <= p->n_samples; ++g) {
            const volatile double q = (double)g / nd;
            if (q >= p->good_fraction_min) { a.good_need = g; break; }
        }
    }
    a.min_score = p->min_human_score;
    a.min_parts = p->min_parts;
    a.counts = counts; a.peaks = peaks;
    a.cap_part = ctx->caps.max_peaks_per_part;
    a.cap_frame = ctx->caps.max_peaks_per_frame;
    a.cap_cands = ctx->caps.max_candidates;
    a.cap_humans = ctx->caps.max_humans_per_frame;
    a.frame_base = frame_base;
    a.frame_first = ctx->d_frame_first; a.frame_count = ctx->d_frame_count;
    a.h_score = ctx->d_hscore; a.h_nparts = ctx->d_hnparts;
    a.kp_x = ctx->d_kpx; a.kp_y = ctx->d_kpy; a.kp_score = ctx->d_kps; a.kp_peak = ctx->d_kpp;
    a.pool_cap = pool_cap;
    a.st = ctx->d_status;
    a.debug = ctx->debug;
    a.dbg_npeaks = ctx->d_dbg_np; a.dbg_peaks = ctx->d_dbg_peaks;
    a.dbg_nconns = ctx->d_dbg_nc; a.dbg_conn_i = ctx->d_dbg_ci; a.dbg_conn_d = ctx->d_dbg_cd;
    a.cand_spill = ctx->d_spill;
    if (ctx->large) {                                // frames past the shared-memory capacities
        int rc = ensure_large_ws(ctx, (size_t)n);
        if (rc) return rc;
        {
            KernelTimer kt(ctx, kParseLarge, 1, s);
            CU(launch_parse_large(a, ctx->lws, n, s));
        }
        if (two) CU(cudaEventRecord(ctx->ev_parsed[sc.set], s));
        return PF_OK;
    }
    const bool psplit = !ctx->count_paf && (ctx->parse_split == 2 || (ctx->parse_split == 1 && n > ctx->sms * PF_WIDE_FRAMES_PER_SM));
    if (ctx->count_paf && L > 0) {
        a.paf_touch = ctx->d_paf_touch;
        a.touch_words = (int)(((size_t)2 * L * h * w + 255) / 256);   // 8 floats per sector, 32 sectors per word
    }
    if (psplit) {
        int rc = ensure_split_ws(ctx, (size_t)n);
        if (rc) return rc;
        a.split = 1;
        a.pk_cell = ctx->d_pk_cell; a.pk_score = ctx->d_pk_score; a.pk_base = ctx->d_pk_base;
        a.pair_pp = ctx->d_pair_pp; a.n_pairs = ctx->d_npairs; a.pair_base = ctx->d_pair_base;
        a.pair_total = ctx->d_pair_base + ctx->split_frames;
        a.ferr = ctx->d_ferr; a.cand_n = ctx->d_cand_n;
        a.crowd_frames = ctx->d_crowd_frames;
        a.crowd_cap = (int)ctx->split_frames;
        CU(cudaMemsetAsync(ctx->d_crowd_frames + ctx->split_frames, 0, sizeof(int), s));
        a.cand_g = reinterpret_cast<Cand *>(ctx->d_spill);
    }
    const int threads = psplit ? kParseFinThreads
                               : (n <= ctx->sms * PF_WIDE_FRAMES_PER_SM && !ctx->count_paf && sc.wide ? kParseWideThreads
                                                                                    : kParseThreads);
    // (the host path keeps the 128-thread form: its PAF read in place over PCIe
    // is request-rate bound, and beside the overlapped NMS stream the narrow
    // CTAs leave room for the next chunk's kernels -- 137-140k vs 131-137k e2e)
    const size_t smem =
        parse_smem_bytes(a.cap_frame, a.cap_part, a.cap_cands, a.cap_humans, K, ctx->topo.L, threads / 32, psplit);
    if (a.split) {
        {
            KernelTimer kt(ctx, kParsePeaks, 2, s);   // k_parse_peaks + k_pair_scan
            CU(launch_parse_peaks(a, n, s));
        }
        KernelTimer kt(ctx, kScorePairs, 1, s);
        CU(launch_score_pairs(a, n, s));
    }
    {
        KernelTimer kt(ctx, kParseFrames, 1, s);
        CU(launch_parse_frames(a, n, threads, smem, s));
    }
    if (two) CU(cudaEventRecord(ctx->ev_parsed[sc.set], s));
    return PF_OK;
}

int check_call(pf_ctx *ctx, int batch, int grid_h, int grid_w, int stride, const pf_params *p)
{
    int rc = validate_params_impl(ctx, p);          // ConfigError first (paf.py:295)
    if (rc) return rc;
    if (!ctx->has_topo) return fail(ctx, PF_ERR_CONTRACT, "topology not set");
    if (batch < 0) return fail(ctx, PF_ERR_CONTRACT, "batch must be >= 0");
    if (grid_h < 0 || grid_w < 0) return fail(ctx, PF_ERR_CONTRACT, "grid extents must be >= 0");
    if (stride < 1) return fail(ctx, PF_ERR_CONTRACT, "stride must be >= 1");   // types.py:194-195
    if (stride % p->upsample != 0)
        return fail(ctx, PF_ERR_CONTRACT, "stride %d not divisible by upsample %d", stride, p->upsample);
    if ((long long)grid_h * p->upsample > 65535 || (long long)grid_w * p->upsample > 65535)
        return fail(ctx, PF_ERR_CONTRACT, "parse grid exceeds 65535 cells per axis");
    return PF_OK;
}

// PF_OPT_COUNT_PAF: one zeroed sampled-sector bitmap per frame of the call.
int prepare_paf_touch(pf_ctx *ctx, int batch, int h, int w)
{
    ctx->touch_used = 0;
    if (!ctx->count_paf || ctx->topo.L == 0 || batch == 0) return PF_OK;
    const size_t words = (size_t)batch * (((size_t)2 * ctx->topo.L * h * w + 255) / 256);
    if (words > ctx->touch_cap) {
        cudaFree(ctx->d_paf_touch);
        ctx->d_paf_touch = nullptr;
        ctx->touch_cap = 0;
        CU(dev_alloc(&ctx->d_paf_touch, words));
        ctx->touch_cap = words;
    }
    CU(cudaMemsetAsync(ctx->d_paf_touch, 0, words * sizeof(uint32_t), ctx->stream));
    ctx->touch_used = words;
    return PF_OK;
}

int begin_call(pf_ctx *ctx, int batch, int pool_cap)
{
    int rc = ensure_frames(ctx, batch > 0 ? batch : 1);
    if (rc) return rc;
    rc = ensure_pool(ctx, pool_cap > 0 ? pool_cap : 1, ctx->topo.K);
    if (rc) return rc;
    rc = ensure_debug(ctx, batch > 0 ? batch : 1);
    if (rc) return rc;
    // status: code 0, frame INT_MAX, pool_used 0
    Status init{};
    init.frame = 0x7fffffff;
    *ctx->h_status = init;
    CU(cudaMemcpyAsync(ctx->d_status, ctx->h_status, sizeof(Status), cudaMemcpyHostToDevice, ctx->stream));
    ctx->results_ready = false;
    ctx->status_ready = false;
    return PF_OK;
}

// Output pool size for a call: the fixed cap if the caller set one, else
// 64 humans per frame, grown (never shrunk) to whatever a previous call needed.
int pool_cap_for(pf_ctx *ctx, int batch)
{
    if (ctx->caps.max_humans_total > 0) return ctx->caps.max_humans_total;
    long long v = 64LL * (batch > 0 ? batch : 1);
    if (v < (long long)ctx->pool_cap) v = (long long)ctx->pool_cap;
    if (v < ctx->pool_need) v = ctx->pool_need;
    return (int)(v > (1LL << 30) ? (1LL << 30) : v);
}

// Grow the automatic capacity a failed call ran out of; false if that
// capacity is fixed by the caller or cannot grow (shared-memory bound).
bool grow_cap(pf_ctx *ctx, const Status &st)
{
    if (!((ctx->auto_caps >> st.what) & 1)) return false;
    pf_caps c = ctx->caps;
    const long long need = st.value > 0 ? st.value : 1;
    // shared-memory / 16-bit bound limits of k_parse_frames; past them the
    // context parses through k_parse_large (HBM workspace, 32-bit indices)
    bool large = ctx->large != 0;
    switch (st.what) {
    case kCapPool:
        if ((long long)st.pool_used <= ctx->pool_need) return false;
        ctx->pool_need = st.pool_used;
        return true;
    case kCapPart: {
        long long v = c.max_peaks_per_part;
        while (v < need) v *= 2;
        if (v > (1 << 20)) return false;
        c.max_peaks_per_part = (int)v;
        if (c.max_peaks_per_part > c.max_peaks_per_frame && ((ctx->auto_caps >> kCapFrame) & 1))
            c.max_peaks_per_frame = c.max_peaks_per_part;
        break;
    }
    case kCapCands: {
        long long v = c.max_candidates;
        while (v < need) v *= 2;
        if (v > (1 << 26)) return false;
        c.max_candidates = (int)v;
        break;
    }
    case kCapFrame: {
        long long v = c.max_peaks_per_frame;
        while (v < need) v *= 2;
        if (v > (1 << 26)) return false;
        c.max_peaks_per_frame = (int)v;
        break;
    }
    case kCapHumans: {
        long long v = c.max_humans_per_frame * 2LL;
        if (v > (1 << 24)) return false;
        c.max_humans_per_frame = (int)v;
        break;
    }
    default:
        return false;
    }
    if (c.max_peaks_per_frame > 32767 || c.max_humans_per_frame > 32767 || c.max_candidates > (1 << 24)) large = true;
    const size_t smem = parse_smem_bytes(c.max_peaks_per_frame, c.max_peaks_per_part, c.max_candidates,
                                         c.max_humans_per_frame, PF_MAX_KEYPOINTS, PF_MAX_LIMBS,
                                         std::max(kParseThreads, kParseFinThreads) / 32, false) + 2048;
    if (smem > (size_t)ctx->max_smem) large = true;
    if (c.max_peaks_per_part == ctx->caps.max_peaks_per_part && c.max_candidates == ctx->caps.max_candidates &&
        c.max_peaks_per_frame == ctx->caps.max_peaks_per_frame &&
        c.max_humans_per_frame == ctx->caps.max_humans_per_frame && large == (ctx->large != 0))
        return false;
    if (large && !ctx->large) {
        ctx->large_auto = 1;
        ctx->caps_usual = ctx->caps;
    }
    ctx->caps = c;
    ctx->large = large ? 1 : 0;
    return true;
}

// A new call (not a capacity replay) after an automatic switch to the
// large-frame path starts on the usual path again.
void reset_large(pf_ctx *ctx)
{
    if (ctx->replaying || !ctx->large_auto) return;
    ctx->caps = ctx->caps_usual;
    ctx->large = 0;
    ctx->large_auto = 0;
}

int prepare_axes(pf_ctx *ctx, int h, int w, const pf_params *p, AxisCache **rows, AxisCache **cols)
{
    *rows = *cols = nullptr;
    if (p->upsample > 1 && h > 0 && w > 0) {
        int rc = get_axis(ctx, h, h * p->upsample, rows);
        if (rc) return rc;
        rc = get_axis(ctx, w, w * p->upsample, cols);
        if (rc) return rc;
    }
    return PF_OK;
}

int chunk_for(pf_ctx *ctx, const pf_params *p, int h, int w)
{
    int chunk = ctx->caps.chunk_frames;
    const bool materialise = (p->blur_sigma > 0.0 && !fused_blur(ctx, p, w * p->upsample)) ||
                             (p->upsample > 1 && (p->nms_window / 2 > kMaxFusedHalf || ctx->materialise));
    if (materialise) {
        // bound the full-resolution workspace ([chunk][K][H][W]) to ~2 GiB
        const size_t per = (size_t)ctx->topo.K * h * w * p->upsample * p->upsample * sizeof(float);
        size_t lim = per ? ((size_t)2 << 30) / per : chunk;
        if (lim < 1) lim = 1;
        if ((size_t)chunk > lim) chunk = (int)lim;
    }
    // bound the per-frame parse workspace (NMS slab, candidate lists, and
    // k_parse_large's tables) to ~4 GiB per chunk
    size_t per = (size_t)ctx->topo.K * ctx->caps.max_peaks_per_part * 8 +
                 (size_t)ctx->caps.max_candidates * cand_record_bytes();
    if (ctx->large) per += large_bytes_per_frame(ctx);
    const size_t lim = std::max<size_t>(1, ((size_t)4 << 30) / std::max<size_t>(per, 1));
    if ((size_t)chunk > lim) chunk = (int)lim;
    return chunk;
}

}  // namespace

extern "C" {

int pf_abi_version(void) { return PF_ABI_VERSION; }

int pf_create(pf_ctx **out, int device, const pf_caps *caps)
{
    if (!out) return fail(nullptr, PF_ERR_CONTRACT, "out is NULL");
    *out = nullptr;
    pf_caps c{};
    if (caps) c = *caps;
    // caps left at 0 are automatic: they start at the defaults and grow (with
    // a replay of the call) when a frame needs more; explicit caps are fixed
    int auto_caps = 0;
    if (c.max_peaks_per_part <= 0) { c.max_peaks_per_part = 128; auto_caps |= 1 << kCapPart; }
    if (c.max_peaks_per_frame <= 0) { c.max_peaks_per_frame = 256; auto_caps |= 1 << kCapFrame; }
    if (c.max_candidates <= 0) { c.max_candidates = 4096; auto_caps |= 1 << kCapCands; }
    if (c.max_humans_per_frame <= 0) { c.max_humans_per_frame = 64; auto_caps |= 1 << kCapHumans; }
    if (c.max_humans_total <= 0) auto_caps |= 1 << kCapPool;
    if (c.chunk_frames <= 0) c.chunk_frames = 8192;
    // bitonic sort over the candidate store needs a power of two
    int pc = 1;
    while (pc < c.max_candidates) pc <<= 1;
    c.max_candidates = pc;
    if (c.max_peaks_per_frame > (1 << 26)) return fail(nullptr, PF_ERR_CONFIG, "max_peaks_per_frame > 2^26");
    if (c.max_humans_per_frame > (1 << 24)) return fail(nullptr, PF_ERR_CONFIG, "max_humans_per_frame > 2^24");
    if (c.max_candidates > (1 << 26)) return fail(nullptr, PF_ERR_CONFIG, "max_candidates > 2^26");
    pf_ctx *ctx = new pf_ctx();
    ctx->device = device;
    ctx->caps = c;
    ctx->auto_caps = auto_caps;
    auto bail = [&](int code) {
        g_create_err = ctx->err;
        pf_destroy(ctx);
        return code;
    };
    if (set_device(ctx)) return bail(PF_ERR_CUDA);
    cudaDeviceProp prop;
    {
        cudaError_t e = cudaGetDeviceProperties(&prop, device);
        if (e != cudaSuccess) { fail(ctx, PF_ERR_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e)); return bail(PF_ERR_CUDA); }
    }
    if (prop.major < 10) {
        fail(ctx, PF_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a", device, prop.major, prop.minor);
        return bail(PF_ERR_CUDA);
    }
    ctx->sms = prop.multiProcessorCount;
    auto cu = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess) fail(ctx, PF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
        return e != cudaSuccess;
    };
    if (cu(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream") ||
        cu(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream") ||
        cu(cudaDeviceGetStreamPriorityRange(&ctx->prio_low, &ctx->prio_high), "stream priorities") ||
        // the parse stream first: its latency-bound CTAs are dispatched ahead of the next NMS stage's
        cu(cudaStreamCreateWithPriority(&ctx->parse_stream, cudaStreamNonBlocking, ctx->prio_high), "parse stream") ||
        cu(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming), "event"))
        return bail(PF_ERR_CUDA);
    for (int k = 0; k < 2; ++k) {
        if (cu(cudaEventCreateWithFlags(&ctx->ev_nms[k], cudaEventDisableTiming), "event") ||
            cu(cudaEventCreateWithFlags(&ctx->ev_parsed[k], cudaEventDisableTiming), "event"))
            return bail(PF_ERR_CUDA);
    }
    ctx->stream = ctx->own_stream;
    for (int k = 0; k < kHostSlots; ++k) {
        if (cu(cudaEventCreateWithFlags(&ctx->ev_copied[k], cudaEventDisableTiming), "event") ||
            cu(cudaEventCreateWithFlags(&ctx->ev_free[k], cudaEventDisableTiming), "event"))
            return bail(PF_ERR_CUDA);
    }
    if (cu(cudaMalloc(&ctx->d_status, sizeof(Status)), "cudaMalloc status") ||
        cu(cudaHostAlloc(&ctx->h_status, sizeof(Status), cudaHostAllocDefault), "cudaHostAlloc status"))
        return bail(PF_ERR_CUDA);
    const int max_smem = prop.sharedMemPerBlockOptin;
    ctx->max_smem = max_smem;
    {
        // explicit caps past k_parse_frames' shared-memory bounds: large path from the start
        const pf_caps &cc = ctx->caps;
        if (cc.max_peaks_per_frame > 32767 || cc.max_humans_per_frame > 32767 || cc.max_candidates > (1 << 24) ||
            parse_smem_bytes(cc.max_peaks_per_frame, cc.max_peaks_per_part, cc.max_candidates, cc.max_humans_per_frame,
                             PF_MAX_KEYPOINTS, PF_MAX_LIMBS, std::max(kParseThreads, kParseFinThreads) / 32, false) +
                    2048 > (size_t)max_smem)
            ctx->large = 1;
    }
    if (cu(configure_nms_kernels(max_smem), "configure k_nms_up") ||
        cu(configure_corner_kernels(max_smem), "configure k_nms_up_corner") ||
        cu(configure_parse_kernels(max_smem), "configure k_parse_frames") ||
        cu(configure_blur_kernels(max_smem), "configure k_up_blur_nms"))
        return bail(PF_ERR_CUDA);
    const size_t need = parse_smem_bytes(c.max_peaks_per_frame, c.max_peaks_per_part, c.max_candidates,
                                         c.max_humans_per_frame, PF_MAX_KEYPOINTS, PF_MAX_LIMBS,
                                         std::max(kParseThreads, kParseFinThreads) / 32, false) + 2048;
    if (need > (size_t)max_smem) {
        fail(ctx, PF_ERR_CONFIG, "caps need %zu B of shared memory per frame CTA (> %d)", need, max_smem);
        return bail(PF_ERR_CONFIG);
    }
    *out = ctx;
    return PF_OK;
}

void pf_destroy(pf_ctx *ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    void *dev[] = {ctx->d_counts, ctx->d_peaks, ctx->d_counts2, ctx->d_peaks2, ctx->d_spill, ctx->d_frame_first, ctx->d_frame_count,
                   ctx->d_hscore, ctx->d_hnparts, ctx->d_kpx, ctx->d_kpy, ctx->d_kps, ctx->d_kpp,
                   ctx->d_status, ctx->d_full, ctx->d_tmp,
                   ctx->d_dbg_np, ctx->d_dbg_nc, ctx->d_dbg_ci, ctx->d_dbg_peaks, ctx->d_dbg_cd,
                   ctx->d_corner_spill, ctx->d_paf_touch, ctx->d_surv, ctx->d_surv_n, ctx->d_crowd, ctx->d_exact, ctx->d_pk_cell, ctx->d_pk_score,
                   ctx->d_pk_base, ctx->d_pair_pp, ctx->d_npairs, ctx->d_pair_base, ctx->d_ferr, ctx->d_cand_n, ctx->d_crowd_frames,
                   ctx->d_owner};
    for (void *p : dev) cudaFree(p);
    {
        LargeWs &w = ctx->lws;
        void *lw[] = {w.pk_cell, w.pk_score, w.owner, w.cand, w.used, w.h_parts, w.h_order, w.h_n, w.h_alive,
                      w.h_mask, w.h_score, w.h_pos};
        for (void *p : lw) cudaFree(p);
    }
    for (float *p : ctx->d_in) cudaFree(p);
    void *host[] = {ctx->h_frame_first, ctx->h_frame_count, ctx->h_hscore, ctx->h_hnparts,
                    ctx->h_kpx, ctx->h_kpy, ctx->h_kps, ctx->h_kpp, ctx->h_status};
    for (void *p : host) cudaFreeHost(p);
    for (auto &kv : ctx->axes) {
        cudaFree(kv.second.d_i0); cudaFree(kv.second.d_i1);
        cudaFree(kv.second.d_t); cudaFree(kv.second.d_omt);
        cudaFree(kv.second.d_first); cudaFree(kv.second.d_last);
        cudaFree(kv.second.d_rec);
        cudaFree(kv.second.d_bands); cudaFree(kv.second.d_band_dt);
    }
    for (auto &p : ctx->pending) { ctx->ev_pool.push_back(p.second.first); ctx->ev_pool.push_back(p.second.second); }
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    for (int k = 0; k < kHostSlots; ++k) {
        if (ctx->ev_copied[k]) cudaEventDestroy(ctx->ev_copied[k]);
        if (ctx->ev_free[k]) cudaEventDestroy(ctx->ev_free[k]);
    }
    for (int k = 0; k < 2; ++k) {
        if (ctx->ev_nms[k]) cudaEventDestroy(ctx->ev_nms[k]);
        if (ctx->ev_parsed[k]) cudaEventDestroy(ctx->ev_parsed[k]);
    }
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->parse_stream) cudaStreamDestroy(ctx->parse_stream);
    delete ctx;
}

const char *pf_last_error(const pf_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int pf_set_stream(pf_ctx *ctx, void *cuda_stream)
{
    if (!ctx) return PF_ERR_CONTRACT;
    ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    return PF_OK;
}

int pf_use_own_stream(pf_ctx *ctx)
{
    if (!ctx) return PF_ERR_CONTRACT;
    ctx->stream = ctx->own_stream;
    return PF_OK;
}

int pf_set_topology(pf_ctx *ctx, int n_keypoints, int n_limbs, const int32_t *limbs,
                    const int32_t *paf_channels)
{
    if (!ctx) return PF_ERR_CONTRACT;
    // SkeletonTopology.validate (types.py:115-143)
    if (n_keypoints < 1) return fail(ctx, PF_ERR_CONTRACT, "topology needs at least one keypoint");
    if (n_keypoints > PF_MAX_KEYPOINTS)
        return fail(ctx, PF_ERR_CONTRACT, "at most %d keypoints supported", PF_MAX_KEYPOINTS);
    if (n_limbs < 0 || n_limbs > PF_MAX_LIMBS)
        return fail(ctx, PF_ERR_CONTRACT, "at most %d limbs supported", PF_MAX_LIMBS);
    if (n_limbs > 0 && (!limbs || !paf_channels)) return fail(ctx, PF_ERR_CONTRACT, "null limb tables");
    Topo t{};
    t.K = n_keypoints;
    t.L = n_limbs;
    std::vector<int> seen(2 * n_limbs + 1, -1);
    for (int l = 0; l < n_limbs; ++l) {
        const int a = limbs[2 * l], b = limbs[2 * l + 1];
        if (a == b) return fail(ctx, PF_ERR_CONTRACT, "limb %d connects keypoint %d to itself", l, a);
        if (a < 0 || a >= n_keypoints || b < 0 || b >= n_keypoints)
            return fail(ctx, PF_ERR_CONTRACT, "limb %d endpoint out of range: (%d, %d)", l, a, b);
        const int cx = paf_channels[2 * l], cy = paf_channels[2 * l + 1];
        for (int ch : {cx, cy}) {
            if (ch < 0 || ch >= 2 * n_limbs)
                return fail(ctx, PF_ERR_CONTRACT, "paf channel %d of limb %d out of range", ch, l);
            if (seen[ch] >= 0)
                return fail(ctx, PF_ERR_CONTRACT, "paf channel %d shared by limbs %d and %d", ch, seen[ch], l);
            seen[ch] = l;
        }
        if (cx == cy) return fail(ctx, PF_ERR_CONTRACT, "limb %d maps both components to channel %d", l, cx);
        t.la[l] = (int8_t)a;
        t.lb[l] = (int8_t)b;
        t.cx[l] = (int16_t)cx;
        t.cy[l] = (int16_t)cy;
    }
    ctx->topo = t;
    ctx->has_topo = true;
    return PF_OK;
}

int pf_validate_params(const pf_params *p) { return validate_params_impl(nullptr, p); }

int pf_set_debug(pf_ctx *ctx, int enable)
{
    if (!ctx) return PF_ERR_CONTRACT;
    ctx->debug = enable ? 1 : 0;
    return PF_OK;
}

int pf_set_option(pf_ctx *ctx, int option, int value)
{
    if (!ctx) return PF_ERR_CONTRACT;
    switch (option) {
    case PF_OPT_DEBUG: ctx->debug = value ? 1 : 0; return PF_OK;
    case PF_OPT_TIMING: ctx->timing = value ? 1 : 0; return PF_OK;
    case PF_OPT_MATERIALISE: ctx->materialise = value ? 1 : 0; return PF_OK;
    case PF_OPT_GENERIC_FUSED: ctx->generic_fused = value ? 1 : 0; return PF_OK;
    case PF_OPT_WIN_VARIANT: ctx->win_variant = (value >= 1 && value <= 4) ? value : 4; return PF_OK;
    case PF_OPT_NO_CHAIN: ctx->no_chain = value ? 1 : 0; return PF_OK;
    case PF_OPT_PAF_ZERO_COPY: ctx->paf_zero_copy = value ? 1 : 0; return PF_OK;
    case PF_OPT_CONF_ZERO_COPY: ctx->conf_zero_copy = value ? 1 : 0; return PF_OK;
    case PF_OPT_CORNER_SPLIT: ctx->corner_split = (value >= 0 && value <= 2) ? value : 1; return PF_OK;
    case PF_OPT_PARSE_SPLIT: ctx->parse_split = (value >= 0 && value <= 2) ? value : 1; return PF_OK;
    case PF_OPT_PDL: g_pdl_mask = value; return PF_OK;
    case PF_OPT_COUNT_PAF: ctx->count_paf = value ? 1 : 0; return PF_OK;
    case PF_OPT_LARGE: ctx->large = value ? 1 : 0; return PF_OK;
    case PF_OPT_HOST_OVERLAP: ctx->host_overlap = value ? 1 : 0; return PF_OK;
    case PF_OPT_EXACT_LIST: ctx->exact_opt = value; return PF_OK;
    default: return fail(ctx, PF_ERR_CONFIG, "unknown option %d", option);
    }
}

const char *pf_kernel_name(int id) { return id >= 0 && id < PF_N_KERNELS ? kKernelNames[id] : ""; }

int pf_get_kernel_times(pf_ctx *ctx, double *ms, int64_t *launches, int reset)
{
    if (!ctx) return PF_ERR_CONTRACT;
    if (!ctx->pending.empty()) {
        CU(cudaStreamSynchronize(ctx->stream));
        for (auto &p : ctx->pending) {
            float t = 0.f;
            CU(cudaEventElapsedTime(&t, p.second.first, p.second.second));
            ctx->kernel_ms[p.first] += t;
            ctx->ev_pool.push_back(p.second.first);
            ctx->ev_pool.push_back(p.second.second);
        }
        ctx->pending.clear();
    }
    for (int k = 0; k < PF_N_KERNELS; ++k) {
        if (ms) ms[k] = ctx->kernel_ms[k];
        if (launches) launches[k] = ctx->kernel_launches[k];
        if (reset) { ctx->kernel_ms[k] = 0.0; ctx->kernel_launches[k] = 0; }
    }
    return PF_OK;
}

int pf_parse_device(pf_ctx *ctx, const float *conf, const float *paf, int batch, int grid_h,
                    int grid_w, int stride, const pf_params *p)
{
    if (!ctx) return PF_ERR_CONTRACT;
    int rc = check_call(ctx, batch, grid_h, grid_w, stride, p);
    if (rc) return rc;
    rc = set_device(ctx);
    if (rc) return rc;
    reset_large(ctx);
    const int K = ctx->topo.K, L = ctx->topo.L;
    const int pool = pool_cap_for(ctx, batch);
    rc = begin_call(ctx, batch, pool);
    if (rc) return rc;
    rc = prepare_paf_touch(ctx, batch, grid_h, grid_w);
    if (rc) return rc;
    ctx->last_batch = batch;
    ctx->last_K = K;
    ctx->last.kind = 1;
    ctx->last.conf = conf; ctx->last.paf = paf;
    ctx->last.batch = batch; ctx->last.h = grid_h; ctx->last.w = grid_w; ctx->last.stride = stride;
    ctx->last.p = *p;
    if (batch == 0) return PF_OK;
    if (grid_h == 0 || grid_w == 0) {
        // no cells, no peaks: every frame parses to [] (nms_peaks on empty maps)
        CU(cudaMemsetAsync(ctx->d_frame_count, 0, sizeof(int) * batch, ctx->stream));
        CU(cudaMemsetAsync(ctx->d_frame_first, 0, sizeof(int) * batch, ctx->stream));
        if (ctx->debug) {
            CU(cudaMemsetAsync(ctx->d_dbg_np, 0, sizeof(int) * batch, ctx->stream));
            CU(cudaMemsetAsync(ctx->d_dbg_nc, 0, sizeof(int) * batch, ctx->stream));
        }
        return PF_OK;
    }
    if (!conf || (L > 0 && !paf)) return fail(ctx, PF_ERR_CONTRACT, "null map pointer");
    AxisCache *rows, *cols;
    rc = prepare_axes(ctx, grid_h, grid_w, p, &rows, &cols);
    if (rc) return rc;
    const int chunk = chunk_for(ctx, p, grid_h, grid_w);
    rc = ensure_nms_ws(ctx, chunk, K);
    if (rc) return rc;
    const size_t conf_frame = (size_t)(K + 1) * grid_h * grid_w;
    const size_t paf_frame = (size_t)2 * L * grid_h * grid_w;
    for (int f0 = 0; f0 < batch; f0 += chunk) {
        const int n = batch - f0 < chunk ? batch - f0 : chunk;
        rc = run_chunk(ctx, conf + (size_t)f0 * conf_frame, paf + (size_t)f0 * paf_frame, n, f0,
                       grid_h, grid_w, stride, p, rows, cols, pool, Sched{ctx->stream, ctx->stream, 0, true});
        if (rc) return rc;
    }
    return PF_OK;
}

int pf_get_results(pf_ctx *ctx, pf_results *out)
{
    if (!ctx || !out) return PF_ERR_CONTRACT;
    int rc = set_device(ctx);
    if (rc) return rc;
    const int B = ctx->last_batch;
    const int K = ctx->last_K;
    if (!ctx->results_ready) {
        CU(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(Status), cudaMemcpyDeviceToHost, ctx->stream));
        if (B > 0) {
            CU(cudaMemcpyAsync(ctx->h_frame_first, ctx->d_frame_first, sizeof(int) * B,
                               cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaMemcpyAsync(ctx->h_frame_count, ctx->d_frame_count, sizeof(int) * B,
                               cudaMemcpyDeviceToHost, ctx->stream));
        }
        CU(cudaStreamSynchronize(ctx->stream));
        const Status st = *ctx->h_status;
        if (st.code == PF_ERR_CAPACITY && ctx->last.kind != 0 && grow_cap(ctx, st)) {
            // an automatic capacity was too small for some frame: it has been
            // grown to the need and the call is replayed (inputs must stay
            // valid until results are fetched)
            const auto L = ctx->last;
            ctx->replaying = 1;
            rc = L.kind == 1 ? pf_parse_device(ctx, L.conf, L.paf, L.batch, L.h, L.w, L.stride, &L.p)
                             : pf_parse_host(ctx, L.conf, L.paf, L.batch, L.h, L.w, L.stride, &L.p, nullptr);
            ctx->replaying = 0;
            if (rc) return rc;
            return pf_get_results(ctx, out);
        }
        if (st.code == PF_ERR_CAPACITY) {
            static const char *what[] = {"?", "max_peaks_per_part", "max_peaks_per_frame",
                                         "max_candidates", "max_humans_per_frame", "max_humans_total"};
            const int wi = st.what >= 1 && st.what <= 5 ? st.what : 0;
            return fail(ctx, PF_ERR_CAPACITY, "frame %d exceeds capacity %s (needs %d)", st.frame,
                        what[wi], st.value);
        }
        const size_t total = (size_t)st.pool_used;
        if (total > 0) {
            CU(cudaMemcpyAsync(ctx->h_hscore, ctx->d_hscore, sizeof(double) * total, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaMemcpyAsync(ctx->h_hnparts, ctx->d_hnparts, sizeof(int) * total, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaMemcpyAsync(ctx->h_kpx, ctx->d_kpx, sizeof(double) * total * K, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaMemcpyAsync(ctx->h_kpy, ctx->d_kpy, sizeof(double) * total * K, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaMemcpyAsync(ctx->h_kps, ctx->d_kps, sizeof(float) * total * K, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaMemcpyAsync(ctx->h_kpp, ctx->d_kpp, sizeof(int) * total * K, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
        }
        ctx->results_ready = true;
    }
    out->n_frames = B;
    out->n_keypoints = K;
    out->total_humans = ctx->h_status->pool_used;
    out->frame_first = ctx->h_frame_first;
    out->frame_count = ctx->h_frame_count;
    out->human_score = ctx->h_hscore;
    out->human_n_parts = ctx->h_hnparts;
    out->kp_x = ctx->h_kpx;
    out->kp_y = ctx->h_kpy;
    out->kp_score = ctx->h_kps;
    out->kp_peak = ctx->h_kpp;
    return PF_OK;
}

int pf_parse_host(pf_ctx *ctx, const float *conf, const float *paf, int batch, int grid_h, int grid_w,
                  int stride, const pf_params *p, pf_results *out)
{
    if (!ctx) return PF_ERR_CONTRACT;
    int rc = check_call(ctx, batch, grid_h, grid_w, stride, p);
    if (rc) return rc;
    rc = set_device(ctx);
    if (rc) return rc;
    reset_large(ctx);
    const int K = ctx->topo.K, L = ctx->topo.L;
    if (batch == 0 || grid_h == 0 || grid_w == 0) {
        rc = pf_parse_device(ctx, nullptr, nullptr, batch, grid_h, grid_w, stride, p);
        if (rc) return rc;
        return out ? pf_get_results(ctx, out) : PF_OK;
    }
    if (!conf || (L > 0 && !paf)) return fail(ctx, PF_ERR_CONTRACT, "null map pointer");
    const int pool = pool_cap_for(ctx, batch);
    rc = begin_call(ctx, batch, pool);
    if (rc) return rc;
    rc = prepare_paf_touch(ctx, batch, grid_h, grid_w);
    if (rc) return rc;
    ctx->last_batch = batch;
    ctx->last_K = K;
    ctx->last.kind = 2;
    ctx->last.conf = conf; ctx->last.paf = paf;
    ctx->last.batch = batch; ctx->last.h = grid_h; ctx->last.w = grid_w; ctx->last.stride = stride;
    ctx->last.p = *p;
    AxisCache *rows, *cols;
    rc = prepare_axes(ctx, grid_h, grid_w, p, &rows, &cols);
    if (rc) return rc;
    int chunk = chunk_for(ctx, p, grid_h, grid_w);
#ifndef PF_HOST_CHUNK
#define PF_HOST_CHUNK 128   // e2e (8192 frames): 131.5-132k at 128-192, 127.6k at 256, 120.6k at 64, 112k at 512
#endif
    if (chunk > PF_HOST_CHUNK) chunk = PF_HOST_CHUNK;   // copy/compute overlap granularity
    // PF_OPT_PAF_ZERO_COPY: a pinned (mapped) host PAF is read in place by
    // k_parse_frames over PCIe -- only the sampled cells cross the link
    // instead of the whole 2L-channel field.
    const float *paf_dev = nullptr, *conf_dev = nullptr;
    if (ctx->paf_zero_copy && L > 0) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, paf) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr)
            paf_dev = static_cast<const float *>(pa.devicePointer);
        cudaGetLastError();
    }
    if (ctx->conf_zero_copy) {        // the NMS kernels stream the planes over PCIe themselves
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, conf) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr)
            conf_dev = static_cast<const float *>(pa.devicePointer);
        cudaGetLastError();
    }
    // PF_OPT_HOST_OVERLAP: the NMS stage of chunk c+1 runs on ctx->stream
    // beside the parse of chunk c on parse_stream (two NMS slab sets); the
    // in-place PAF parse is bound by the PCIe read-request rate, the NMS
    // stage by the SMs, so they overlap
    const bool ov = ctx->host_overlap && !ctx->count_paf && !ctx->large && batch > chunk;
    rc = ensure_nms_ws(ctx, chunk, K, ov ? 2 : 1);
    if (rc) return rc;
    const size_t plane = (size_t)grid_h * grid_w;
    const size_t conf_frame = (size_t)(K + 1) * plane, paf_frame = (size_t)2 * L * plane;
    const size_t slot = (size_t)chunk * (conf_frame + paf_frame);
    if (slot > ctx->in_elems) {
        for (float *&p : ctx->d_in) {
            cudaFree(p);
            p = nullptr;
        }
        for (float *&p : ctx->d_in) CU(dev_alloc(&p, slot));
        ctx->in_elems = slot;
    }
    // a PAF read in place over PCIe: the one-kernel parse keeps each frame's
    // gathers on one SM (measured 131k vs 120k frames/s for the split parse)
    const int saved_split = ctx->parse_split;
    if (paf_dev) ctx->parse_split = 0;
    struct Restore {
        pf_ctx *c;
        int v;
        ~Restore() { c->parse_split = v; }
    } restore{ctx, saved_split};
    // slots start free
    for (int k = 0; k < kHostSlots; ++k) CU(cudaEventRecord(ctx->ev_free[k], ctx->stream));
    struct Join {                       // the parse stream rejoins ctx->stream on every exit
        pf_ctx *c;
        bool on;
        void now()
        {
            if (on && cudaEventRecord(c->ev_join, c->parse_stream) == cudaSuccess)
                cudaStreamWaitEvent(c->stream, c->ev_join, 0);
            on = false;
        }
        ~Join() { now(); }
    } join{ctx, ov};
    if (ov) {
        CU(cudaEventRecord(ctx->ev_join, ctx->stream));
        CU(cudaStreamWaitEvent(ctx->parse_stream, ctx->ev_join, 0));
        for (int k = 0; k < 2; ++k) CU(cudaEventRecord(ctx->ev_parsed[k], ctx->parse_stream));
    }
    int ci = 0;
    for (int f0 = 0; f0 < batch; f0 += chunk, ++ci) {
        const int n = batch - f0 < chunk ? batch - f0 : chunk;
        const int sl = ci % kHostSlots;
        float *dconf = ctx->d_in[sl];
        float *dpaf = dconf + (size_t)n * conf_frame;
        CU(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_free[sl], 0));
        // the background channel (index K) is never read: copy K of K+1 planes per frame
        if (!conf_dev)
            CU(cudaMemcpy2DAsync(dconf, conf_frame * sizeof(float), conf + (size_t)f0 * conf_frame,
                                 conf_frame * sizeof(float), (size_t)K * plane * sizeof(float), n,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
        if (L > 0 && !paf_dev)
            CU(cudaMemcpyAsync(dpaf, paf + (size_t)f0 * paf_frame, (size_t)n * paf_frame * sizeof(float),
                               cudaMemcpyHostToDevice, ctx->copy_stream));
        CU(cudaEventRecord(ctx->ev_copied[sl], ctx->copy_stream));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[sl], 0));
        rc = run_chunk(ctx, conf_dev ? conf_dev + (size_t)f0 * conf_frame : dconf,
                       paf_dev ? paf_dev + (size_t)f0 * paf_frame : dpaf, n, f0, grid_h, grid_w,
                       stride, p, rows, cols, pool,
                       ov ? Sched{ctx->stream, ctx->parse_stream, ci & 1, false}
                          : Sched{ctx->stream, ctx->stream, 0, false});
        if (rc) return rc;
        // the slot is free once its last reader is done: the NMS stage, or the
        // parse when the PAF was copied into the slot
        CU(cudaEventRecord(ctx->ev_free[sl], ov && !paf_dev ? ctx->parse_stream : ctx->stream));
    }
    join.now();
    return out ? pf_get_results(ctx, out) : PF_OK;
}

int pf_get_paf_sectors(pf_ctx *ctx, long long *sectors)
{
    if (!ctx || !sectors) return PF_ERR_CONTRACT;
    *sectors = 0;
    if (!ctx->count_paf) return fail(ctx, PF_ERR_CONTRACT, "PF_OPT_COUNT_PAF is off");
    int rc = set_device(ctx);
    if (rc) return rc;
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->touch_used == 0) return PF_OK;
    std::vector<uint32_t> bm(ctx->touch_used);
    CU(cudaMemcpy(bm.data(), ctx->d_paf_touch, bm.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    long long n = 0;
    for (uint32_t v : bm) n += __builtin_popcount(v);
    *sectors = n;
    return PF_OK;
}

// pf_parse_batch's scatter: warp per frame, the frame's humans from the
// context pool (frame_first / frame_count) into the caller's [B][Hmax] slots.
__global__ void k_scatter_out(const Status *__restrict__ st, int B, int K, const int *__restrict__ first,
                              const int *__restrict__ count, const double *__restrict__ hs,
                              const int *__restrict__ hn, const double *__restrict__ kx,
                              const double *__restrict__ ky, const float *__restrict__ ks,
                              const int *__restrict__ kp, pf_out o)
{
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int code = st->code;
    if (code != 0 && warp == 0 && lane == 0) {                 // internal capacity: nothing is valid
        atomicMax(o.status, code);
        atomicMin(reinterpret_cast<unsigned *>(o.status + 1), (unsigned)st->frame);
    }
    for (int f = warp; f < B; f += nwarps) {
        const int n = code != 0 ? 0 : count[f];
        if (lane == 0) {
            o.n_humans[f] = n;
            if (n > o.max_humans) {
                atomicMax(o.status, PF_ERR_CAPACITY);
                atomicMin(reinterpret_cast<unsigned *>(o.status + 1), (unsigned)f);
            }
        }
        const int nh = min(n, o.max_humans), h0 = first[f];
        const size_t slot0 = (size_t)f * o.max_humans;
        for (int h = lane; h < nh; h += kWarp) {
            o.human_score[slot0 + h] = hs[h0 + h];
            o.n_parts[slot0 + h] = hn[h0 + h];
        }
        for (int e = lane; e < nh * K; e += kWarp) {
            const size_t src = (size_t)h0 * K + e, dst = slot0 * K + e;
            const bool present = kp[src] >= 0;
            o.kp_xy[2 * dst] = present ? kx[src] : 0.0;
            o.kp_xy[2 * dst + 1] = present ? ky[src] : 0.0;
            o.kp_score[dst] = present ? ks[src] : 0.f;
            o.kp_present[dst] = present ? 1 : 0;
        }
    }
}

int pf_parse_batch(pf_ctx *ctx, const float *conf, const float *paf, int batch, int grid_h, int grid_w,
                   int stride, const pf_params *p, const pf_out *out, void *cuda_stream)
{
    if (!ctx) return PF_ERR_CONTRACT;
    if (!out || !out->status) return fail(ctx, PF_ERR_CONTRACT, "pf_parse_batch: null output / status");
    if (out->max_humans < 0) return fail(ctx, PF_ERR_CONTRACT, "pf_parse_batch: max_humans must be >= 0");
    if (batch > 0 && (!out->n_humans || (out->max_humans > 0 && (!out->human_score || !out->n_parts ||
                                                                  !out->kp_xy || !out->kp_score ||
                                                                  !out->kp_present))))
        return fail(ctx, PF_ERR_CONTRACT, "pf_parse_batch: null output array");
    struct Restore {
        pf_ctx *c;
        cudaStream_t s;
        ~Restore() { c->stream = s; }
    } restore{ctx, ctx->stream};
    if (cuda_stream) ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    int rc = pf_parse_device(ctx, conf, paf, batch, grid_h, grid_w, stride, p);
    ctx->last.kind = 0;                                  // never replayed: inputs only for the call
    if (rc) return rc;
    CU(cudaMemsetAsync(out->status, 0, sizeof(int32_t), ctx->stream));
    CU(cudaMemsetAsync(out->status + 1, 0xff, sizeof(int32_t), ctx->stream));   // -1: no frame
    if (batch == 0) return PF_OK;
    const int threads = 256;
    const int blocks = std::min((batch * kWarp + threads - 1) / threads, ctx->sms * 8);
    {
        KernelTimer kt(ctx, kScatterOut);
        k_scatter_out<<<blocks, threads, 0, ctx->stream>>>(ctx->d_status, batch, ctx->topo.K, ctx->d_frame_first,
                                                            ctx->d_frame_count, ctx->d_hscore, ctx->d_hnparts,
                                                            ctx->d_kpx, ctx->d_kpy, ctx->d_kps, ctx->d_kpp, *out);
        CU(cudaGetLastError());
    }
    return PF_OK;
}

int pf_get_results_into(pf_ctx *ctx, const pf_host_out *dst, int32_t *n_frames, int32_t *total_humans)
{
    if (!ctx || !dst || !n_frames || !total_humans) return PF_ERR_CONTRACT;
    if (dst->capacity < 0) return fail(ctx, PF_ERR_CONTRACT, "pf_get_results_into: negative capacity");
    int rc = set_device(ctx);
    if (rc) return rc;
    // the status (and, on a capacity overflow, the grow + replay) as pf_get_results
    if (!ctx->results_ready && !ctx->status_ready) {
        CU(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(Status), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        const Status st = *ctx->h_status;
        if (st.code == PF_ERR_CAPACITY) {
            pf_results tmp;                      // grows, replays and reports exactly like pf_get_results
            rc = pf_get_results(ctx, &tmp);
            if (rc) return rc;
        }
        ctx->status_ready = true;
    }
    const int B = ctx->last_batch;
    const int K = ctx->last_K;
    const int total = ctx->h_status->pool_used;
    *n_frames = B;
    *total_humans = total;
    if (total > dst->capacity) return PF_ERR_CAPACITY;   // no message: the caller grows its arrays
    if (B > 0 && (!dst->frame_first || !dst->frame_count))
        return fail(ctx, PF_ERR_CONTRACT, "pf_get_results_into: null frame arrays");
    if (total > 0 && (!dst->human_score || !dst->human_n_parts || !dst->kp_x || !dst->kp_y || !dst->kp_score ||
                      !dst->kp_peak))
        return fail(ctx, PF_ERR_CONTRACT, "pf_get_results_into: null human arrays");
    if (B > 0) {
        CU(cudaMemcpyAsync(dst->frame_first, ctx->d_frame_first, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(dst->frame_count, ctx->d_frame_count, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (total > 0) {
        const size_t t = (size_t)total;
        CU(cudaMemcpyAsync(dst->human_score, ctx->d_hscore, sizeof(double) * t, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(dst->human_n_parts, ctx->d_hnparts, sizeof(int) * t, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(dst->kp_x, ctx->d_kpx, sizeof(double) * t * K, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(dst->kp_y, ctx->d_kpy, sizeof(double) * t * K, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(dst->kp_score, ctx->d_kps, sizeof(float) * t * K, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(dst->kp_peak, ctx->d_kpp, sizeof(int) * t * K, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    return PF_OK;
}

int pf_sync(pf_ctx *ctx)
{
    if (!ctx) return PF_ERR_CONTRACT;
    CU(cudaStreamSynchronize(ctx->stream));
    return PF_OK;
}

int pf_get_peaks(pf_ctx *ctx, int frame, int *n_peaks, int32_t *part, int32_t *row, int32_t *col,
                 float *score)
{
    if (!ctx || !n_peaks) return PF_ERR_CONTRACT;
    if (!ctx->debug || !ctx->d_dbg_np) return fail(ctx, PF_ERR_CONTRACT, "debug capture not enabled");
    if (frame < 0 || frame >= ctx->last_batch) return fail(ctx, PF_ERR_CONTRACT, "frame out of range");
    CU(cudaStreamSynchronize(ctx->stream));
    int n = 0;
    CU(cudaMemcpy(&n, ctx->d_dbg_np + frame, sizeof(int), cudaMemcpyDeviceToHost));
    *n_peaks = n;
    if (!part && !row && !col && !score) return PF_OK;
    std::vector<int4> buf(n > 0 ? n : 1);
    if (n > 0)
        CU(cudaMemcpy(buf.data(), ctx->d_dbg_peaks + (size_t)frame * ctx->caps.max_peaks_per_frame,
                      sizeof(int4) * n, cudaMemcpyDeviceToHost));
    for (int q = 0; q < n; ++q) {
        if (part) part[q] = buf[q].x;
        if (row) row[q] = buf[q].y;
        if (col) col[q] = buf[q].z;
        if (score) { int bits = buf[q].w; std::memcpy(&score[q], &bits, sizeof(float)); }
    }
    return PF_OK;
}

int pf_get_connections(pf_ctx *ctx, int frame, int *n_conns, int32_t *limb, int32_t *id_a,
                       int32_t *id_b, double *score, double *good)
{
    if (!ctx || !n_conns) return PF_ERR_CONTRACT;
    if (!ctx->debug || !ctx->d_dbg_nc) return fail(ctx, PF_ERR_CONTRACT, "debug capture not enabled");
    if (frame < 0 || frame >= ctx->last_batch) return fail(ctx, PF_ERR_CONTRACT, "frame out of range");
    CU(cudaStreamSynchronize(ctx->stream));
    int n = 0;
    CU(cudaMemcpy(&n, ctx->d_dbg_nc + frame, sizeof(int), cudaMemcpyDeviceToHost));
    *n_conns = n;
    if (!limb && !id_a && !id_b && !score && !good) return PF_OK;
    std::vector<int> ci((size_t)(n > 0 ? n : 1) * 3);
    std::vector<double> cd((size_t)(n > 0 ? n : 1) * 2);
    if (n > 0) {
        const size_t o = (size_t)frame * ctx->caps.max_candidates;
        CU(cudaMemcpy(ci.data(), ctx->d_dbg_ci + o * 3, sizeof(int) * 3 * n, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(cd.data(), ctx->d_dbg_cd + o * 2, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    }
    for (int q = 0; q < n; ++q) {
        if (limb) limb[q] = ci[q * 3 + 0];
        if (id_a) id_a[q] = ci[q * 3 + 1];
        if (id_b) id_b[q] = ci[q * 3 + 2];
        if (score) score[q] = cd[q * 2 + 0];
        if (good) good[q] = cd[q * 2 + 1];
    }
    return PF_OK;
}

static int preprocess_impl(pf_ctx *ctx, const void *src, int is_f32, int batch, int h, int w,
                           float *dst, int out_h, int out_w)
{
    if (!ctx) return PF_ERR_CONTRACT;
    // operators.py:120-121 zero-area frame; operators.py:83 positive extents
    if (h < 1 || w < 1) return fail(ctx, PF_ERR_CONTRACT, "zero-area frame");
    if (out_h < 1 || out_w < 1) return fail(ctx, PF_ERR_CONTRACT, "resize requires positive extents");
    if (batch < 0) return fail(ctx, PF_ERR_CONTRACT, "batch must be >= 0");
    if (batch == 0) return PF_OK;
    if (!src || !dst) return fail(ctx, PF_ERR_CONTRACT, "null image pointer");
    int rc = set_device(ctx);
    if (rc) return rc;
    const AxisRec *rt = nullptr, *ct = nullptr;
    if (h != out_h || w != out_w) {
        if (h > 65535 || w > 65535) return fail(ctx, PF_ERR_CONTRACT, "source extents exceed 65535");
        AxisCache *r, *c;
        rc = get_axis(ctx, h, out_h, &r);
        if (rc) return rc;
        rc = get_axis(ctx, w, out_w, &c);
        if (rc) return rc;
        rt = r->d_rec;
        ct = c->d_rec;
    }
    KernelTimer kt(ctx, kPreprocess);
    CU(launch_preprocess(src, is_f32, batch, h, w, dst, out_h, out_w, rt, ct, ctx->stream));
    return PF_OK;
}

int pf_preprocess_device(pf_ctx *ctx, const uint8_t *src, int batch, int h, int w, float *dst,
                         int out_h, int out_w)
{
    return preprocess_impl(ctx, src, 0, batch, h, w, dst, out_h, out_w);
}

int pf_preprocess_f32_device(pf_ctx *ctx, const float *src, int batch, int h, int w, float *dst,
                             int out_h, int out_w)
{
    return preprocess_impl(ctx, src, 1, batch, h, w, dst, out_h, out_w);
}

int pf_resize_device(pf_ctx *ctx, const float *src, int n_planes, int in_h, int in_w, float *dst,
                     int out_h, int out_w)
{
    if (!ctx) return PF_ERR_CONTRACT;
    if (in_h < 1 || in_w < 1 || out_h < 1 || out_w < 1)
        return fail(ctx, PF_ERR_CONTRACT, "resize requires positive extents");
    if (n_planes < 0) return fail(ctx, PF_ERR_CONTRACT, "n_planes must be >= 0");
    if (n_planes == 0) return PF_OK;
    if (!src || !dst) return fail(ctx, PF_ERR_CONTRACT, "null plane pointer");
    int rc = set_device(ctx);
    if (rc) return rc;
    if (in_h == out_h && in_w == out_w) {   // operators.py:84-85 exact copy
        CU(cudaMemcpyAsync(dst, src, sizeof(float) * (size_t)n_planes * in_h * in_w,
                           cudaMemcpyDeviceToDevice, ctx->stream));
        return PF_OK;
    }
    AxisCache *r, *c;
    rc = get_axis(ctx, in_h, out_h, &r);
    if (rc) return rc;
    rc = get_axis(ctx, in_w, out_w, &c);
    if (rc) return rc;
    KernelTimer kt(ctx, kResize);
    CU(launch_resize_planes(src, (long long)in_h * in_w, 1, n_planes, in_h, in_w, dst, out_h, out_w, r->d_rec,
                            c->d_rec, ctx->stream));
    return PF_OK;
}

int pf_overlay(pf_ctx *ctx, const pf_overlay_prim *prims, const int32_t *prim_first, int n_prims, int frames,
               int h, int w, float *img)
{
    if (!ctx) return PF_ERR_CONTRACT;
    if (frames < 0 || h < 0 || w < 0 || n_prims < 0) return fail(ctx, PF_ERR_CONTRACT, "negative extents");
    if ((long long)frames * h * w == 0) return PF_OK;
    if (!img || !prim_first || (n_prims > 0 && !prims)) return fail(ctx, PF_ERR_CONTRACT, "null pointer");
    int rc = set_device(ctx);
    if (rc) return rc;
    const size_t px = (size_t)frames * h * w;
    if (px > ctx->overlay_px) {
        cudaFree(ctx->d_owner);
        ctx->d_owner = nullptr;
        ctx->overlay_px = 0;
        CU(dev_alloc(&ctx->d_owner, px));
        ctx->overlay_px = px;
    }
    CU(launch_overlay(prims, prim_first, n_prims, frames, h, w, ctx->d_owner, img, ctx->sms, ctx->stream));
    return PF_OK;
}

int pf_render_maps(pf_ctx *ctx, const double *kp_cells, const int32_t *n_humans, int frames, int max_humans,
                   int grid_h, int grid_w, double sigma, double halfwidth, float *conf, float *paf)
{
    if (!ctx) return PF_ERR_CONTRACT;
    if (!ctx->has_topo) return fail(ctx, PF_ERR_CONTRACT, "topology not set");
    if (frames < 0 || max_humans < 0 || grid_h < 0 || grid_w < 0)
        return fail(ctx, PF_ERR_CONTRACT, "negative extents");
    if (!(sigma > 0.0) || !(halfwidth > 0.0)) return fail(ctx, PF_ERR_CONFIG, "sigma and halfwidth must be > 0");
    if ((long long)frames * grid_h * grid_w == 0) return PF_OK;
    if (!kp_cells || !n_humans || !conf || !paf) return fail(ctx, PF_ERR_CONTRACT, "null pointer");
    int rc = set_device(ctx);
    if (rc) return rc;
    RenderArgs a{};
    a.topo = ctx->topo;
    a.kp = kp_cells; a.n_humans = n_humans;
    a.F = frames; a.hmax = max_humans; a.gh = grid_h; a.gw = grid_w;
    a.sigma = sigma; a.halfwidth = halfwidth;
    a.conf = conf; a.paf = paf;
    CU(launch_render_maps(a, ctx->sms, ctx->stream));
    return PF_OK;
}

int pf_gaussian_taps(double sigma, double *taps, int cap)
{
    if (!(sigma > 0.0) || !std::isfinite(sigma) || (int)std::ceil(3.0 * sigma) > kMaxBlurRadius) return -1;
    BlurTaps t;
    make_taps(sigma, t);
    for (int k = 0; k <= 2 * t.r && taps && k < cap; ++k) taps[k] = t.w[k];
    return t.r;
}

void *pf_host_alloc(size_t bytes)
{
    void *p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    return p;
}

void pf_host_free(void *p)
{
    if (p) cudaFreeHost(p);
}

int64_t pf_launch_count(const pf_ctx *ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
