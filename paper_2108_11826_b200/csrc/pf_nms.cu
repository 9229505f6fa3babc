// pf_nms.cu — peak extraction (paf.py:74-109 nms_peaks) on sm_100a.
//
// Two kernels, both writing unsorted peak records into per-(frame, part)
// slabs with a per-slab counter; k_parse_frames sorts them into the
// reference order (score desc, row, col) and assigns ids, so the atomic
// arrival order never shows in the results.
//
//  k_nms_plane — NMS over materialised maps (Mode R: the feature grid as-is;
//    also the upsampled/blurred maps when those are materialised).  One CTA
//    per plane streams the plane with 16-byte loads; only cells >= thr look
//    at their (2h+1)^2-1 neighbours, through L1.  HBM-read bound.
//
//  k_nms_up — fused x`up` bilinear upsample + NMS (Mode U).  The low-res
//    plane (or a row band of it) is staged in shared memory as fp64; the
//    output band is cut into 8x32 tiles and a tile is evaluated only if the
//    max of its low-res source rectangle reaches the fp32 threshold — exact,
//    because every upsampled value is a convex combination of its four
//    sources and rounds to <= their max.  A hot
//    tile's values plus an NMS halo are computed in fp64 (reference op
//    order) into a warp-private shared tile, then tested.  The upsampled
//    maps never touch HBM.
#include "pf_launch.h"

namespace pf {

#ifndef PF_NMS_STAGE
#define PF_NMS_STAGE 1
#endif

__device__ __forceinline__ bool plane_is_peak(const float *__restrict__ p, int H, int W,
                                              int i, int j, float v, int half)
{
    for (int di = -half; di <= half; ++di) {
        const int ni = i + di;
        if (ni < 0 || ni >= H) continue;
        for (int dj = -half; dj <= half; ++dj) {
            const int nj = j + dj;
            if ((di | dj) == 0 || nj < 0 || nj >= W) continue;
            if (!nms_beats(v, __ldg(p + (size_t)ni * W + nj), di, dj)) return false;
        }
    }
    return true;
}

__device__ __forceinline__ void emit_peak(int *counts, uint2 *peaks, int plane, int cap,
                                          float v, int i, int j)
{
    const int slot = atomicAdd(counts + plane, 1);
    if (slot < cap) peaks[(size_t)plane * cap + slot] = pack_peak(v, i, j);
}

// The same with the plane's counter in shared memory (one CTA per plane).
__device__ __forceinline__ void emit_peak_s(int *npk, uint2 *peaks, int plane, int cap, float v, int i, int j)
{
    const int slot = atomicAdd(npk, 1);
    if (slot < cap) peaks[(size_t)plane * cap + slot] = pack_peak(v, i, j);
}

// conf: [B][C][H][W]; planes are (b, k) for k < K; plane index = b*K + k.
// One CTA per plane: the peak count lives in shared memory (crowded planes
// emit tens of peaks; a global atomic each serialised them) and is stored
// once at the end.
__global__ void __launch_bounds__(256)
k_nms_plane(const float *__restrict__ conf, int C, int K, int H, int W, float thr, int half,
            int cap, int *__restrict__ counts, uint2 *__restrict__ peaks)
{
    __shared__ int s_npk;
    if (threadIdx.x == 0) s_npk = 0;
    __syncthreads();
    int *const npk = &s_npk;
    const int plane = blockIdx.x;
    const int b = plane / K, k = plane - b * K;
    const float *p = conf + ((size_t)b * C + k) * (size_t)H * W;
    const int HW = H * W;
    if ((HW & 3) == 0 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
        // HBM-read bound: kNmsUnroll 16-byte loads in flight per thread, the
        // (rare) cells >= thr then look at their neighbours through L1
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        const int n4 = HW >> 2;
        constexpr int kNmsUnroll = 4;
        const int lane = threadIdx.x & 31;
        // warp-uniform trip count (the row-neighbour shuffles need every lane)
        for (int bw = threadIdx.x - lane; bw < n4; bw += kNmsUnroll * blockDim.x) {
            const int b4 = bw + lane;
            float4 v4[kNmsUnroll];
#pragma unroll
            for (int u = 0; u < kNmsUnroll; ++u) {
                const int e4 = b4 + u * blockDim.x;
                v4[u] = e4 < n4 ? __ldg(p4 + e4) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
#pragma unroll
            for (int u = 0; u < kNmsUnroll; ++u) {
                const float vs[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
                const int e4 = b4 + u * blockDim.x;
                // 3x3 window: the row neighbours come from registers (the
                // adjacent lanes hold the adjacent float4s) and must not beat
                // the centre (paf.py:95-99: left strictly, right non-strictly)
                // before the other six neighbours are read
                const float lft = __shfl_up_sync(0xffffffffu, vs[3], 1);
                const float rgt = __shfl_down_sync(0xffffffffu, vs[0], 1);
                if (!(vs[0] >= thr || vs[1] >= thr || vs[2] >= thr || vs[3] >= thr)) continue;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!(vs[q] >= thr)) continue;
                    const int e = e4 * 4 + q, i = e / W, j = e - i * W;
                    if (half == 1) {
                        // flat neighbours e -/+ 1 are the row neighbours unless j is
                        // at a row end (then the reference pads -inf); lane 0's left
                        // and lane 31's right float4 are not in this warp: unknown
                        const bool have_l = j == 0 || q > 0 || lane > 0, have_r = j == W - 1 || q < 3 || lane < 31;
                        const float l = j == 0 ? -INFINITY : (q > 0 ? vs[q - 1] : lft);
                        const float r = j == W - 1 ? -INFINITY : (q < 3 ? vs[q + 1] : rgt);
                        if ((have_l && !(vs[q] > l)) || (have_r && !(vs[q] >= r))) continue;
                    }
                    if (plane_is_peak(p, H, W, i, j, vs[q], half)) emit_peak_s(npk, peaks, plane, cap, vs[q], i, j);
                }
            }
        }
    } else {
        for (int e = threadIdx.x; e < HW; e += blockDim.x) {
            const float v = __ldg(p + e);
            if (!(v >= thr)) continue;
            const int i = e / W, j = e - i * W;
            if (plane_is_peak(p, H, W, i, j, v, half)) emit_peak_s(npk, peaks, plane, cap, v, i, j);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) counts[plane] = s_npk;
}

// Small planes (Mode R feature grids, <= kNmsStageBytes): the plane is
// staged in shared memory with 16-byte loads, then every cell >= thr reads
// its neighbours from there — no L1 round trip per neighbour and no integer
// division per hot cell (crowded Mode R planes are mostly hot).  Same
// predicate (nms_beats, -inf outside the plane) as k_nms_plane.
constexpr int kNmsStageBytes = 24 * 1024;

__global__ void __launch_bounds__(256)
k_nms_plane_s(const float *__restrict__ conf, int C, int K, int H, int W, float thr, int half,
              int cap, int *__restrict__ counts, uint2 *__restrict__ peaks)
{
    extern __shared__ __align__(16) float sp[];
    __shared__ int s_npk;
    if (threadIdx.x == 0) s_npk = 0;
    const int plane = blockIdx.x;
    const int b = plane / K, k = plane - b * K;
    const float *p = conf + ((size_t)b * C + k) * (size_t)H * W;
    const int HW = H * W;
    if ((HW & 3) == 0 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        float4 *s4 = reinterpret_cast<float4 *>(sp);
        for (int e4 = threadIdx.x; e4 < (HW >> 2); e4 += blockDim.x) s4[e4] = __ldg(p4 + e4);
    } else {
        for (int e = threadIdx.x; e < HW; e += blockDim.x) sp[e] = __ldg(p + e);
    }
    __syncthreads();
    const float inv_w = 1.0f / (float)W;
    for (int e = threadIdx.x; e < HW; e += blockDim.x) {
        const float v = sp[e];
        if (!(v >= thr)) continue;
        const int i = (int)(((float)e + 0.5f) * inv_w), j = e - i * W;   // exact: HW < 2^16
        bool peak = true;
        if (half == 1) {
            // 3x3 unrolled (nms_beats: the row above and the left neighbour
            // strictly, the right neighbour and the row below non-strictly)
            const float *c = sp + e;
            const bool lf = j > 0, rt = j < W - 1;
            peak = (!lf || v > c[-1]) && (!rt || v >= c[1]);
            if (peak && i > 0) peak = (!lf || v > c[-W - 1]) && v > c[-W] && (!rt || v > c[-W + 1]);
            if (peak && i < H - 1) peak = (!lf || v >= c[W - 1]) && v >= c[W] && (!rt || v >= c[W + 1]);
            if (peak) emit_peak_s(&s_npk, peaks, plane, cap, v, i, j);
            continue;
        }
        for (int di = -half; di <= half && peak; ++di) {
            const int ni = i + di;
            if (ni < 0 || ni >= H) continue;
            for (int dj = -half; dj <= half; ++dj) {
                const int nj = j + dj;
                if ((di | dj) == 0 || nj < 0 || nj >= W) continue;
                if (!nms_beats(v, sp[ni * W + nj], di, dj)) { peak = false; break; }
            }
        }
        if (peak) emit_peak_s(&s_npk, peaks, plane, cap, v, i, j);
    }
    __syncthreads();
    if (threadIdx.x == 0) counts[plane] = s_npk;
}

constexpr int kTH = 8;    // tile rows
constexpr int kTW = 32;   // tile cols (one per lane)

// Shared memory: low-res band as fp64 [n_src][w] | per-warp value tiles
// [(kTH+2h)][(kTW+2h)] f32 | hot-tile list.
__global__ void __launch_bounds__(256)
k_nms_up(const UpArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int plane = blockIdx.x / a.n_bands;
    const int band = blockIdx.x - plane * a.n_bands;
    const int b = plane / a.K, k = plane - b * a.K;
    const float *src = a.conf + ((size_t)b * a.C + k) * (size_t)a.h * a.w;

    const int r0 = band * a.band_rows;
    const int r1 = min(a.H, r0 + a.band_rows);
    const int ev_lo = max(0, r0 - a.half), ev_hi = min(a.H, r1 + a.half);  // rows evaluated
    const int s_lo = __ldg(a.rows.i0 + ev_lo);
    const int s_hi = __ldg(a.rows.i1 + ev_hi - 1);
    const int n_src = s_hi - s_lo + 1;

    double *lo = reinterpret_cast<double *>(smem_raw);
    const int RW = kTW + 2 * a.half, RH = kTH + 2 * a.half;
    float *tiles = reinterpret_cast<float *>(lo + (size_t)n_src * a.w);
    const int n_warps = blockDim.x / kWarp;
    int *hot = reinterpret_cast<int *>(tiles + (size_t)n_warps * RH * RW);
    __shared__ int n_hot;

    // Stage the low-res rows (coalesced) as fp64.
    const float *srow = src + (size_t)s_lo * a.w;
    for (int e = threadIdx.x; e < n_src * a.w; e += blockDim.x) lo[e] = (double)__ldg(srow + e);
    if (threadIdx.x == 0) n_hot = 0;
    __syncthreads();

    // Phase 1: hot-tile detection.
    const int tiles_y = (r1 - r0 + kTH - 1) / kTH;
    const int tiles_x = (a.W + kTW - 1) / kTW;
    const double thr_d = (double)a.thr;
    for (int t = threadIdx.x; t < tiles_y * tiles_x; t += blockDim.x) {
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int y0 = r0 + ty * kTH, y1 = min(r1, y0 + kTH);
        const int x0 = tx * kTW, x1 = min(a.W, x0 + kTW);
        const int si0 = __ldg(a.rows.i0 + y0) - s_lo, si1 = __ldg(a.rows.i1 + y1 - 1) - s_lo;
        const int sj0 = __ldg(a.cols.i0 + x0), sj1 = __ldg(a.cols.i1 + x1 - 1);
        bool is_hot = false;
        for (int si = si0; si <= si1 && !is_hot; ++si)
            for (int sj = sj0; sj <= sj1; ++sj)
                if (lo[si * a.w + sj] >= thr_d) { is_hot = true; break; }
        if (is_hot) hot[atomicAdd(&n_hot, 1)] = t;
    }
    __syncthreads();

    // Phase 2: one warp per hot tile.
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    float *vt = tiles + (size_t)warp * RH * RW;
    for (int q = warp; q < n_hot; q += n_warps) {
        const int t = hot[q];
        const int ty = t / tiles_x, tx = t - ty * tiles_x;
        const int y0 = r0 + ty * kTH, y1 = min(r1, y0 + kTH);
        const int x0 = tx * kTW, x1 = min(a.W, x0 + kTW);
        const int ry0 = max(0, y0 - a.half), ry1 = min(a.H, y1 + a.half);
        const int rx0 = max(0, x0 - a.half), rx1 = min(a.W, x1 + a.half);
        for (int c = lane; c < rx1 - rx0; c += kWarp) {
            const int xo = rx0 + c;
            const int j0 = __ldg(a.cols.i0 + xo), j1 = __ldg(a.cols.i1 + xo);
            const double txv = __ldg(a.cols.t + xo), omtx = __ldg(a.cols.omt + xo);
            for (int r = 0; r < ry1 - ry0; ++r) {
                const int yo = ry0 + r;
                const int i0 = __ldg(a.rows.i0 + yo) - s_lo, i1 = __ldg(a.rows.i1 + yo) - s_lo;
                const double tyv = __ldg(a.rows.t + yo), omty = __ldg(a.rows.omt + yo);
                vt[r * RW + c] = bilerp(lo[i0 * a.w + j0], lo[i0 * a.w + j1],
                                        lo[i1 * a.w + j0], lo[i1 * a.w + j1],
                                        txv, omtx, tyv, omty);
            }
        }
        __syncwarp();
        const int xo = x0 + lane;
        if (xo < x1) {
            const int c = xo - rx0;
            for (int yo = y0; yo < y1; ++yo) {
                const int r = yo - ry0;
                const float v = vt[r * RW + c];
                if (!(v >= a.thr)) continue;
                bool peak = true;
                for (int di = -a.half; di <= a.half && peak; ++di) {
                    const int ny = yo + di;
                    if (ny < 0 || ny >= a.H) continue;
                    for (int dj = -a.half; dj <= a.half; ++dj) {
                        const int nx = xo + dj;
                        if ((di | dj) == 0 || nx < 0 || nx >= a.W) continue;
                        if (!nms_beats(v, vt[(ny - ry0) * RW + (nx - rx0)], di, dj)) { peak = false; break; }
                    }
                }
                if (peak) emit_peak(a.counts, a.peaks, plane, a.cap, v, yo, xo);
            }
        }
        __syncwarp();
    }
}

// Host-side launch helpers (called from pf_capi.cu).
cudaError_t launch_nms_plane(const float *conf, int B, int C, int K, int H, int W, float thr,
                             int half, int cap, int *counts, uint2 *peaks, cudaStream_t s)
{
    if (B * K == 0) return cudaSuccess;
#if PF_NMS_STAGE
    const size_t bytes = (size_t)H * W * sizeof(float);
    if (bytes <= (size_t)kNmsStageBytes) {
        k_nms_plane_s<<<B * K, 256, bytes, s>>>(conf, C, K, H, W, thr, half, cap, counts, peaks);
        return cudaGetLastError();
    }
#endif
    k_nms_plane<<<B * K, 256, 0, s>>>(conf, C, K, H, W, thr, half, cap, counts, peaks);
    return cudaGetLastError();
}

size_t nms_up_smem(int n_src_max, int w, int half, int band_rows, int W)
{
    const int RW = kTW + 2 * half, RH = kTH + 2 * half;
    const int tiles = ((band_rows + kTH - 1) / kTH) * ((W + kTW - 1) / kTW);
    return (size_t)n_src_max * w * sizeof(double) + (size_t)8 * RH * RW * sizeof(float) +
           (size_t)tiles * sizeof(int);
}

cudaError_t launch_nms_up(const UpArgs &a, int B, size_t smem, cudaStream_t s)
{
    const long long grid = (long long)B * a.K * a.n_bands;
    if (grid == 0) return cudaSuccess;
    k_nms_up<<<(unsigned)grid, 256, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_nms_up_win2<HALF> — register-window fused upsample + NMS (windows 3 and 5):
// the strip path for maps the corner kernels do not take (wider than 255
// cells per axis, non-canonical bands, window 5, or PF_OPT_WIN_VARIANT != 4).
//
// One CTA (4 warps) per (frame, part) plane.
//  phase 1: the low-res plane is streamed once (16-byte loads) and turned into
//           per-row "cell >= thr" bitmasks in shared memory (the compulsory
//           HBM read of the path; later reads hit L1).  The output-row
//           interpolation parameters (operators.py:87-96) go to a shared table.
//  phase 2: a warp owns a strip of 60 output columns, two per lane (lanes 0
//           and 31 carry the NMS halo).  From the bitmasks it derives the
//           strip's hot source rows and walks only the output rows whose
//           values can reach thr (+/- HALF halo rows), top to bottom, with an
//           inner row loop per source-row pair: each lane keeps the
//           horizontal interpolants of the pair's two source rows (the
//           reference's `top`/`bot`, operators.py:104-105 — they depend on the
//           source row only, so reuse is bit-exact) and per output row spends
//           one broadcast LDS.128 (the row weights), 4 DMUL + 2 DADD + 2 F2F
//           for its two outputs, 2*HALF shuffles and a few maxima.
//  NMS (paf.py:87-99) as two maxima: the centre must beat max(earlier
//           neighbours) strictly and max(later neighbours) non-strictly.  The
//           maxima propagate NaN (max.NaN.f32), so a NaN neighbour suppresses
//           the centre exactly as numpy's compares do; out-of-grid neighbours
//           are -inf, the reference's padding.  Row maxima are formed once per
//           row from warp shuffles and kept in a register window.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void axis_at(int o, double ratio, int n_in, int &i0, int &i1, double &t,
                                        double &omt)
{
    // operators.py:87-96, same fp64 op order as the host tables
    const double s = dadd(dmul(dadd((double)o, 0.5), ratio), -0.5);
    const double f = floor(s);
    const int fi = (int)f;
    t = __dsub_rn(s, f);
    omt = __dsub_rn(1.0, t);
    i0 = min(max(fi, 0), n_in - 1);
    i1 = min(max(fi + 1, 0), n_in - 1);
}

__device__ __forceinline__ float max_nan(float a, float b)
{
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// ---------------------------------------------------------------------------
template <int HALF>
__global__ void __launch_bounds__(128)
k_nms_up_win2(const UpWinArgs a)
{
    static_assert(HALF >= 1 && HALF <= 2, "halo lanes carry at most two columns");
    constexpr int SW = 2 * (kWarp - 2);      // useful columns per strip (lanes 1..30)
    constexpr int WIN = 2 * HALF + 1;
    extern __shared__ __align__(16) uint32_t sm[];
    const int plane = blockIdx.x;
    const int b = plane / a.K, k = plane - b * a.K;
    const float *p = a.conf + ((size_t)b * a.C + k) * (size_t)a.h * a.w;
    const int h = a.h, w = a.w, H = a.H;
    const int n_cw = (w + 31) >> 5;
    const int n_rw = (h + 31) >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_warps = blockDim.x >> 5;
    // shared: row weights [H] | row source pair [H] | last row of the pair [H] |
    //         hot bytes [h*w] | row masks [h][n_cw] | strip masks [warps][n_rw]
    double2 *rt_w = reinterpret_cast<double2 *>(sm);
    uint32_t *rt_idx = reinterpret_cast<uint32_t *>(rt_w + H);
    int *rt_gend = reinterpret_cast<int *>(rt_idx + H);
    uint8_t *hot = reinterpret_cast<uint8_t *>(rt_gend + H);
    uint32_t *rowmask = reinterpret_cast<uint32_t *>(hot + ((h * w + 15) & ~15));
    uint32_t *srcmask = rowmask + h * n_cw + warp * n_rw;

    // ---- phase 1: stream the plane -> hot bytes; row table ----
    const int hw = h * w;
    if ((hw & 3) == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        uchar4 *hot4 = reinterpret_cast<uchar4 *>(hot);
        for (int e = threadIdx.x; e < (hw >> 2); e += blockDim.x) {
            const float4 v = __ldg(p4 + e);
            hot4[e] = make_uchar4(v.x >= a.thr, v.y >= a.thr, v.z >= a.thr, v.w >= a.thr);
        }
    } else {
        for (int e = threadIdx.x; e < hw; e += blockDim.x) hot[e] = __ldg(p + e) >= a.thr;
    }
    for (int y = threadIdx.x; y < H; y += blockDim.x) {
        int i0, i1;
        double t, omt;
        axis_at(y, a.ry, h, i0, i1, t, omt);
        rt_w[y] = make_double2(t, omt);
        rt_idx[y] = uint32_t(i0) | (uint32_t(i1) << 16);
    }
    __syncthreads();
    for (int y = threadIdx.x; y < H; y += blockDim.x) {
        int e = y;                               // source pairs are monotone in y
        while (e + 1 < H && rt_idx[e + 1] == rt_idx[y]) ++e;
        rt_gend[y] = e;
    }
    for (int r = warp; r < h; r += n_warps) {
        for (int q = 0; q < n_cw; ++q) {
            const int col = (q << 5) + lane;
            const uint32_t m = __ballot_sync(0xffffffffu, col < w && hot[r * w + col]);
            if (lane == 0) rowmask[r * n_cw + q] = m;
        }
    }
    __syncthreads();

    // ---- phase 2: strips of SW columns, two per lane ----
    const int n_strips = (a.W + SW - 1) / SW;
    for (int s = warp; s < n_strips; s += n_warps) {
        const int x0 = s * SW;
        int xc[2], j0[2], j1[2];
        double tx[2], omtx[2];
        bool in_grid[2], useful[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            xc[c] = x0 + 2 * (lane - 1) + c;
            in_grid[c] = xc[c] >= 0 && xc[c] < a.W;
            useful[c] = lane >= 1 && lane <= kWarp - 2 && in_grid[c];
            axis_at(min(max(xc[c], 0), a.W - 1), a.rx, w, j0[c], j1[c], tx[c], omtx[c]);
        }
        // source-column span of the strip's useful columns
        const int last_x = min(x0 + SW, a.W) - 1;
        int cj0, cj1, dmy;
        double dt, domt;
        axis_at(x0, a.rx, w, cj0, dmy, dt, domt);
        axis_at(last_x, a.rx, w, dmy, cj1, dt, domt);
        for (int r0 = 0; r0 < h; r0 += 32) {
            const int r = r0 + lane;
            bool any = false;
            if (r < h) {
                for (int q = cj0 >> 5; q <= (cj1 >> 5) && !any; ++q) {
                    const uint32_t m = rowmask[r * n_cw + q];
                    const int lo = max(cj0 - (q << 5), 0), hi = min(cj1 - (q << 5), 31);
                    const uint32_t span = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
                    any = (m & span) != 0u;
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, any);
            if (lane == 0) srcmask[r0 >> 5] = bal;
        }
        __syncwarp();

        int run_lo = -1, run_hi = -2;
        for (int q = 0; q <= n_rw; ++q) {
            uint32_t m = q < n_rw ? srcmask[q] : 0u;
            bool flush_final = q == n_rw;
            while (m || flush_final) {
                int lo = 0, hi = -1;
                if (m) {
                    const int r = (q << 5) + __ffs(m) - 1;
                    m &= m - 1u;
                    lo = max(__ldg(a.first_out + r) - HALF, 0);
                    hi = min(__ldg(a.last_out + r) + HALF, H - 1);
                    if (run_hi >= run_lo && lo <= run_hi + 1) {
                        run_hi = max(run_hi, hi);
                        continue;
                    }
                } else {
                    flush_final = false;
                }
                if (run_hi >= run_lo) {
                    // window per column: 0 = oldest row, HALF = centre
                    float full[2][WIN], cv[2][WIN], lm[2][WIN], rm[2][WIN];
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int t = 0; t < WIN; ++t) full[c][t] = cv[c][t] = lm[c][t] = rm[c][t] = -INFINITY;
                    const int test_lo = run_lo == 0 ? 0 : run_lo + HALF;
                    const int test_hi = run_hi == H - 1 ? H - 1 : run_hi - HALF;
                    const int last_eval = run_hi == H - 1 ? run_hi + HALF : run_hi;
                    double hA[2] = {0.0, 0.0}, hB[2] = {0.0, 0.0};
                    int y = run_lo;
                    while (y <= last_eval) {
                        int yend;
                        if (y < H) {
                            // refresh the two source-row interpolants (uniform branch)
                            const uint32_t idx = rt_idx[y];
                            const int i0 = int(idx & 0xffffu), i1 = int(idx >> 16);
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                hA[c] = dadd(dmul((double)__ldg(p + i0 * w + j0[c]), omtx[c]),
                                             dmul((double)__ldg(p + i0 * w + j1[c]), tx[c]));
                                hB[c] = dadd(dmul((double)__ldg(p + i1 * w + j0[c]), omtx[c]),
                                             dmul((double)__ldg(p + i1 * w + j1[c]), tx[c]));
                            }
                            yend = min(rt_gend[y], last_eval);
                        } else {
                            yend = last_eval;       // virtual -inf rows below the grid
                        }
                        for (; y <= yend; ++y) {
                            float v[2];
                            if (y < H) {
                                const double2 wy = rt_w[y];
#pragma unroll
                                for (int c = 0; c < 2; ++c) {
                                    const float val = __double2float_rn(dadd(dmul(hA[c], wy.y), dmul(hB[c], wy.x)));
                                    v[c] = in_grid[c] ? val : -INFINITY;
                                }
                            } else {
                                v[0] = v[1] = -INFINITY;
                            }
                            // neighbour columns: x0c-1 = lane-1's col 1, x1c+1 = lane+1's col 0,
                            // x0c-2 = lane-1's col 0, x1c+2 = lane+1's col 1
                            const float l1 = __shfl_up_sync(0xffffffffu, v[1], 1);
                            const float r1 = __shfl_down_sync(0xffffffffu, v[0], 1);
                            float lmax0, rmax0, lmax1, rmax1;
                            if (HALF == 1) {
                                lmax0 = l1;    rmax0 = v[1];
                                lmax1 = v[0];  rmax1 = r1;
                            } else {
                                const float l2 = __shfl_up_sync(0xffffffffu, v[0], 1);
                                const float r2 = __shfl_down_sync(0xffffffffu, v[1], 1);
                                lmax0 = max_nan(l1, l2);       rmax0 = max_nan(v[1], r1);
                                lmax1 = max_nan(v[0], l1);     rmax1 = max_nan(r1, r2);
                            }
                            const float lmx[2] = {lmax0, lmax1}, rmx[2] = {rmax0, rmax1};
                            const int yc = y - HALF;
                            const bool row_ok = yc >= test_lo && yc <= test_hi;
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
#pragma unroll
                                for (int t = 0; t < WIN - 1; ++t) {
                                    full[c][t] = full[c][t + 1]; cv[c][t] = cv[c][t + 1];
                                    lm[c][t] = lm[c][t + 1]; rm[c][t] = rm[c][t + 1];
                                }
                                full[c][WIN - 1] = max_nan(max_nan(lmx[c], v[c]), rmx[c]);
                                cv[c][WIN - 1] = v[c]; lm[c][WIN - 1] = lmx[c]; rm[c][WIN - 1] = rmx[c];
                                float earlier = lm[c][HALF], later = rm[c][HALF];
#pragma unroll
                                for (int t = 0; t < HALF; ++t) {
                                    earlier = max_nan(earlier, full[c][t]);
                                    later = max_nan(later, full[c][HALF + 1 + t]);
                                }
                                const float cc = cv[c][HALF];
                                if (useful[c] && row_ok && cc >= a.thr && cc > earlier && cc >= later)
                                    emit_peak(a.counts, a.peaks, plane, a.cap, cc, yc, xc[c]);
                            }
                        }
                    }
                }
                if (hi >= lo) { run_lo = lo; run_hi = hi; }
                else { run_lo = -1; run_hi = -2; }
            }
        }
        __syncwarp();
    }
}


size_t nms_up_win_smem(int h, int w, int H, int threads)
{
    const int n_cw = (w + 31) >> 5, n_rw = (h + 31) >> 5;
    return (size_t)H * (16 + 4 + 4) + (size_t)((h * w + 15) & ~15) + (size_t)h * n_cw * 4 +
           (size_t)(threads / 32) * n_rw * 4 + 16;
}

cudaError_t launch_nms_up_win(const UpWinArgs &a, int B, cudaStream_t s)
{
    const long long grid = (long long)B * a.K;
    if (grid == 0) return cudaSuccess;
    const size_t smem = nms_up_win_smem(a.h, a.w, a.H, 128);
    if (a.half == 1) k_nms_up_win2<1><<<(unsigned)grid, 128, smem, s>>>(a);
    else if (a.half == 2) k_nms_up_win2<2><<<(unsigned)grid, 128, smem, s>>>(a);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

template <typename F>
static cudaError_t raise_smem_limit(F *fn, int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - (int)fa.sharedSizeBytes);
}

cudaError_t configure_nms_kernels(int max_smem)
{
    {
        cudaError_t e;
        if ((e = raise_smem_limit(k_nms_up_win2<1>, max_smem)) != cudaSuccess) return e;
        if ((e = raise_smem_limit(k_nms_up_win2<2>, max_smem)) != cudaSuccess) return e;
    }
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_nms_up);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_nms_up, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - (int)fa.sharedSizeBytes);
}

}  // namespace pf
