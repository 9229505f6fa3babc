// pf_blur.cu — k_up_blur_nms: fused x`up` bilinear upsample (operators.py:
// 79-107) -> separable Gaussian smoothing (HyperPose's heatmap blur; no
// reference) -> 3x3 NMS (paf.py:74-109) of the smoothed maps.
//
// Nothing full-resolution touches HBM: each CTA owns a column tile of one
// part plane and rolls down its output rows once, keeping a ring of the
// (2r+1) most recent horizontally smoothed rows and of the last smoothed
// rows in shared memory.  Per output row u:
//   U  the upsampled row: thread j owns output column j of the tile halo and
//      keeps top/bot (the column-interpolated source rows, operators.py:104-
//      105) in registers for the whole row band, so a row costs 3 fp64 ops;
//      U = fp32(top*(1-ty) + bot*ty) (operators.py:106-107 op order);
//   T  horizontal pass: T = sum_k w_k U[clamp(x+k)], fp32 fma chain in
//      ascending k from 0.0f, w_k = (float)taps[k];
//   B  vertical pass of row u - r from the ring, same chain, clamped rows;
//   N  the reference peak test of row u - r - 1 on B (earlier neighbours
//      strictly, later ones non-strictly, -inf outside the grid), peaks into
//      the plane's slab (global atomic per peak: several CTAs per plane).
// Kept for radii beyond k_up_blur_tile's (R > 8).  HBM traffic is the
// low-res part planes (read through L1/L2) and the peaks.
#include <algorithm>

#include "pf_launch.h"

namespace pf {

constexpr int kBlurThreads = 256;
#ifndef PF_BLUR_MINB
#define PF_BLUR_MINB 5
#endif

__global__ void __launch_bounds__(kBlurThreads, PF_BLUR_MINB)
k_up_blur_nms(const __grid_constant__ UpBlurArgs a)
{
    extern __shared__ __align__(16) unsigned char smb[];
    const int r = a.taps.r, R = 2 * r + 1;
    const int tw = a.tw;
    const int NB = tw + 2, NU = tw + 2 + 2 * r;
    float *Ud = reinterpret_cast<float *>(smb);                // [NU]
    float *Tr = Ud + NU;                                        // [R][NB]
    float *Br = Tr + (size_t)R * NB;                            // [4][NB]
    __shared__ float wt[2 * kMaxBlurRadius + 1];

    const int tile = blockIdx.x % a.tiles;
    const int plane = blockIdx.x / a.tiles;
    const int fb = plane / a.K, k = plane - fb * a.K;
    const float *S = a.conf + ((size_t)fb * a.C + k) * (size_t)a.h * a.w;
    const int H = a.H, W = a.W, w = a.w;
    const int x0 = tile * tw;
    const int j = threadIdx.x;
    for (int t = j; t < R; t += kBlurThreads) wt[t] = (float)a.taps.w[t];

    // this thread's U column (clamped): its axis record, kept for all rows
    int cj0 = 0, cj1 = 0;
    double tx = 0.0, omtx = 0.0;
    if (j < NU) {
        const int xu = min(max(x0 - 1 - r + j, 0), W - 1);
        const int4 v = __ldg(reinterpret_cast<const int4 *>(a.crec + xu));
        cj0 = v.x & 0xffff;
        cj1 = v.x >> 16;
        tx = __hiloint2double(v.w, v.z);
        omtx = __dsub_rn(1.0, tx);
    }
    // this thread's T / B column
    const int xb = x0 - 1 + j;
    const bool b_in = j < NB && xb >= 0 && xb < W;
    const bool n_in = j >= 1 && j <= tw && xb < W;            // NMS columns: the tile itself
    __syncthreads();

    double top = 0.0, bot = 0.0;
    int band0 = -1, band1 = -1;
    for (int u = 0; u <= H + r; ++u) {
        if (u < H) {
            const int4 ry = __ldg(reinterpret_cast<const int4 *>(a.rrec + u));
            const int i0 = ry.x & 0xffff, i1 = ry.x >> 16;
            const double ty = __hiloint2double(ry.w, ry.z);
            if (j < NU) {
                if (i0 != band0 || i1 != band1) {               // new source row pair: top / bot
                    const float *s0 = S + (size_t)i0 * w, *s1 = S + (size_t)i1 * w;
                    top = dadd(dmul((double)__ldg(s0 + cj0), omtx), dmul((double)__ldg(s0 + cj1), tx));
                    bot = dadd(dmul((double)__ldg(s1 + cj0), omtx), dmul((double)__ldg(s1 + cj1), tx));
                }
                Ud[j] = __double2float_rn(dadd(dmul(top, __dsub_rn(1.0, ty)), dmul(bot, ty)));
            }
            band0 = i0;
            band1 = i1;
            __syncthreads();
            if (b_in) {                                          // T row u (horizontal pass)
                float acc = 0.0f;
                for (int t = 0; t < R; ++t) acc = __fmaf_rn(wt[t], Ud[j + t], acc);
                Tr[(size_t)(u % R) * NB + j] = acc;
            }
            __syncthreads();
        }
        const int y = u - r;                                     // B row y (vertical pass)
        if (y >= 0 && y < H) {
            if (j < NB) {
                float bv = -INFINITY;
                if (b_in) {
                    // rows y-r .. y+r clamped to the grid; the ring slot
                    // advances with the row (clamped rows repeat a slot)
                    int row = max(y - r, 0), sl = row % R;
                    float acc = 0.0f;
                    for (int t = 0; t < R; ++t) {
                        acc = __fmaf_rn(wt[t], Tr[(size_t)sl * NB + j], acc);
                        const int nrow = min(max(y - r + t + 1, 0), H - 1);
                        if (nrow != row) {
                            row = nrow;
                            sl = sl + 1 == R ? 0 : sl + 1;
                        }
                    }
                    bv = acc;
                }
                Br[(y & 3) * NB + j] = bv;
            }
            __syncthreads();
        }
        const int yn = y - 1;                                    // NMS of row yn
        if (yn >= 0 && yn < H && n_in) {
            const float *cur = Br + (yn & 3) * NB;
            const float v = cur[j];
            if (v >= a.thr) {
                bool ok = v > cur[j - 1] && v >= cur[j + 1];
                if (ok && yn > 0) {
                    const float *up = Br + ((yn - 1) & 3) * NB;
                    ok = v > up[j - 1] && v > up[j] && v > up[j + 1];
                }
                if (ok && yn + 1 < H) {
                    const float *dn = Br + ((yn + 1) & 3) * NB;
                    ok = v >= dn[j - 1] && v >= dn[j] && v >= dn[j + 1];
                }
                if (ok) {
                    const int slot = atomicAdd(a.counts + plane, 1);
                    if (slot < a.cap) a.peaks[(size_t)plane * a.cap + slot] = pack_peak(v, yn, xb);
                }
            }
        }
    }
}


// ---------------------------------------------------------------------------
// k_up_blur_tile<R> — the same computation on 2-D tiles (radius R <= 8): a
// CTA owns a th x tw block of one part plane's output and computes, each
// stage over the whole block, every thread on four independent outputs at
// once (interleaved fma chains, taps unrolled, no per-row barriers):
//   H  per (source row, U column): top/bot halves of operators.py:104-105,
//      fl(S[i][j0]*(1-tx) + S[i][j1]*tx) — shared by every output row whose
//      i0 or i1 is that source row (bit-identical to recomputing it);
//   U  the upsampled value fp32(H[i0]*(1-ty) + H[i1]*ty) (operators.py:106-107)
//      on the block plus the blur and NMS halo (R + 1), clamped coordinates;
//   T  horizontal pass, fp32 fma chain in ascending k from 0.0f (a thread:
//      4 adjacent columns from one 4 + 2R window of U);
//   B  vertical pass over T, same chain (4 adjacent rows per thread);
//   N  the reference 3x3 peak test (paf.py:95-99) on B, -inf off the grid.
// Block rows / columns of B are padded to multiples of 4 (the pad computes
// clamped duplicates that nothing reads).
constexpr int kTileThreads = 256;
constexpr int kTileMaxR = 8;
constexpr int kTileTarget = 64;      // output rows / columns per block (before balancing)
constexpr int kVec = 4;              // outputs per thread per pass

struct TileDims {
    int th, tw, tiles_y, tiles_x;
};

static TileDims tile_dims(int H, int W)
{
    TileDims d;
    d.tiles_y = (H + kTileTarget - 1) / kTileTarget;
    d.tiles_x = (W + kTileTarget - 1) / kTileTarget;
    d.th = (H + d.tiles_y - 1) / d.tiles_y;
    d.tw = (W + d.tiles_x - 1) / d.tiles_x;
    return d;
}

struct TileLayout {
    int NRB, NCB, NR, NCU, NS;
    size_t wt, colj, colt, rowi, rowt, hrow, u, t, total;
};

__host__ __device__ inline TileLayout tile_layout(int th, int tw, int r, int up)
{
    TileLayout L;
    L.NRB = (th + 2 + kVec - 1) / kVec * kVec;   // B rows: block +- 1, padded
    L.NCB = (tw + kVec - 1) / kVec * kVec + kVec; // T / B columns: block +- 1, padded (N reads 4g .. 4g+5)
    L.NR = L.NRB + 2 * r;                        // U / T rows
    L.NCU = (L.NCB + 2 * r + kVec - 1) / kVec * kVec;   // U columns, padded
    L.NS = (L.NR + up - 1) / up + 3;             // source rows the U rows can read
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o = (o + bytes + 15) & ~(size_t)15; return at; };
    L.wt = take((size_t)(2 * kTileMaxR + 1) * sizeof(float));
    L.colj = take((size_t)L.NCU * sizeof(int2));
    L.colt = take((size_t)L.NCU * sizeof(double2));   // (tx, 1 - tx)
    L.rowi = take((size_t)L.NR * sizeof(int2));
    L.rowt = take((size_t)L.NR * sizeof(double2));    // (ty, 1 - ty)
    L.hrow = take((size_t)L.NS * L.NCU * sizeof(double));
    L.u = take((size_t)L.NR * L.NCU * sizeof(float));   // later B (NRB x NCB)
    L.t = take((size_t)L.NR * L.NCB * sizeof(float));
    L.total = o;
    return L;
}

// Row-major walk of an n_rows x n_cols block by a CTA, element tid, tid +
// kTileThreads, ...: one division per thread, then carries.
struct Walk2D {
    int q, c, dq, dc, n_cols;
    __device__ Walk2D(int n_cols_, int tid) : n_cols(n_cols_)
    {
        q = tid / n_cols;
        c = tid - q * n_cols;
        dq = kTileThreads / n_cols;
        dc = kTileThreads - dq * n_cols;
    }
    __device__ void next()
    {
        q += dq;
        c += dc;
        if (c >= n_cols) { c -= n_cols; ++q; }
    }
};

template <int R>
__global__ void __launch_bounds__(kTileThreads, 4)
k_up_blur_tile(const __grid_constant__ UpBlurArgs a)
{
    constexpr int NT = 2 * R + 1;
    extern __shared__ __align__(16) unsigned char smt[];
    const int th = a.th, tw = a.tw;
    const int H = a.H, W = a.W, w = a.w, h = a.h;
    const TileLayout L = tile_layout(th, tw, R, a.up);
    float *wt = reinterpret_cast<float *>(smt + L.wt);
    int2 *colj = reinterpret_cast<int2 *>(smt + L.colj);
    double2 *colt = reinterpret_cast<double2 *>(smt + L.colt);
    int2 *rowi = reinterpret_cast<int2 *>(smt + L.rowi);
    double2 *rowt = reinterpret_cast<double2 *>(smt + L.rowt);
    double *Hr = reinterpret_cast<double *>(smt + L.hrow);
    float *U = reinterpret_cast<float *>(smt + L.u);
    float *T = reinterpret_cast<float *>(smt + L.t);
    float *Bv = reinterpret_cast<float *>(smt + L.u);           // aliases U once T is done

    const int NR = L.NR, NCU = L.NCU, NCB = L.NCB, NRB = L.NRB;
    const int tid = threadIdx.x;
    for (int t = tid; t < NT; t += kTileThreads) wt[t] = (float)a.taps.w[t];
    // per-thread walks of the stages (the divisions once per CTA)
    const int gx = NCB / kVec, gy = NRB / kVec, gn = (tw + kVec - 1) / kVec;
    const Walk2D wH(NCU, tid), wU(NCU / kVec, tid), wT(gx, tid), wB(NCB, tid), wN(gn, tid);
    const int per_plane = a.tiles_y * a.tiles_x;
    const int n_blocks = a.B * a.K * per_plane;
    __syncthreads();
    float wr[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) wr[t] = wt[t];

    // persistent: blocks round-robin over the resident CTAs
    for (int blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const int plane = blk / per_plane, tile = blk - plane * per_plane;
    const int ty_ = tile / a.tiles_x;
    const int y0 = ty_ * th, x0 = (tile - ty_ * a.tiles_x) * tw;
    const int fb = plane / a.K, k = plane - fb * a.K;
    const float *S = a.conf + ((size_t)fb * a.C + k) * (size_t)h * w;

    // Cold block: every source the block's U region reads lies in [0, X)
    // with X = thr (1 - 2^-10).  U (a convex combination, rounded) stays in
    // [0, X); each fp32 fma pass of positive taps (sum <= 1 + 17 * 2^-24)
    // grows the bound by < 2^-17, so every B < thr: no peak in the block
    // (paf.py:89 needs v >= thr).  NaN, negative or hot sources: computed.
    {
        const int yl = min(max(y0 - 1 - R + NR - 1, 0), H - 1);
        const int xf = min(max(x0 - 1 - R, 0), W - 1), xl = min(max(x0 - 1 - R + NCU - 1, 0), W - 1);
        const int r0 = __ldg(&a.rrec[min(max(y0 - 1 - R, 0), H - 1)].i01) & 0xffff;
        const int r1 = __ldg(&a.rrec[yl].i01) >> 16;
        const int c0 = __ldg(&a.crec[xf].i01) & 0xffff, c1 = __ldg(&a.crec[xl].i01) >> 16;
        const int nc = c1 - c0 + 1, n = (r1 - r0 + 1) * nc;
        const float X = a.thr > 0.f ? a.thr - a.thr * 0.0009765625f : -INFINITY;
        bool hot = false;
        for (int e = tid; e < n; e += kTileThreads) {
            const int rr = e / nc;
            const float v = __ldg(S + (size_t)(r0 + rr) * w + c0 + (e - rr * nc));
            hot |= !(v >= 0.f && v < X);
        }
        if (!__syncthreads_or(hot)) continue;
    }
    // records of the previous block were last read before its U stage ended
    for (int c = tid; c < NCU; c += kTileThreads) {             // U column records (clamped)
        const int xx = min(max(x0 - 1 - R + c, 0), W - 1);
        const int4 v = __ldg(reinterpret_cast<const int4 *>(a.crec + xx));
        const double tx = __hiloint2double(v.w, v.z);
        colj[c] = make_int2(v.x & 0xffff, v.x >> 16);
        colt[c] = make_double2(tx, __dsub_rn(1.0, tx));
    }
    // source row window: i0 of the first row .. i1 of the last (rows are monotone)
    const int yfirst = min(max(y0 - 1 - R, 0), H - 1);
    const int s0 = __ldg(&a.rrec[yfirst].i01) & 0xffff;
    for (int q = tid; q < NR; q += kTileThreads) {
        const int yy = min(max(y0 - 1 - R + q, 0), H - 1);
        const int4 v = __ldg(reinterpret_cast<const int4 *>(a.rrec + yy));
        const double ty = __hiloint2double(v.w, v.z);
        rowi[q] = make_int2(((v.x & 0xffff) - s0) * NCU, ((v.x >> 16) - s0) * NCU);
        rowt[q] = make_double2(ty, __dsub_rn(1.0, ty));
    }
    __syncthreads();
    // H: the column-interpolated source rows (operators.py:104-105 halves)
    const int ns = min(L.NS, h - s0);
    for (Walk2D it = wH; it.q < ns; it.next()) {
        const int sr = it.q, c = it.c, e = sr * NCU + c;
        const float *row = S + (size_t)(s0 + sr) * w;
        const int2 j = colj[c];
        const double2 t = colt[c];
        Hr[e] = dadd(dmul((double)__ldg(row + j.x), t.y), dmul((double)__ldg(row + j.y), t.x));
    }
    __syncthreads();
    // U, 4 adjacent columns per thread (the previous block's N stage is over)
    for (Walk2D it = wU; it.q < NR; it.next()) {
        const int q = it.q, c = it.c * kVec;
        const int2 i = rowi[q];
        const double2 t = rowt[q];
        // 16-byte shared loads: a lane's four columns are contiguous
        const double2 a0 = *reinterpret_cast<const double2 *>(Hr + i.x + c);
        const double2 a1 = *reinterpret_cast<const double2 *>(Hr + i.x + c + 2);
        const double2 b0 = *reinterpret_cast<const double2 *>(Hr + i.y + c);
        const double2 b1 = *reinterpret_cast<const double2 *>(Hr + i.y + c + 2);
        const double hi[kVec] = {a0.x, a0.y, a1.x, a1.y}, lo[kVec] = {b0.x, b0.y, b1.x, b1.y};
        float o[kVec];
#pragma unroll
        for (int v = 0; v < kVec; ++v) o[v] = __double2float_rn(dadd(dmul(hi[v], t.y), dmul(lo[v], t.x)));
        *reinterpret_cast<float4 *>(U + q * NCU + c) = make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    // T: horizontal pass, 4 adjacent columns per thread (U column of output
    // column cb, tap t: cb + t)
    for (Walk2D it = wT; it.q < NR; it.next()) {
        const int q = it.q, cb = it.c * kVec;
        const float *u = U + q * NCU + cb;
        constexpr int NW = (kVec + 2 * R + 3) / 4 * 4;
        float win[NW];
#pragma unroll
        for (int m = 0; m < NW; m += 4) {      // 16-byte shared loads (U rows are padded to NW)
            const float4 f = *reinterpret_cast<const float4 *>(u + m);
            win[m] = f.x; win[m + 1] = f.y; win[m + 2] = f.z; win[m + 3] = f.w;
        }
        float acc[kVec];
#pragma unroll
        for (int v = 0; v < kVec; ++v) acc[v] = 0.0f;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int v = 0; v < kVec; ++v) acc[v] = __fmaf_rn(wr[t], win[v + t], acc[v]);
        *reinterpret_cast<float4 *>(T + q * NCB + cb) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
    __syncthreads();
    // B: vertical pass for block rows -1 .. th (+ pad), 4 adjacent rows per
    // thread (T row of output row q', tap t: q' + t)
    for (Walk2D it = wB; it.q < gy; it.next()) {
        const int cb = it.c, q = it.q * kVec;
        const float *tc = T + q * NCB + cb;
        float win[kVec + 2 * R];
#pragma unroll
        for (int m = 0; m < kVec + 2 * R; ++m) win[m] = tc[m * NCB];
        float acc[kVec];
#pragma unroll
        for (int v = 0; v < kVec; ++v) acc[v] = 0.0f;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int v = 0; v < kVec; ++v) acc[v] = __fmaf_rn(wr[t], win[v + t], acc[v]);
        const int xb = x0 - 1 + cb;
        const bool xin = xb >= 0 && xb < W;
#pragma unroll
        for (int v = 0; v < kVec; ++v) {
            const int yb = y0 - 1 + q + v;
            Bv[(q + v) * NCB + cb] = (xin && yb >= 0 && yb < H) ? acc[v] : -INFINITY;
        }
    }
    __syncthreads();
    // N: the block's own pixels, 4 adjacent columns per thread (B columns
    // 4g .. 4g+5 of three rows: a float4 and a float2 each); the centre row
    // first — a group with no centre >= thr is done
    for (Walk2D it = wN; it.q < th; it.next()) {
        const int qy = it.q, qx = it.c * kVec;
        const int y = y0 + qy;
        const float *rb = Bv + qy * NCB + qx;
        float m[3][kVec + 2];
        auto load_row = [&](int rr) {
            const float4 lo = *reinterpret_cast<const float4 *>(rb + rr * NCB);
            const float2 hi = *reinterpret_cast<const float2 *>(rb + rr * NCB + kVec);
            m[rr][0] = lo.x; m[rr][1] = lo.y; m[rr][2] = lo.z; m[rr][3] = lo.w; m[rr][4] = hi.x; m[rr][5] = hi.y;
        };
        load_row(1);
        if (!(m[1][1] >= a.thr || m[1][2] >= a.thr || m[1][3] >= a.thr || m[1][4] >= a.thr) || y >= H) continue;
        load_row(0);
        load_row(2);
#pragma unroll
        for (int v = 0; v < kVec; ++v) {
            const float c = m[1][v + 1];
            const int x = x0 + qx + v;
            if (!(c >= a.thr) || qx + v >= tw || x >= W) continue;
            if (c > m[0][v] && c > m[0][v + 1] && c > m[0][v + 2] && c > m[1][v] && c >= m[1][v + 2] &&
                c >= m[2][v] && c >= m[2][v + 1] && c >= m[2][v + 2]) {
                const int slot = atomicAdd(a.counts + plane, 1);
                if (slot < a.cap) a.peaks[(size_t)plane * a.cap + slot] = pack_peak(c, y, x);
            }
        }
    }
    }
}

static size_t up_blur_tile_smem(int H, int W, int r, int up)
{
    const TileDims d = tile_dims(H, W);
    return tile_layout(d.th, d.tw, r, up).total;
}

size_t up_blur_smem(int tw, int r)
{
    const int NB = tw + 2, NU = tw + 2 + 2 * r;
    return (size_t)NU * sizeof(float) + (size_t)(2 * r + 1) * NB * sizeof(float) + (size_t)4 * NB * sizeof(float);
}

int up_blur_tile_width(int W, int r)
{
    const int max_tw = kBlurThreads - 2 - 2 * r;
    if (max_tw < 1) return 0;
    const int tiles = (W + max_tw - 1) / max_tw;
    return (W + tiles - 1) / tiles;
}

cudaError_t launch_up_blur_nms(const UpBlurArgs &a_in, cudaStream_t s)
{
    UpBlurArgs a = a_in;
    const long long P = (long long)a.B * a.K;
    if (P == 0) return cudaSuccess;
    int dev = 0, max_smem = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    if (a.taps.r <= kTileMaxR && up_blur_tile_smem(a.H, a.W, a.taps.r, a.up) <= (size_t)max_smem) {
        const TileDims d = tile_dims(a.H, a.W);
        a.th = d.th; a.tw = d.tw; a.tiles_y = d.tiles_y; a.tiles_x = d.tiles_x;
        const size_t smem = tile_layout(d.th, d.tw, a.taps.r, a.up).total;
        // persistent: the resident CTAs take the blocks round-robin
        int sms = 0, occ = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_up_blur_tile<3>, kTileThreads, smem);
        if (e != cudaSuccess) return e;
        const unsigned grid = (unsigned)std::min<long long>(P * d.tiles_y * d.tiles_x, (long long)std::max(occ, 1) * sms);
        switch (a.taps.r) {
        case 1: k_up_blur_tile<1><<<grid, kTileThreads, smem, s>>>(a); break;
        case 2: k_up_blur_tile<2><<<grid, kTileThreads, smem, s>>>(a); break;
        case 3: k_up_blur_tile<3><<<grid, kTileThreads, smem, s>>>(a); break;
        case 4: k_up_blur_tile<4><<<grid, kTileThreads, smem, s>>>(a); break;
        case 5: k_up_blur_tile<5><<<grid, kTileThreads, smem, s>>>(a); break;
        case 6: k_up_blur_tile<6><<<grid, kTileThreads, smem, s>>>(a); break;
        case 7: k_up_blur_tile<7><<<grid, kTileThreads, smem, s>>>(a); break;
        default: k_up_blur_tile<8><<<grid, kTileThreads, smem, s>>>(a); break;
        }
        return cudaGetLastError();
    }
    a.tw = up_blur_tile_width(a.W, a.taps.r);
    if (a.tw < 1) return cudaErrorInvalidValue;
    a.tiles = (a.W + a.tw - 1) / a.tw;
    const size_t smem = up_blur_smem(a.tw, a.taps.r);
    k_up_blur_nms<<<(unsigned)(P * a.tiles), kBlurThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int R>
static cudaError_t configure_tile(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_up_blur_tile<R>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_up_blur_tile<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    return e;
}

cudaError_t configure_blur_kernels(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_up_blur_nms);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_up_blur_nms, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = configure_tile<1>(max_smem);
    if (e == cudaSuccess) e = configure_tile<2>(max_smem);
    if (e == cudaSuccess) e = configure_tile<3>(max_smem);
    if (e == cudaSuccess) e = configure_tile<4>(max_smem);
    if (e == cudaSuccess) e = configure_tile<5>(max_smem);
    if (e == cudaSuccess) e = configure_tile<6>(max_smem);
    if (e == cudaSuccess) e = configure_tile<7>(max_smem);
    if (e == cudaSuccess) e = configure_tile<8>(max_smem);
    return e;
}

}  // namespace pf
