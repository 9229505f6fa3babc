// pf_corner.cu — k_nms_up_corner: fused x`up` bilinear upsample + 3x3 NMS
// (paf.py:74-109 on operators.py:79-107 maps) that evaluates only the
// output pixels that can possibly be peaks.  Exact, by the argument below.
//
// Cells.  Output rows sharing the same source pair (i0, i1) form a row band;
// output columns likewise.  A cell = (row band p, column band q).  Inside a
// cell every output is v = RN32(F), F = the reference's fp64 expression
// (operators.py:104-107) of the same four sources, and the exact value
// G = P*(1-tx) + Q*tx (P, Q the row-weighted source columns) is affine in tx
// along a row and affine in ty along a column.  With M = max |source|,
// |v - G| <= 2^-24 M + ~5*2^-53 M < 2^-23 M, so two outputs whose exact
// values differ by more than 2^-22 M compare the same way after rounding.
//
// Interior exclusion.  Along a row of cell (p, q) the exact step between
// adjacent outputs is D_h * dtx (+ <= 2^-52 M), D_h = (A1-A0)(1-ty) + (B1-B0) ty.
// If |D_h| * dtx_min > 2^-22 M the row is strictly monotone, so no output
// with both horizontal neighbours in the cell can be "> left and >= right"
// (paf.py:95-99): a peak needs its column at the band's first or last column
// ("h_ok").  D_h is affine in ty, so the band's first and last rows (same
// sign) bound every row; vertically the same with D_v ("v_ok": a peak needs a
// boundary row).  Slopes are evaluated in fp32 (error <= 2^-21 M) against
// n = 2^-17 M, which leaves the needed 2^-22 M with margin.
//   h_ok && v_ok        -> "normal": only the 4 corner pixels can be peaks;
//   otherwise           -> "partial": the pixels on boundary columns (if h_ok)
//                          x boundary rows (if v_ok), all rows/columns else.
// Border bands count as flat in their border direction (the clamped bands
// have D = 0 there anyway), so grid-edge pixels are always examined.  Cold
// cells (all four sources < thr) cannot reach thr (convex combination,
// monotone rounding) and are never touched.
//
// Corner pruning.  A normal cell's corner can only hold a peak if the cell's
// own slopes rise toward it (at most one corner per cell passes).  For that
// corner the exact values around the shared source point are piecewise
// affine; the step across the cell boundary is m_q (1-tx(x1)) + m_{q+1} tx(x2)
// (x1 = last column of band q, x2 = first of q+1), which decides ">= right"
// ("> left" for x2) whenever it clears n, and likewise vertically.  Every
// surviving pixel (a few per plane) gets the exact 3x3 test on exactly
// computed values.
#include "pf_launch.h"

namespace pf {

constexpr float kNoise = 7.62939453125e-06f;   // 2^-17

__device__ __forceinline__ void emit_peak_c(int *counts, uint2 *peaks, int plane, int cap, float v, int i, int j)
{
    const int slot = atomicAdd(counts + plane, 1);
    if (slot < cap) peaks[(size_t)plane * cap + slot] = pack_peak(v, i, j);
}

// Row or column interpolation parameters of one output coordinate.
struct Ax {
    int i0, i1;
    double t, omt;
    bool in;
};

__device__ __forceinline__ Ax ax_load(const AxisTab &tab, int o, int n_out)
{
    Ax r;
    r.in = o >= 0 && o < n_out;
    const int oc = min(max(o, 0), n_out - 1);
    r.i0 = __ldg(tab.i0 + oc);
    r.i1 = __ldg(tab.i1 + oc);
    r.t = __ldg(tab.t + oc);
    r.omt = __ldg(tab.omt + oc);
    return r;
}

// Exact upsampled value (operators.py:104-107 op order); -inf off-grid.
__device__ __forceinline__ float up_val(const float *S, int w, const Ax &ry, const Ax &cx)
{
    if (!(ry.in && cx.in)) return -INFINITY;
    return bilerp(S[ry.i0 * w + cx.i0], S[ry.i0 * w + cx.i1], S[ry.i1 * w + cx.i0], S[ry.i1 * w + cx.i1],
                  cx.t, cx.omt, ry.t, ry.omt);
}

// The reference predicate (paf.py:87-99) on exactly computed values; each row
// and column parameter is loaded once.
__device__ __noinline__ bool exact_peak(const UpCornerArgs &a, const float *S, int y, int x, float &v)
{
    const Ax ym = ax_load(a.rows, y - 1, a.H), yc = ax_load(a.rows, y, a.H), yp = ax_load(a.rows, y + 1, a.H);
    const Ax xm = ax_load(a.cols, x - 1, a.W), xc = ax_load(a.cols, x, a.W), xp = ax_load(a.cols, x + 1, a.W);
    v = up_val(S, a.w, yc, xc);
    if (!(v >= a.thr)) return false;
    // earlier neighbours: strictly greater; later: greater or equal
    if (!(v > up_val(S, a.w, ym, xm))) return false;
    if (!(v > up_val(S, a.w, ym, xc))) return false;
    if (!(v > up_val(S, a.w, ym, xp))) return false;
    if (!(v > up_val(S, a.w, yc, xm))) return false;
    if (!(v >= up_val(S, a.w, yc, xp))) return false;
    if (!(v >= up_val(S, a.w, yp, xm))) return false;
    if (!(v >= up_val(S, a.w, yp, xc))) return false;
    return v >= up_val(S, a.w, yp, xp);
}

struct CellF {
    float a0, a1, b0, b1;    // S[r0][c0], S[r0][c1], S[r1][c0], S[r1][c1]
};

__device__ __forceinline__ CellF cellf(const float *S, int w, int4 rb, int4 cb)
{
    return CellF{S[rb.z * w + cb.z], S[rb.z * w + cb.w], S[rb.w * w + cb.z], S[rb.w * w + cb.w]};
}
__device__ __forceinline__ float mag(const CellF &c)
{
    return fmaxf(fmaxf(fabsf(c.a0), fabsf(c.a1)), fmaxf(fabsf(c.b0), fabsf(c.b1)));
}
// slopes per unit t along a row (row weights) and along a column (column weights)
__device__ __forceinline__ float sl_h(const CellF &c, float omty, float ty)
{
    return (c.a1 - c.a0) * omty + (c.b1 - c.b0) * ty;
}
__device__ __forceinline__ float sl_v(const CellF &c, float omtx, float tx)
{
    return (c.b0 - c.a0) * omtx + (c.b1 - c.a1) * tx;
}

// Cross-boundary part of the corner test for the corner pixel (row role i,
// column role j) of corner (P, Q): the pixel is (i ? first(P+1) : last(P),
// j ? first(Q+1) : last(Q)) in cell (P+i, Q+j).  The own-cell in-band
// neighbours were checked by the caller.
__device__ __forceinline__ bool corner_cross_ok(const UpCornerArgs &a, const float *S, int P, int Q, int i, int j)
{
    const int4 R0 = __ldg(a.rband + P), R1 = __ldg(a.rband + P + 1);
    const int4 C0 = __ldg(a.cband + Q), C1 = __ldg(a.cband + Q + 1);
    const CellF c00 = cellf(S, a.w, R0, C0), c01 = cellf(S, a.w, R0, C1);
    const CellF c10 = cellf(S, a.w, R1, C0), c11 = cellf(S, a.w, R1, C1);
    const float n = fmaxf(fmaxf(mag(c00), mag(c01)), fmaxf(mag(c10), mag(c11))) * kNoise;
    const int y1 = R0.y, y2 = R1.x, x1 = C0.y, x2 = C1.x;
    const int yy = i ? y2 : y1, xx = j ? x2 : x1;
    if (C0.w == C1.z) {              // bands share the source column: piecewise affine across it
        const float omty = (float)__ldg(a.rows.omt + yy), ty = (float)__ldg(a.rows.t + yy);
        const float mq = sl_h(i ? c10 : c00, omty, ty), mq1 = sl_h(i ? c11 : c01, omty, ty);
        const float cross = mq * (float)__ldg(a.cols.omt + x1) + mq1 * (float)__ldg(a.cols.t + x2);
        if (j == 0 ? cross > n : cross < -n) return false;     // ~ G(x2) - G(x1)
    }
    if (R0.w == R1.z) {
        const float omtx = (float)__ldg(a.cols.omt + xx), tx = (float)__ldg(a.cols.t + xx);
        const float mp = sl_v(j ? c01 : c00, omtx, tx), mp1 = sl_v(j ? c11 : c10, omtx, tx);
        const float cross = mp * (float)__ldg(a.rows.omt + y1) + mp1 * (float)__ldg(a.rows.t + y2);
        if (i == 0 ? cross > n : cross < -n) return false;     // ~ G(y2) - G(y1)
    }
    return true;
}

// Classify a hot cell.  Returns bit 0 = h_ok, bit 1 = v_ok (3 = normal) and,
// for the own-cell corner tests, a bitmask of corners (bit 2*i + j) whose
// in-band neighbours do not strictly beat them.
__device__ __forceinline__ unsigned classify_cell(const UpCornerArgs &a, const float *S, int p, int q, int4 rb,
                                                  int4 cb, unsigned &corners)
{
    corners = 0u;
    const CellF c = cellf(S, a.w, rb, cb);
    const float n = mag(c) * kNoise;
    if (!(n <= 3.0e38f)) return 0u;                                     // NaN / inf sources: all pixels
    const float d_first = sl_h(c, (float)__ldg(a.rows.omt + rb.x), (float)__ldg(a.rows.t + rb.x));
    const float d_last = sl_h(c, (float)__ldg(a.rows.omt + rb.y), (float)__ldg(a.rows.t + rb.y));
    const float e_first = sl_v(c, (float)__ldg(a.cols.omt + cb.x), (float)__ldg(a.cols.t + cb.x));
    const float e_last = sl_v(c, (float)__ldg(a.cols.omt + cb.y), (float)__ldg(a.cols.t + cb.y));
    bool h_ok = q != 0 && q != a.nbc - 1, v_ok = p != 0 && p != a.nbr - 1;   // border bands: flat
    if (h_ok && cb.y - cb.x >= 2) {                                     // interior columns exist
        h_ok = ((d_first > 0.f && d_last > 0.f) || (d_first < 0.f && d_last < 0.f)) &&
               fminf(fabsf(d_first), fabsf(d_last)) * (float)__ldg(a.cdt + q) > n;
    }
    if (v_ok && rb.y - rb.x >= 2) {                                     // interior rows exist
        v_ok = ((e_first > 0.f && e_last > 0.f) || (e_first < 0.f && e_last < 0.f)) &&
               fminf(fabsf(e_first), fabsf(e_last)) * (float)__ldg(a.rdt + p) > n;
    }
    if (h_ok && v_ok) {
        // in-band neighbour steps of each corner (i = 1 top row, j = 1 left column)
        const float sxl = (float)(__ldg(a.cols.t + cb.y) - __ldg(a.cols.t + max(cb.y - 1, cb.x)));
        const float sxr = (float)(__ldg(a.cols.t + min(cb.x + 1, cb.y)) - __ldg(a.cols.t + cb.x));
        const float syu = (float)(__ldg(a.rows.t + rb.y) - __ldg(a.rows.t + max(rb.y - 1, rb.x)));
        const float syd = (float)(__ldg(a.rows.t + min(rb.x + 1, rb.y)) - __ldg(a.rows.t + rb.x));
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float d = i ? d_first : d_last, e = j ? e_first : e_last;
                bool ok = true;
                if (cb.y > cb.x) ok = ok && (j == 0 ? !(d * sxl < -n) : !(d * sxr > n));
                if (rb.y > rb.x) ok = ok && (i == 0 ? !(e * syu < -n) : !(e * syd > n));
                if (ok) corners |= 1u << (2 * i + j);
            }
    }
    return (h_ok ? 1u : 0u) | (v_ok ? 2u : 0u);
}

// Candidate pixels of a partial cell, exactly tested by the warp's lanes.
__device__ __forceinline__ void process_partial(const UpCornerArgs &a, const float *S, int plane, int p, int q,
                                                unsigned ok, int lane)
{
    const int4 rb = __ldg(a.rband + p), cb = __ldg(a.cband + q);
    const int bh = rb.y - rb.x + 1, bw = cb.y - cb.x + 1;
    // candidate rows: the two boundary rows when v_ok, else all rows; same for columns
    const int nr = (ok & 2u) ? min(bh, 2) : bh, nc = (ok & 1u) ? min(bw, 2) : bw;
    for (int e = lane; e < nr * nc; e += kWarp) {
        const int r = e / nc, c = e - r * nc;
        const int y = (ok & 2u) ? (r ? rb.y : rb.x) : rb.x + r;
        const int x = (ok & 1u) ? (c ? cb.y : cb.x) : cb.x + c;
        float v;
        if (exact_peak(a, S, y, x, v)) emit_peak_c(a.counts, a.peaks, plane, a.cap, v, y, x);
    }
}

__global__ void __launch_bounds__(128, 8)
k_nms_up_corner(const UpCornerArgs a)
{
    extern __shared__ __align__(16) unsigned char smc[];
    const int plane = blockIdx.x;
    const int b = plane / a.K, k = plane - b * a.K;
    const float *p = a.conf + ((size_t)b * a.C + k) * (size_t)a.h * a.w;
    const int h = a.h, w = a.w, hw = h * w;
    const int nbc = a.nbc, ncell = a.nbr * nbc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_bw = ((hw + 127) & ~127) >> 5;
    const int n_cw = (ncell + 31) >> 5;
    float *S = reinterpret_cast<float *>(smc);                                     // [h*w]
    uint32_t *hotbits = reinterpret_cast<uint32_t *>(S + ((hw + 3) & ~3));         // [n_bw]
    uint32_t *cellbits = hotbits + n_bw;                                           // [n_cw]
    uint16_t *list = reinterpret_cast<uint16_t *>(cellbits + n_cw);                // [ncell] hot cells
    __shared__ int n_hot;

    // ---- phase 1: the plane (the compulsory HBM read) -> shared memory + hot bitmap
    for (int c = threadIdx.x; c < n_cw; c += blockDim.x) cellbits[c] = 0u;
    if (threadIdx.x == 0) n_hot = 0;
    if ((hw & 3) == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        float4 *s4 = reinterpret_cast<float4 *>(S);
        const int n4 = hw >> 2, n4_pad = (n4 + 31) & ~31;
        constexpr int U = 8;
        for (int e0 = threadIdx.x; e0 < n4_pad; e0 += U * blockDim.x) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * blockDim.x;
                v[u] = e < n4 ? __ldg(p4 + e) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * blockDim.x;
                if (e - lane >= n4_pad) break;                                     // warp-uniform tail
                if (e < n4) s4[e] = v[u];
                uint32_t nib = uint32_t(v[u].x >= a.thr) | (uint32_t(v[u].y >= a.thr) << 1) |
                               (uint32_t(v[u].z >= a.thr) << 2) | (uint32_t(v[u].w >= a.thr) << 3);
                nib = (e < n4 ? nib : 0u) << (4 * (lane & 7));
                nib |= __shfl_xor_sync(0xffffffffu, nib, 1);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 2);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 4);
                if ((lane & 7) == 0) hotbits[e >> 3] = nib;
            }
        }
    } else {
        for (int q = threadIdx.x; q < n_bw; q += blockDim.x) hotbits[q] = 0u;
        __syncthreads();
        for (int e = threadIdx.x; e < hw; e += blockDim.x) {
            const float v = __ldg(p + e);
            S[e] = v;
            if (v >= a.thr) atomicOr(hotbits + (e >> 5), 1u << (e & 31));
        }
    }
    __syncthreads();

    // ---- phase 2: hot cells = the cells reading a hot source (bitmap, then a dense list)
    for (int q = threadIdx.x; q < n_bw; q += blockDim.x) {
        uint32_t m = hotbits[q];
        if (!m) continue;
        const int base = q << 5;
        int r = base / w;                    // a 32-bit word spans at most ceil(32/w)+1 rows
        int c0 = base - r * w;
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1u;
            int rr = r, c = c0 + bit;
            while (c >= w) { c -= w; ++rr; }
            const int2 br = __ldg(a.src_rband + rr), bc = __ldg(a.src_cband + c);
            for (int pp = br.x; pp <= br.y; ++pp)
                for (int qq = bc.x; qq <= bc.y; ++qq) {
                    const int cell = pp * nbc + qq;
                    atomicOr(cellbits + (cell >> 5), 1u << (cell & 31));
                }
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n_cw; q += blockDim.x) {
        uint32_t m = cellbits[q];
        if (!m) continue;
        int slot = atomicAdd(&n_hot, __popc(m));
        while (m) {
            list[slot++] = uint16_t((q << 5) + __ffs(m) - 1);
            m &= m - 1u;
        }
    }
    __syncthreads();

    // ---- phase 3: a warp takes 32 hot cells at a time (lane = cell): classify;
    // corners of normal cells per lane; then the warp's partial cells, one at a
    // time with all lanes over the candidate pixels.  No CTA barrier after this.
    const int nh = n_hot;
    for (int base = warp * kWarp; base < nh; base += blockDim.x) {
        const int idx = base + lane;
        unsigned ok = 3u;
        int pr = 0, q = 0;
        if (idx < nh) {
            const int cell = list[idx];
            pr = cell / nbc;
            q = cell - pr * nbc;
            const int4 rb = __ldg(a.rband + pr), cb = __ldg(a.cband + q);
            unsigned corners;
            ok = classify_cell(a, S, pr, q, rb, cb, corners);
            if (ok == 3u) {
                while (corners) {
                    const int bit = __ffs(corners) - 1;
                    corners &= corners - 1u;
                    const int i = bit >> 1, j = bit & 1;
                    if (i == 1 && rb.x == rb.y) continue;     // a 1-row band's pixel is visited once
                    if (j == 1 && cb.x == cb.y) continue;
                    if (!corner_cross_ok(a, S, i ? pr - 1 : pr, j ? q - 1 : q, i, j)) continue;
                    const int yy = i ? rb.x : rb.y, xx = j ? cb.x : cb.y;
                    float v;
                    if (exact_peak(a, S, yy, xx, v)) emit_peak_c(a.counts, a.peaks, plane, a.cap, v, yy, xx);
                }
            }
        }
        uint32_t part = __ballot_sync(0xffffffffu, idx < nh && ok != 3u);
        while (part) {
            const int src = __ffs(part) - 1;
            part &= part - 1u;
            const int ppr = __shfl_sync(0xffffffffu, pr, src);
            const int pq = __shfl_sync(0xffffffffu, q, src);
            const unsigned pok_ = __shfl_sync(0xffffffffu, ok, src);
            process_partial(a, S, plane, ppr, pq, pok_, lane);
        }
    }
}

size_t nms_up_corner_smem(int h, int w, int nbr, int nbc, int scr_rows, int scr_cols)
{
    (void)scr_rows;
    (void)scr_cols;
    const int hw = h * w, ncell = nbr * nbc;
    return (size_t)((hw + 3) & ~3) * sizeof(float) + (size_t)(((hw + 127) & ~127) >> 5) * 4 +
           (size_t)((ncell + 31) >> 5) * 4 + (size_t)((ncell + 7) & ~7) * 2 + 16;
}

cudaError_t launch_nms_up_corner(const UpCornerArgs &a, int B, cudaStream_t s)
{
    const long long grid = (long long)B * a.K;
    if (grid == 0) return cudaSuccess;
    const size_t smem = nms_up_corner_smem(a.h, a.w, a.nbr, a.nbc, a.scr_rows, a.scr_cols);
    k_nms_up_corner<<<(unsigned)grid, 128, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t configure_corner_kernels(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_nms_up_corner);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_nms_up_corner, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - (int)fa.sharedSizeBytes);
}

}  // namespace pf
