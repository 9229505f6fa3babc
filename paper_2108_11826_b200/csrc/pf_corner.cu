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
//
// Pipeline (B200).  Persistent CTAs (grid = resident CTAs, planes
// round-robin).  Each low-res plane is one contiguous h*w fp32 block, so it
// is fetched by a single 1-D bulk copy (cp.async.bulk, the TMA unit) into a
// ring of shared-memory stages signalled by mbarriers; the next plane lands
// while the current one is processed, so the kernel never waits on HBM
// latency.  Per plane: (A) the hot-source bitmap from shared memory, (B) the
// hot cells as row-band bit masks — with integer upsampling the bands are
// canonical (band b reads sources b-1, b), so cell (p, q) is hot iff
// M_p bit q-1 or bit q, M_p = hot row p-1 | hot row p — compacted into a list,
// (C) one warp per 32 hot cells: classify, test surviving corners, and walk
// partial cells with all lanes.  The per-band slope weights live in shared
// memory for the whole kernel.
#include <algorithm>

#include "pf_launch.h"

namespace pf {

constexpr float kNoise = 7.62939453125e-06f;   // 2^-17
constexpr int kCornerThreads = 128;
constexpr int kCornerCands = 512;    // candidate pixels per plane kept in shared memory
constexpr int kCornerList = 1024;    // hot cells per plane kept in shared memory

// Per band, fp32 copies of the axis weights the classification uses.
struct BandT {
    float omt_f, t_f, omt_l, t_l;   // (1 - t), t at the band's first and last output
    float s_l, s_f, dt, pad;        // t step into the last output, out of the first; min step
};

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

// Shared-memory view of one CTA's band tables.
struct Bands {
    const int4 *rb, *cb;      // (first, last, src0, src1)
    const BandT *rt, *ct;
};

// Cross-boundary part of the corner test for the corner pixel (row role i,
// column role j) of corner (P, Q): the pixel is (i ? first(P+1) : last(P),
// j ? first(Q+1) : last(Q)) in cell (P+i, Q+j).  The own-cell in-band
// neighbours were checked by the caller.  Canonical bands: the four cells
// around the corner read the 3x3 sources rows (R0.z, R0.w = R1.z, R1.w) x
// columns (C0.z, C0.w = C1.z, C1.w), so both boundaries are piecewise affine.
__device__ __forceinline__ bool corner_cross_ok(const Bands &bd, const float *S, int w, int P, int Q, int i, int j)
{
    const int4 R0 = bd.rb[P], R1 = bd.rb[P + 1];
    const int4 C0 = bd.cb[Q], C1 = bd.cb[Q + 1];
    const float *s0 = S + R0.z * w, *s1 = S + R0.w * w, *s2 = S + R1.w * w;
    const float v00 = s0[C0.z], v01 = s0[C0.w], v02 = s0[C1.w];
    const float v10 = s1[C0.z], v11 = s1[C0.w], v12 = s1[C1.w];
    const float v20 = s2[C0.z], v21 = s2[C0.w], v22 = s2[C1.w];
    const float n = fmaxf(fmaxf(fmaxf(fabsf(v00), fabsf(v01)), fmaxf(fabsf(v02), fabsf(v10))),
                          fmaxf(fmaxf(fabsf(v11), fabsf(v12)), fmaxf(fmaxf(fabsf(v20), fabsf(v21)), fabsf(v22)))) *
                    kNoise;
    const BandT &rt0 = bd.rt[P], &rt1 = bd.rt[P + 1], &ct0 = bd.ct[Q], &ct1 = bd.ct[Q + 1];
    {
        // horizontal step across the column boundary, on row yy of cell row P+i
        const float omty = i ? rt1.omt_f : rt0.omt_l, ty = i ? rt1.t_f : rt0.t_l;
        const float ua0 = i ? v10 : v00, ua1 = i ? v11 : v01, ua2 = i ? v12 : v02;   // upper source row
        const float ub0 = i ? v20 : v10, ub1 = i ? v21 : v11, ub2 = i ? v22 : v12;   // lower source row
        const float mq = (ua1 - ua0) * omty + (ub1 - ub0) * ty;
        const float mq1 = (ua2 - ua1) * omty + (ub2 - ub1) * ty;
        const float cross = mq * ct0.omt_l + mq1 * ct1.t_f;                           // ~ G(x2) - G(x1)
        if (j == 0 ? cross > n : cross < -n) return false;
    }
    {
        const float omtx = j ? ct1.omt_f : ct0.omt_l, tx = j ? ct1.t_f : ct0.t_l;
        const float la0 = j ? v01 : v00, la1 = j ? v11 : v10, la2 = j ? v21 : v20;   // left source column
        const float lb0 = j ? v02 : v01, lb1 = j ? v12 : v11, lb2 = j ? v22 : v21;   // right source column
        const float mp = (la1 - la0) * omtx + (lb1 - lb0) * tx;
        const float mp1 = (la2 - la1) * omtx + (lb2 - lb1) * tx;
        const float cross = mp * rt0.omt_l + mp1 * rt1.t_f;                           // ~ G(y2) - G(y1)
        if (i == 0 ? cross > n : cross < -n) return false;
    }
    return true;
}

// Classify a hot cell.  Returns bit 0 = h_ok, bit 1 = v_ok (3 = normal) and,
// for the own-cell corner tests, a bitmask of corners (bit 2*i + j) whose
// in-band neighbours do not strictly beat them.
__device__ __forceinline__ unsigned classify_cell(const Bands &bd, const float *S, int w, int nbr, int nbc,
                                                  int p, int q, int4 rb, int4 cb, unsigned &corners)
{
    corners = 0u;
    const CellF c = cellf(S, w, rb, cb);
    const float n = mag(c) * kNoise;
    if (!(n <= 3.0e38f)) return 0u;                                     // NaN / inf sources: all pixels
    const BandT rt = bd.rt[p], ct = bd.ct[q];
    const float d_first = sl_h(c, rt.omt_f, rt.t_f), d_last = sl_h(c, rt.omt_l, rt.t_l);
    const float e_first = sl_v(c, ct.omt_f, ct.t_f), e_last = sl_v(c, ct.omt_l, ct.t_l);
    bool h_ok = q != 0 && q != nbc - 1, v_ok = p != 0 && p != nbr - 1;   // border bands: flat
    if (h_ok && cb.y - cb.x >= 2) {                                     // interior columns exist
        h_ok = ((d_first > 0.f && d_last > 0.f) || (d_first < 0.f && d_last < 0.f)) &&
               fminf(fabsf(d_first), fabsf(d_last)) * ct.dt > n;
    }
    if (v_ok && rb.y - rb.x >= 2) {                                     // interior rows exist
        v_ok = ((e_first > 0.f && e_last > 0.f) || (e_first < 0.f && e_last < 0.f)) &&
               fminf(fabsf(e_first), fabsf(e_last)) * rt.dt > n;
    }
    if (h_ok && v_ok) {
        // in-band neighbour steps of each corner (i = 1 top row, j = 1 left column)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float d = i ? d_first : d_last, e = j ? e_first : e_last;
                bool ok = true;
                if (cb.y > cb.x) ok = ok && (j == 0 ? !(d * ct.s_l < -n) : !(d * ct.s_f > n));
                if (rb.y > rb.x) ok = ok && (i == 0 ? !(e * rt.s_l < -n) : !(e * rt.s_f > n));
                if (ok) corners |= 1u << (2 * i + j);
            }
    }
    return (h_ok ? 1u : 0u) | (v_ok ? 2u : 0u);
}

// Candidate list of one plane (shared memory): packed (y << 16 | x).
struct CandList {
    uint32_t *c;
    int *n;
    int cap;
};

__device__ __forceinline__ void push_cand(const CandList &cl, int y, int x)
{
    const int slot = atomicAdd(cl.n, 1);
    if (slot < cl.cap) cl.c[slot] = (uint32_t(y) << 16) | uint32_t(x);   // beyond: plane redone (slow path)
}

// Candidate pixels of a partial cell.  Rows restricted to the boundary rows
// when v_ok, columns to the boundary columns when h_ok; further, a row whose
// own slope clears the noise bound is strictly monotone inside the cell, so
// only its rising-end column can be "> left and >= right" (and likewise a
// monotone column keeps only its rising-end row).
__device__ __forceinline__ void partial_cands(const UpCornerArgs &a, const Bands &bd, const CandList &cl,
                                              const float *S, int plane, int p, int q, unsigned ok)
{
    const int4 rb = bd.rb[p], cb = bd.cb[q];
    const CellF c = cellf(S, a.w, rb, cb);
    const float n = mag(c) * kNoise;              // NaN / inf: no compare passes, nothing pruned
    const float cdt = bd.ct[q].dt, rdt = bd.rt[p].dt;
    const bool q_in = q != 0 && q != a.nbc - 1 && cb.y > cb.x;
    const bool p_in = p != 0 && p != a.nbr - 1 && rb.y > rb.x;
    const int bh = rb.y - rb.x + 1, bw = cb.y - cb.x + 1;
    const int nr = (ok & 2u) ? min(bh, 2) : bh, nc = (ok & 1u) ? min(bw, 2) : bw;
    for (int r = 0; r < nr; ++r) {
        const int y = (ok & 2u) ? (r ? rb.y : rb.x) : rb.x + r;
        int only_x = -1;
        if (q_in) {
            const float d = sl_h(c, (float)__ldg(a.rows.omt + y), (float)__ldg(a.rows.t + y));
            if (fabsf(d) * cdt > n) only_x = d > 0.f ? cb.y : cb.x;
        }
        for (int k = 0; k < nc; ++k) {
            const int x = (ok & 1u) ? (k ? cb.y : cb.x) : cb.x + k;
            if (only_x >= 0 && x != only_x) continue;
            if (p_in) {
                const float e = sl_v(c, (float)__ldg(a.cols.omt + x), (float)__ldg(a.cols.t + x));
                if (fabsf(e) * rdt > n && y != (e > 0.f ? rb.y : rb.x)) continue;
            }
            push_cand(cl, y, x);
        }
    }
}

// One hot cell: classify; a normal cell pushes its surviving corner, a partial
// cell its candidate pixels.
__device__ __forceinline__ void process_cell(const UpCornerArgs &a, const Bands &bd, const CandList &cl,
                                             const float *S, int plane, int pr, int q)
{
    const int4 rb = bd.rb[pr], cb = bd.cb[q];
    unsigned corners;
    const unsigned ok = classify_cell(bd, S, a.w, a.nbr, a.nbc, pr, q, rb, cb, corners);
    if (ok == 3u) {
        while (corners) {
            const int bit = __ffs(corners) - 1;
            corners &= corners - 1u;
            const int i = bit >> 1, j = bit & 1;
            if (i == 1 && rb.x == rb.y) continue;     // a 1-row band's pixel is visited once
            if (j == 1 && cb.x == cb.y) continue;
            if (!corner_cross_ok(bd, S, a.w, i ? pr - 1 : pr, j ? q - 1 : q, i, j)) continue;
            push_cand(cl, i ? rb.x : rb.y, j ? cb.x : cb.y);
        }
    } else {
        partial_cands(a, bd, cl, S, plane, pr, q, ok);
    }
}

// Exact value of output pixel (y, x); -inf off the grid (paf.py:87-93 pads).
__device__ __forceinline__ float exact_value(const UpCornerArgs &a, const float *S, int y, int x)
{
    return up_val(S, a.w, ax_load(a.rows, y, a.H), ax_load(a.cols, x, a.W));
}

// ---- mbarrier + 1-D bulk copy (TMA) helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// Shared-memory layout of one CTA (byte offsets).
struct CornerLayout {
    int plane_floats;    // h*w rounded up to 128 (padding = -inf)
    int n_hw;            // hot-bitmap words per plane
    size_t planes, bars, rb, cb, rt, ct, hot, list, cand, total;
};

__host__ __device__ inline CornerLayout corner_layout(int h, int w, int nbr, int nbc, int nst)
{
    CornerLayout L;
    const int hw = h * w;
    L.plane_floats = (hw + 127) & ~127;
    L.n_hw = L.plane_floats >> 5;
    size_t o = 0;
    L.planes = o; o += (size_t)nst * L.plane_floats * sizeof(float);
    L.bars = o;   o += (size_t)nst * 8;
    o = (o + 15) & ~(size_t)15;
    L.rb = o;     o += (size_t)nbr * sizeof(int4);
    L.cb = o;     o += (size_t)nbc * sizeof(int4);
    L.rt = o;     o += (size_t)nbr * sizeof(BandT);
    L.ct = o;     o += (size_t)nbc * sizeof(BandT);
    L.hot = o;    o += (size_t)(L.n_hw + 4) * sizeof(uint32_t);
    L.list = o;   o += (size_t)kCornerList * sizeof(uint16_t);
    L.cand = o;   o += (size_t)kCornerCands * sizeof(uint32_t);
    L.total = (o + 15) & ~(size_t)15;
    return L;
}

__device__ __forceinline__ void fill_band(const AxisTab &tab, const double *dt, const int4 *bands, int b, int4 &B,
                                          BandT &T)
{
    B = __ldg(bands + b);
    const int f = B.x, l = B.y;
    T.omt_f = (float)__ldg(tab.omt + f);
    T.t_f = (float)__ldg(tab.t + f);
    T.omt_l = (float)__ldg(tab.omt + l);
    T.t_l = (float)__ldg(tab.t + l);
    T.s_l = (float)(__ldg(tab.t + l) - __ldg(tab.t + max(l - 1, f)));
    T.s_f = (float)(__ldg(tab.t + min(f + 1, l)) - __ldg(tab.t + f));
    T.dt = (float)__ldg(dt + b);
    T.pad = 0.f;
}

// Hot bits of source row r, columns [32j, 32j+32), from the
// linear hot bitmap (bits beyond the row masked off).
__device__ __forceinline__ uint32_t row_word(const uint32_t *hot, int h, int w, int r, int j)
{
    const int c0 = j << 5;
    if (r < 0 || r >= h || c0 >= w) return 0u;
    const int o = r * w + c0;
    uint32_t v = __funnelshift_r(hot[o >> 5], hot[(o >> 5) + 1], o & 31);
    const int rem = w - c0;
    if (rem < 32) v &= (1u << rem) - 1u;
    return v;
}

// Slow path for a plane whose hot cells or candidates overflowed the shared
// lists: forget its peaks and exactly test every pixel of every hot cell.
__device__ __noinline__ void redo_plane(const UpCornerArgs &a, const Bands &bd, const float *S,
                                        const uint32_t *hot, int plane)
{
    if (threadIdx.x == 0) a.counts[plane] = 0;
    __syncthreads();
    const int h = a.h, w = a.w, nwc = (w + 32) >> 5;
    for (int t = threadIdx.x; t < (h + 1) * nwc; t += kCornerThreads) {
        const int p = t / nwc, j = t - p * nwc;
        const uint32_t m = row_word(hot, h, w, p - 1, j) | row_word(hot, h, w, p, j);
        uint32_t c = m | (m << 1);
        if (j) c |= (row_word(hot, h, w, p - 1, j - 1) | row_word(hot, h, w, p, j - 1)) >> 31;
        while (c) {
            const int q = (j << 5) + __ffs(c) - 1;
            c &= c - 1u;
            const int4 rb = bd.rb[p], cb = bd.cb[q];
            for (int y = rb.x; y <= rb.y; ++y)
                for (int x = cb.x; x <= cb.y; ++x) {
                    float v;
                    if (exact_peak(a, S, y, x, v)) emit_peak_c(a.counts, a.peaks, plane, a.cap, v, y, x);
                }
        }
    }
}

__global__ void __launch_bounds__(kCornerThreads, 5)
k_nms_up_corner(const UpCornerArgs a)
{
    extern __shared__ __align__(128) unsigned char smc[];
    const int h = a.h, w = a.w, hw = h * w;
    const int nbr = a.nbr, nbc = a.nbc, nst = a.nst;
    const CornerLayout L = corner_layout(h, w, nbr, nbc, nst);
    float *planes = reinterpret_cast<float *>(smc + L.planes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smc + L.bars);
    int4 *RB = reinterpret_cast<int4 *>(smc + L.rb);
    int4 *CB = reinterpret_cast<int4 *>(smc + L.cb);
    BandT *RT = reinterpret_cast<BandT *>(smc + L.rt);
    BandT *CT = reinterpret_cast<BandT *>(smc + L.ct);
    uint32_t *hot = reinterpret_cast<uint32_t *>(smc + L.hot);
    uint16_t *list = reinterpret_cast<uint16_t *>(smc + L.list);
    uint32_t *cand = reinterpret_cast<uint32_t *>(smc + L.cand);
    __shared__ int n_hot, n_cand;
    const CandList cl{cand, &n_cand, kCornerCands};
    const Bands bd{RB, CB, RT, CT};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long P = (long long)a.B * a.K;
    const uint32_t plane_bytes = (uint32_t)hw * 4u;

    // ---- prologue: band tables, -inf plane padding, barriers, first loads
    for (int b = threadIdx.x; b < nbr + nbc; b += kCornerThreads) {
        if (b < nbr) fill_band(a.rows, a.rdt, a.rband, b, RB[b], RT[b]);
        else fill_band(a.cols, a.cdt, a.cband, b - nbr, CB[b - nbr], CT[b - nbr]);
    }
    for (int s = 0; s < nst; ++s)
        for (int e = hw + threadIdx.x; e < L.plane_floats; e += kCornerThreads) planes[s * L.plane_floats + e] = -INFINITY;
    for (int e = L.n_hw + threadIdx.x; e < L.n_hw + 4; e += kCornerThreads) hot[e] = 0u;
    if (threadIdx.x == 0) {
        n_hot = 0;
        n_cand = 0;
        if (a.bulk) {
            for (int s = 0; s < nst; ++s) mbar_init(bars + s, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int s = 0; s < nst; ++s) {
                const long long pl = blockIdx.x + (long long)s * gridDim.x;
                if (pl < P) {
                    const long long b = pl / a.K, k = pl - b * a.K;
                    bulk_load(planes + s * L.plane_floats, a.conf + ((size_t)b * a.C + k) * (size_t)hw, plane_bytes,
                              bars + s);
                }
            }
        }
    }
    __syncthreads();

    int it = 0;
    for (long long pl = blockIdx.x; pl < P; pl += gridDim.x, ++it) {
        const int stage = it % nst;
        float *S = planes + stage * L.plane_floats;
        const int plane = (int)pl;
        if (a.bulk) {
            mbar_wait(bars + stage, (uint32_t)(it / nst) & 1u);
        } else {
            const long long b = pl / a.K, k = pl - b * a.K;
            const float *src = a.conf + ((size_t)b * a.C + k) * (size_t)hw;
            for (int e = threadIdx.x; e < hw; e += kCornerThreads) S[e] = __ldg(src + e);
            __syncthreads();
        }

        // ---- (A) hot-source bitmap: 8 lanes x float4 = one 32-bit word
        {
            const float4 *s4 = reinterpret_cast<const float4 *>(S);
            const int n4 = L.plane_floats >> 2;            // multiple of 32: warp-uniform trip count
            for (int e = threadIdx.x; e < n4; e += kCornerThreads) {
                const float4 v = s4[e];
                uint32_t nib = uint32_t(v.x >= a.thr) | (uint32_t(v.y >= a.thr) << 1) |
                               (uint32_t(v.z >= a.thr) << 2) | (uint32_t(v.w >= a.thr) << 3);
                nib <<= 4 * (lane & 7);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 1);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 2);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 4);
                if ((lane & 7) == 0) hot[e >> 3] = nib;
            }
        }
        __syncthreads();

        // ---- (B) hot cells of canonical bands: C_p = M_p | M_p << 1 (+ carry)
        {
            const int nwc = (w + 32) >> 5;                  // words per band row (nbc = w + 1 bits)
            const int ntask = (h + 1) * nwc;
            for (int t = threadIdx.x; t < ntask; t += kCornerThreads) {
                const int p = t / nwc, j = t - p * nwc;
                const uint32_t m = row_word(hot, h, w, p - 1, j) | row_word(hot, h, w, p, j);
                uint32_t c = m | (m << 1);
                if (j) c |= (row_word(hot, h, w, p - 1, j - 1) | row_word(hot, h, w, p, j - 1)) >> 31;
                if (c) {
                    int slot = atomicAdd(&n_hot, __popc(c));
                    while (c) {
                        const int q = (j << 5) + __ffs(c) - 1;
                        c &= c - 1u;
                        if (slot < kCornerList) list[slot] = uint16_t(p * nbc + q);   // beyond: slow path
                        ++slot;
                    }
                }
            }
        }
        __syncthreads();

        // ---- (C1) lane = hot cell: classify; normal cells push their surviving
        // corner, partial cells their candidate pixels
        const int nh = min(n_hot, kCornerList);
        for (int idx = threadIdx.x; idx < nh; idx += kCornerThreads) {
            const int cell = list[idx];
            const int pr = cell / nbc;
            process_cell(a, bd, cl, S, plane, pr, cell - pr * nbc);
        }
        __syncthreads();

        // ---- (C2) the exact 3x3 test, 9 lanes per candidate (one pixel each),
        // three candidates per warp, gathered by shuffles
        {
            const int nc = min(n_cand, kCornerCands);
            const int grp = lane / 9, nb = lane - grp * 9;
            const int src = min(grp, 2) * 9;
            for (int base = warp * 3; base < nc; base += 3 * (kCornerThreads / kWarp)) {
                const int ci = base + grp;
                const bool act = grp < 3 && ci < nc;
                int y = 0, x = 0;
                float val = -INFINITY;
                if (act) {
                    const uint32_t yx = cand[ci];
                    y = (int)(yx >> 16);
                    x = (int)(yx & 0xffffu);
                    val = exact_value(a, S, y + nb / 3 - 1, x + nb % 3 - 1);
                }
                float nv[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) nv[k] = __shfl_sync(0xffffffffu, val, src + k);
                if (act && nb == 4) {
                    const float v = nv[4];
                    // paf.py:95-99: earlier neighbours strictly, later ones non-strictly
                    if (v >= a.thr && v > nv[0] && v > nv[1] && v > nv[2] && v > nv[3] && v >= nv[5] &&
                        v >= nv[6] && v >= nv[7] && v >= nv[8])
                        emit_peak_c(a.counts, a.peaks, plane, a.cap, v, y, x);
                }
            }
        }
        __syncthreads();
        if (n_hot > kCornerList || n_cand > kCornerCands) {    // CTA-uniform: a list overflowed
            redo_plane(a, bd, S, hot, plane);
        }
        __syncthreads();                                     // stage + list free again
        if (threadIdx.x == 0) {
            n_hot = 0;
            n_cand = 0;
            const long long nx = pl + (long long)nst * gridDim.x;
            if (a.bulk && nx < P) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const long long b = nx / a.K, k = nx - b * a.K;
                bulk_load(S, a.conf + ((size_t)b * a.C + k) * (size_t)hw, plane_bytes, bars + stage);
            }
        }
    }
}

size_t nms_up_corner_smem(int h, int w, int nbr, int nbc, int nst)
{
    return corner_layout(h, w, nbr, nbc, nst).total;
}

cudaError_t launch_nms_up_corner(const UpCornerArgs &a_in, cudaStream_t s)
{
    UpCornerArgs a = a_in;
    const long long P = (long long)a.B * a.K;
    if (P == 0) return cudaSuccess;
    const size_t smem = nms_up_corner_smem(a.h, a.w, a.nbr, a.nbc, a.nst);
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_up_corner, kCornerThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    // bulk copies need 16-byte aligned, 16-byte multiple planes
    a.bulk = ((size_t)a.h * a.w * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(a.conf) & 15) == 0;
    const long long grid = std::min<long long>(P, (long long)occ * sms);
    k_nms_up_corner<<<(unsigned)grid, kCornerThreads, smem, s>>>(a);
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
