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

// Chain pre-filter: true if provably no output pixel of interior-direction
// cell (p, q) is a peak.  Cheap (4-6 shared loads, no band tables), so it
// runs on every hot cell and only the survivors pay for classify_cell.
//
// hR: both source rows rise to the right, fl(a1 - a0) > d and fl(b1 - b0) > d
// with d = 2^-16 * max|sources involved|.  Then D_h >= d for every ty in the
// band, adjacent outputs of a row differ by >= d * (1/u) >= 2^-20 M exactly
// (u <= 16, checked by the launcher: a.chain), which beats the rounding of
// both values (< 2^-23 M each, see the header), so every output but the
// band's last column has a strictly larger right neighbour (fails ">= right",
// paf.py:99).  If the next cell (q+1) rises to the right too, the last column
// fails as well: its right neighbour is first(q+1) and
// G(first(q+1)) - G(last(q)) = (R1-R0)(1-t_l) + (R2-R1) t_f >= d/u.  So the
// whole cell is excluded.  hL / vD / vU are the mirror and vertical cases
// (the strict "> left/up" rules fail instead).  Border bands in the tested
// direction are never pruned in that direction (their sources coincide, so
// the differences are 0 and the strict compares fail by themselves).
// NaN/inf sources make every compare false: nothing is pruned.
__device__ __forceinline__ bool chain_pruned(const Bands &bd, const float *S, int w, int nbr, int nbc, int p, int q)
{
    const int4 rb = bd.rb[p], cb = bd.cb[q];
    const float *r0 = S + rb.z * w, *r1 = S + rb.w * w;
    const float a0 = r0[cb.z], a1 = r0[cb.w], b0 = r1[cb.z], b1 = r1[cb.w];
    const float m4 = fmaxf(fmaxf(fabsf(a0), fabsf(a1)), fmaxf(fabsf(b0), fabsf(b1)));
    if (!(m4 >= 8.673617379884035e-19f)) return false;   // 2^-60: tiny or NaN -> exact path
    const float d4 = m4 * 1.52587890625e-05f;              // 2^-16 (exact scaling)
    const float ha = a1 - a0, hb = b1 - b0, va = b0 - a0, vb = b1 - a1;
    const bool hR = ha > d4 && hb > d4, hL = ha < -d4 && hb < -d4;
    const bool vD = va > d4 && vb > d4, vU = va < -d4 && vb < -d4;
    if (hR || hL) {
        // the neighbouring cell in the rising direction: column pair (c1, c2) or (c_-1, c0)
        const int qn = hR ? q + 1 : q - 1;
        if (qn >= 0 && qn < nbc) {
            const int4 cn = bd.cb[qn];
            const float e0 = r0[cn.z], e1 = r0[cn.w], f0 = r1[cn.z], f1 = r1[cn.w];
            const float m = fmaxf(m4, fmaxf(fmaxf(fabsf(e0), fabsf(e1)), fmaxf(fabsf(f0), fabsf(f1))));
            const float d = m * 1.52587890625e-05f;
            const float ea = e1 - e0, eb = f1 - f0;
            const bool ok = hR ? (ha > d && hb > d && ea > d && eb > d) : (ha < -d && hb < -d && ea < -d && eb < -d);
            if (ok) return true;
        }
    }
    if (vD || vU) {
        const int pn = vD ? p + 1 : p - 1;
        if (pn >= 0 && pn < nbr) {
            const int4 rn = bd.rb[pn];
            const float *s0 = S + rn.z * w, *s1 = S + rn.w * w;
            const float e0 = s0[cb.z], e1 = s0[cb.w], f0 = s1[cb.z], f1 = s1[cb.w];
            const float m = fmaxf(m4, fmaxf(fmaxf(fabsf(e0), fabsf(e1)), fmaxf(fabsf(f0), fabsf(f1))));
            const float d = m * 1.52587890625e-05f;
            const float ea = f0 - e0, eb = f1 - e1;
            const bool ok = vD ? (va > d && vb > d && ea > d && eb > d) : (va < -d && vb < -d && ea < -d && eb < -d);
            if (ok) return true;
        }
    }
    return false;
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
    L.list = o;   o += (size_t)kCornerList * sizeof(uint32_t);
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
    uint32_t *list = reinterpret_cast<uint32_t *>(smc + L.list);
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
                        if (slot < kCornerList) list[slot] = (uint32_t(p) << 16) | uint32_t(q);   // beyond: slow path
                        ++slot;
                    }
                }
            }
        }
        __syncthreads();

        // ---- (C1) lane = hot cell.  Each warp owns a contiguous slice of the
        // hot list: the chain pre-filter runs on every cell and compacts the
        // survivors in place at the front of the slice (warp-synchronous: a
        // write index never passes the read index), then the survivors are
        // classified; normal cells push their surviving corner, partial cells
        // their candidate pixels.
        {
            const int nh = min(n_hot, kCornerList);
            const int chunk = (nh + 3) >> 2;
            const int lo = warp * chunk, hi = min(nh, lo + chunk);
            int ns = hi - lo;
            if (a.chain) {
                ns = 0;
                for (int base = lo; base < hi; base += kWarp) {
                    const int idx = base + lane;
                    uint32_t cell = 0u;
                    bool keep = false;
                    if (idx < hi) {
                        cell = list[idx];
                        keep = !chain_pruned(bd, S, w, nbr, nbc, int(cell >> 16), int(cell & 0xffffu));
                    }
                    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                    __syncwarp();
                    if (keep) list[lo + ns + __popc(bal & ((1u << lane) - 1u))] = cell;
                    ns += __popc(bal);
                }
                __syncwarp();
            }
            for (int idx = lo + lane; idx < lo + ns; idx += kWarp) {
                const uint32_t cell = list[idx];
                process_cell(a, bd, cl, S, plane, int(cell >> 16), int(cell & 0xffffu));
            }
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

// ---------------------------------------------------------------------------
// k_nms_up_corner_w — the same exact algorithm, reorganised so that the four
// warps of a CTA never wait for each other inside a plane.  Warp w owns the
// band rows [w*R, (w+1)*R) of the plane in the stage buffer and runs, on its
// own, the whole chain for them:
//   hot rows    — ballot(S[r][32j + lane] >= thr): one row-aligned hot word
//                 per (source row, 32 columns), carried in registers from one
//                 band row to the next (band p reads source rows p-1, p);
//   hot cells   — C = M | M << 1 (+ carry), M = hot(p-1) | hot(p): lane q of
//                 word j is cell (p, 32j + q); compacted into a per-warp list;
//   chain prune — on full lanes, survivors compacted in place (chain_pruned);
//   classify    — survivors only (process_cell) -> per-warp candidate list;
//   exact test  — 9 lanes per candidate, as in k_nms_up_corner.
// The only CTA barrier per plane is the one that frees the stage buffer.
constexpr int kWList = 256;      // hot cells per warp before a flush
constexpr int kWCand = 128;      // candidate pixels per warp per plane
constexpr int kMaxRowWords = 8;  // w <= 255

struct CornerWLayout {
    int plane_floats;
    size_t planes, bars, rb, cb, rt, ct, list, cand, total;
};

__host__ __device__ inline CornerWLayout corner_w_layout(int h, int w, int nbr, int nbc, int nst)
{
    CornerWLayout L;
    L.plane_floats = (h * w + 127) & ~127;
    size_t o = 0;
    L.planes = o; o += (size_t)nst * L.plane_floats * sizeof(float);
    L.bars = o;   o += (size_t)nst * 8;
    o = (o + 15) & ~(size_t)15;
    L.rb = o;     o += (size_t)nbr * sizeof(int4);
    L.cb = o;     o += (size_t)nbc * sizeof(int4);
    L.rt = o;     o += (size_t)nbr * sizeof(BandT);
    L.ct = o;     o += (size_t)nbc * sizeof(BandT);
    L.list = o;   o += (size_t)(kCornerThreads / kWarp) * kWList * sizeof(uint32_t);
    L.cand = o;   o += (size_t)(kCornerThreads / kWarp) * kWCand * sizeof(uint32_t);
    L.total = (o + 15) & ~(size_t)15;
    return L;
}

// Hot word of source row r, columns [32j, 32j + 32) (warp-uniform result).
__device__ __forceinline__ uint32_t hot_word(const float *S, int h, int w, int r, int j, int lane, float thr)
{
    const int c = (j << 5) + lane;
    const bool hot = r >= 0 && r < h && c < w && S[r * w + c] >= thr;
    return __ballot_sync(0xffffffffu, hot);
}

// Prune the warp's hot list (full lanes, in place) and classify the survivors.
__device__ __forceinline__ void flush_cells(const UpCornerArgs &a, const Bands &bd, const CandList &cl,
                                            const float *S, int plane, uint32_t *list, int nl, int lane)
{
    int ns = nl;
    if (a.chain) {
        ns = 0;
        for (int base = 0; base < nl; base += kWarp) {
            const int idx = base + lane;
            uint32_t cell = 0u;
            bool keep = false;
            if (idx < nl) {
                cell = list[idx];
                keep = !chain_pruned(bd, S, a.w, a.nbr, a.nbc, int(cell >> 16), int(cell & 0xffffu));
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) list[ns + __popc(bal & ((1u << lane) - 1u))] = cell;
            ns += __popc(bal);
        }
        __syncwarp();
    }
    for (int idx = lane; idx < ns; idx += kWarp) {
        const uint32_t cell = list[idx];
        process_cell(a, bd, cl, S, plane, int(cell >> 16), int(cell & 0xffffu));
    }
    __syncwarp();
}

// Slow path (a per-warp candidate list overflowed): exact test of every
// pixel of every hot cell of the plane, straight from the sources.
__device__ __noinline__ void redo_plane_w(const UpCornerArgs &a, const Bands &bd, const float *S, int plane)
{
    if (threadIdx.x == 0) a.counts[plane] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < a.nbr * a.nbc; t += kCornerThreads) {
        const int p = t / a.nbc, q = t - p * a.nbc;
        const int4 rb = bd.rb[p], cb = bd.cb[q];
        const CellF c = cellf(S, a.w, rb, cb);
        if (!(c.a0 >= a.thr || c.a1 >= a.thr || c.b0 >= a.thr || c.b1 >= a.thr)) continue;
        for (int y = rb.x; y <= rb.y; ++y)
            for (int x = cb.x; x <= cb.y; ++x) {
                float v;
                if (exact_peak(a, S, y, x, v)) emit_peak_c(a.counts, a.peaks, plane, a.cap, v, y, x);
            }
    }
}

__global__ void __launch_bounds__(kCornerThreads, 5)
k_nms_up_corner_w(const UpCornerArgs a)
{
    extern __shared__ __align__(128) unsigned char smc[];
    const int h = a.h, w = a.w, hw = h * w;
    const int nbr = a.nbr, nbc = a.nbc, nst = a.nst;
    const CornerWLayout L = corner_w_layout(h, w, nbr, nbc, nst);
    float *planes = reinterpret_cast<float *>(smc + L.planes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smc + L.bars);
    int4 *RB = reinterpret_cast<int4 *>(smc + L.rb);
    int4 *CB = reinterpret_cast<int4 *>(smc + L.cb);
    BandT *RT = reinterpret_cast<BandT *>(smc + L.rt);
    BandT *CT = reinterpret_cast<BandT *>(smc + L.ct);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *list = reinterpret_cast<uint32_t *>(smc + L.list) + warp * kWList;
    uint32_t *cand = reinterpret_cast<uint32_t *>(smc + L.cand) + warp * kWCand;
    __shared__ int n_cand[kCornerThreads / kWarp];
    __shared__ int overflow;
    const CandList cl{cand, &n_cand[warp], kWCand};
    const Bands bd{RB, CB, RT, CT};
    const int P = a.B * a.K;
    const uint32_t plane_bytes = (uint32_t)hw * 4u;
    const int nws = (w + 31) >> 5;                 // source-row words
    const int nwc = (nbc + 31) >> 5;               // band-row cell words
    const int rpw = (nbr + 3) >> 2;                // band rows per warp
    const int p_lo = warp * rpw, p_hi = min(nbr, p_lo + rpw);

    for (int b = threadIdx.x; b < nbr + nbc; b += kCornerThreads) {
        if (b < nbr) fill_band(a.rows, a.rdt, a.rband, b, RB[b], RT[b]);
        else fill_band(a.cols, a.cdt, a.cband, b - nbr, CB[b - nbr], CT[b - nbr]);
    }
    if (lane == 0) n_cand[warp] = 0;
    if (threadIdx.x == 0) {
        overflow = 0;
        if (a.bulk) {
            for (int s = 0; s < nst; ++s) mbar_init(bars + s, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int s = 0; s < nst; ++s) {
                const int pl = blockIdx.x + s * gridDim.x;
                if (pl < P) {
                    const int b = pl / a.K, k = pl - b * a.K;
                    bulk_load(planes + s * L.plane_floats, a.conf + ((size_t)b * a.C + k) * (size_t)hw, plane_bytes,
                              bars + s);
                }
            }
        }
    }
    __syncthreads();

    int it = 0, stage = 0;
    for (int pl = blockIdx.x; pl < P; pl += gridDim.x, ++it) {
        float *S = planes + stage * L.plane_floats;
        if (a.bulk) {
            mbar_wait(bars + stage, (uint32_t)(it / nst) & 1u);
        } else {
            const int b = pl / a.K, k = pl - b * a.K;
            const float *src = a.conf + ((size_t)b * a.C + k) * (size_t)hw;
            for (int e = threadIdx.x; e < hw; e += kCornerThreads) S[e] = __ldg(src + e);
            __syncthreads();
        }

        // ---- hot cells of this warp's band rows -> list (flushed when full)
        uint32_t prev[kMaxRowWords], cur[kMaxRowWords];
#pragma unroll
        for (int j = 0; j < kMaxRowWords; ++j)
            prev[j] = j < nws ? hot_word(S, h, w, p_lo - 1, j, lane, a.thr) : 0u;
        int nl = 0;
        for (int p = p_lo; p < p_hi; ++p) {
            uint32_t carry = 0u;
#pragma unroll
            for (int j = 0; j < kMaxRowWords; ++j) {
                if (j >= nwc) break;
                cur[j] = j < nws ? hot_word(S, h, w, p, j, lane, a.thr) : 0u;
                const uint32_t m = prev[j] | cur[j];
                uint32_t c = m | (m << 1) | carry;
                carry = m >> 31;
                if ((j << 5) + 32 > nbc) c &= (1u << (nbc - (j << 5))) - 1u;
                if (c) {
                    if (nl > kWList - kWarp) {
                        flush_cells(a, bd, cl, S, pl, list, nl, lane);
                        nl = 0;
                    }
                    if ((c >> lane) & 1u)
                        list[nl + __popc(c & ((1u << lane) - 1u))] = (uint32_t(p) << 16) | uint32_t((j << 5) + lane);
                    nl += __popc(c);
                }
            }
#pragma unroll
            for (int j = 0; j < kMaxRowWords; ++j) prev[j] = cur[j];
        }
        __syncwarp();
        if (nl) flush_cells(a, bd, cl, S, pl, list, nl, lane);

        // ---- exact 3x3 test of this warp's candidates: 9 lanes each
        {
            const int ncd = n_cand[warp];
            const int nc = min(ncd, kWCand);
            const int grp = lane / 9, nb = lane - grp * 9;
            const int src = min(grp, 2) * 9;
            for (int base = 0; base < nc; base += 3) {
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
                        emit_peak_c(a.counts, a.peaks, pl, a.cap, v, y, x);
                }
            }
            __syncwarp();
            if (lane == 0) {
                if (ncd > kWCand) overflow = 1;
                n_cand[warp] = 0;
            }
        }
        __syncthreads();                                     // every warp done with the stage
        if (overflow) {                                      // CTA-uniform
            redo_plane_w(a, bd, S, pl);
            __syncthreads();
            if (threadIdx.x == 0) overflow = 0;
        }
        if (threadIdx.x == 0) {
            const int nx = pl + nst * gridDim.x;
            if (a.bulk && nx < P) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const int b = nx / a.K, k = nx - b * a.K;
                bulk_load(S, a.conf + ((size_t)b * a.C + k) * (size_t)hw, plane_bytes, bars + stage);
            }
        }
        if (!a.bulk) __syncthreads();
        stage = stage + 1 == nst ? 0 : stage + 1;
    }
}

size_t nms_up_corner_w_smem(int h, int w, int nbr, int nbc, int nst)
{
    return corner_w_layout(h, w, nbr, nbc, nst).total;
}

// ---------------------------------------------------------------------------
// k_nms_up_corner_g — warp per plane, sources read through L1/L2 instead of
// a shared-memory copy.  A shared plane buffer (15 KB at 46x82) caps a CTA
// design at ~5 resident CTAs per SM, and the per-plane chain (hot words ->
// hot cells -> chain prune -> classify -> exact test) is latency bound, so
// residency is what sets the speed.  Here a warp needs ~2 KB of shared
// memory, 32 warps stay resident per SM, and every warp runs its planes
// start to finish with warp-synchronous steps only:
//   hot words  — batches of kGwBatch row-aligned loads in flight per lane
//                (lane = column), one ballot per (source row, 32 columns);
//                the warp's next plane is prefetched into L2 meanwhile;
//   hot cells  — lane = band row p: C_j = M | M << 1 (+ carry),
//                M = hot(p-1) | hot(p); a warp scan places every lane's
//                cells into the warp's list (flushed whenever it fills);
//   flush      — chain_pruned on full lanes, process_cell on the survivors;
//   exact test — 9 lanes per candidate.  A candidate-list overflow sends the
//                plane to an exact warp-level rescan instead.
constexpr int kGwThreads = 256;
constexpr int kGwWarps = kGwThreads / kWarp;
constexpr int kGwList = 256;
constexpr int kGwCand = 64;
constexpr int kGwBatch = 16;

__host__ __device__ inline int gw_row_stride(int w)
{
    const int nws = (w + 31) >> 5;
    return nws | 1;                      // odd: conflict-free lane-per-row reads
}

__host__ __device__ inline size_t gw_smem(int h, int w)
{
    return (size_t)kGwWarps * ((size_t)h * gw_row_stride(w) + kGwList + kGwCand) * sizeof(uint32_t);
}

__device__ __noinline__ void redo_plane_g(const UpCornerArgs &a, const Bands &bd, const float *S, int plane,
                                          int lane)
{
    for (int t = lane; t < a.nbr * a.nbc; t += kWarp) {
        const int p = t / a.nbc, q = t - p * a.nbc;
        const int4 rb = bd.rb[p], cb = bd.cb[q];
        const CellF c = cellf(S, a.w, rb, cb);
        if (!(c.a0 >= a.thr || c.a1 >= a.thr || c.b0 >= a.thr || c.b1 >= a.thr)) continue;
        for (int y = rb.x; y <= rb.y; ++y)
            for (int x = cb.x; x <= cb.y; ++x) {
                float v;
                if (exact_peak(a, S, y, x, v)) emit_peak_c(a.counts, a.peaks, plane, a.cap, v, y, x);
            }
    }
}

__global__ void __launch_bounds__(kGwThreads, 4)
k_nms_up_corner_g(const UpCornerArgs a)
{
    extern __shared__ __align__(16) uint32_t smg[];
    const int h = a.h, w = a.w, hw = h * w;
    const int nbr = a.nbr, nbc = a.nbc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rs = gw_row_stride(w);
    uint32_t *R = smg + (size_t)warp * h * rs;
    uint32_t *list = smg + (size_t)kGwWarps * h * rs + warp * kGwList;
    uint32_t *cand = smg + (size_t)kGwWarps * (h * rs + kGwList) + warp * kGwCand;
    __shared__ int n_cand[kGwWarps];
    const CandList cl{cand, &n_cand[warp], kGwCand};
    const Bands bd{a.rband, a.cband, a.rbt, a.cbt};
    const int P = a.B * a.K;
    const int nws = (w + 31) >> 5;               // source-row words
    const int nwc = (nbc + 31) >> 5;             // band-row cell words
    const int U = h * nws;
    const int nwarps = gridDim.x * kGwWarps;
    if (lane == 0) n_cand[warp] = 0;
    __syncwarp();

    for (int pl = blockIdx.x * kGwWarps + warp; pl < P; pl += nwarps) {
        const int fb = pl / a.K, k = pl - fb * a.K;
        const float *S = a.conf + ((size_t)fb * a.C + k) * (size_t)hw;
        {
            const int nx = pl + nwarps;          // this warp's next plane -> L2
            if (nx < P) {
                const int nb = nx / a.K, nk = nx - nb * a.K;
                const char *Sn = reinterpret_cast<const char *>(a.conf + ((size_t)nb * a.C + nk) * (size_t)hw);
                for (int o = lane * 128; o < hw * 4; o += kWarp * 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(Sn + o));
            }
        }

        // ---- hot words R[r][j] (bit = column 32j + lane >= thr)
        {
            int r = 0, j = 0;
            for (int u0 = 0; u0 < U; u0 += kGwBatch) {
                float v[kGwBatch];
                int rr = r, jj = j;
#pragma unroll
                for (int i = 0; i < kGwBatch; ++i) {
                    const int col = (jj << 5) + lane;
                    v[i] = (u0 + i < U && col < w) ? __ldg(S + rr * w + col) : -INFINITY;
                    if (++jj == nws) { jj = 0; ++rr; }
                }
                uint32_t mine = 0u;
#pragma unroll
                for (int i = 0; i < kGwBatch; ++i) {
                    const uint32_t word = __ballot_sync(0xffffffffu, v[i] >= a.thr);
                    if (lane == i) mine = word;
                }
                const int u = u0 + lane;
                if (lane < kGwBatch && u < U) {
                    const int ur = u / nws;
                    R[ur * rs + (u - ur * nws)] = mine;
                }
                r = rr; j = jj;
            }
        }
        __syncwarp();

        // ---- hot cells: lane = band row, warp scan into the list
        int nl = 0;
        for (int pg = 0; pg < nbr; pg += kWarp) {
            const int p = pg + lane;
            uint32_t cw[kMaxRowWords];
            int cnt = 0;
            uint32_t carry = 0u;
#pragma unroll
            for (int jw = 0; jw < kMaxRowWords; ++jw) {
                uint32_t c = 0u;
                if (jw < nwc && p < nbr) {
                    uint32_t m = 0u;
                    if (jw < nws) {
                        if (p >= 1) m |= R[(p - 1) * rs + jw];
                        if (p < h) m |= R[p * rs + jw];
                    }
                    c = m | (m << 1) | carry;
                    carry = m >> 31;
                    const int left = nbc - (jw << 5);
                    if (left < 32) c &= (1u << left) - 1u;
                }
                cw[jw] = c;
                cnt += __popc(c);
            }
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < kWarp; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t;
            }
            const int total = __shfl_sync(0xffffffffu, incl, kWarp - 1);
            if (total == 0) continue;
            const int excl = incl - cnt;
            int w0 = 0;
            while (true) {
                const int room = kGwList - nl;
                int idx = excl;
#pragma unroll
                for (int jw = 0; jw < kMaxRowWords; ++jw) {
                    uint32_t c = cw[jw];
                    while (c) {
                        const int bit = __ffs(c) - 1;
                        c &= c - 1u;
                        if (idx >= w0 && idx < w0 + room)
                            list[nl + idx - w0] = (uint32_t(p) << 16) | uint32_t((jw << 5) + bit);
                        ++idx;
                    }
                }
                const int wrote = min(total - w0, room);
                nl += wrote;
                w0 += wrote;
                __syncwarp();
                if (w0 >= total) break;
                flush_cells(a, bd, cl, S, pl, list, nl, lane);
                nl = 0;
            }
        }
        if (nl) flush_cells(a, bd, cl, S, pl, list, nl, lane);

        // ---- exact 3x3 test of the candidates, 9 lanes each
        const int ncd = n_cand[warp];
        __syncwarp();
        if (lane == 0) n_cand[warp] = 0;
        if (ncd > kGwCand) {
            redo_plane_g(a, bd, S, pl, lane);    // nothing of this plane was emitted yet
        } else {
            const int grp = lane / 9, nb = lane - grp * 9;
            const int src = min(grp, 2) * 9;
            for (int base = 0; base < ncd; base += 3) {
                const int ci = base + grp;
                const bool act = grp < 3 && ci < ncd;
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
                for (int kk = 0; kk < 9; ++kk) nv[kk] = __shfl_sync(0xffffffffu, val, src + kk);
                if (act && nb == 4) {
                    const float v = nv[4];
                    // paf.py:95-99: earlier neighbours strictly, later ones non-strictly
                    if (v >= a.thr && v > nv[0] && v > nv[1] && v > nv[2] && v > nv[3] && v >= nv[5] &&
                        v >= nv[6] && v >= nv[7] && v >= nv[8])
                        emit_peak_c(a.counts, a.peaks, pl, a.cap, v, y, x);
                }
            }
        }
        __syncwarp();
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
    if (a.variant == 1 && a.w <= 32 * kMaxRowWords && a.nbc <= 32 * kMaxRowWords && P < (1ll << 30)) {
        int dev = 0, sms = 0, occ = 0;
        const size_t smem = gw_smem(a.h, a.w);
        cudaError_t e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_up_corner_g, kGwThreads, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        const long long grid = std::min<long long>((P + kGwWarps - 1) / kGwWarps, (long long)occ * sms);
        k_nms_up_corner_g<<<(unsigned)grid, kGwThreads, smem, s>>>(a);
        return cudaGetLastError();
    }
    const bool wk = a.warp_rows && a.w <= 32 * kMaxRowWords && a.nbc <= 32 * kMaxRowWords;
    const size_t smem = wk ? nms_up_corner_w_smem(a.h, a.w, a.nbr, a.nbc, a.nst)
                           : nms_up_corner_smem(a.h, a.w, a.nbr, a.nbc, a.nst);
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = wk ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_up_corner_w, kCornerThreads, smem)
               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_up_corner, kCornerThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    // bulk copies need 16-byte aligned, 16-byte multiple planes
    a.bulk = ((size_t)a.h * a.w * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(a.conf) & 15) == 0;
    const long long grid = std::min<long long>(P, (long long)occ * sms);
    if (wk) k_nms_up_corner_w<<<(unsigned)grid, kCornerThreads, smem, s>>>(a);
    else k_nms_up_corner<<<(unsigned)grid, kCornerThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t configure_corner_kernels(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_nms_up_corner);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_nms_up_corner, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_nms_up_corner_g);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_nms_up_corner_g, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_nms_up_corner_w);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_nms_up_corner_w, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    return e;
}

}  // namespace pf
