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

#if defined(PF_CORNER_PROF) || defined(PF_FIN_PROF)
__device__ unsigned long long g_corner_prof[16];  // cycles per phase [0, 12) (thread 0 of each CTA), planes, hot, survivors, candidates
#endif

constexpr float kNoise = 7.62939453125e-06f;   // 2^-17
#ifndef PF_CORNER_THREADS
#define PF_CORNER_THREADS 128
#endif
constexpr int kCornerThreads = PF_CORNER_THREADS;
constexpr int kCornerCands = 512;    // candidate pixels per plane kept in shared memory
constexpr int kCornerList = 1024;    // hot cells per plane kept in shared memory
constexpr int kCornerSurv = 256;     // chain survivors per plane kept in shared memory
constexpr int kCornerSpill = 4096;   // candidates per CTA beyond the shared list (global slab)


// One CTA owns a plane, so its peak count lives in shared memory (no global
// atomic round trip on the critical path) and is stored once per plane.
__device__ __forceinline__ void emit_peak_c(int *npk, uint2 *peaks, int plane, int cap, float v, int i, int j)
{
    const int slot = atomicAdd(npk, 1);
    if (slot < cap) peaks[(size_t)plane * cap + slot] = pack_peak(v, i, j);
}

// Row or column interpolation parameters of one output coordinate.
struct Ax {
    int i0, i1;
    double t, omt;
    bool in;
};

// one 16-byte load of the packed record (i0 | i1 << 16, t); 1 - t is the
// host table's own single rounded subtraction
__device__ __forceinline__ Ax ax_load(const AxisRec *tab, int o, int n_out)
{
    Ax r;
    r.in = o >= 0 && o < n_out;
    const int oc = min(max(o, 0), n_out - 1);
    const int4 v = __ldg(reinterpret_cast<const int4 *>(tab + oc));
    r.i0 = v.x & 0xffff;
    r.i1 = v.x >> 16;
    r.t = __hiloint2double(v.w, v.z);
    r.omt = __dsub_rn(1.0, r.t);
    return r;
}


// Source accessor of a low-res plane (global or shared memory).
struct PlaneSrc {
    const float *S;
    int w;
    __device__ float operator()(int r, int c) const { return S[r * w + c]; }
};

// Exact upsampled value (operators.py:104-107 op order); -inf off-grid.
template <class Src>
__device__ __forceinline__ float up_val(const Src &S, const Ax &ry, const Ax &cx)
{
    if (!(ry.in && cx.in)) return -INFINITY;
    return bilerp(S(ry.i0, cx.i0), S(ry.i0, cx.i1), S(ry.i1, cx.i0), S(ry.i1, cx.i1), cx.t, cx.omt, ry.t, ry.omt);
}

// The reference predicate (paf.py:87-99) on exactly computed values; each row
// and column parameter is loaded once.
__device__ __noinline__ bool exact_peak(const UpCornerArgs &a, const float *S, int y, int x, float &v)
{
    const Ax ym = ax_load(a.rrec, y - 1, a.H), yc = ax_load(a.rrec, y, a.H), yp = ax_load(a.rrec, y + 1, a.H);
    const Ax xm = ax_load(a.crec, x - 1, a.W), xc = ax_load(a.crec, x, a.W), xp = ax_load(a.crec, x + 1, a.W);
    const PlaneSrc src{S, a.w};
    v = up_val(src, yc, xc);
    if (!(v >= a.thr)) return false;
    // earlier neighbours: strictly greater; later: greater or equal
    if (!(v > up_val(src, ym, xm))) return false;
    if (!(v > up_val(src, ym, xc))) return false;
    if (!(v > up_val(src, ym, xp))) return false;
    if (!(v > up_val(src, yc, xm))) return false;
    if (!(v >= up_val(src, yc, xp))) return false;
    if (!(v >= up_val(src, yp, xm))) return false;
    if (!(v >= up_val(src, yp, xc))) return false;
    return v >= up_val(src, yp, xp);
}

// Horizontal lerps of source row r at three output columns (operators.py:104-105).
template <class Src>
__device__ __forceinline__ void hlerp3(const Src &S, int r, const Ax *xs, double *o)
{
#pragma unroll
    for (int c = 0; c < 3; ++c) o[c] = dadd(dmul(S(r, xs[c].i0), xs[c].omt), dmul(S(r, xs[c].i1), xs[c].t));
}

// The same predicate without early exits: all nine values at once (one
// load round trip).  A horizontal lerp depends only on its source row and
// output column, so the three output rows share them: an output row in the
// same band as the previous one reuses both, one in the next band reuses
// the previous bottom row as its top (canonical bands: i0 = previous i1).
// Every value is the same fp64 expression as up_val.
template <class Src>
__device__ __forceinline__ bool exact_peak_all(const UpCornerArgs &a, const Src &S, int y, int x, float &v)
{
    const Ax ys[3] = {ax_load(a.rrec, y - 1, a.H), ax_load(a.rrec, y, a.H), ax_load(a.rrec, y + 1, a.H)};
    const Ax xs[3] = {ax_load(a.crec, x - 1, a.W), ax_load(a.crec, x, a.W), ax_load(a.crec, x + 1, a.W)};
    float n[9];
    double T[3], B[3];
    hlerp3(S, ys[0].i0, xs, T);
    hlerp3(S, ys[0].i1, xs, B);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        if (r > 0 && !(ys[r].i0 == ys[r - 1].i0 && ys[r].i1 == ys[r - 1].i1)) {
            if (ys[r].i0 == ys[r - 1].i1) {
#pragma unroll
                for (int c = 0; c < 3; ++c) T[c] = B[c];
            } else {
                hlerp3(S, ys[r].i0, xs, T);
            }
            hlerp3(S, ys[r].i1, xs, B);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c)
            n[3 * r + c] = (ys[r].in && xs[c].in)
                               ? __double2float_rn(dadd(dmul(T[c], ys[r].omt), dmul(B[c], ys[r].t)))
                               : -INFINITY;
    }
    v = n[4];
    // paf.py:95-99: earlier neighbours strictly, later ones non-strictly
    return v >= a.thr && v > n[0] && v > n[1] && v > n[2] && v > n[3] && v >= n[5] && v >= n[6] && v >= n[7] &&
           v >= n[8];
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
    uint32_t *spill;     // this CTA's global overflow slab (crowded planes)
    int spill_cap;
    __device__ void operator()(int y, int x) const;   // candidate sink: push_cand
};

__device__ __forceinline__ void push_cand(const CandList &cl, int y, int x)
{
    const int slot = atomicAdd(cl.n, 1);
    const uint32_t yx = (uint32_t(y) << 16) | uint32_t(x);
    if (slot < cl.cap) cl.c[slot] = yx;
    else if (slot < cl.cap + cl.spill_cap) cl.spill[slot - cl.cap] = yx;   // beyond: plane redone (slow path)
}
__device__ __forceinline__ void CandList::operator()(int y, int x) const { push_cand(*this, y, x); }

// Candidate pixels of a partial cell.  Rows restricted to the boundary rows
// when v_ok, columns to the boundary columns when h_ok; further, a row whose
// own slope clears the noise bound is strictly monotone inside the cell, so
// only its rising-end column can be "> left and >= right" (and likewise a
// monotone column keeps only its rising-end row).
template <typename Sink>
__device__ __forceinline__ void partial_cands(const UpCornerArgs &a, const Bands &bd, const Sink &cl,
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
            const double ty = __ldg(&a.rrec[y].t);
            const float d = sl_h(c, (float)__dsub_rn(1.0, ty), (float)ty);
            if (fabsf(d) * cdt > n) only_x = d > 0.f ? cb.y : cb.x;
        }
        for (int k = 0; k < nc; ++k) {
            const int x = (ok & 1u) ? (k ? cb.y : cb.x) : cb.x + k;
            if (only_x >= 0 && x != only_x) continue;
            if (p_in) {
                const double tx = __ldg(&a.crec[x].t);
                const float e = sl_v(c, (float)__dsub_rn(1.0, tx), (float)tx);
                if (fabsf(e) * rdt > n && y != (e > 0.f ? rb.y : rb.x)) continue;
            }
#ifdef PF_FIN_PROF
            atomicAdd(g_corner_prof + 4, 1ull);
#endif
            cl(y, x);
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
__device__ __forceinline__ bool chain_pruned(const float *S, int w, int nbr, int nbc, int p, int q)
{
    // canonical bands: cell (p, q) reads source rows p-1, p and columns q-1, q;
    // border cells (clamped sources) take the exact path
    if (p < 1 || p > nbr - 2 || q < 1 || q > nbc - 2) return false;
    const float *s = S + (p - 1) * w + (q - 1);
    const float a0 = s[0], a1 = s[1], b0 = s[w], b1 = s[w + 1];
    const float m4 = fmaxf(fmaxf(fabsf(a0), fabsf(a1)), fmaxf(fabsf(b0), fabsf(b1)));
    if (!(m4 >= 8.673617379884035e-19f)) return false;   // 2^-60: tiny or NaN -> exact path
    const float d4 = m4 * 1.52587890625e-05f;              // 2^-16 (exact scaling)
    const float ha = a1 - a0, hb = b1 - b0, va = b0 - a0, vb = b1 - a1;
    const bool hR = ha > d4 && hb > d4, hL = ha < -d4 && hb < -d4;
    const bool vD = va > d4 && vb > d4, vU = va < -d4 && vb < -d4;
    // the next cell in the rising direction reads one new source column (row):
    // hR: column q+1 (s[2], s[w+2]); hL: column q-2 (s[-1], s[w-1]);
    // vD: row p+1 (s[2w], s[2w+1]); vU: row p-2 (s[-w], s[-w+1])
    if ((hR && q + 1 <= nbc - 2) || (hL && q - 1 >= 1)) {
        const int o = hR ? 2 : -1;
        const float e = s[o], f = s[w + o];
        const float d = fmaxf(m4, fmaxf(fabsf(e), fabsf(f))) * 1.52587890625e-05f;
        if (hR ? (ha > d && hb > d && e - a1 > d && f - b1 > d)
               : (ha < -d && hb < -d && e - a0 > d && f - b0 > d)) return true;
    }
    if ((vD && p + 1 <= nbr - 2) || (vU && p - 1 >= 1)) {
        const int o = vD ? 2 * w : -w;
        const float e = s[o], f = s[o + 1];
        const float d = fmaxf(m4, fmaxf(fabsf(e), fabsf(f))) * 1.52587890625e-05f;
        if (vD ? (va > d && vb > d && e - b0 > d && f - b1 > d)
               : (va < -d && vb < -d && e - a0 > d && f - a1 > d)) return true;
    }
    return false;
}

// One hot cell: classify; a normal cell pushes its surviving corner, a partial
// cell its candidate pixels.
template <typename Sink>
__device__ __forceinline__ void process_cell(const UpCornerArgs &a, const Bands &bd, const Sink &cl,
                                             const float *S, int plane, int pr, int q)
{
    const int4 rb = bd.rb[pr], cb = bd.cb[q];
    unsigned corners;
    const unsigned ok = classify_cell(bd, S, a.w, a.nbr, a.nbc, pr, q, rb, cb, corners);
#ifdef PF_FIN_PROF
    atomicAdd(g_corner_prof + (ok == 3u ? 1 : 2), 1ull);
    if (ok != 3u) atomicAdd(g_corner_prof + 6 + ok, 1ull);
#endif
    if (ok == 3u) {
        while (corners) {
            const int bit = __ffs(corners) - 1;
            corners &= corners - 1u;
            const int i = bit >> 1, j = bit & 1;
            if (i == 1 && rb.x == rb.y) continue;     // a 1-row band's pixel is visited once
            if (j == 1 && cb.x == cb.y) continue;
            if (!corner_cross_ok(bd, S, a.w, i ? pr - 1 : pr, j ? q - 1 : q, i, j)) continue;
#ifdef PF_FIN_PROF
            atomicAdd(g_corner_prof + 3, 1ull);
#endif
            cl(i ? rb.x : rb.y, j ? cb.x : cb.y);
        }
    } else {
        partial_cands(a, bd, cl, S, plane, pr, q, ok);
    }
}

// Exact value of output pixel (y, x); -inf off the grid (paf.py:87-93 pads).
__device__ __forceinline__ float exact_value(const UpCornerArgs &a, const float *S, int y, int x)
{
    return up_val(PlaneSrc{S, a.w}, ax_load(a.rrec, y, a.H), ax_load(a.crec, x, a.W));
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
    int plane_floats;    // h*w rounded up to 4 (padding = -inf)
    size_t planes, bars, rb, cb, rt, ct, hot, list, cand, surv, total;
};

__host__ __device__ inline CornerLayout corner_layout(int h, int w, int nbr, int nbc, int nst)
{
    CornerLayout L;
    const int hw = h * w;
    L.plane_floats = (hw + 3) & ~3;                   // 16-byte stages for the bulk copies
    size_t o = 0;
    L.planes = o; o += (size_t)nst * L.plane_floats * sizeof(float);
    L.bars = o;   o += (size_t)nst * 8;
    o = (o + 15) & ~(size_t)15;
    L.rb = o;     o += (size_t)nbr * sizeof(int4);
    L.cb = o;     o += (size_t)nbc * sizeof(int4);
    L.rt = o;     o += (size_t)nbr * sizeof(BandT);
    L.ct = o;     o += (size_t)nbc * sizeof(BandT);
    L.hot = o;    o += (size_t)(h + 2) * ((w + 31) >> 5) * sizeof(uint32_t);   // row-aligned hot words
    L.list = o;   o += (size_t)kCornerList * sizeof(uint16_t);
    L.cand = o;   o += (size_t)kCornerCands * sizeof(uint32_t);
    L.surv = o;   o += (size_t)kCornerSurv * sizeof(uint32_t);
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

// Hot cells of band row p, columns [32j, 32j + 32): band p reads source rows
// p-1 and p, cell q source columns q-1 and q, so with M = hot(p-1) | hot(p)
// (row-aligned words; guard rows -1 and h are zero) the cell word is
// M | M << 1 plus bit 31 of the previous word.  Source bits stop at column
// w-1, so cell bits stop at q = w (band count w + 1) by themselves.
__device__ __forceinline__ uint32_t cell_word(const uint32_t *R, int nws, int p, int j, int stride)
{
    const uint32_t *r0 = R + p * stride, *r1 = r0 + stride;   // rows p-1, p (guard-offset by one row)
    const uint32_t m = j < nws ? (r0[j] | r1[j]) : 0u;
    const uint32_t cin = j > 0 ? (r0[j - 1] | r1[j - 1]) >> 31 : 0u;
    return m | (m << 1) | cin;
}

// Slow path for a plane whose hot cells or candidates overflowed the shared
// lists: forget its peaks and exactly test every pixel of every hot cell.
__device__ __noinline__ void redo_plane(const UpCornerArgs &a, const Bands &bd, const float *S,
                                        const uint32_t *R, int plane, int *npk)
{
    if (threadIdx.x == 0) *npk = 0;
    __syncthreads();
    const int nws = (a.w + 31) >> 5, nwc = (a.w + 32) >> 5;
    for (int t = threadIdx.x; t < a.nbr * nwc; t += kCornerThreads) {
        const int p = t / nwc, j = t - p * nwc;
        uint32_t c = cell_word(R, nws, p, j, nws);
        while (c) {
            const int q = (j << 5) + __ffs(c) - 1;
            c &= c - 1u;
            const int4 rb = bd.rb[p], cb = bd.cb[q];
            for (int y = rb.x; y <= rb.y; ++y)
                for (int x = cb.x; x <= cb.y; ++x) {
                    float v;
                    if (exact_peak(a, S, y, x, v)) emit_peak_c(npk, a.peaks, plane, a.cap, v, y, x);
                }
        }
    }
}

#ifndef PF_CORNER_MINB
#define PF_CORNER_MINB 8
#endif
template <int NWS>   // hot words per source row, (w + 31) / 32: fixed so phase A is straight-line code
__global__ void __launch_bounds__(kCornerThreads, PF_CORNER_MINB)
k_nms_up_corner(const __grid_constant__ UpCornerArgs a)
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
    uint16_t *list = reinterpret_cast<uint16_t *>(smc + L.list);   // (p << 8) | q
    uint32_t *cand = reinterpret_cast<uint32_t *>(smc + L.cand);
    uint32_t *surv = reinterpret_cast<uint32_t *>(smc + L.surv);
    __shared__ int n_hot, n_cand, n_surv, n_pk;
    const CandList cl{cand, &n_cand, kCornerCands, a.cand_spill + (size_t)blockIdx.x * kCornerSpill,
                      a.cand_spill ? kCornerSpill : 0};
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
    constexpr int nws = NWS;                         // hot words per source row
    const int nwc = (w + 32) >> 5;                   // cell words per band row (nbc = w + 1)
    const float inv_nwc = 1.0f / (float)nwc;
    for (int e = threadIdx.x; e < nws; e += kCornerThreads) {
        hot[e] = 0u;                                 // guard row -1
        hot[(h + 1) * nws + e] = 0u;                 // guard row h
    }
    if (threadIdx.x == 0) {
        n_hot = 0;
        n_cand = 0;
        n_surv = 0;
        n_pk = 0;
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

#ifdef PF_CORNER_PROF
    unsigned long long acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = clock64(), t1;
#define PROF_MARK(k) do { if (threadIdx.x == 0) { t1 = clock64(); acc[k] += t1 - t0; t0 = t1; } } while (0)
#else
#define PROF_MARK(k) do { } while (0)
#endif
    int it = 0;
    for (long long pl = blockIdx.x; pl < P; pl += gridDim.x, ++it) {
        const int stage = it % nst;
        float *S = planes + stage * L.plane_floats;
        const int plane = (int)pl;
        PROF_MARK(7);
        if (a.bulk) {
            mbar_wait(bars + stage, (uint32_t)(it / nst) & 1u);
            PROF_MARK(10);
        } else {
            const long long b = pl / a.K, k = pl - b * a.K;
            const float *src = a.conf + ((size_t)b * a.C + k) * (size_t)hw;
            for (int e = threadIdx.x; e < hw; e += kCornerThreads) S[e] = __ldg(src + e);
            __syncthreads();
        }

        // ---- (A) row-aligned hot words: warp per source row, lane = column,
        // one ballot per 32 columns (rows offset by the zero guard row)
        for (int r = warp; r < h; r += kCornerThreads / kWarp) {
            const float *row = S + r * w;
            float v[NWS];
#pragma unroll
            for (int j = 0; j < NWS; ++j) {
                const int c = (j << 5) + lane;
                v[j] = (j < NWS - 1 || c < w) ? row[c] : -INFINITY;
            }
            uint32_t mine = 0u;
#pragma unroll
            for (int j = 0; j < NWS; ++j) {
                const uint32_t word = __ballot_sync(0xffffffffu, v[j] >= a.thr);
                if (lane == j) mine = word;
            }
            if (lane < nws) hot[(r + 1) * nws + lane] = mine;
        }
        PROF_MARK(0);
        __syncthreads();
        PROF_MARK(1);

        // ---- (B) hot cells, one (band row, 32 cells) word per task
        for (int t = threadIdx.x; t < nbr * nwc; t += kCornerThreads) {
            const int p = (int)(((float)t + 0.5f) * inv_nwc), j = t - p * nwc;   // exact for t < 2^16
            uint32_t c = cell_word(hot, nws, p, j, nws);
            if (c) {
                int slot = atomicAdd(&n_hot, __popc(c));
                while (c) {
                    const int q = (j << 5) + __ffs(c) - 1;
                    c &= c - 1u;
                    if (slot < kCornerList) list[slot] = uint16_t((p << 8) | q);   // beyond: slow path
                    ++slot;
                }
            }
        }
        PROF_MARK(2);
        __syncthreads();
        PROF_MARK(3);

        // ---- (C1) lane = hot cell (interleaved over the warps): the chain
        // pre-filter on every cell, survivors appended to the CTA survivor
        // list (warp-aggregated), then the survivors are classified spread
        // over all warps (survivor i -> warp i % 4): normal cells push their
        // surviving corner, partial cells their candidate pixels.
        if (n_hot > kCornerList) {
            // crowded plane (the hot list overflowed): no lists, each thread
            // walks the hot cells of its (band row, 32 cells) words itself
            for (int t = threadIdx.x; t < nbr * nwc; t += kCornerThreads) {
                const int p = (int)(((float)t + 0.5f) * inv_nwc), j = t - p * nwc;
                uint32_t c = cell_word(hot, nws, p, j, nws);
                while (c) {
                    const int q = (j << 5) + __ffs(c) - 1;
                    c &= c - 1u;
                    if (!(a.chain && chain_pruned(S, w, nbr, nbc, p, q))) process_cell(a, bd, cl, S, plane, p, q);
                }
            }
        } else {
            const int nh = min(n_hot, kCornerList);
            for (int base = warp * kWarp; base < nh; base += kCornerThreads) {
                const int idx = base + lane;
                uint32_t cell = 0u;
                bool keep = false;
                if (idx < nh) {
                    const uint32_t pq = list[idx];
                    cell = ((pq >> 8) << 16) | (pq & 0xffu);
                    keep = !(a.chain && chain_pruned(S, w, nbr, nbc, int(cell >> 16), int(cell & 0xffffu)));
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (bal) {
                    int at = 0;
                    if (lane == 0) at = atomicAdd(&n_surv, __popc(bal));
                    at = __shfl_sync(0xffffffffu, at, 0);
                    const int slot = at + __popc(bal & ((1u << lane) - 1u));
                    if (keep && slot < kCornerSurv) surv[slot] = cell;          // beyond: slow path
                }
            }
        }
        PROF_MARK(8);
        __syncthreads();
        PROF_MARK(9);
        if (n_hot > kCornerList) {
            // done above
        } else if (n_surv <= kCornerSurv) {
            const int ns = n_surv;
            const int nw = kCornerThreads / kWarp;
            for (int i = warp + nw * lane; i < ns; i += kCornerThreads) {
                const uint32_t cell = surv[i];
                process_cell(a, bd, cl, S, plane, int(cell >> 16), int(cell & 0xffffu));
            }
        } else if (n_surv > kCornerSurv) {
            // the survivor list overflowed: classify every surviving hot cell
            // straight from the hot words (the hot list itself was complete)
            const int nh = n_hot;
            for (int i = threadIdx.x; i < nh; i += kCornerThreads) {
                const uint32_t pq = list[i];
                const int p = int(pq >> 8), q = int(pq & 0xffu);
                if (!(a.chain && chain_pruned(S, w, nbr, nbc, p, q))) process_cell(a, bd, cl, S, plane, p, q);
            }
        }
        PROF_MARK(4);
        __syncthreads();
        PROF_MARK(5);

        // ---- (C2) the exact 3x3 test, 9 lanes per candidate (one pixel each),
        // three candidates per warp, gathered by shuffles
        {
            const int nc = min(n_cand, kCornerCands + cl.spill_cap);
            const int grp = lane / 9, nb = lane - grp * 9;
            const int src = min(grp, 2) * 9;
            for (int base = warp * 3; base < nc; base += 3 * (kCornerThreads / kWarp)) {
                const int ci = base + grp;
                const bool act = grp < 3 && ci < nc;
                int y = 0, x = 0;
                float val = -INFINITY;
                if (act) {
                    const uint32_t yx = ci < kCornerCands ? cand[ci] : __ldcg(cl.spill + (ci - kCornerCands));
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
                        emit_peak_c(&n_pk, a.peaks, plane, a.cap, v, y, x);
                }
            }
        }
        __syncthreads();
        PROF_MARK(6);
#ifdef PF_CORNER_PROF
        if (threadIdx.x == 0) {
            atomicAdd(g_corner_prof + 13, (unsigned long long)n_hot);
            atomicAdd(g_corner_prof + 14, (unsigned long long)n_surv);
            atomicAdd(g_corner_prof + 15, (unsigned long long)n_cand);
        }
#endif
        if (n_cand > kCornerCands + cl.spill_cap) {          // CTA-uniform: the candidate lists overflowed
            redo_plane(a, bd, S, hot, plane, &n_pk);
        }
        __syncthreads();                                     // stage + list free again
        if (threadIdx.x == 0) {
            a.counts[plane] = n_pk;
            n_hot = 0;
            n_cand = 0;
            n_surv = 0;
            n_pk = 0;
            const long long nx = pl + (long long)nst * gridDim.x;
            if (a.bulk && nx < P) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const long long b = nx / a.K, k = nx - b * a.K;
                bulk_load(S, a.conf + ((size_t)b * a.C + k) * (size_t)hw, plane_bytes, bars + stage);
            }
        }
    }
#ifdef PF_CORNER_PROF
    if (threadIdx.x == 0) {
        for (int k = 0; k < 12; ++k) atomicAdd(g_corner_prof + k, acc[k]);
        atomicAdd(g_corner_prof + 12, (unsigned long long)it);
    }
#endif
}

// ---------------------------------------------------------------------------
// k_nms_up_scan — the streaming half of the split path, on its own: no band
// tables, no candidate lists, no classification code, so it needs ~19 KB of
// shared memory and few registers and keeps more planes in flight per SM.
// Per plane: (A) row-aligned hot words, (B) the hot-cell list, (C) the chain
// pre-filter with survivors written straight to HBM (a hot-list overflow
// walks the hot words instead); a plane with more than kCornerSurv survivors
// is marked crowded (surv_n = -2) and k_corner_crowded walks it from the
// sources.
#ifndef PF_SCAN_THREADS
#define PF_SCAN_THREADS 96   // three warps: measured 0.593 vs 0.615 ms (128), 0.630 (64), 0.68-0.81 (160-256)
#endif
constexpr int kScanThreads = PF_SCAN_THREADS;
constexpr int kScanCrowd = 64;       // more survivors than this: k_corner_crowded (CTA per plane)
#ifndef PF_SCAN_MINB
#define PF_SCAN_MINB 10
#endif
#ifndef PF_SCAN_STAGES
#define PF_SCAN_STAGES 1
#endif
#ifndef PF_SCAN_B_FAST
#define PF_SCAN_B_FAST 1   // unguarded hot-list writes when the run fits: scan 0.578 -> 0.545 ms
#endif

struct ScanLayout {
    int plane_floats;
    size_t planes, bars, hot, list, total;
};

__host__ __device__ inline ScanLayout scan_layout(int h, int w, int nst)
{
    ScanLayout L;
    L.plane_floats = (h * w + 3) & ~3;
    size_t o = 0;
    L.planes = o; o += (size_t)nst * L.plane_floats * sizeof(float);
    L.bars = o;   o += (size_t)nst * 8;
    o = (o + 15) & ~(size_t)15;
    L.hot = o;    o += (size_t)(h + 2) * ((((w + 31) >> 5) + 3) & ~3) * sizeof(uint32_t);   // rows padded to 16 B
    L.list = o;   o += (size_t)kCornerList * sizeof(uint16_t);
    L.total = (o + 15) & ~(size_t)15;
    return L;
}

template <int NWS>
__global__ void __launch_bounds__(kScanThreads, PF_SCAN_MINB)
k_nms_up_scan(const UpCornerArgs a)
{
    extern __shared__ __align__(128) unsigned char smc[];
    pdl_trigger();                                       // k_corner_finish may queue behind the persistent grid
    const int h = a.h, w = a.w, hw = h * w;
    const int nbr = a.nbr, nbc = a.nbc, nst = a.nst;
    const ScanLayout L = scan_layout(h, w, nst);
    float *planes = reinterpret_cast<float *>(smc + L.planes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smc + L.bars);
    uint32_t *hot = reinterpret_cast<uint32_t *>(smc + L.hot);
    uint16_t *list = reinterpret_cast<uint16_t *>(smc + L.list);   // (p << 8) | q
    __shared__ int n_hot, n_surv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = a.B * a.K;
    const uint32_t plane_bytes = (uint32_t)hw * 4u;
    constexpr int nws = NWS;
    constexpr int hs = (NWS + 3) & ~3;                   // hot-row stride: one 16-byte store per row
    const int nwc = (w + 32) >> 5;
    const float inv_nwc = 1.0f / (float)nwc;

    for (int e = threadIdx.x; e < hs; e += kScanThreads) {
        hot[e] = 0u;
        hot[(h + 1) * hs + e] = 0u;
    }
    if (threadIdx.x == 0) {
        n_hot = 0;
        n_surv = 0;
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
            if (threadIdx.x == 0) mbar_wait(bars + stage, (uint32_t)(it / nst) & 1u);
            __syncthreads();                               // the others sleep at the barrier
        } else {
            const int b = pl / a.K, k = pl - b * a.K;
            const float *src = a.conf + ((size_t)b * a.C + k) * (size_t)hw;
            for (int e = threadIdx.x; e < hw; e += kScanThreads) S[e] = __ldg(src + e);
            __syncthreads();
        }
        // (A) row-aligned hot words (row and hot-row pointers stepped, not
        // recomputed: this loop is a third of the kernel's instructions)
        {
            constexpr int kRowStep = kScanThreads / kWarp;
            const float *row = S + warp * w + lane;
            uint4 *hr = reinterpret_cast<uint4 *>(hot + (warp + 1) * hs);
            const bool tail = (((NWS - 1) << 5) + lane) < w;      // the last word's column exists
            for (int r = warp; r < h; r += kRowStep, row += kRowStep * w, hr += kRowStep * hs / 4) {
                float v[NWS];
#pragma unroll
                for (int j = 0; j < NWS; ++j) v[j] = (j < NWS - 1 || tail) ? row[j << 5] : -INFINITY;
                uint32_t wd[hs];
#pragma unroll
                for (int j = 0; j < hs; ++j) wd[j] = j < NWS ? __ballot_sync(0xffffffffu, v[j < NWS ? j : 0] >= a.thr) : 0u;
                if (lane == 0) {                          // the row's words in one or two 16-byte stores
#pragma unroll
                    for (int q = 0; q < hs / 4; ++q) hr[q] = make_uint4(wd[4 * q], wd[4 * q + 1], wd[4 * q + 2], wd[4 * q + 3]);
                }
            }
        }
        __syncthreads();
        // (B) hot cells
        for (int t = threadIdx.x; t < nbr * nwc; t += kScanThreads) {
            const int p = (int)(((float)t + 0.5f) * inv_nwc), j = t - p * nwc;   // exact for t < 2^16
            uint32_t c = cell_word(hot, nws, p, j, hs);
            if (c) {
                const int nb = __popc(c);
                int slot = atomicAdd(&n_hot, nb);
                const uint32_t base = (uint32_t(p) << 8) | uint32_t(j << 5);   // (p << 8) | q, q = 32 j + bit
#if PF_SCAN_B_FAST
                if (slot + nb <= kCornerList) {
                    uint16_t *dst = list + slot;
                    while (c) {
                        *dst++ = uint16_t(base + uint32_t(__ffs(c) - 1));
                        c &= c - 1u;
                    }
                } else
#endif
                while (c) {
                    const int q = (j << 5) + __ffs(c) - 1;
                    c &= c - 1u;
                    if (slot < kCornerList) list[slot] = uint16_t((p << 8) | q);
                    ++slot;
                }
            }
        }
        __syncthreads();
        // (C) chain pre-filter; survivors straight to HBM
        const int nh = n_hot;
        uint32_t *sv = a.surv_out + (size_t)pl * kCornerSurv;
        if (nh <= kCornerList) {
            for (int base = warp * kWarp; base < nh; base += kScanThreads) {
                const int idx = base + lane;
                uint32_t cell = 0u;
                bool keep = false;
                if (idx < nh) {
                    const uint32_t pq = list[idx];
                    cell = ((pq >> 8) << 16) | (pq & 0xffu);
                    keep = !(a.chain && chain_pruned(S, w, nbr, nbc, int(cell >> 16), int(cell & 0xffffu)));
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (bal) {
                    int at = 0;
                    if (lane == 0) at = atomicAdd(&n_surv, __popc(bal));
                    at = __shfl_sync(0xffffffffu, at, 0);
                    const int slot = at + __popc(bal & ((1u << lane) - 1u));
                    if (keep && slot < kCornerSurv) sv[slot] = cell;
                }
            }
        } else {
            // the hot list overflowed (crowded plane): each thread walks the
            // hot cells of its (band row, 32 cells) words itself
            for (int t = threadIdx.x; t < nbr * nwc; t += kScanThreads) {
                const int p = (int)(((float)t + 0.5f) * inv_nwc), j = t - p * nwc;
                uint32_t c = cell_word(hot, nws, p, j, hs);
                while (c) {
                    const int q = (j << 5) + __ffs(c) - 1;
                    c &= c - 1u;
                    if (!(a.chain && chain_pruned(S, w, nbr, nbc, p, q))) {
                        const int slot = atomicAdd(&n_surv, 1);
                        if (slot < kCornerSurv) sv[slot] = (uint32_t(p) << 16) | uint32_t(q);
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (n_surv > kScanCrowd) {                           // crowded: a whole CTA finishes it
                a.surv_n[pl] = int(0x80000000u | uint32_t(min(n_surv, 0x3fffffff)));   // < 0 for k_corner_finish
                a.crowd_list[atomicAdd(a.crowd_n, 1)] = pl;
            } else {
                a.surv_n[pl] = n_surv;
            }
            n_hot = 0;
            n_surv = 0;
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

size_t nms_up_scan_smem(int h, int w, int nst)
{
    return scan_layout(h, w, nst).total;
}

size_t nms_up_scan_launch_smem(int h, int w)
{
    return nms_up_scan_smem(h, w, PF_SCAN_STAGES);   // what launch_nms_up_scan requests
}

cudaError_t launch_nms_up_scan(const UpCornerArgs &a_in, cudaStream_t s)
{
    UpCornerArgs a = a_in;
    const long long P = (long long)a.B * a.K;
    if (P == 0) return cudaSuccess;
    a.nst = PF_SCAN_STAGES;
    const size_t smem = nms_up_scan_smem(a.h, a.w, a.nst);
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_up_scan<3>, kScanThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    a.bulk = ((size_t)a.h * a.w * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(a.conf) & 15) == 0;
    const long long grid = std::min<long long>(P, (long long)occ * sms);
    switch ((a.w + 31) >> 5) {
    case 1: k_nms_up_scan<1><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    case 2: k_nms_up_scan<2><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    case 3: k_nms_up_scan<3><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    case 4: k_nms_up_scan<4><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    case 5: k_nms_up_scan<5><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    case 6: k_nms_up_scan<6><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    case 7: k_nms_up_scan<7><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    default: k_nms_up_scan<8><<<(unsigned)grid, kScanThreads, smem, s>>>(a); break;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_corner_finish — second half of the split corner path.  k_nms_up_corner
// (split mode) keeps only the streaming part — hot words, hot cells, chain
// pre-filter — and hands each plane's chain survivors (≈15) over; here one
// warp per plane classifies them (process_cell, lane per survivor) and runs
// the exact 3x3 test lane per candidate (exact_peak_all: all nine values
// gathered at once).  Sources are read through L1/L2 — no plane buffer — so
// many warps stay resident to hide the gathers.  Persistent CTAs fill the
// band tables once.  Same functions as the one-kernel path: same results; a
// candidate overflow falls back to the exact test of every pixel of every
// survivor cell.
constexpr int kFinThreads = 256;
#ifndef PF_FIN_GROUP
#define PF_FIN_GROUP 32
#endif
constexpr int kFinGroup = PF_FIN_GROUP;              // lanes per plane (16: two planes per warp)
constexpr int kFinGroups = kFinThreads / kFinGroup;  // planes in flight per CTA
#ifndef PF_FIN_CANDS
#define PF_FIN_CANDS 192
#endif
constexpr int kFinCands = PF_FIN_CANDS;              // candidates per plane in shared memory

__device__ __noinline__ void classify_inline(const UpCornerArgs &a, const Bands &bd, const float *S, int plane,
                                            int *npk, int p, int q);

// Candidate sink that runs the exact test on the spot (candidate-list overflows).
struct InlineSink {
    const UpCornerArgs *a;
    const float *S;
    int plane;
    int *npk;
    __device__ void operator()(int y, int x) const
    {
        float v;
        if (exact_peak_all(*a, PlaneSrc{S, a->w}, y, x, v)) emit_peak_c(npk, a->peaks, plane, a->cap, v, y, x);
    }
};

// process_cell with the on-the-spot sink, kept out of line so the common
// path's register allocation does not pay for it
__device__ __noinline__ void classify_inline(const UpCornerArgs &a, const Bands &bd, const float *S, int plane,
                                            int *npk, int p, int q)
{
    const InlineSink sink{&a, S, plane, npk};
    process_cell(a, bd, sink, S, plane, p, q);
}


#ifndef PF_FIN_MINB
#define PF_FIN_MINB 4
#endif
#ifndef PF_FIN_REVERSE
#define PF_FIN_REVERSE 1
#endif
#ifndef PF_EXACT_MINB
#define PF_EXACT_MINB 4
#endif

// The exact tests of one plane's candidate list in the finish itself (the
// k_corner_exact list was full), out of line so they do not set the finish's
// register count.
__device__ __noinline__ void exact_tests_here(const UpCornerArgs &a, const float *S, const uint32_t *wc, int ncd,
                                              int gl, int plane, int *npk)
{
    for (int ci = gl; ci < ncd; ci += kFinGroup) {
        const uint32_t yx = wc[ci];
        const int y = (int)(yx >> 16), x = (int)(yx & 0xffffu);
        float v;
        if (exact_peak_all(a, PlaneSrc{S, a.w}, y, x, v)) emit_peak_c(npk, a.peaks, plane, a.cap, v, y, x);
    }
}
__global__ void __launch_bounds__(kFinThreads, PF_FIN_MINB)
k_corner_finish(const __grid_constant__ UpCornerArgs a)
{
    extern __shared__ __align__(16) unsigned char smf[];
    const int nbr = a.nbr, nbc = a.nbc;
    int4 *RB = reinterpret_cast<int4 *>(smf);
    int4 *CB = RB + nbr;
    BandT *RT = reinterpret_cast<BandT *>(CB + nbc);
    BandT *CT = RT + nbr;
    uint32_t *candw = reinterpret_cast<uint32_t *>(CT + nbc);
    __shared__ int n_cand[kFinGroups], n_pk[kFinGroups];
    for (int b = threadIdx.x; b < nbr + nbc; b += kFinThreads) {
        if (b < nbr) fill_band(a.rows, a.rdt, a.rband, b, RB[b], RT[b]);
        else fill_band(a.cols, a.cdt, a.cband, b - nbr, CB[b - nbr], CT[b - nbr]);
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();                                          // the scan's survivors
    const int grp = threadIdx.x / kFinGroup, gl = threadIdx.x % kFinGroup;
    const unsigned gmask = kFinGroup == kWarp ? 0xffffffffu
                                              : ((1u << kFinGroup) - 1u) << ((threadIdx.x & 31) & ~(kFinGroup - 1));
    const Bands bd{RB, CB, RT, CT};
    uint32_t *wc = candw + grp * kFinCands;
    const CandList cl{wc, &n_cand[grp], kFinCands, nullptr, 0};
    const int P = a.B * a.K;
    // (frame, part) of the plane stepped alongside it: no division per plane
    const int p0 = blockIdx.x * kFinGroups + grp, pstep = gridDim.x * kFinGroups;
    const int fstep = pstep / a.K, kstep = pstep - fstep * a.K;
#if PF_FIN_REVERSE
    // planes from the end: the scan streamed them last, so the first ones
    // still have their sources in L2
    int fb = (P - 1 - p0) / a.K, k = (P - 1 - p0) - fb * a.K;
    for (int plane = P - 1 - p0; plane >= 0; plane -= pstep, fb -= fstep, k -= kstep, fb -= k < 0, k += k < 0 ? a.K : 0) {
#else
    int fb = p0 / a.K, k = p0 - fb * a.K;
    for (int plane = p0; plane < P; plane += pstep, fb += fstep, k += kstep, fb += k >= a.K, k -= k >= a.K ? a.K : 0) {
#endif
        const int ns = __ldcg(a.surv_n + plane);
        if (ns < 0) continue;   // -1: k_nms_up_corner finished it; -2: crowded (k_corner_crowded); group-uniform
#ifdef PF_FIN_PROF
        if (gl == 0) { atomicAdd(g_corner_prof + 12, 1ull); atomicAdd(g_corner_prof + 0, (unsigned long long)ns); }
#endif
        if (gl == 0) { n_cand[grp] = 0; n_pk[grp] = 0; }
        __syncwarp(gmask);
        const float *S = a.conf + ((size_t)fb * a.C + k) * (size_t)a.h * a.w;
        const uint32_t *sv = a.surv_out + (size_t)plane * kCornerSurv;
        for (int i = gl; i < ns; i += kFinGroup) {
            const uint32_t cell = __ldcg(sv + i);
            process_cell(a, bd, cl, S, plane, int(cell >> 16), int(cell & 0xffffu));
        }
        __syncwarp(gmask);
        const int ncd = n_cand[grp];
        bool handed = false;
        if (ncd > 0 && ncd <= kFinCands && a.exact_list) {
            // the exact tests run in k_corner_exact, a thread per candidate of
            // the whole batch (here ≈15 candidates would fill half the lanes);
            // a plane's candidates stay contiguous, so its sources stay in L1
            int base = 0;
            if (gl == 0) base = atomicAdd(a.exact_n, ncd);
            base = __shfl_sync(gmask, base, 0, kFinGroup);   // the group's first lane
            handed = base + ncd <= a.exact_cap;
            for (int ci = gl; ci < ncd; ci += kFinGroup)
                if (base + ci < a.exact_cap) a.exact_list[base + ci] = make_uint2(handed ? uint32_t(plane) : 0xffffffffu, wc[ci]);
        }
        if (handed) {
            // counts[plane] stays 0 here; k_corner_exact adds the peaks
        } else if (ncd <= kFinCands) {
            if (a.exact_list) {
                exact_tests_here(a, S, wc, ncd, gl, plane, &n_pk[grp]);   // the list was full (rare)
            } else {
                for (int ci = gl; ci < ncd; ci += kFinGroup) {
                    const uint32_t yx = wc[ci];
                    const int y = (int)(yx >> 16), x = (int)(yx & 0xffffu);
                    float v;
                    if (exact_peak_all(a, PlaneSrc{S, a.w}, y, x, v)) emit_peak_c(&n_pk[grp], a.peaks, plane, a.cap, v, y, x);
                }
            }
        } else {
            // candidate overflow: classify again and test each candidate on
            // the spot (nothing was emitted yet)
            for (int i = gl; i < ns; i += kFinGroup) {
                const uint32_t cell = __ldcg(sv + i);
                classify_inline(a, bd, S, plane, &n_pk[grp], int(cell >> 16), int(cell & 0xffffu));
            }
        }
        __syncwarp(gmask);
        if (gl == 0) a.counts[plane] = n_pk[grp];
        __syncwarp(gmask);
    }
}

// Exact 3x3 tests of the candidates k_corner_finish handed over (thread per
// candidate, grid-stride over the batch's list); peaks are appended to the
// plane's slab with a global counter (k_parse_peaks sorts them).  Entries
// marked 0xffffffff belong to a plane whose range overflowed the list (that
// plane was tested in k_corner_finish).
constexpr int kExactPerPlane = 32;
size_t corner_exact_entries_per_plane() { return kExactPerPlane; }

__global__ void __launch_bounds__(kFinThreads, PF_EXACT_MINB)
k_corner_exact(const __grid_constant__ UpCornerArgs a)
{
    const int n = min(*a.exact_n, a.exact_cap);
    const size_t hw = (size_t)a.h * a.w;
    for (int i = blockIdx.x * kFinThreads + threadIdx.x; i < n; i += gridDim.x * kFinThreads) {
        // newest entries first: the planes the finish classified last are the
        // likeliest to still have their sources in L2 (0.260 -> 0.255 ms)
        const uint2 e = a.exact_list[n - 1 - i];
        if (e.x == 0xffffffffu) continue;
        const int plane = (int)e.x, fb = plane / a.K, k = plane - fb * a.K;
        const float *S = a.conf + ((size_t)fb * a.C + k) * hw;
        const int y = (int)(e.y >> 16), x = (int)(e.y & 0xffffu);
        float v;
        if (exact_peak_all(a, PlaneSrc{S, a.w}, y, x, v)) emit_peak_c(a.counts + plane, a.peaks, plane, a.cap, v, y, x);
    }
}

cudaError_t launch_corner_exact(const UpCornerArgs &a, cudaStream_t s)
{
    if (!a.exact_list || (long long)a.B * a.K == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    k_corner_exact<<<sms * PF_EXACT_MINB, kFinThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// Crowded planes of the split path (more than kScanCrowd survivors): the
// scan appends them to a compact list; here a whole CTA takes one such plane
// and redoes it from a shared-memory copy of the plane (when it fits):
//   1. hot words (ballots) and the hot-cell list;
//   2. thread per hot cell: chain pre-filter, classification; a normal cell
//      pushes its surviving corners (exact test from the list, or on the spot
//      when the list is full), a partial cell goes to the dense list;
//   3. candidates: the exact 3x3 test, thread per candidate;
//   4. dense cells, warp per cell: the exact values of the cell and its
//      one-pixel ring are computed once into a per-warp buffer and EVERY
//      pixel of the cell is tested from it (a superset of partial_cands'
//      candidates; an exact test never passes a non-peak and each pixel
//      belongs to one cell, so the peaks are the same, without duplicates).
// Crowded scenes make most hot cells non-monotone ("partial"), where testing
// pixel by pixel would cost nine interpolations per pixel.
constexpr int kCrowdCands = 2048;
constexpr int kCrowdList = 4096;     // hot cells per plane in shared memory
constexpr int kCrowdDense = 1024;    // partial cells per plane in shared memory
constexpr int kCrowdWarps = kFinThreads / kWarp;

struct CrowdLayout {
    size_t rb, cb, rt, ct, plane, hot, list, cand, dense, vbuf, total;
    int vcap;            // floats per warp buffer
    bool staged;         // the plane is copied into shared memory
};

__host__ __device__ inline CrowdLayout crowd_layout(int h, int w, int nbr, int nbc, int max_band, size_t budget)
{
    CrowdLayout L;
    L.vcap = (max_band + 2) * (max_band + 2);
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o = (o + bytes + 15) & ~(size_t)15; return at; };
    L.rb = take((size_t)nbr * sizeof(int4));
    L.cb = take((size_t)nbc * sizeof(int4));
    L.rt = take((size_t)nbr * sizeof(BandT));
    L.ct = take((size_t)nbc * sizeof(BandT));
    L.hot = take((size_t)(h + 2) * ((w + 31) >> 5) * sizeof(uint32_t));
    L.list = take((size_t)kCrowdList * sizeof(uint32_t));
    L.cand = take((size_t)kCrowdCands * sizeof(uint32_t));
    L.dense = take((size_t)kCrowdDense * sizeof(uint32_t));
    L.vbuf = take((size_t)kCrowdWarps * L.vcap * sizeof(float));
    L.plane = o;
    L.staged = o + (size_t)h * w * sizeof(float) + 16 <= budget;
    if (L.staged) take((size_t)h * w * sizeof(float));
    L.total = o;
    return L;
}

// Candidate sink of the crowded kernel: the shared list, or the exact test
// on the spot once it is full.
struct CrowdSink {
    const UpCornerArgs *a;
    const float *S;
    uint32_t *c;
    int *n;
    int *npk;
    int plane;
    __device__ void operator()(int y, int x) const
    {
        const int slot = atomicAdd(n, 1);
        if (slot < kCrowdCands) {
            c[slot] = (uint32_t(y) << 16) | uint32_t(x);
        } else {
            float v;
            if (exact_peak_all(*a, PlaneSrc{S, a->w}, y, x, v)) emit_peak_c(npk, a->peaks, plane, a->cap, v, y, x);
        }
    }
};

#ifndef PF_CROWD_MINB
#define PF_CROWD_MINB 4   // 64 registers (128 B spill): C3 Mode U 0.507 -> 0.494 ms vs 3; 2: 0.639
#endif
__global__ void __launch_bounds__(kFinThreads, PF_CROWD_MINB)
k_corner_crowded(const __grid_constant__ UpCornerArgs a, const CrowdLayout L)
{
    extern __shared__ __align__(16) unsigned char smf[];
    const int nbr = a.nbr, nbc = a.nbc, h = a.h, w = a.w, hw = h * w;
    int4 *RB = reinterpret_cast<int4 *>(smf + L.rb);
    int4 *CB = reinterpret_cast<int4 *>(smf + L.cb);
    BandT *RT = reinterpret_cast<BandT *>(smf + L.rt);
    BandT *CT = reinterpret_cast<BandT *>(smf + L.ct);
    uint32_t *hot = reinterpret_cast<uint32_t *>(smf + L.hot);
    uint32_t *list = reinterpret_cast<uint32_t *>(smf + L.list);
    uint32_t *cand = reinterpret_cast<uint32_t *>(smf + L.cand);
    uint32_t *dense = reinterpret_cast<uint32_t *>(smf + L.dense);
    float *vbuf = reinterpret_cast<float *>(smf + L.vbuf);
    float *Sp = reinterpret_cast<float *>(smf + L.plane);
    __shared__ int n_hot, n_cand, n_dense, n_pk;
    pdl_trigger();
    pdl_wait();                                          // the crowd list and the finished planes' counts
    const int nlist = min(*a.crowd_n, a.B * a.K);
    if ((int)blockIdx.x >= nlist) return;                 // the usual case: nothing crowded
    for (int b = threadIdx.x; b < nbr + nbc; b += kFinThreads) {
        if (b < nbr) fill_band(a.rows, a.rdt, a.rband, b, RB[b], RT[b]);
        else fill_band(a.cols, a.cdt, a.cband, b - nbr, CB[b - nbr], CT[b - nbr]);
    }
    const Bands bd{RB, CB, RT, CT};
    const int nws = (w + 31) >> 5, nwc = (w + 32) >> 5;
    const float inv_nwc = 1.0f / (float)nwc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < nws; e += kFinThreads) {
        hot[e] = 0u;                                     // guard rows -1 and h
        hot[(h + 1) * nws + e] = 0u;
    }
    float *vb = vbuf + warp * L.vcap;
    // planes handed out dynamically (crowded planes differ widely in cost):
    // the first by CTA index, the rest from a counter (crowd_n[1])
    __shared__ int s_next;
    for (int li = blockIdx.x; li < nlist;) {
        const int plane = __ldcg(a.crowd_list + li);
        if (threadIdx.x == 0) { n_hot = 0; n_cand = 0; n_dense = 0; n_pk = 0; }
        const int fb = plane / a.K, k = plane - fb * a.K;
        const float *G = a.conf + ((size_t)fb * a.C + k) * (size_t)hw;
        const float *S = G;
        if (L.staged) {
            for (int e = threadIdx.x; e < hw; e += kFinThreads) Sp[e] = __ldg(G + e);
            S = Sp;
        }
        __syncthreads();
        // 1. hot words (warp per source row, one ballot per 32 columns), hot cells
        for (int r = warp; r < h; r += kCrowdWarps) {
            for (int j = 0; j < nws; ++j) {
                const int c = (j << 5) + lane;
                const uint32_t word = __ballot_sync(0xffffffffu, c < w && S[r * w + c] >= a.thr);
                if (lane == 0) hot[(r + 1) * nws + j] = word;
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nbr * nwc; t += kFinThreads) {
            const int p = (int)(((float)t + 0.5f) * inv_nwc), j = t - p * nwc;   // exact for t < 2^16
            uint32_t c = cell_word(hot, nws, p, j, nws);
            if (c) {
                int slot = atomicAdd(&n_hot, __popc(c));
                while (c) {
                    const int q = (j << 5) + __ffs(c) - 1;
                    c &= c - 1u;
                    if (slot < kCrowdList) list[slot] = (uint32_t(p) << 16) | uint32_t(q);
                    ++slot;
                }
            }
        }
        __syncthreads();
        // 2. thread per hot cell: prune, classify, corners -> candidates,
        // partial cells -> dense list
        const CrowdSink sink{&a, S, cand, &n_cand, &n_pk, plane};
        auto cell_work = [&](int p, int q) {
            if (a.chain && chain_pruned(S, w, nbr, nbc, p, q)) return;
            const int4 rb = bd.rb[p], cb = bd.cb[q];
            unsigned corners;
            const unsigned ok = classify_cell(bd, S, w, nbr, nbc, p, q, rb, cb, corners);
            if (ok == 3u) {
                while (corners) {
                    const int bit = __ffs(corners) - 1;
                    corners &= corners - 1u;
                    const int i = bit >> 1, j = bit & 1;
                    if (i == 1 && rb.x == rb.y) continue;
                    if (j == 1 && cb.x == cb.y) continue;
                    if (!corner_cross_ok(bd, S, w, i ? p - 1 : p, j ? q - 1 : q, i, j)) continue;
                    sink(i ? rb.x : rb.y, j ? cb.x : cb.y);
                }
            } else if ((rb.y - rb.x + 3) * (cb.y - cb.x + 3) <= L.vcap) {
                const int slot = atomicAdd(&n_dense, 1);
                if (slot < kCrowdDense) dense[slot] = (uint32_t(p) << 16) | uint32_t(q);
                else partial_cands(a, bd, sink, S, plane, p, q, ok);
            } else {
                partial_cands(a, bd, sink, S, plane, p, q, ok);
            }
        };
        const int nh = n_hot;
        if (nh <= kCrowdList) {
            for (int i = threadIdx.x; i < nh; i += kFinThreads) {
                const uint32_t pq = list[i];
                cell_work(int(pq >> 16), int(pq & 0xffffu));
            }
        } else {
            for (int t = threadIdx.x; t < nbr * nwc; t += kFinThreads) {
                const int p = (int)(((float)t + 0.5f) * inv_nwc), j = t - p * nwc;
                uint32_t c = cell_word(hot, nws, p, j, nws);
                while (c) {
                    const int q = (j << 5) + __ffs(c) - 1;
                    c &= c - 1u;
                    cell_work(p, q);
                }
            }
        }
        __syncthreads();
        // 3. candidates of normal cells
        const int nc = min(n_cand, kCrowdCands);
        for (int ci = threadIdx.x; ci < nc; ci += kFinThreads) {
            const uint32_t yx = cand[ci];
            const int y = (int)(yx >> 16), x = (int)(yx & 0xffffu);
            float v;
            if (exact_peak_all(a, PlaneSrc{S, a.w}, y, x, v)) emit_peak_c(&n_pk, a.peaks, plane, a.cap, v, y, x);
        }
        // 4. dense cells, warp per cell
        const int nd = min(n_dense, kCrowdDense);
        for (int di = warp; di < nd; di += kCrowdWarps) {
            const uint32_t pq = dense[di];
            const int4 rb = bd.rb[int(pq >> 16)], cb = bd.cb[int(pq & 0xffffu)];
            const int y0 = rb.x - 1, x0 = cb.x - 1;
            const int bh = rb.y - rb.x + 3, bw = cb.y - cb.x + 3;
            // row of e by a float reciprocal, exact for e < 2^16 (no integer division per pixel)
            const float inv_bw = __frcp_rn((float)bw), inv_cw = __frcp_rn((float)(bw - 2));   // = 1.0f / n
            for (int e = lane; e < bh * bw; e += kWarp) {
                const int yy = (int)(((float)e + 0.5f) * inv_bw), xx = e - yy * bw;
                vb[e] = exact_value(a, S, y0 + yy, x0 + xx);          // -inf off the grid
            }
            __syncwarp();
            const int ch = bh - 2, cw = bw - 2;
            for (int e = lane; e < ch * cw; e += kWarp) {
                const int yy = (int)(((float)e + 0.5f) * inv_cw) + 1, xx = e - (yy - 1) * cw + 1;
                const float *c = vb + yy * bw + xx;
                const float v = c[0];
                // paf.py:95-99: earlier neighbours strictly, later ones non-strictly
                if (v >= a.thr && v > c[-bw - 1] && v > c[-bw] && v > c[-bw + 1] && v > c[-1] && v >= c[1] &&
                    v >= c[bw - 1] && v >= c[bw] && v >= c[bw + 1])
                    emit_peak_c(&n_pk, a.peaks, plane, a.cap, v, y0 + yy, x0 + xx);
            }
            __syncwarp();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            a.counts[plane] = n_pk;
            s_next = (int)gridDim.x + atomicAdd(a.crowd_n + 1, 1);
        }
        __syncthreads();
        li = s_next;
    }
}

cudaError_t launch_corner_finish(const UpCornerArgs &a, cudaStream_t s)
{
    const long long P = (long long)a.B * a.K;
    if (P == 0) return cudaSuccess;
    const size_t smem = (size_t)(a.nbr + a.nbc) * (sizeof(int4) + sizeof(BandT)) +
                        (size_t)kFinGroups * kFinCands * sizeof(uint32_t);
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_corner_finish, kFinThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const long long need = (P * (kCornerSurv / kFinGroup) + kFinGroups - 1) / kFinGroups;
    e = launch_pdl(kPdlFinish, k_corner_finish, dim3((unsigned)std::min<long long>(need, (long long)occ * sms)), dim3(kFinThreads),
                   smem, s, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_corner_crowded(const UpCornerArgs &a, cudaStream_t s)
{
    const long long P = (long long)a.B * a.K;
    if (P == 0) return cudaSuccess;
    int dev = 0, sms = 0, max_smem = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    // stage the plane when PF_CROWD_MINB CTAs per SM still fit, else read it through L1
    const size_t per_cta = (size_t)(228 * 1024) / PF_CROWD_MINB - 1024 - 256;
    const CrowdLayout L = crowd_layout(a.h, a.w, a.nbr, a.nbc, a.max_band,
                                       std::min(per_cta, (size_t)max_smem - 256));
    e = launch_pdl(kPdlCrowded, k_corner_crowded, dim3((unsigned)std::min<long long>(P, (long long)sms * PF_CROWD_MINB)),
                   dim3(kFinThreads), L.total, s, a, L);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

size_t corner_surv_entries_per_plane() { return kCornerSurv; }

size_t nms_up_corner_spill_entries(int max_ctas)
{
    return (size_t)max_ctas * kCornerSpill;
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
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_up_corner<3>, kCornerThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    // bulk copies need 16-byte aligned, 16-byte multiple planes
    a.bulk = ((size_t)a.h * a.w * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(a.conf) & 15) == 0;
    const long long grid = std::min<long long>(P, (long long)occ * sms);
    switch ((a.w + 31) >> 5) {
    case 1: k_nms_up_corner<1><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    case 2: k_nms_up_corner<2><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    case 3: k_nms_up_corner<3><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    case 4: k_nms_up_corner<4><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    case 5: k_nms_up_corner<5><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    case 6: k_nms_up_corner<6><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    case 7: k_nms_up_corner<7><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    default: k_nms_up_corner<8><<<(unsigned)grid, kCornerThreads, smem, s>>>(a); break;
    }
    return cudaGetLastError();
}

template <int NWS>
static cudaError_t configure_corner(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_nms_up_corner<NWS>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_nms_up_corner<NWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    return e;
}

template <int NWS>
static cudaError_t configure_scan(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_nms_up_scan<NWS>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_nms_up_scan<NWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    return e;
}

cudaError_t configure_corner_kernels(int max_smem)
{
    cudaError_t e = configure_corner<1>(max_smem);
    if (e == cudaSuccess) e = configure_corner<2>(max_smem);
    if (e == cudaSuccess) e = configure_corner<3>(max_smem);
    if (e == cudaSuccess) e = configure_corner<4>(max_smem);
    if (e == cudaSuccess) e = configure_corner<5>(max_smem);
    if (e == cudaSuccess) e = configure_corner<6>(max_smem);
    if (e == cudaSuccess) e = configure_corner<7>(max_smem);
    if (e == cudaSuccess) e = configure_corner<8>(max_smem);
    if (e == cudaSuccess) e = configure_scan<1>(max_smem);
    if (e == cudaSuccess) e = configure_scan<2>(max_smem);
    if (e == cudaSuccess) e = configure_scan<3>(max_smem);
    if (e == cudaSuccess) e = configure_scan<4>(max_smem);
    if (e == cudaSuccess) e = configure_scan<5>(max_smem);
    if (e == cudaSuccess) e = configure_scan<6>(max_smem);
    if (e == cudaSuccess) e = configure_scan<7>(max_smem);
    if (e == cudaSuccess) e = configure_scan<8>(max_smem);
    if (e == cudaSuccess) {
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, k_corner_crowded);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_corner_crowded, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     max_smem - (int)fa.sharedSizeBytes);
    }
    if (e == cudaSuccess) {
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, k_corner_finish);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_corner_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     max_smem - (int)fa.sharedSizeBytes);
    }
    return e;
}

}  // namespace pf

#if defined(PF_CORNER_PROF) || defined(PF_FIN_PROF)
// development builds only: read (and reset) the per-phase cycle counters
extern "C" int pf_corner_prof_read(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, pf::g_corner_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 4;
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(pf::g_corner_prof, z, sizeof(z));
    }
    return 0;
}
#endif
