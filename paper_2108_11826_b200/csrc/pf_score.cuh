// pf_score.cuh — the limb line integral (score_limb, paf.py:112-146) and
// CPython's float sum, shared by the parse kernels (pf_parse.cu) and the
// large-frame parse (pf_large.cu).
#pragma once

#include "pf_launch.h"

namespace pf {

constexpr int kParseTTab = 64;     // sample positions kept in shared memory

// PAF value pair at parse-grid cell (ci, cj): the feature grid itself
// (up == 1), or the x`up` bilinear value of operators.py:102-107 re-derived
// from the low-res PAF with one packed axis record per axis.  Loads (fetch)
// and arithmetic (finish) are separate steps; software-pipelining the next
// sample's loads was measured slower (registers -> residency).
struct SampleRaw {
    float x00, x01, x10, x11, y00, y01, y10, y11;
    double tx, ty;
};

__device__ __forceinline__ void fetch_sample(const ParseArgs &a, const float *__restrict__ chx,
                                             const float *__restrict__ chy, int ci, int cj, SampleRaw &r)
{
    if (a.up == 1) {
        const size_t o = (size_t)ci * a.w + cj;
        r.x00 = __ldg(chx + o);
        r.y00 = __ldg(chy + o);
        return;
    }
    const int4 ry = __ldg(reinterpret_cast<const int4 *>(a.rrec + ci));
    const int4 rx = __ldg(reinterpret_cast<const int4 *>(a.crec + cj));
    const int i0 = ry.x & 0xffff, i1 = ry.x >> 16, j0 = rx.x & 0xffff, j1 = rx.x >> 16;
    r.ty = __hiloint2double(ry.w, ry.z);
    r.tx = __hiloint2double(rx.w, rx.z);
    const size_t o00 = (size_t)i0 * a.w + j0, o01 = (size_t)i0 * a.w + j1;
    const size_t o10 = (size_t)i1 * a.w + j0, o11 = (size_t)i1 * a.w + j1;
    r.x00 = __ldg(chx + o00); r.x01 = __ldg(chx + o01); r.x10 = __ldg(chx + o10); r.x11 = __ldg(chx + o11);
    r.y00 = __ldg(chy + o00); r.y01 = __ldg(chy + o01); r.y10 = __ldg(chy + o10); r.y11 = __ldg(chy + o11);
}

// dot of the sampled PAF vector with the unit limb direction (paf.py:142-143)
__device__ __forceinline__ double finish_sample(const ParseArgs &a, const SampleRaw &r, double vx, double vy)
{
    double px, py;
    if (a.up == 1) {
        px = (double)r.x00;
        py = (double)r.y00;
    } else {
        const double omty = __dsub_rn(1.0, r.ty), omtx = __dsub_rn(1.0, r.tx);
        px = (double)bilerp(r.x00, r.x01, r.x10, r.x11, r.tx, omtx, r.ty, omty);
        py = (double)bilerp(r.y00, r.y01, r.y10, r.y11, r.tx, omtx, r.ty, omty);
    }
    return dadd(dmul(px, vx), dmul(py, vy));
}

// score_limb + gate of one (limb, a, b) pair (paf.py:131-165): the samples in
// order, so the fp64 running total is the reference's `total += d`; the pair
// is left as soon as it can no longer pass (more failing samples than
// max_fail = n - good_need).  True if gated (good >= good_min, score > 0).
// COUNT: also mark, in this frame's bitmap (a.paf_touch), every 32-byte
// sector of the PAF the sample reads — the instrumented pass that measures
// the bytes an in-place (zero-copy) PAF moves over PCIe.
__device__ __forceinline__ void touch_sector(uint32_t *bm, const float *base, const float *p)
{
    const size_t sec = (size_t)(p - base) >> 3;                  // 8 floats per 32-byte sector
    atomicOr(bm + (sec >> 5), 1u << (sec & 31));
}

template <bool COUNT = false>
__device__ __forceinline__ bool score_pair(const ParseArgs &a, const float *__restrict__ paf_f, int l, uint32_t ca,
                                           uint32_t cbp, const double *t_tab, int max_fail, double &score, int &ngood,
                                           uint32_t *touch = nullptr)
{
    const int n = a.n_samples;
    const int ai = int(ca >> 16), aj = int(ca & 0xffff);
    const int di = int(cbp >> 16) - ai, dj = int(cbp & 0xffff) - aj;
    if ((di | dj) == 0) return false;                     // coincident cells score (0, 0): never gated
    const double norm = __dsqrt_rn((double)((long long)di * di + (long long)dj * dj));   // exact (Python ints)
    const double vx = __ddiv_rn((double)dj, norm);
    const double vy = __ddiv_rn((double)di, norm);
    const float *chx = paf_f + (size_t)a.topo.cx[l] * a.h * a.w;
    const float *chy = paf_f + (size_t)a.topo.cy[l] * a.h * a.w;
    const double den = (double)(n - 1);
    double total = 0.0;
    int nfail = 0;
    ngood = 0;
    for (int u = 0; u < n; ++u) {
        // nearest cell of sample u (paf.py:139-141)
        const double t = u < kParseTTab ? t_tab[u] : __ddiv_rn((double)u, den);
        const int ci = (int)floor(dadd(dadd((double)ai, dmul(t, (double)di)), 0.5));
        const int cj = (int)floor(dadd(dadd((double)aj, dmul(t, (double)dj)), 0.5));
        SampleRaw r;
        fetch_sample(a, chx, chy, ci, cj, r);
        if (COUNT) {
            if (a.up == 1) {
                touch_sector(touch, paf_f, chx + (size_t)ci * a.w + cj);
                touch_sector(touch, paf_f, chy + (size_t)ci * a.w + cj);
            } else {
                const int4 ry = __ldg(reinterpret_cast<const int4 *>(a.rrec + ci));
                const int4 rx = __ldg(reinterpret_cast<const int4 *>(a.crec + cj));
                const int i0 = ry.x & 0xffff, i1 = ry.x >> 16, j0 = rx.x & 0xffff, j1 = rx.x >> 16;
                for (const float *ch : {chx, chy}) {
                    touch_sector(touch, paf_f, ch + (size_t)i0 * a.w + j0);
                    touch_sector(touch, paf_f, ch + (size_t)i0 * a.w + j1);
                    touch_sector(touch, paf_f, ch + (size_t)i1 * a.w + j0);
                    touch_sector(touch, paf_f, ch + (size_t)i1 * a.w + j1);
                }
            }
        }
        const double d = finish_sample(a, r, vx, vy);
        total = dadd(total, d);
        if (d >= a.dot_thr) ++ngood;
        else if (++nfail > max_fail) return false;
    }
    score = __ddiv_rn(total, (double)n);
    return score > 0.0;                                   // paf.py:162 (good already passed)
}

// CPython 3.12 builtin sum() over floats starting from int 0 (Neumaier).
__device__ __forceinline__ void neumaier_add(double &f, double &c, double v)
{
    const double t = dadd(f, v);
    if (fabs(f) >= fabs(v)) c = dadd(c, dadd(__dsub_rn(f, t), v));
    else c = dadd(c, dadd(__dsub_rn(v, t), f));
    f = t;
}


}  // namespace pf
