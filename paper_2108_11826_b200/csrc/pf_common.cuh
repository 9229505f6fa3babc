// pf_common.cuh — shared device helpers for the sm_100a pose-parsing kernels.
//
// Bit-exactness rules (SURVEY.md §7 "hard parts"):
//  * fp64 products and sums go through __dmul_rn/__dadd_rn so nvcc can never
//    contract them into DFMA (the library is also built with -fmad=false);
//  * the confidence threshold is compared in fp32 (numpy >= 2, NEP 50);
//  * u8/255 is an IEEE fp32 division (__fdiv_rn), never a reciprocal multiply.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pf_b200.h"

namespace pf {

constexpr int kWarp = 32;

// Skeleton tables, passed by value as a kernel parameter (constant bank).
struct Topo {
    int K;                       // keypoints (conf channels 0..K-1 are parts)
    int L;                       // limbs
    int8_t la[PF_MAX_LIMBS];     // limb endpoint parts
    int8_t lb[PF_MAX_LIMBS];
    int16_t cx[PF_MAX_LIMBS];    // PAF channel pair of each limb
    int16_t cy[PF_MAX_LIMBS];
};

// One axis of operators.bilinear_resize (operators.py:86-96), precomputed on
// the host in fp64 with the reference operation order.
struct AxisTab {
    const int32_t *i0;   // clip(floor(s), 0, in-1)
    const int32_t *i1;   // clip(floor(s)+1, 0, in-1)
    const double *t;     // s - floor(s)
    const double *omt;   // 1 - t, as its own rounded op
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// operators.py:102-107: top = a*(1-tx) + b*tx ; bot = c*(1-tx) + d*tx ;
// out = float32(top*(1-ty) + bot*ty), every op separately rounded.
__device__ __forceinline__ float bilerp(double a, double b, double c, double d,
                                        double tx, double omtx, double ty, double omty)
{
    const double top = dadd(dmul(a, omtx), dmul(b, tx));
    const double bot = dadd(dmul(c, omtx), dmul(d, tx));
    return __double2float_rn(dadd(dmul(top, omty), dmul(bot, ty)));
}

// operators.py:87-96 for one output coordinate, evaluated in registers with
// the same fp64 op order as the host tables: s = (o + 0.5) * ratio - 0.5,
// f = floor(s), t = s - f, 1 - t, indices clipped to [0, n_in - 1].
__device__ __forceinline__ void axis_coord(int o, double ratio, int n_in, int &i0, int &i1, double &t,
                                           double &omt)
{
    const double s = dadd(dmul(dadd((double)o, 0.5), ratio), -0.5);
    const double f = floor(s);
    const int fi = (int)f;
    t = __dsub_rn(s, f);
    omt = __dsub_rn(1.0, t);
    i0 = min(max(fi, 0), n_in - 1);
    i1 = min(max(fi + 1, 0), n_in - 1);
}

// Peak record produced by the NMS kernels: fp32 score bits + packed cell.
__device__ __forceinline__ uint2 pack_peak(float v, int i, int j)
{
    return make_uint2(__float_as_uint(v), (uint32_t(i) << 16) | uint32_t(j));
}

// paf.py:95-99 — centre must beat lexicographically-earlier neighbours
// strictly and later ones (di>0, or di==0 && dj>0) non-strictly.  NaN in
// either operand fails both compares, as in numpy.
__device__ __forceinline__ bool nms_beats(float v, float nv, int di, int dj)
{
    const bool later = di > 0 || (di == 0 && dj > 0);
    return later ? (v >= nv) : (v > nv);
}

// Device-side status words (one per context).
struct Status {
    int code;          // max error code seen (PF_ERR_CAPACITY)
    int frame;         // smallest offending global frame index
    int what;          // which capacity (see pf_capi.cu kCap*)
    int value;         // offending count
    int pool_used;     // humans written to the output pool
    int pad[3];
};

__device__ __forceinline__ void report_capacity(Status *st, int frame, int what, int value)
{
    atomicMax(&st->code, PF_ERR_CAPACITY);
    const int prev = atomicMin(&st->frame, frame);
    if (frame < prev || prev == frame) {
        // best effort detail for the earliest frame
        atomicExch(&st->what, what);
        atomicExch(&st->value, value);
    }
}

}  // namespace pf
