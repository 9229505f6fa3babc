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
//   T  horizontal pass: T = fp32(sum_k w_k U[clamp(x+k)]), fp64 fma chain in
//      ascending k from 0.0;
//   B  vertical pass of row u - r from the ring, same chain, clamped rows;
//   N  the reference peak test of row u - r - 1 on B (earlier neighbours
//      strictly, later ones non-strictly, -inf outside the grid), peaks into
//      the plane's slab (global atomic per peak: several CTAs per plane).
// The work is fp64-pipe bound (~18 fp64 instructions per output pixel);
// HBM traffic is the low-res part planes (read through L1/L2) and the peaks.
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
    double *Ud = reinterpret_cast<double *>(smb);              // [NU]
    double *Tr = Ud + NU;                                       // [R][NB]
    float *Br = reinterpret_cast<float *>(Tr + (size_t)R * NB); // [4][NB]
    __shared__ double wt[2 * kMaxBlurRadius + 1];

    const int tile = blockIdx.x % a.tiles;
    const int plane = blockIdx.x / a.tiles;
    const int fb = plane / a.K, k = plane - fb * a.K;
    const float *S = a.conf + ((size_t)fb * a.C + k) * (size_t)a.h * a.w;
    const int H = a.H, W = a.W, w = a.w;
    const int x0 = tile * tw;
    const int j = threadIdx.x;
    for (int t = j; t < R; t += kBlurThreads) wt[t] = a.taps.w[t];

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
                Ud[j] = (double)__double2float_rn(dadd(dmul(top, __dsub_rn(1.0, ty)), dmul(bot, ty)));
            }
            band0 = i0;
            band1 = i1;
            __syncthreads();
            if (b_in) {                                          // T row u (horizontal pass)
                double acc = 0.0;
                for (int t = 0; t < R; ++t) acc = __fma_rn(wt[t], Ud[j + t], acc);
                Tr[(size_t)(u % R) * NB + j] = (double)__double2float_rn(acc);
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
                    double acc = 0.0;
                    for (int t = 0; t < R; ++t) {
                        acc = __fma_rn(wt[t], Tr[(size_t)sl * NB + j], acc);
                        const int nrow = min(max(y - r + t + 1, 0), H - 1);
                        if (nrow != row) {
                            row = nrow;
                            sl = sl + 1 == R ? 0 : sl + 1;
                        }
                    }
                    bv = __double2float_rn(acc);
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

size_t up_blur_smem(int tw, int r)
{
    const int NB = tw + 2, NU = tw + 2 + 2 * r;
    return (size_t)NU * sizeof(double) + (size_t)(2 * r + 1) * NB * sizeof(double) + (size_t)4 * NB * sizeof(float);
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
    a.tw = up_blur_tile_width(a.W, a.taps.r);
    if (a.tw < 1) return cudaErrorInvalidValue;
    a.tiles = (a.W + a.tw - 1) / a.tw;
    const size_t smem = up_blur_smem(a.tw, a.taps.r);
    k_up_blur_nms<<<(unsigned)(P * a.tiles), kBlurThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t configure_blur_kernels(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_up_blur_nms);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_up_blur_nms, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    return e;
}

}  // namespace pf
