// pf_image.cu — dense image/map kernels: pre-processing, materialised
// bilinear resize of planes, separable Gaussian smoothing.  All three are
// HBM-streaming kernels (no reuse beyond the 2x2 / (2r+1) stencils, which
// L1 absorbs); stores are 16-byte vectors where the row width allows.
#include "pf_launch.h"

namespace pf {

// operators.py:114-131 (+ formats.py:116-117 for u8 input): HWC -> f32 CHW.
// u8 input: v = float32(u8) / 255.0f (IEEE division, tabulated with the same
// division); f32 input: the value as-is (an already-normalised Frame image).
// Unless the size is unchanged (pure layout permutation, operators.py:123-124)
// the fp64 bilinear formula of operators.py:97-101 (3-D branch) is applied and
// rounded once to fp32.
template <typename Tin>
struct PixelLoad;

template <>
struct PixelLoad<uint8_t> {
    const float *lut;
    __device__ float operator()(const uint8_t *p) const { return lut[*p]; }
};

template <>
struct PixelLoad<float> {
    __device__ float operator()(const float *p) const { return __ldg(p); }
};

// Same size (operators.py:123-124: layout only): 4 pixels per thread, one
// 12-byte (u8) or 48-byte (f32) load, one 16-byte store per channel plane.
template <typename Tin>
__global__ void __launch_bounds__(256)
k_preprocess_same(const Tin *__restrict__ src, int hw, float *__restrict__ dst, int vec)
{
    __shared__ float lut[256];
    if constexpr (sizeof(Tin) == 1) {
        for (int u = threadIdx.x; u < 256; u += blockDim.x) lut[u] = __fdiv_rn((float)u, 255.0f);
        __syncthreads();
    }
    const long long b = blockIdx.y;
    const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (p0 >= hw) return;
    const Tin *s = src + b * (long long)hw * 3 + (long long)p0 * 3;
    float *d = dst + b * 3LL * hw + p0;
    float v[12];
    if (vec) {
        if constexpr (sizeof(Tin) == 1) {
            const uint32_t *s4 = reinterpret_cast<const uint32_t *>(s);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const uint32_t wd = __ldg(s4 + k);
#pragma unroll
                for (int q = 0; q < 4; ++q) v[4 * k + q] = lut[(wd >> (8 * q)) & 0xffu];
            }
        } else {
            const float4 *s4 = reinterpret_cast<const float4 *>(s);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float4 f = __ldg(s4 + k);
                v[4 * k] = f.x; v[4 * k + 1] = f.y; v[4 * k + 2] = f.z; v[4 * k + 3] = f.w;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c)
            __stcs(reinterpret_cast<float4 *>(d + (long long)c * hw),
                   make_float4(v[c], v[3 + c], v[6 + c], v[9 + c]));
    } else {
        for (int q = 0; q < 4 && p0 + q < hw; ++q)
            for (int c = 0; c < 3; ++c) {
                const Tin x = s[3 * q + c];
                d[(long long)c * hw + q] = sizeof(Tin) == 1 ? lut[(int)x] : (float)x;
            }
    }
}

// Resize (operators.py:97-101, 3-D branch): thread per output pixel, packed
// axis records, fp64 bilinear per channel rounded once to fp32.
template <typename Tin>
__global__ void __launch_bounds__(128)
k_preprocess_resize(const Tin *__restrict__ src, int h, int w, float *__restrict__ dst, int H, int W,
                    const AxisRec *__restrict__ rrec, const AxisRec *__restrict__ crec)
{
    __shared__ float lut[256];
    if constexpr (sizeof(Tin) == 1) {
        for (int u = threadIdx.x; u < 256; u += blockDim.x) lut[u] = __fdiv_rn((float)u, 255.0f);
        __syncthreads();
    }
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const long long b = blockIdx.z;
    if (x >= W) return;
    const int4 ry = __ldg(reinterpret_cast<const int4 *>(rrec + y));
    const int4 rx = __ldg(reinterpret_cast<const int4 *>(crec + x));
    const int i0 = ry.x & 0xffff, i1 = ry.x >> 16, j0 = rx.x & 0xffff, j1 = rx.x >> 16;
    const double ty = __hiloint2double(ry.w, ry.z), tx = __hiloint2double(rx.w, rx.z);
    const double omty = __dsub_rn(1.0, ty), omtx = __dsub_rn(1.0, tx);
    const Tin *s = src + b * (long long)h * w * 3;
    const Tin *p00 = s + ((size_t)i0 * w + j0) * 3, *p01 = s + ((size_t)i0 * w + j1) * 3;
    const Tin *p10 = s + ((size_t)i1 * w + j0) * 3, *p11 = s + ((size_t)i1 * w + j1) * 3;
    auto ld = [&](const Tin *q) -> float {
        if constexpr (sizeof(Tin) == 1) return lut[*q];
        else return __ldg(q);
    };
    const long long HW = (long long)H * W;
    float *d = dst + b * 3 * HW + (long long)y * W + x;
#pragma unroll
    for (int c = 0; c < 3; ++c)
        d[c * HW] = bilerp(ld(p00 + c), ld(p01 + c), ld(p10 + c), ld(p11 + c), tx, omtx, ty, omty);
}

// operators.py:102-107 (2-D branch) applied per plane: [P][h][w] -> [P][H][W]
// (source plane p at (p / K) * src_frame + (p % K) * h * w, so the part
// channels can be taken out of a [K+1]-channel tensor).  HBM-write bound: a
// thread owns 4 adjacent output columns of a band of kResizeRows output
// rows; its column records are loaded once, and the row interpolants
// top = a*(1-tx) + b*tx, bot = c*(1-tx) + d*tx are recomputed only when the
// source row pair changes (8 output rows share one at x8), so an output costs
// 2 DMUL + 1 DADD + 1 F2F and a 16-byte store.  Same op order as bilerp().
constexpr int kResizeRows = 32;
constexpr int kResizeThreads = 128;

__global__ void __launch_bounds__(kResizeThreads)
k_resize_planes(const float *__restrict__ src, long long src_frame, int K, int h, int w,
                float *__restrict__ dst, int H, int W, const AxisRec *__restrict__ rrec,
                const AxisRec *__restrict__ crec, int n_row_blocks)
{
    const int x0 = (blockIdx.x * kResizeThreads + threadIdx.x) * 4;
    if (x0 >= W) return;
    const long long plane = blockIdx.y / n_row_blocks;
    const int y_lo = (int)(blockIdx.y - plane * n_row_blocks) * kResizeRows;
    const int y_hi = min(H, y_lo + kResizeRows);
    const float *s = src + (plane / K) * src_frame + (plane % K) * (long long)h * w;
    float *d = dst + plane * (long long)H * W;
    int j0[4], j1[4];
    double tx[4], omtx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int4 r = __ldg(reinterpret_cast<const int4 *>(crec + min(x0 + k, W - 1)));
        j0[k] = r.x & 0xffff;
        j1[k] = r.x >> 16;
        tx[k] = __hiloint2double(r.w, r.z);
        omtx[k] = __dsub_rn(1.0, tx[k]);
    }
    int cur = -1;
    double top[4], bot[4];
    const bool vec = (W & 3) == 0 && x0 + 3 < W;
    for (int y = y_lo; y < y_hi; ++y) {
        const int4 r = __ldg(reinterpret_cast<const int4 *>(rrec + y));
        if (r.x != cur) {
            cur = r.x;
            const float *r0 = s + (size_t)(r.x & 0xffff) * w, *r1 = s + (size_t)(r.x >> 16) * w;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                top[k] = dadd(dmul((double)__ldg(r0 + j0[k]), omtx[k]), dmul((double)__ldg(r0 + j1[k]), tx[k]));
                bot[k] = dadd(dmul((double)__ldg(r1 + j0[k]), omtx[k]), dmul((double)__ldg(r1 + j1[k]), tx[k]));
            }
        }
        const double ty = __hiloint2double(r.w, r.z), omty = __dsub_rn(1.0, ty);
        float out[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = __double2float_rn(dadd(dmul(top[k], omty), dmul(bot[k], ty)));
        float *o = d + (size_t)y * W + x0;
        if (vec) {
            __stcs(reinterpret_cast<float4 *>(o), make_float4(out[0], out[1], out[2], out[3]));
        } else {
            for (int k = 0; k < 4 && x0 + k < W; ++k) o[k] = out[k];
        }
    }
}

// Separable Gaussian (no reference): taps k=-r..r, clamped
// edges, fp32 fma chain in ascending k from 0.0f with w_k = (float)taps[k].
// The materialised form (Mode R blur, wide NMS windows); Mode U with the 3x3
// window takes the fused k_up_blur_nms (pf_blur.cu).
// Source and destination planes are addressed as (plane / K) * src_frame +
// (plane % K) * HW so the blur can read part channels out of a [K+1]-channel
// tensor.

__global__ void __launch_bounds__(256)
k_blur_rows(const float *__restrict__ src, long long src_frame, float *__restrict__ dst,
            long long dst_frame, int K, int H, int W, const BlurTaps taps, long long total)
{
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long HW = (long long)H * W;
        const long long plane = e / HW;
        const int rem = int(e - plane * HW);
        const int y = rem / W, x = rem - y * W;
        const long long fb = plane / K;
        const int k = int(plane - fb * K);
        const float *s = src + fb * src_frame + (long long)k * HW + (long long)y * W;
        float acc = 0.0f;
        for (int t = -taps.r; t <= taps.r; ++t) {
            const int xx = min(max(x + t, 0), W - 1);
            acc = __fmaf_rn((float)taps.w[t + taps.r], __ldg(s + xx), acc);
        }
        dst[fb * dst_frame + (long long)k * HW + rem] = acc;
    }
}

__global__ void __launch_bounds__(256)
k_blur_cols(const float *__restrict__ src, long long src_frame, float *__restrict__ dst,
            long long dst_frame, int K, int H, int W, const BlurTaps taps, long long total)
{
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long HW = (long long)H * W;
        const long long plane = e / HW;
        const int rem = int(e - plane * HW);
        const int y = rem / W, x = rem - y * W;
        const long long fb = plane / K;
        const int k = int(plane - fb * K);
        const float *s = src + fb * src_frame + (long long)k * HW + x;
        float acc = 0.0f;
        for (int t = -taps.r; t <= taps.r; ++t) {
            const int yy = min(max(y + t, 0), H - 1);
            acc = __fmaf_rn((float)taps.w[t + taps.r], __ldg(s + (long long)yy * W), acc);
        }
        dst[fb * dst_frame + (long long)k * HW + rem] = acc;
    }
}

static unsigned grid_for(long long total, int threads, int sms)
{
    long long blocks = (total + threads - 1) / threads;
    const long long cap = (long long)sms * 16;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_preprocess(const void *src, int src_is_f32, int B, int h, int w, float *dst,
                              int H, int W, const AxisRec *rrec, const AxisRec *crec, cudaStream_t s)
{
    if ((long long)B * H * W == 0) return cudaSuccess;
    for (int b0 = 0; b0 < B; b0 += 65535) {           // grid.y / grid.z <= 65535
        const int nb = B - b0 < 65535 ? B - b0 : 65535;
        if (h == H && w == W) {
            const int hw = h * w;
            const dim3 grid((unsigned)((hw / 4 + 256) / 256), (unsigned)nb);
            // 16-byte vectors need hw % 4 == 0 and aligned bases
            const int vec = (hw & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
                            (reinterpret_cast<uintptr_t>(src) & (src_is_f32 ? 15 : 3)) == 0;
            if (src_is_f32)
                k_preprocess_same<float><<<grid, 256, 0, s>>>(static_cast<const float *>(src) + (size_t)b0 * hw * 3,
                                                             hw, dst + (size_t)b0 * 3 * hw, vec);
            else
                k_preprocess_same<uint8_t><<<grid, 256, 0, s>>>(static_cast<const uint8_t *>(src) + (size_t)b0 * hw * 3,
                                                               hw, dst + (size_t)b0 * 3 * hw, vec);
        } else {
            if (H > 65535) return cudaErrorInvalidConfiguration;
            const dim3 grid((unsigned)((W + 127) / 128), (unsigned)H, (unsigned)nb);
            const size_t so = (size_t)b0 * h * w * 3, dof = (size_t)b0 * 3 * H * W;
            if (src_is_f32)
                k_preprocess_resize<float><<<grid, 128, 0, s>>>(static_cast<const float *>(src) + so, h, w, dst + dof,
                                                               H, W, rrec, crec);
            else
                k_preprocess_resize<uint8_t><<<grid, 128, 0, s>>>(static_cast<const uint8_t *>(src) + so, h, w,
                                                                 dst + dof, H, W, rrec, crec);
        }
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_resize_planes(const float *src, long long src_frame, int K, long long P, int h, int w,
                                 float *dst, int H, int W, const AxisRec *rrec, const AxisRec *crec,
                                 cudaStream_t s)
{
    if (P == 0 || H == 0 || W == 0) return cudaSuccess;
    const int nrb = (H + kResizeRows - 1) / kResizeRows;
    const unsigned gx = (unsigned)(((W + 3) / 4 + kResizeThreads - 1) / kResizeThreads);
    // grid.y <= 65535: launch whole frames (K planes) at a time
    long long per = (65535 / nrb) / K * K;
    if (per < K) return cudaErrorInvalidConfiguration;
    for (long long p0 = 0; p0 < P; p0 += per) {      // P is a multiple of K
        const long long n = P - p0 < per ? P - p0 : per;
        k_resize_planes<<<dim3(gx, (unsigned)(n * nrb)), kResizeThreads, 0, s>>>(
            src + (p0 / K) * src_frame, src_frame, K, h, w, dst + p0 * (long long)H * W, H, W, rrec, crec, nrb);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_blur(const float *src, long long src_frame, float *tmp, float *dst,
                        long long dst_frame, int B, int K, int H, int W, const BlurTaps &taps,
                        int sms, cudaStream_t s)
{
    const long long total = (long long)B * K * H * W;
    if (total == 0) return cudaSuccess;
    const long long tmp_frame = (long long)K * H * W;
    k_blur_rows<<<grid_for(total, 256, sms), 256, 0, s>>>(src, src_frame, tmp, tmp_frame, K, H, W, taps, total);
    k_blur_cols<<<grid_for(total, 256, sms), 256, 0, s>>>(tmp, tmp_frame, dst, dst_frame, K, H, W, taps, total);
    return cudaGetLastError();
}

}  // namespace pf
