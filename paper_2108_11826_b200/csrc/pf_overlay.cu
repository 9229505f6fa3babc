// pf_overlay.cu — GPU overlay rasteriser: the
// reference's visualize (operators.py:173-290) — limbs as Bresenham lines
// stamped with discs, then keypoint discs, then optional score labels, in a
// fixed order where later draws overwrite earlier ones.
//
// "Later overwrites earlier" is resolved without serialising the drawing:
// every primitive carries its draw-order index, (1) one thread per primitive
// rasterises it (the reference's exact integer Bresenham walk and disc test)
// and records atomicMax(index + 1) in the pixel's owner word, (2) one thread
// per pixel copies its owner's colour into the frame copy.  The pixel set and
// the colour of each primitive are the reference's, so the image is
// identical.  Host code (Python) places the keypoints (round-half-up of the
// scaled coordinates, operators.py:270-277) and expands label glyphs into
// points, so the device only does integer raster work.
#include <algorithm>

#include "pf_launch.h"

namespace pf {

__device__ __forceinline__ void own(unsigned *owner, int h, int w, int x, int y, unsigned tag)
{
    if (0 <= y && y < h && 0 <= x && x < w) atomicMax(owner + (size_t)y * w + x, tag);
}

// _draw_disc (operators.py:178-188): dx*dx + dy*dy <= r*r, clipped
__device__ __forceinline__ void disc(unsigned *owner, int h, int w, int cx, int cy, int r, unsigned tag)
{
    for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx)
            if (dx * dx + dy * dy <= r * r) own(owner, h, w, cx + dx, cy + dy, tag);
}

__global__ void __launch_bounds__(128)
k_overlay_raster(const OverlayPrim *__restrict__ prims, const int *__restrict__ prim_first, int frames, int h, int w,
                 unsigned *__restrict__ owner)
{
    const int total = prim_first[frames];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const OverlayPrim pr = prims[i];
        unsigned *ow = owner + (size_t)pr.frame * h * w;
        const unsigned tag = (unsigned)(i - prim_first[pr.frame]) + 1u;   // draw order within the frame
        if (pr.kind == 0) {
            // _draw_line (operators.py:191-216): Bresenham stamped with a disc of radius thickness // 2
            int x = pr.x0, y = pr.y0;
            const int dx = abs(pr.x1 - pr.x0), dy = -abs(pr.y1 - pr.y0);
            const int sx = pr.x0 < pr.x1 ? 1 : -1, sy = pr.y0 < pr.y1 ? 1 : -1;
            int err = dx + dy;
            while (true) {
                if (pr.r == 0) own(ow, h, w, x, y, tag);
                else disc(ow, h, w, x, y, pr.r, tag);
                if (x == pr.x1 && y == pr.y1) break;
                const int e2 = 2 * err;
                if (e2 >= dy) { err += dy; x += sx; }
                if (e2 <= dx) { err += dx; y += sy; }
            }
        } else {
            disc(ow, h, w, pr.x0, pr.y0, pr.r, tag);             // keypoint disc; r = 0: a label pixel
        }
    }
}

__global__ void __launch_bounds__(256)
k_overlay_paint(const OverlayPrim *__restrict__ prims, const int *__restrict__ prim_first, int frames, int h, int w,
                const unsigned *__restrict__ owner, float *__restrict__ img)
{
    const long long n = (long long)frames * h * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const unsigned tag = owner[e];
        if (!tag) continue;
        const int f = (int)(e / ((long long)h * w));
        const OverlayPrim pr = prims[prim_first[f] + (int)tag - 1];
        img[e * 3 + 0] = pr.rgb[0];
        img[e * 3 + 1] = pr.rgb[1];
        img[e * 3 + 2] = pr.rgb[2];
    }
}

cudaError_t launch_overlay(const OverlayPrim *prims, const int *prim_first, int n_prims, int frames, int h, int w,
                           unsigned *owner, float *img, int sms, cudaStream_t s)
{
    if ((long long)frames * h * w == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(owner, 0, sizeof(unsigned) * (size_t)frames * h * w, s);
    if (e != cudaSuccess) return e;
    if (n_prims > 0) {
        const int blocks = std::min((n_prims + 127) / 128, sms * 8);
        k_overlay_raster<<<blocks, 128, 0, s>>>(prims, prim_first, frames, h, w, owner);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const long long n = (long long)frames * h * w;
    const long long blocks = std::min<long long>((n + 255) / 256, (long long)sms * 16);
    k_overlay_paint<<<(unsigned)blocks, 256, 0, s>>>(prims, prim_first, frames, h, w, owner, img);
    return cudaGetLastError();
}

}  // namespace pf
