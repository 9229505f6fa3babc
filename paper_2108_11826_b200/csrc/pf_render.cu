// pf_render.cu — k_render_maps: the synthetic backend's renderer on the GPU
// ("GPU-resident producer"): reference synth.py:93-183
// (render_feature_maps + _paint_limb), restated in paper_2108_11826_b200/synth.py.
// One thread per (frame, cell):
//   conf[k]  = max over humans of exp(-((i - ci)^2 + (j - cj)^2) / (2 sigma^2)),
//              background = 1 - max over parts (max with initial 0);
//   paf      = per limb, the sum over humans (in scene order) of the unit limb
//              vector at cells within `halfwidth` of the segment, divided by
//              the count, clamped to unit length;
// all in fp64 with the reference's operation order, stored as fp32.  fp64
// exp() is the only operation whose last bit may differ from numpy's; the
// fp32 maps agree except where a value lies on an fp32 rounding boundary.
#include "pf_launch.h"

namespace pf {

__global__ void __launch_bounds__(256)
k_render_maps(const RenderArgs a)
{
    const int gh = a.gh, gw = a.gw, K = a.topo.K, L = a.topo.L;
    const long long cells = (long long)a.F * gh * gw;
    const double inv = __ddiv_rn(1.0, dmul(dmul(2.0, a.sigma), a.sigma));
    const double hw2 = dmul(a.halfwidth, a.halfwidth);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cells;
         e += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(e / ((long long)gh * gw));
        const int rem = (int)(e - (long long)f * gh * gw);
        const int i = rem / gw, j = rem - i * gw;
        const double row = (double)i, col = (double)j;
        const int nh = a.n_humans[f];
        const double *kp = a.kp + (size_t)f * a.hmax * K * 2;
        float *conf = a.conf + (size_t)f * (K + 1) * gh * gw + rem;
        float *paf = a.paf + (size_t)f * 2 * L * gh * gw + rem;
        double cmax = 0.0;                                 // max over parts, initial 0
        for (int k = 0; k < K; ++k) {
            double m = 0.0;                                // conf starts at zeros
            for (int hh = 0; hh < nh; ++hh) {
                const double ci = kp[((size_t)hh * K + k) * 2], cj = kp[((size_t)hh * K + k) * 2 + 1];
                if (ci != ci) continue;                    // missing keypoint (NaN)
                const double di = __dsub_rn(row, ci), dj = __dsub_rn(col, cj);
                const double g = exp(dmul(-dadd(dmul(di, di), dmul(dj, dj)), inv));
                m = fmax(m, g);
            }
            conf[(size_t)k * gh * gw] = (float)m;
            cmax = fmax(cmax, m);
        }
        conf[(size_t)K * gh * gw] = (float)__dsub_rn(1.0, cmax);
        for (int l = 0; l < L; ++l) {
            const int pa = a.topo.la[l], pb = a.topo.lb[l];
            double sx = 0.0, sy = 0.0;
            int cnt = 0;
            for (int hh = 0; hh < nh; ++hh) {
                const double ai = kp[((size_t)hh * K + pa) * 2], aj = kp[((size_t)hh * K + pa) * 2 + 1];
                const double bi = kp[((size_t)hh * K + pb) * 2], bj = kp[((size_t)hh * K + pb) * 2 + 1];
                if (ai != ai || bi != bi) continue;
                const double dli = __dsub_rn(bi, ai), dlj = __dsub_rn(bj, aj);
                const double len_sq = dadd(dmul(dli, dli), dmul(dlj, dlj));
                if (len_sq == 0.0) continue;
                const double len = __dsqrt_rn(len_sq);
                const double ux = __ddiv_rn(dlj, len), uy = __ddiv_rn(dli, len);
                double t = __ddiv_rn(dadd(dmul(__dsub_rn(row, ai), dli), dmul(__dsub_rn(col, aj), dlj)), len_sq);
                t = fmin(fmax(t, 0.0), 1.0);               // np.clip
                const double ei = __dsub_rn(row, dadd(ai, dmul(t, dli)));
                const double ej = __dsub_rn(col, dadd(aj, dmul(t, dlj)));
                if (dadd(dmul(ei, ei), dmul(ej, ej)) <= hw2) {
                    sx = dadd(sx, ux);
                    sy = dadd(sy, uy);
                    ++cnt;
                }
            }
            double vx = 0.0, vy = 0.0;
            if (cnt > 0) {
                vx = __ddiv_rn(sx, (double)cnt);
                vy = __ddiv_rn(sy, (double)cnt);
                const double mag = __dsqrt_rn(dadd(dmul(vx, vx), dmul(vy, vy)));
                if (mag > 1.0) {
                    vx = __ddiv_rn(vx, mag);
                    vy = __ddiv_rn(vy, mag);
                }
            }
            paf[(size_t)a.topo.cx[l] * gh * gw] = (float)vx;
            paf[(size_t)a.topo.cy[l] * gh * gw] = (float)vy;
        }
    }
}

cudaError_t launch_render_maps(const RenderArgs &a, int sms, cudaStream_t s)
{
    const long long cells = (long long)a.F * a.gh * a.gw;
    if (cells == 0) return cudaSuccess;
    long long blocks = (cells + 255) / 256;
    if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
    k_render_maps<<<(unsigned)blocks, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace pf
