// pf_large.cu — k_parse_large: the parse of frames past the shared-memory
// bound capacities of k_parse_frames (more than 32767 peaks per frame, peak
// ids past 16 bits, per-part bitmaps or human tables that no longer fit in
// shared memory).  The reference has no such limits (paf.py:100-109,
// :231-289); a context switches to this path for a call when an automatic
// capacity cannot grow any further on the usual path (pf_capi.cu grow_cap).
//
// One 1024-thread CTA per frame, every table in a per-frame HBM workspace with
// 32-bit indices; the same steps and the same exactness rules as
// k_parse_frames (paf.py:292-305):
//   1. peak counts per part (NMS slab), ids as a prefix over parts (:298-303);
//   2. each part's peaks ranked by (-score, i, j) (paf.py:104), thread per peak;
//   3. every (limb, a, b) pair scored by score_pair (paf.py:112-165), gated
//      candidates appended (local peak indices: ids differ by a per-limb
//      constant, so the order of local indices is the order of ids);
//   4. one bitonic sort of the candidates by (limb, -score, id_a, id_b)
//      (paf.py:173) through HBM;
//   5. greedy per limb, thread per limb, used-bitmaps in HBM (paf.py:174-181);
//   6. assemble_humans replayed by one thread (paf.py:241-271);
//   7. Neumaier score sums, filters, stable rank, pool write (paf.py:273-289).
// Throughput is not the point here; exactness and the absence of limits are.
#include <algorithm>

#include "pf_score.cuh"

namespace pf {

constexpr int kLargeThreads = 1024;
constexpr uint32_t kLargeAccepted = 0x80000000u;

struct CandL {
    double score;
    uint32_t ia, ib;     // peak indices within the limb's parts
    uint32_t lg;         // limb << 24 | n_good; kLargeAccepted marks greedy acceptance
    uint32_t pad;
};

__device__ __forceinline__ bool candl_less(const CandL &x, const CandL &y)
{
    const uint32_t lx = (x.lg >> 24) & 0x7f, ly = (y.lg >> 24) & 0x7f;
    if (lx != ly) return lx < ly;
    if (x.score != y.score) return x.score > y.score;
    if (x.ia != y.ia) return x.ia < y.ia;
    return x.ib < y.ib;
}

__device__ __forceinline__ bool part_less(uint2 u, uint2 v)
{
    const float us = __uint_as_float(u.x), vs = __uint_as_float(v.x);
    return (us > vs) || (us == vs && u.y < v.y);
}

__global__ void __launch_bounds__(kLargeThreads, 1)
k_parse_large(const ParseArgs a, const LargeWs ws)
{
    const int K = a.topo.K, L = a.topo.L;
    const int b = blockIdx.x, gframe = a.frame_base + b;
    const int tid = threadIdx.x, nthr = blockDim.x;
    __shared__ int s_base[PF_MAX_KEYPOINTS + 1];
    __shared__ long long s_pp[PF_MAX_LIMBS + 1];
    __shared__ int s_seg[PF_MAX_LIMBS + 1];
    __shared__ int s_err, s_val, s_nh, s_pool;
    __shared__ unsigned long long s_nc;
    __shared__ double s_t[kParseTTab];
    __shared__ int8_t s_la[PF_MAX_LIMBS], s_lb[PF_MAX_LIMBS];

    uint32_t *pk_cell = ws.pk_cell + (size_t)b * ws.cap_peaks;
    float *pk_score = ws.pk_score + (size_t)b * ws.cap_peaks;
    int *owner = ws.owner + (size_t)b * ws.cap_peaks;
    CandL *cand = reinterpret_cast<CandL *>(ws.cand) + (size_t)b * ws.cap_cands;
    uint32_t *used = ws.used + (size_t)b * ws.used_words;
    int *h_parts = ws.h_parts + (size_t)b * ws.cap_humans * K;
    int8_t *h_order = ws.h_order + (size_t)b * ws.cap_humans * K;
    int8_t *h_n = ws.h_n + (size_t)b * ws.cap_humans;
    int8_t *h_alive = ws.h_alive + (size_t)b * ws.cap_humans;
    uint32_t *h_mask = ws.h_mask + (size_t)b * ws.cap_humans;
    double *h_score = ws.h_score + (size_t)b * ws.cap_humans;
    int *h_pos = ws.h_pos + (size_t)b * ws.cap_humans;

    for (int u = tid; u < kParseTTab && u < a.n_samples; u += nthr)
        s_t[u] = __ddiv_rn((double)u, (double)(a.n_samples - 1));
    for (int l = tid; l < L; l += nthr) { s_la[l] = a.topo.la[l]; s_lb[l] = a.topo.lb[l]; }
    // ---- 1. counts, prefix, capacities ----
    if (tid == 0) {
        int err = 0, val = 0, acc = 0;
        s_base[0] = 0;
        for (int k = 0; k < K; ++k) {
            const int c = a.counts[(size_t)b * K + k];
            if (c > a.cap_part && !err) { err = kCapPart; val = c; }
            acc += c;
            s_base[k + 1] = acc;
        }
        if (!err && acc > ws.cap_peaks) { err = kCapFrame; val = acc; }
        s_err = err; s_val = val; s_nc = 0;
    }
    __syncthreads();
    for (int k = tid; k < K; k += nthr) a.counts[(size_t)b * K + k] = 0;    // ready for the next launch
    if (s_err) {
        if (tid == 0) {
            report_capacity(a.st, gframe, s_err, s_val);
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
            if (a.debug) { a.dbg_npeaks[gframe] = 0; a.dbg_nconns[gframe] = 0; }
        }
        return;
    }
    const int P = s_base[K];

    // ---- 2. rank each part's peaks (paf.py:104) ----
    for (int e = tid; e < P; e += nthr) {
        int part = 0;
        while (e >= s_base[part + 1]) ++part;
        const uint2 *slab = a.peaks + ((size_t)b * K + part) * a.cap_part;
        const int np = s_base[part + 1] - s_base[part];
        const uint2 v = __ldg(slab + (e - s_base[part]));
        int rank = 0;
        for (int q = 0; q < np; ++q) rank += part_less(__ldg(slab + q), v);
        pk_cell[s_base[part] + rank] = v.y;
        pk_score[s_base[part] + rank] = __uint_as_float(v.x);
        owner[e] = -1;
    }
    if (tid == 0) {
        long long acc = 0;
        for (int l = 0; l < L; ++l) {
            s_pp[l] = acc;
            acc += (long long)(s_base[s_la[l] + 1] - s_base[s_la[l]]) * (s_base[s_lb[l] + 1] - s_base[s_lb[l]]);
        }
        s_pp[L] = acc;
    }
    __syncthreads();
    if (a.debug) {
        for (int e = tid; e < P; e += nthr) {
            int part = 0;
            while (e >= s_base[part + 1]) ++part;
            a.dbg_peaks[(size_t)gframe * a.cap_frame + e] =
                make_int4(part, int(pk_cell[e] >> 16), int(pk_cell[e] & 0xffff), __float_as_int(pk_score[e]));
        }
        if (tid == 0) a.dbg_npeaks[gframe] = P;
    }

    // ---- 3. line integrals of every pair (paf.py:149-165) ----
    const float *paf_f = a.paf + (size_t)b * (2 * L) * a.h * a.w;
    const long long n_pairs = s_pp[L];
    const int max_fail = a.n_samples - a.good_need;
    if (max_fail >= 0) {
        for (long long p = tid; p < n_pairs; p += nthr) {
            int l = 0;
            while (p >= s_pp[l + 1]) ++l;
            const int na = s_base[s_la[l] + 1] - s_base[s_la[l]], nb = s_base[s_lb[l] + 1] - s_base[s_lb[l]];
            (void)na;
            const long long local = p - s_pp[l];
            const int qa = int(local / nb), qb = int(local - (long long)qa * nb);
            double score;
            int ngood;
            if (!score_pair(a, paf_f, l, pk_cell[s_base[s_la[l]] + qa], pk_cell[s_base[s_lb[l]] + qb], s_t, max_fail,
                            score, ngood))
                continue;
            const unsigned long long slot = atomicAdd(&s_nc, 1ull);
            if (slot < (unsigned long long)ws.cap_cands) {
                CandL c;
                c.score = score;
                c.ia = uint32_t(qa);
                c.ib = uint32_t(qb);
                c.lg = (uint32_t(l) << 24) | uint32_t(ngood);
                c.pad = 0;
                cand[slot] = c;
            }
        }
    }
    __syncthreads();
    if (s_nc > (unsigned long long)ws.cap_cands) {
        if (tid == 0) {
            report_capacity(a.st, gframe, kCapCands, (int)min(s_nc, 0x7fffffffull));
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
            if (a.debug) a.dbg_nconns[gframe] = 0;
        }
        return;
    }
    const int nc = (int)s_nc;

    // ---- 4. sort by (limb, -score, id_a, id_b) (paf.py:173) ----
    int n2 = 1;
    while (n2 < nc) n2 <<= 1;
    for (int e = nc + tid; e < n2; e += nthr) {
        CandL pad;
        pad.score = 0.0; pad.ia = 0xffffffffu; pad.ib = 0xffffffffu; pad.lg = 0x7f000000u; pad.pad = 0;
        cand[e] = pad;
    }
    __syncthreads();
    for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int i = tid; i < n2; i += nthr) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const CandL x = cand[i], y = cand[ixj];
                    const bool asc = (i & kk) == 0;
                    if (asc ? candl_less(y, x) : candl_less(x, y)) { cand[i] = y; cand[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
    for (int l = tid; l <= L; l += nthr) s_seg[l] = nc;
    __syncthreads();
    for (int e = tid; e < nc; e += nthr) {
        const int l = int(cand[e].lg >> 24);
        const int prev = e ? int(cand[e - 1].lg >> 24) : -1;
        for (int q = prev + 1; q <= l; ++q) s_seg[q] = e;
    }
    __syncthreads();

    // ---- 5. greedy per limb (paf.py:174-181), thread per limb ----
    for (int q = tid; q < ws.used_words; q += nthr) used[q] = 0u;
    __syncthreads();
    for (int l = tid; l < L; l += nthr) {
        uint32_t *ua = used + (size_t)l * 2 * ws.part_words, *ub = ua + ws.part_words;
        for (int e = s_seg[l]; e < s_seg[l + 1]; ++e) {
            CandL &c = cand[e];
            if ((ua[c.ia >> 5] >> (c.ia & 31)) & 1u) continue;
            if ((ub[c.ib >> 5] >> (c.ib & 31)) & 1u) continue;
            ua[c.ia >> 5] |= 1u << (c.ia & 31);
            ub[c.ib >> 5] |= 1u << (c.ib & 31);
            c.lg |= kLargeAccepted;
        }
    }
    __syncthreads();
    if (a.debug && tid == 0) {
        int q = 0;
        for (int e = 0; e < nc; ++e) {
            const CandL c = cand[e];
            if (!(c.lg & kLargeAccepted)) continue;
            const int l = int((c.lg >> 24) & 0x7f);
            if (q < a.cap_cands) {
                const size_t o = (size_t)gframe * a.cap_cands + q;
                a.dbg_conn_i[o * 3 + 0] = l;
                a.dbg_conn_i[o * 3 + 1] = s_base[s_la[l]] + int(c.ia);
                a.dbg_conn_i[o * 3 + 2] = s_base[s_lb[l]] + int(c.ib);
                a.dbg_conn_d[o * 2 + 0] = c.score;
                a.dbg_conn_d[o * 2 + 1] = __ddiv_rn((double)(c.lg & 0xffffffu), (double)a.n_samples);
            }
            ++q;
        }
        a.dbg_nconns[gframe] = min(q, a.cap_cands);
    }

    // ---- 6. assemble_humans (paf.py:241-271), one thread, limb-major order ----
    if (tid == 0) {
        int nh = 0, err = 0;
        for (int e = 0; e < nc && !err; ++e) {
            const CandL c = cand[e];
            if (!(c.lg & kLargeAccepted)) continue;
            const int l = int((c.lg >> 24) & 0x7f);
            const int a_part = s_la[l], b_part = s_lb[l];
            const int pa = s_base[a_part] + int(c.ia), pb = s_base[b_part] + int(c.ib);
            const int ha = owner[pa], hb = owner[pb];
            if (ha < 0 && hb < 0) {                                  // paf.py:246-253
                if (nh >= ws.cap_humans) { err = 1; break; }
                int *parts = h_parts + (size_t)nh * K;
                for (int k = 0; k < K; ++k) parts[k] = -1;
                parts[a_part] = pa;
                parts[b_part] = pb;
                h_order[(size_t)nh * K + 0] = int8_t(a_part);
                h_order[(size_t)nh * K + 1] = int8_t(b_part);
                h_n[nh] = 2;
                h_mask[nh] = (1u << a_part) | (1u << b_part);
                h_score[nh] = c.score;
                h_alive[nh] = 1;
                owner[pa] = nh;
                owner[pb] = nh;
                ++nh;
            } else if (ha >= 0 && hb >= 0) {
                if (ha == hb) {                                      // paf.py:255-256
                    h_score[ha] = dadd(h_score[ha], c.score);
                } else if ((h_mask[ha] & h_mask[hb]) == 0u) {        // paf.py:257-262
                    const int nB = h_n[hb];
                    int nA = h_n[ha];
                    for (int q = 0; q < nB; ++q) {
                        const int part = h_order[(size_t)hb * K + q];
                        const int pid = h_parts[(size_t)hb * K + part];
                        h_parts[(size_t)ha * K + part] = pid;
                        h_order[(size_t)ha * K + nA++] = int8_t(part);
                        owner[pid] = ha;
                    }
                    h_n[ha] = int8_t(nA);
                    h_mask[ha] |= h_mask[hb];
                    h_score[ha] = dadd(h_score[ha], dadd(h_score[hb], c.score));
                    h_alive[hb] = 0;
                }                                                    // else paf.py:263
            } else {                                                 // paf.py:264-271
                const int hidx = ha >= 0 ? ha : hb;
                const int part = ha >= 0 ? b_part : a_part;
                const int pid = ha >= 0 ? pb : pa;
                if (!((h_mask[hidx] >> part) & 1u)) {
                    const int nn = h_n[hidx];
                    h_parts[(size_t)hidx * K + part] = pid;
                    h_order[(size_t)hidx * K + nn] = int8_t(part);
                    h_n[hidx] = int8_t(nn + 1);
                    h_mask[hidx] |= 1u << part;
                    h_score[hidx] = dadd(h_score[hidx], c.score);
                    owner[pid] = hidx;
                }
            }
        }
        s_nh = nh;
        s_err = err;
    }
    __syncthreads();
    if (s_err) {
        if (tid == 0) {
            report_capacity(a.st, gframe, kCapHumans, ws.cap_humans + 1);
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
        }
        return;
    }
    const int nh = s_nh;

    // ---- 7. filters, scores (paf.py:273-287), stable rank (paf.py:288), output ----
    for (int hh = tid; hh < nh; hh += nthr) {
        bool keep = h_alive[hh] && h_n[hh] >= a.min_parts;
        double score = 0.0;
        if (keep) {
            const int np = h_n[hh];
            double f = 0.0, c = 0.0;
            for (int q = 0; q < np; ++q) {
                const double v = (double)pk_score[h_parts[(size_t)hh * K + h_order[(size_t)hh * K + q]]];
                if (q == 0) f = dadd(0.0, v);
                else neumaier_add(f, c, v);
            }
            if (c != 0.0 && isfinite(c)) f = dadd(f, c);
            score = __ddiv_rn(dadd(f, h_score[hh]), (double)np);
            keep = !(score < a.min_score);
        }
        h_score[hh] = score;
        h_pos[hh] = keep ? 1 : 0;
    }
    __syncthreads();
    if (tid == 0) {
        int nk = 0;
        for (int hh = 0; hh < nh; ++hh) nk += h_pos[hh];
        int base = nk ? atomicAdd(&a.st->pool_used, nk) : 0;
        if (base + nk > a.pool_cap) {
            report_capacity(a.st, gframe, kCapPool, base + nk);
            base = -1;
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
        } else {
            a.frame_first[gframe] = base;
            a.frame_count[gframe] = nk;
        }
        s_pool = base;
    }
    __syncthreads();
    if (s_pool < 0) return;
    for (int hh = tid; hh < nh; hh += nthr) {
        if (!h_pos[hh]) continue;
        const double s = h_score[hh];
        int pos = 0;
        for (int g = 0; g < nh; ++g) {
            if (!h_pos[g]) continue;
            const double sg = h_score[g];
            pos += (sg > s) || (sg == s && g < hh);
        }
        const size_t o = (size_t)(s_pool + pos);
        a.h_score[o] = s;
        a.h_nparts[o] = h_n[hh];
        const double sd = (double)a.stride_eff;
        for (int k = 0; k < K; ++k) {
            const int pid = h_parts[(size_t)hh * K + k];
            const size_t ok = o * K + k;
            if (pid < 0) {
                a.kp_x[ok] = 0.0; a.kp_y[ok] = 0.0; a.kp_score[ok] = 0.0f; a.kp_peak[ok] = -1;
            } else {
                const uint32_t cell = pk_cell[pid];
                const double i = (double)(cell >> 16), j = (double)(cell & 0xffff);
                a.kp_x[ok] = dadd(dmul(dadd(j, 0.5), sd), -0.5);
                a.kp_y[ok] = dadd(dmul(dadd(i, 0.5), sd), -0.5);
                a.kp_score[ok] = pk_score[pid];
                a.kp_peak[ok] = pid;
            }
        }
    }
}

size_t large_cand_bytes() { return sizeof(CandL); }

cudaError_t launch_parse_large(const ParseArgs &a, const LargeWs &ws, int B, cudaStream_t s)
{
    if (B == 0) return cudaSuccess;
    k_parse_large<<<B, kLargeThreads, 0, s>>>(a, ws);
    return cudaGetLastError();
}

}  // namespace pf
