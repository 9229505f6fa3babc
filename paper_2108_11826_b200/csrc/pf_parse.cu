// pf_parse.cu — per-frame limb scoring, greedy matching and human assembly.
//
// One CTA (4 warps) per frame (frames are independent; paf.py:292-305 is
// pure).  Everything after peak extraction happens on chip:
//
//   1. peak ids      — rank-sort each part's peaks by (score desc, row, col)
//                      (paf.py:104) straight from the NMS slab and prefix the
//                      parts (paf.py:298-303)
//   2. line integral — a 16-lane group scores one (limb, a, b) pair: lane u
//                      takes sample u (nearest cell, paf.py:138-145), so all
//                      PAF reads of a pair are in flight together; the fp64
//                      mean is then summed in sample order through shuffles
//                      (paf.py:144 `total += d`, the reference's rounding
//                      order) and the good count is a ballot.  Gate
//                      good >= min && score > 0 (paf.py:162).  In Mode U the
//                      PAF value of a full-res cell is re-derived from the
//                      low-res PAF with the operators.py:102-107 fp64 formula.
//   3. greedy        — bitonic sort of the gated candidates by
//                      (limb, -score, id_a, id_b) (paf.py:173) in shared
//                      memory (crowded frames spill past kCandSmem entries to
//                      a per-frame global slab), then one warp per limb walks
//                      its segment with used-bitmaps (paf.py:174-181)
//   4. assembly      — one thread replays assemble_humans' order-dependent
//                      branches exactly (paf.py:241-271) on shared tables
//                      (owner per peak, part slots + dict insertion order +
//                      part bitmask per human)
//   5. finalise      — per-human Neumaier keypoint sum (CPython 3.12 sum()),
//                      filters (paf.py:276-281), stable rank by -score
//                      (paf.py:288), cell_to_pixel (types.py:233-235), and a
//                      compact write into the output pool.
#include <algorithm>

#include "pf_score.cuh"

namespace pf {

#ifndef PF_PAR_ASM_MIN
#define PF_PAR_ASM_MIN 96
#endif
constexpr int kParAsmMin = PF_PAR_ASM_MIN;   // accepted connections from which the assembly runs limb-parallel

struct Cand {
    double score;
    uint32_t ab;     // id_a << 16 | id_b ; bit 31 = accepted
    uint32_t lg;     // limb << 24 | n_good
};

constexpr uint32_t kAccepted = 0x80000000u;

__device__ __forceinline__ bool cand_less(const Cand &x, const Cand &y)
{
    const uint32_t lx = x.lg >> 24, ly = y.lg >> 24;
    if (lx != ly) return lx < ly;
    if (x.score != y.score) return x.score > y.score;
    return (x.ab & 0x7fffffffu) < (y.ab & 0x7fffffffu);  // (id_a, id_b) lexicographic
}

// Candidate storage: the first kCandSmem entries in shared memory, the rest
// (crowded frames only) in this frame's global spill slab.
// An accepted connection, parts resolved, for the serial assembly.
struct ConnRec {
    uint16_t pa, pb;
    uint8_t a_part, b_part;
    uint16_t pad;
    double score;
};

struct CandStore {
    Cand *s;
    Cand *g;
    int ns;              // entries in shared memory
    __device__ __forceinline__ Cand &operator[](int i) const { return i < ns ? s[i] : g[i - ns]; }
};

// Crowded frames (candidates past the shared-memory part): the accepted
// connections, as ConnRec records, compacted in place over the sorted
// candidates in windows (every read of a window happens before its writes,
// which never pass the window's end).  Kept out of line so the usual path's
// register allocation is not disturbed.  Returns the number of records.
__device__ __noinline__ int compact_crowded(const CandStore cand, int nc, const int8_t *s_la, const int8_t *s_lb,
                                            int *s_wacc)
{
    constexpr int kWin = 4;
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, n_warps = nthr >> 5;
    int kbase = 0;                                           // block-uniform
    for (int w0 = 0; w0 < nc; w0 += nthr * kWin) {
        Cand v[kWin];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
            const int e = w0 + tid * kWin + j;
            if (e < nc) v[j] = cand[e];
            else v[j].ab = 0u;
            cnt += (v[j].ab & kAccepted) ? 1 : 0;
        }
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += x;
        }
        if (lane == kWarp - 1) s_wacc[warp] = incl;
        __syncthreads();
        int off = kbase + incl - cnt, tot = 0;
        for (int w2 = 0; w2 < n_warps; ++w2) {
            if (w2 < warp) off += s_wacc[w2];
            tot += s_wacc[w2];
        }
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
            if (!(v[j].ab & kAccepted)) continue;
            const int l = int(v[j].lg >> 24);
            ConnRec r;
            r.pa = uint16_t((v[j].ab >> 16) & 0x7fff);
            r.pb = uint16_t(v[j].ab & 0xffff);
            r.a_part = uint8_t(s_la[l]);
            r.b_part = uint8_t(s_lb[l]);
            r.pad = 0;
            r.score = v[j].score;
            *reinterpret_cast<ConnRec *>(&cand[off++]) = r;
        }
        kbase += tot;
        __syncthreads();
    }
    return kbase;
}

#ifndef PF_PARSE_MINB
#define PF_PARSE_MINB 8
#endif
#ifndef PF_PARSE_FIN_MINB
#define PF_PARSE_FIN_MINB 16
#endif
// SPLIT = false: the whole parse of a frame in this CTA.  SPLIT = true: peaks
// ranked by k_parse_peaks and pairs scored by k_score_pairs (all frames'
// pairs spread over the whole GPU); this CTA takes the frame's gated
// candidates from HBM and runs steps 4-7 (sort, greedy, assembly, scores).
// CROWD (split only): a frame whose gated candidates exceed the 64-thread
// CTA's shared store (kCandSmemSplit) is listed by k_parse_frames<true> and
// finished here instead — 512 threads, kCandSmemCrowd candidates and their
// connection records in shared memory — so crowded frames (C3: ~2k
// candidates) rank per limb in shared memory instead of a bitonic sort
// through L2 by 64 threads.
template <bool SPLIT, bool COUNT, bool CROWD>
__device__ __forceinline__ void parse_frame(const ParseArgs &a, const int b)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int K = a.topo.K, L = a.topo.L;
    const int gframe = a.frame_base + b;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int warp = tid / kWarp, lane = tid % kWarp, n_warps = nthr / kWarp;

    __shared__ int s_base[PF_MAX_KEYPOINTS + 1];
    __shared__ int s_pp[PF_MAX_LIMBS + 1];      // pair prefix per limb
    __shared__ int s_seg[PF_MAX_LIMBS + 1];     // candidate segment start per limb
    __shared__ int s_err, s_errval, s_ncand, s_nh, s_pool_base, s_nacc;
    __shared__ int s_wacc[kParseMaxThreads / kWarp];
    __shared__ int s_lcnt[PF_MAX_LIMBS], s_lcur[PF_MAX_LIMBS];
    __shared__ int s_aseg[PF_MAX_LIMBS + 1];    // accepted connections per limb, then their prefix
    // split: fewer candidates in shared memory and the peak table read from
    // the k_parse_peaks slab, so more frames stay resident per SM
    constexpr int CS = CROWD ? kCandSmemCrowd : (SPLIT ? kCandSmemSplit : kCandSmem);
    __shared__ uint16_t s_bucket[CS], s_order[CS];   // by limb; sorted within limb
    __shared__ int8_t s_la[PF_MAX_LIMBS], s_lb[PF_MAX_LIMBS];
    __shared__ int16_t s_cx[PF_MAX_LIMBS], s_cy[PF_MAX_LIMBS];
    __shared__ double s_t[kParseTTab];          // u / (n - 1), paf.py:139
    for (int u = tid; u < kParseTTab && u < a.n_samples; u += nthr)
        s_t[u] = __ddiv_rn((double)u, (double)(a.n_samples - 1));
    for (int l = tid; l < L; l += nthr) {
        s_la[l] = a.topo.la[l]; s_lb[l] = a.topo.lb[l];
        s_cx[l] = a.topo.cx[l]; s_cy[l] = a.topo.cy[l];
    }

    // ---- shared layout (sizes from the caps; see parse_smem_bytes) ----
    Cand *cand_s = reinterpret_cast<Cand *>(smem_raw);                       // CS
    double *h_score = reinterpret_cast<double *>(cand_s + CS);               // cap_humans (conn, then final)
    uint32_t *p_cell = SPLIT ? const_cast<uint32_t *>(a.pk_cell) + (size_t)b * a.cap_frame
                             : reinterpret_cast<uint32_t *>(h_score + a.cap_humans);   // cap_frame
    float *p_score = SPLIT ? const_cast<float *>(a.pk_score) + (size_t)b * a.cap_frame
                           : reinterpret_cast<float *>(p_cell + a.cap_frame);          // cap_frame
    uint32_t *h_mask = SPLIT ? reinterpret_cast<uint32_t *>(h_score + a.cap_humans)
                             : reinterpret_cast<uint32_t *>(p_score + a.cap_frame);    // cap_humans
    int *h_pos = reinterpret_cast<int *>(h_mask + a.cap_humans);             // cap_humans
    const int pm_words = (a.cap_part + 31) / 32;
    uint32_t *used = reinterpret_cast<uint32_t *>(h_pos + a.cap_humans);     // used_words(), see parse_smem_bytes
    int16_t *owner = reinterpret_cast<int16_t *>(used + L * 2 * pm_words);  // cap_frame
    int16_t *h_parts = owner + a.cap_frame;                                   // cap_humans*K
    int8_t *h_order = reinterpret_cast<int8_t *>(h_parts + a.cap_humans * K); // cap_humans*K
    int8_t *h_n = h_order + a.cap_humans * K;                                 // cap_humans
    int8_t *h_alive = h_n + a.cap_humans;                                     // cap_humans
    ConnRec *conn = reinterpret_cast<ConnRec *>((reinterpret_cast<uintptr_t>(h_alive + a.cap_humans) + 15) &
                                                ~uintptr_t(15));                 // CS accepted connections
    // split: the frame's candidates already sit in cand_g; entries past the
    // shared part are used (and sorted) in place there
    const CandStore cand{cand_s,
                         SPLIT ? a.cand_g + (size_t)b * a.cap_cands + CS
                               : reinterpret_cast<Cand *>(a.cand_spill) + (size_t)b * (a.cap_cands - kCandSmem),
                         CS};

    // ---- 1. peak counts, prefix, capacity checks; reset counters ----
    if (tid == 0) { s_err = 0; s_ncand = 0; }
    if (SPLIT) {
        for (int k = tid; k <= K; k += nthr) s_base[k] = a.pk_base[(size_t)b * (K + 1) + k];
        if (tid == 0) {
            const int2 e = a.ferr[b];
            s_err = e.x; s_errval = e.y;
            s_ncand = __ldcg(a.cand_n + b);
        }
    } else if (tid < K) {
        const int c = a.counts[(size_t)b * K + tid];
        a.counts[(size_t)b * K + tid] = 0;   // ready for the next launch
        s_base[tid + 1] = c;
    }
    __syncthreads();
    if (!SPLIT && tid == 0) {
        s_base[0] = 0;
        int err = 0, val = 0;
        for (int k = 0; k < K; ++k) {
            const int c = s_base[k + 1];
            if (c > a.cap_part && !err) { err = kCapPart; val = c; }
            s_base[k + 1] = s_base[k] + c;
        }
        if (!err && s_base[K] > a.cap_frame) { err = kCapFrame; val = s_base[K]; }
        s_err = err; s_errval = val;
    }
    __syncthreads();
    if (s_err) {
        if (tid == 0) {
            report_capacity(a.st, gframe, s_err, s_errval);
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
            if (a.debug) { a.dbg_npeaks[gframe] = 0; a.dbg_nconns[gframe] = 0; }
        }
        return;
    }
    if (SPLIT && !CROWD && a.crowd_frames && s_ncand > CS) {   // block-uniform: k_parse_crowd finishes it
        if (tid == 0) a.crowd_frames[atomicAdd(a.crowd_frames + a.crowd_cap, 1)] = b;
        return;
    }
    const int P = s_base[K];

    // ---- 2. rank-sort each part's peaks (read straight from the NMS slab) ----
    if (SPLIT) {
        for (int e = tid; e < P; e += nthr) owner[e] = -1;
    }
    for (int e = tid; !SPLIT && e < P; e += nthr) {
        int part = 0;
        while (e >= s_base[part + 1]) ++part;
        const uint2 *slab = a.peaks + ((size_t)b * K + part) * a.cap_part;
        const int np = s_base[part + 1] - s_base[part];
        const uint2 v = __ldg(slab + (e - s_base[part]));
        const float vs = __uint_as_float(v.x);
        int rank = 0;
        for (int q = 0; q < np; ++q) {
            const uint2 u = __ldg(slab + q);
            const float us = __uint_as_float(u.x);
            rank += (us > vs) || (us == vs && u.y < v.y);
        }
        p_cell[s_base[part] + rank] = v.y;
        p_score[s_base[part] + rank] = vs;
        owner[e] = -1;
    }
    if (!SPLIT && tid == 0) {
        int acc = 0;
        for (int l = 0; l < L; ++l) {
            s_pp[l] = acc;
            const int na = s_base[s_la[l] + 1] - s_base[s_la[l]];
            const int nb = s_base[s_lb[l] + 1] - s_base[s_lb[l]];
            acc += na * nb;
        }
        s_pp[L] = acc;
    }
    for (int l = tid; l <= L; l += nthr) s_seg[l] = 0x7fffffff;
    for (int l = tid; l < L; l += nthr) s_lcnt[l] = 0;
    __syncthreads();
    if (!SPLIT && a.debug) {
        for (int e = tid; e < P; e += nthr) {
            int part = 0;
            while (e >= s_base[part + 1]) ++part;
            a.dbg_peaks[(size_t)gframe * a.cap_frame + e] =
                make_int4(part, int(p_cell[e] >> 16), int(p_cell[e] & 0xffff), __float_as_int(p_score[e]));
        }
        if (tid == 0) a.dbg_npeaks[gframe] = P;
    }

    // ---- 3. line integral: a lane per (limb, a, b) pair (paf.py:149-165).
    // The lane walks the samples in order (paf.py:138-145), so the fp64
    // running total is the reference's `total += d` exactly, and it leaves a
    // pair as soon as the pair can no longer pass the gate (more failing
    // samples than n - good_need): such pairs are never candidates.
    const float *paf_f = a.paf + (size_t)b * (2 * L) * a.h * a.w;
    const int n_pairs = s_pp[L];
    const int n = a.n_samples;
    const int max_fail = n - a.good_need;            // < 0: nothing can pass
    if (!SPLIT && max_fail >= 0) {
        for (int p = tid; p < n_pairs; p += nthr) {
            int l = 0;
            while (p >= s_pp[l + 1]) ++l;
            const int pa_part = s_la[l], pb_part = s_lb[l];
            const int nb = s_base[pb_part + 1] - s_base[pb_part];
            const int local = p - s_pp[l];
            const int qa = local / nb;
            const int ia = s_base[pa_part] + qa;
            const int ib = s_base[pb_part] + (local - qa * nb);
            double score;
            int ngood;
            if (!score_pair<COUNT>(a, paf_f, l, p_cell[ia], p_cell[ib], s_t, max_fail, score, ngood,
                                   COUNT ? a.paf_touch + (size_t)gframe * a.touch_words : nullptr))
                continue;
            const int slot = atomicAdd(&s_ncand, 1);
            atomicAdd(&s_lcnt[l], 1);
            if (slot < a.cap_cands) {
                Cand c;
                c.score = score;
                c.ab = (uint32_t(ia) << 16) | uint32_t(ib);
                c.lg = (uint32_t(l) << 24) | uint32_t(ngood);
                cand[slot] = c;
            }
        }
    }
    if (SPLIT) {
        const int ncg = __ldcg(a.cand_n + b);
        const Cand *cg = a.cand_g + (size_t)b * a.cap_cands;
        for (int i = tid; i < ncg && i < a.cap_cands; i += nthr) {
            const Cand c = cg[i];
            if (i < CS) cand_s[i] = c;
            atomicAdd(&s_lcnt[c.lg >> 24], 1);
        }
        if (tid == 0) s_ncand = ncg;
    }
    __syncthreads();
    const int nc = s_ncand;
    if (nc > a.cap_cands) {
        if (tid == 0) {
            report_capacity(a.st, gframe, kCapCands, nc);
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
            if (a.debug) a.dbg_nconns[gframe] = 0;
        }
        return;
    }

    // ---- 4+5. order candidates by (limb, -score, id_a, id_b) (paf.py:173)
    // and run the greedy per limb (paf.py:174-181).  Usual frames (all
    // candidates in shared memory): bucket by limb, then one warp per limb
    // ranks its bucket (the key is a total order, so ranks are distinct) and
    // its lane 0 walks the ranks with used-bitmaps — no CTA-wide sort.
    // Crowded frames (spill slab): bitonic sort over the whole store.
    const bool fast = nc <= CS;
    if (fast) {
        if (tid == 0) {
            int acc = 0;
            for (int l = 0; l < L; ++l) {
                s_seg[l] = acc;
                s_lcur[l] = acc;
                acc += s_lcnt[l];
            }
            s_seg[L] = acc;
        }
        __syncthreads();
        for (int i = tid; i < nc; i += nthr) {
            const int l = int(cand_s[i].lg >> 24);
            s_bucket[atomicAdd(&s_lcur[l], 1)] = uint16_t(i);
        }
        __syncthreads();
    } else {
        int n2 = 1;
        while (n2 < nc) n2 <<= 1;
        for (int e = nc + tid; e < n2; e += nthr) {
            Cand pad;
            pad.score = 0.0; pad.ab = 0x7fffffffu; pad.lg = 0xff000000u;
            cand[e] = pad;
        }
        __syncthreads();
        for (int kk = 2; kk <= n2; kk <<= 1) {
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                for (int i = tid; i < n2; i += nthr) {
                    const int ixj = i ^ jj;
                    if (ixj > i) {
                        const Cand x = cand[i], y = cand[ixj];
                        const bool asc = (i & kk) == 0;
                        if (asc ? cand_less(y, x) : cand_less(x, y)) { cand[i] = y; cand[ixj] = x; }
                    }
                }
                __syncthreads();
            }
        }
        // segment starts: first index of each limb
        for (int e = tid; e < nc; e += nthr) {
            const int l = int(cand[e].lg >> 24);
            const int prev = e ? int(cand[e - 1].lg >> 24) : -1;
            for (int q = prev + 1; q <= l; ++q) s_seg[q] = e;
        }
        __syncthreads();
        if (tid == 0) {
            int next = nc;
            for (int l = L; l >= 0; --l) {
                if (s_seg[l] == 0x7fffffff) s_seg[l] = next;
                next = s_seg[l];
            }
        }
        __syncthreads();
    }
    // sorted position e -> candidate
    auto at = [&](int e) -> Cand & { return fast ? cand_s[s_order[e]] : cand[e]; };

    if (fast) {
        // rank within the limb, thread per candidate (the key is a total
        // order, so ranks are distinct) ...
        for (int k = tid; k < nc; k += nthr) {
            const int i = s_bucket[k];
            const Cand c = cand_s[i];
            const int l = int(c.lg >> 24);
            const int s0 = s_seg[l], s1 = s_seg[l + 1];
            int rank = 0;
            for (int k2 = s0; k2 < s1; ++k2) rank += cand_less(cand_s[s_bucket[k2]], c);
            s_order[s0 + rank] = uint16_t(i);
        }
    }
    // every limb's greedy walk at once, thread per limb (used bitmaps over
    // the peak's index within its part)
    for (int q = tid; q < L * 2 * pm_words; q += nthr) used[q] = 0u;
    __syncthreads();
    if (fast) {
        for (int l = tid; l < L; l += nthr) {
            uint32_t *used_a = used + l * 2 * pm_words, *used_b = used_a + pm_words;
            const int ba = s_base[s_la[l]], bb = s_base[s_lb[l]];
            int acc = 0;
            for (int e = s_seg[l], e1 = s_seg[l + 1]; e < e1; ++e) {
                Cand &c = cand_s[s_order[e]];
                const uint32_t ab = c.ab;
                const int ia = int((ab >> 16) & 0x7fff) - ba, ib = int(ab & 0xffff) - bb;
                if ((used_a[ia >> 5] >> (ia & 31)) & 1u) continue;
                if ((used_b[ib >> 5] >> (ib & 31)) & 1u) continue;
                used_a[ia >> 5] |= 1u << (ia & 31);
                used_b[ib >> 5] |= 1u << (ib & 31);
                c.ab = ab | kAccepted;
                ++acc;
            }
            s_aseg[l] = acc;
        }
    } else {                                                 // crowded: the bitonic-sorted store
        for (int l = tid; l < L; l += nthr) {
            uint32_t *used_a = used + l * 2 * pm_words, *used_b = used_a + pm_words;
            const int ba = s_base[s_la[l]], bb = s_base[s_lb[l]];
            int acc = 0;
            for (int e = s_seg[l], e1 = s_seg[l + 1]; e < e1; ++e) {
                Cand &c = cand[e];
                const uint32_t ab = c.ab;
                const int ia = int((ab >> 16) & 0x7fff) - ba, ib = int(ab & 0xffff) - bb;
                if ((used_a[ia >> 5] >> (ia & 31)) & 1u) continue;
                if ((used_b[ib >> 5] >> (ib & 31)) & 1u) continue;
                used_a[ia >> 5] |= 1u << (ia & 31);
                used_b[ib >> 5] |= 1u << (ib & 31);
                c.ab = ab | kAccepted;
                ++acc;
            }
            s_aseg[l] = acc;
        }
    }
    __syncthreads();
    if (a.debug && tid == 0) {
        int q = 0;
        for (int e = 0; e < nc; ++e) {
            const Cand ce = at(e);
            if (!(ce.ab & kAccepted)) continue;
            const size_t o = (size_t)gframe * a.cap_cands + q;
            a.dbg_conn_i[o * 3 + 0] = int(ce.lg >> 24);
            a.dbg_conn_i[o * 3 + 1] = int((ce.ab >> 16) & 0x7fff);
            a.dbg_conn_i[o * 3 + 2] = int(ce.ab & 0xffff);
            a.dbg_conn_d[o * 2 + 0] = ce.score;
            a.dbg_conn_d[o * 2 + 1] = __ddiv_rn((double)(ce.lg & 0xffffffu), (double)n);
            ++q;
        }
        a.dbg_nconns[gframe] = q;
    }

    // ---- 6. assembly: exact sequential replay (paf.py:241-271) ----
    // Usual frames: the accepted connections are first compacted in sorted
    // order into self-contained records (parts resolved), so the serial
    // replay reads one record per connection at an address that does not
    // depend on the state it is updating.
    if (fast) {
        const int per = (nc + nthr - 1) / nthr;             // consecutive sorted positions per thread
        const int e0 = tid * per;
        int cnt = 0;
        for (int j = 0; j < per; ++j)
            cnt += (e0 + j < nc) && (cand_s[s_order[e0 + j]].ab & kAccepted) ? 1 : 0;
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        if (lane == kWarp - 1) s_wacc[warp] = incl;
        __syncthreads();
        int off = incl - cnt;
        for (int w2 = 0; w2 < warp; ++w2) off += s_wacc[w2];
        if (tid == nthr - 1) s_nacc = off + cnt;
        for (int j = 0; j < per && e0 + j < nc; ++j) {
            const Cand c = cand_s[s_order[e0 + j]];
            if (!(c.ab & kAccepted)) continue;
            const int l = int(c.lg >> 24);
            ConnRec r;
            r.pa = uint16_t((c.ab >> 16) & 0x7fff);
            r.pb = uint16_t(c.ab & 0xffff);
            r.a_part = uint8_t(s_la[l]);
            r.b_part = uint8_t(s_lb[l]);
            r.score = c.score;
            conn[off++] = r;
        }
        __syncthreads();
    } else {
        const int kb = compact_crowded(cand, nc, s_la, s_lb, s_wacc);
        if (tid == 0) s_nacc = kb;
        __syncthreads();
    }
    // one replay step of paf.py:241-271 (shared by the serial replay and the
    // serial fallback of a conflicting limb)
    auto step = [&](const ConnRec r, int &nh, int &err) {
        const int a_part = r.a_part, b_part = r.b_part, pa = r.pa, pb = r.pb;
        const double cscore = r.score;
        const int ha = owner[pa], hb = owner[pb];
        if (ha < 0 && hb < 0) {                                  // paf.py:246-253
            if (nh >= a.cap_humans) { err = 1; return; }
            int16_t *parts = h_parts + nh * K;
            for (int k = 0; k < K; ++k) parts[k] = -1;
            parts[a_part] = int16_t(pa);
            parts[b_part] = int16_t(pb);
            h_order[nh * K + 0] = int8_t(a_part);
            h_order[nh * K + 1] = int8_t(b_part);
            h_n[nh] = 2;
            h_mask[nh] = (1u << a_part) | (1u << b_part);
            h_score[nh] = cscore;
            h_alive[nh] = 1;
            owner[pa] = int16_t(nh);
            owner[pb] = int16_t(nh);
            ++nh;
        } else if (ha >= 0 && hb >= 0) {
            if (ha == hb) {                                      // paf.py:255-256
                h_score[ha] = dadd(h_score[ha], cscore);
            } else if ((h_mask[ha] & h_mask[hb]) == 0u) {        // paf.py:257-262
                const int nB = h_n[hb];
                int nA = h_n[ha];
                for (int q = 0; q < nB; ++q) {
                    const int part = h_order[hb * K + q];
                    const int pid = h_parts[hb * K + part];
                    h_parts[ha * K + part] = int16_t(pid);
                    h_order[ha * K + nA++] = int8_t(part);
                    owner[pid] = int16_t(ha);
                }
                h_n[ha] = int8_t(nA);
                h_mask[ha] |= h_mask[hb];
                h_score[ha] = dadd(h_score[ha], dadd(h_score[hb], cscore));
                h_alive[hb] = 0;
            }                                                    // else paf.py:263
        } else {                                                 // paf.py:264-271
            const int hidx = ha >= 0 ? ha : hb;
            const int part = ha >= 0 ? b_part : a_part;
            const int pid = ha >= 0 ? pb : pa;
            // one round of independent loads, then the stores
            const uint32_t m = h_mask[hidx];
            const int nn = h_n[hidx];
            const double hs = h_score[hidx];
            if (!((m >> part) & 1u)) {
                h_parts[hidx * K + part] = int16_t(pid);
                h_order[hidx * K + nn] = int8_t(part);
                h_n[hidx] = int8_t(nn + 1);
                h_mask[hidx] = m | (1u << part);
                h_score[hidx] = dadd(hs, cscore);
                owner[pid] = int16_t(hidx);
            }
        }
    };
    auto rec = [&](int e) -> ConnRec {
        return fast ? conn[e] : *reinterpret_cast<const ConnRec *>(&cand[e]);
    };
    const int n_it = s_nacc;
    if (n_it < kParAsmMin) {
        if (tid == 0) {
            int nh = 0, err = 0;
            if (fast) {
                for (int e = 0; e < n_it && !err; ++e) step(conn[e], nh, err);
            } else {
                for (int e = 0; e < n_it && !err; ++e) step(*reinterpret_cast<const ConnRec *>(&cand[e]), nh, err);
            }
            s_nh = nh;
            s_err = err;
        }
    } else {
        // Limb-parallel replay (crowded frames).  Connections of one limb
        // are a matching (distinct peaks), so two of them interact only if
        // they touch the same human: when the humans they touch are pairwise
        // distinct, every one's effect stays inside its own humans and peaks,
        // new humans take their indices in acceptance order (a prefix sum)
        // and the result equals the sequential replay.  A limb where two
        // connections share a human is replayed serially.  h_pos counts the
        // touches (it is free until step 7).
        if (tid == 0) {
            int acc = 0;
            for (int l = 0; l < L; ++l) {
                const int c = s_aseg[l];
                s_aseg[l] = acc;
                acc += c;
            }
            s_aseg[L] = acc;
        }
        for (int hh = tid; hh < a.cap_humans; hh += nthr) h_pos[hh] = 0;
        __syncthreads();
        int nh = 0, err = 0;
        for (int l = 0; l < L && !err; ++l) {
            const int e0 = s_aseg[l], m = s_aseg[l + 1] - e0;
            if (m == 0) continue;
            const int per = (m + nthr - 1) / nthr, i0 = tid * per;
            int n_new = 0;
            for (int j = 0; j < per && i0 + j < m; ++j) {
                const ConnRec r = rec(e0 + i0 + j);
                const int ha = owner[r.pa], hb = owner[r.pb];
                if (ha >= 0) atomicAdd(&h_pos[ha], 1);
                if (hb >= 0 && hb != ha) atomicAdd(&h_pos[hb], 1);
                n_new += (ha < 0 && hb < 0) ? 1 : 0;
            }
            int incl = n_new;
#pragma unroll
            for (int d = 1; d < kWarp; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            if (lane == kWarp - 1) s_wacc[warp] = incl;
            __syncthreads();
            bool clash = false;
            for (int j = 0; j < per && i0 + j < m; ++j) {
                const ConnRec r = rec(e0 + i0 + j);
                const int ha = owner[r.pa], hb = owner[r.pb];
                clash |= (ha >= 0 && h_pos[ha] > 1) || (hb >= 0 && h_pos[hb] > 1);
            }
            int off = incl - n_new, tot = 0;
            for (int w2 = 0; w2 < n_warps; ++w2) {
                if (w2 < warp) off += s_wacc[w2];
                tot += s_wacc[w2];
            }
            const bool any_clash = __syncthreads_or(clash);
            // touches back to zero (nothing has moved yet: same owners)
            for (int j = 0; j < per && i0 + j < m; ++j) {
                const ConnRec r = rec(e0 + i0 + j);
                const int ha = owner[r.pa], hb = owner[r.pb];
                if (ha >= 0) h_pos[ha] = 0;
                if (hb >= 0) h_pos[hb] = 0;
            }
            __syncthreads();
            if (any_clash) {
                if (tid == 0) {
                    int nh0 = nh, e0r = 0;
                    for (int e = e0; e < e0 + m && !e0r; ++e) step(rec(e), nh0, e0r);
                    s_nh = nh0;
                    s_err = e0r;
                }
                __syncthreads();
                nh = s_nh;
                err = s_err;
                __syncthreads();
                continue;
            }
            if (nh + tot > a.cap_humans) {                       // block-uniform
                err = 1;
                break;
            }
            int idx = nh + off;
            for (int j = 0; j < per && i0 + j < m; ++j) {
                const ConnRec r = rec(e0 + i0 + j);
                const int ha = owner[r.pa], hb = owner[r.pb];
                int nh_local = idx, e_local = 0;
                step(r, nh_local, e_local);                      // touches only its own humans
                idx += (ha < 0 && hb < 0) ? 1 : 0;
            }
            nh += tot;
            __syncthreads();
        }
        if (tid == 0) {
            s_nh = nh;
            s_err = err;
        }
    }
    __syncthreads();
    if (s_err) {
        if (tid == 0) {
            report_capacity(a.st, gframe, kCapHumans, a.cap_humans + 1);
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
        }
        return;
    }
    const int nh = s_nh;

    // ---- 7. filters and scores (paf.py:273-287) ----
    for (int hh = tid; hh < nh; hh += nthr) {
        bool keep = h_alive[hh] && h_n[hh] >= a.min_parts;
        double score = 0.0;
        if (keep) {
            const int np = h_n[hh];
            double f = 0.0, c = 0.0;
            for (int q = 0; q < np; ++q) {
                const double v = (double)p_score[h_parts[hh * K + h_order[hh * K + q]]];
                if (q == 0) f = dadd(0.0, v);
                else neumaier_add(f, c, v);
            }
            if (c != 0.0 && isfinite(c)) f = dadd(f, c);
            score = __ddiv_rn(dadd(f, h_score[hh]), (double)np);
            keep = !(score < a.min_score);
        }
        h_score[hh] = score;          // connection sum no longer needed
        h_pos[hh] = keep ? 1 : 0;
    }
    __syncthreads();
    // the frame's slice of the pool: thread 0's atomic is in flight while
    // the ranks are computed
    int pool_base = 0, nk = 0;
    if (tid == 0) {
        for (int hh = 0; hh < nh; ++hh) nk += h_pos[hh];
        if (nk) pool_base = atomicAdd(&a.st->pool_used, nk);
    }
    // stable rank by -score among kept humans (paf.py:288)
    for (int hh = tid; hh < nh; hh += nthr) {
        if (!h_pos[hh]) continue;
        const double s = h_score[hh];
        int pos = 0;
        for (int g = 0; g < nh; ++g) {
            if (!h_pos[g]) continue;
            const double sg = h_score[g];
            pos += (sg > s) || (sg == s && g < hh);
        }
        h_mask[hh] = uint32_t(pos);   // part mask no longer needed; reuse as rank
    }
    __syncthreads();
    if (tid == 0) {
        const int base = pool_base;
        if (base + nk > a.pool_cap) {
            report_capacity(a.st, gframe, kCapPool, base + nk);
            s_pool_base = -1;
            a.frame_first[gframe] = 0;
            a.frame_count[gframe] = 0;
        } else {
            s_pool_base = base;
            a.frame_first[gframe] = base;
            a.frame_count[gframe] = nk;
        }
    }
    __syncthreads();
    if (s_pool_base < 0) return;
    const int base = s_pool_base;
    const double sd = (double)a.stride_eff;
    for (int x = tid; x < nh * K; x += nthr) {
        const int hh = x / K, k = x - hh * K;
        if (!h_pos[hh]) continue;
        const size_t o = (size_t)(base + int(h_mask[hh]));
        if (k == 0) {
            a.h_score[o] = h_score[hh];
            a.h_nparts[o] = h_n[hh];
        }
        const int pid = h_parts[hh * K + k];
        const size_t ok = o * K + k;
        if (pid < 0) {
            a.kp_x[ok] = 0.0; a.kp_y[ok] = 0.0; a.kp_score[ok] = 0.0f; a.kp_peak[ok] = -1;
        } else {
            const uint32_t cell = p_cell[pid];
            const double i = (double)(cell >> 16), j = (double)(cell & 0xffff);
            a.kp_x[ok] = dadd(dmul(dadd(j, 0.5), sd), -0.5);
            a.kp_y[ok] = dadd(dmul(dadd(i, 0.5), sd), -0.5);
            a.kp_score[ok] = p_score[pid];
            a.kp_peak[ok] = pid;
        }
    }
}

template <bool SPLIT, bool COUNT = false>
__global__ void __launch_bounds__(SPLIT ? kParseFinThreads : kParseThreads, SPLIT ? PF_PARSE_FIN_MINB : PF_PARSE_MINB)
k_parse_frames(const ParseArgs a)
{
    pdl_wait();                                          // peaks / candidates of the previous kernels
    parse_frame<SPLIT, COUNT, false>(a, blockIdx.x);
}

// Small batches (fewer frames than SMs): the one-kernel parse with a wide
// CTA per frame, so the line integrals of a frame's pairs run in one round
// instead of several (single-frame latency; same function, same results).
__global__ void __launch_bounds__(kParseWideThreads, 1)
k_parse_frames_wide(const ParseArgs a)
{
    pdl_wait();
    parse_frame<false, false, false>(a, blockIdx.x);
}

// Crowded frames listed by k_parse_frames<true> (persistent over the list).
__global__ void __launch_bounds__(kParseCrowdThreads, 1)
k_parse_crowd(const ParseArgs a)
{
    const int n = __ldcg(a.crowd_frames + a.crowd_cap);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        parse_frame<true, false, true>(a, __ldcg(a.crowd_frames + i));
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Split parse (PF_OPT_PARSE_SPLIT): the per-frame CTA no longer carries the
// gather-bound line integral.
//   k_parse_peaks  — warp per frame: peak counts, capacity checks, rank sort
//                    of each part (paf.py:104), ids, pair prefix per limb;
//   k_pair_scan    — exclusive scan of the frames' pair counts;
//   k_score_pairs  — thread per (frame, limb, a, b) pair over ALL frames
//                    (score_pair), gated candidates appended to the frame's
//                    list in HBM (order irrelevant: the finish step sorts);
//   k_parse_frames<true> — steps 4-7 per frame.
constexpr int kPeakWarps = 4;        // warps per k_parse_peaks CTA
constexpr int kScoreThreads = 256;

// WPF warps per frame, kPeakWarps / WPF frames per CTA.  Large batches keep a
// warp per frame (WPF = 1); batches of at most a few frames per SM (C3's 256
// crowded frames: ≈720 peaks per frame, 22 rank loops of ≈40 peaks per
// lane at WPF = 1) spread each frame's rank sort over the CTA (WPF = 4).
template <int WPF>
__global__ void __launch_bounds__(kPeakWarps * kWarp)
k_parse_peaks(const ParseArgs a, int B)
{
    constexpr int kFrames = kPeakWarps / WPF;
    const int K = a.topo.K, L = a.topo.L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fw = warp / WPF, sub = warp - fw * WPF;    // frame slot in the CTA, warp within the frame
    const int b = blockIdx.x * kFrames + fw;
    __shared__ int s_base[kFrames][PF_MAX_KEYPOINTS + 1];
    __shared__ int s_err[kFrames];
    pdl_trigger();
    pdl_wait();                                          // the NMS slabs
    const bool live = b < B;                             // no early return: the CTA meets at one barrier
    const int gframe = a.frame_base + b;
    if (live && sub == 0) {
        int c = 0;
        if (lane < K) {
            c = a.counts[(size_t)b * K + lane];
            a.counts[(size_t)b * K + lane] = 0;           // ready for the next launch
        }
        int incl = c;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        const int P = __shfl_sync(0xffffffffu, incl, K - 1);
        const uint32_t over = __ballot_sync(0xffffffffu, lane < K && c > a.cap_part);
        int err = 0, val = 0;
        if (over) { err = kCapPart; val = __shfl_sync(0xffffffffu, c, __ffs(over) - 1); }
        else if (P > a.cap_frame) { err = kCapFrame; val = P; }
        {   // exclusive prefix: s_base[k] = incl of lane k - 1 (every lane takes part in the shuffle)
            const int prev = __shfl_sync(0xffffffffu, incl, min(max(lane - 1, 0), 31));
            if (lane <= K) s_base[fw][lane] = lane == 0 ? 0 : prev;
            if (lane == 0 && K == kWarp) s_base[fw][K] = P;   // K = 32: the total has no lane of its own
        }
        if (lane == 0) {
            s_err[fw] = err;
            a.ferr[b] = make_int2(err, val);
            a.cand_n[b] = 0;
            if (err) {
                a.n_pairs[b] = 0;
                if (a.debug) { a.dbg_npeaks[gframe] = 0; a.dbg_nconns[gframe] = 0; }
            }
        }
    }
    if (WPF > 1) __syncthreads();
    else __syncwarp();
    if (!live || s_err[fw]) return;
    const int *sb = s_base[fw];
    const int P = sb[K];
    if (sub == 0)
        for (int k = lane; k <= K; k += kWarp) a.pk_base[(size_t)b * (K + 1) + k] = sb[k];
    // rank sort of each part's peaks by (score desc, cell asc) straight from the slab
    for (int e = sub * kWarp + lane; e < P; e += WPF * kWarp) {
        int part = 0;
        while (e >= sb[part + 1]) ++part;
        const uint2 *slab = a.peaks + ((size_t)b * K + part) * a.cap_part;
        const int np = sb[part + 1] - sb[part];
        const uint2 v = __ldg(slab + (e - sb[part]));
        const float vs = __uint_as_float(v.x);
        int rank = 0;
        for (int q = 0; q < np; ++q) {
            const uint2 u = __ldg(slab + q);
            const float us = __uint_as_float(u.x);
            rank += (us > vs) || (us == vs && u.y < v.y);
        }
        const size_t o = (size_t)b * a.cap_frame + sb[part] + rank;
        a.pk_cell[o] = v.y;
        a.pk_score[o] = vs;
        if (a.debug)
            a.dbg_peaks[(size_t)gframe * a.cap_frame + sb[part] + rank] =
                make_int4(part, int(v.y >> 16), int(v.y & 0xffff), __float_as_int(vs));
    }
    if (sub == 0 && lane == 0) {
        if (a.debug) a.dbg_npeaks[gframe] = P;
        int acc = 0;
        int *pp = a.pair_pp + (size_t)b * (L + 1);
        for (int l = 0; l < L; ++l) {
            pp[l] = acc;
            const int na = sb[a.topo.la[l] + 1] - sb[a.topo.la[l]];
            const int nb = sb[a.topo.lb[l] + 1] - sb[a.topo.lb[l]];
            acc += na * nb;
        }
        pp[L] = acc;
        a.n_pairs[b] = a.n_samples - a.good_need < 0 ? 0 : acc;   // nothing can pass: no pairs to score
    }
}

// exclusive scan of the frames' pair counts (one CTA; B is a launch chunk)
__global__ void __launch_bounds__(1024)
k_pair_scan(const ParseArgs a, int B)
{
    __shared__ long long wsum[32];
    __shared__ long long carry;
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b0 = 0; b0 < B; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const long long v = b < B ? a.n_pairs[b] : 0;
        long long incl = v;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            long long w = wsum[lane];
#pragma unroll
            for (int d = 1; d < kWarp; d <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += t;
            }
            wsum[lane] = w;                                // inclusive over warps
        }
        __syncthreads();
        const long long before = carry + (warp ? wsum[warp - 1] : 0);
        if (b < B) a.pair_base[b] = before + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *a.pair_total = carry;
}

#ifndef PF_SCORE_BSEARCH
#define PF_SCORE_BSEARCH 1
#endif
#ifndef PF_SCORE_MINB
#define PF_SCORE_MINB 4   // 64 registers: 0.27 ms; 79 (1): 0.315, 48 (5): 0.318, 40 (6): 0.386
#endif
__global__ void __launch_bounds__(kScoreThreads, PF_SCORE_MINB)
k_score_pairs(const ParseArgs a, int B)
{
    __shared__ double s_t[kParseTTab];                     // u / (n - 1), paf.py:139
    for (int u = threadIdx.x; u < kParseTTab && u < a.n_samples; u += blockDim.x)
        s_t[u] = __ddiv_rn((double)u, (double)(a.n_samples - 1));
    __syncthreads();
    pdl_trigger();
    pdl_wait();                                          // pair offsets of k_pair_scan
    const int K = a.topo.K, L = a.topo.L;
    const long long total = *a.pair_total;
    const int max_fail = a.n_samples - a.good_need;
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long gw = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); gw < total; gw += stride) {
        // frame of the warp's first pair: last b with pair_base[b] <= gw
        // (frames with no pairs share bases), a 32-way search (3 rounds of
        // one load per lane for 8192 frames instead of 13 dependent loads)
        int lo = 0, hi = B - 1;
        while (lo < hi) {                                    // warp-uniform
            const int idx = lo + (int)(((long long)(hi - lo) * (lane + 1) + 31) / 32);
            const uint32_t le = __ballot_sync(0xffffffffu, __ldg(a.pair_base + idx) <= gw);
            const int c = __popc(le);                        // the probes are increasing: a prefix holds
            const int nlo = c ? __shfl_sync(0xffffffffu, idx, c - 1) : lo;
            const int nhi = c < 32 ? __shfl_sync(0xffffffffu, idx, c < 32 ? c : 31) - 1 : hi;
            lo = nlo;
            hi = nhi;
        }
        const long long g = gw + lane;
        if (g >= total) continue;
        int b = lo;                                          // this lane's pair may lie a few frames on
        while (b + 1 < B && __ldg(a.pair_base + b + 1) <= g) ++b;
        const int local0 = (int)(g - __ldg(a.pair_base + b));
        const int *pp = a.pair_pp + (size_t)b * (L + 1);
        // the pair's limb: the last l with pp[l] <= local0 (binary search over
        // the L + 1 prefix entries instead of a linear walk of dependent loads)
        int l = 0;
#if PF_SCORE_BSEARCH
        for (int hi = L; hi - l > 1;) {
            const int mid = (l + hi) >> 1;
            if (__ldg(pp + mid) <= local0) l = mid;
            else hi = mid;
        }
#else
        while (local0 >= __ldg(pp + l + 1)) ++l;
#endif
        const int *base = a.pk_base + (size_t)b * (K + 1);
        const int pa_part = a.topo.la[l], pb_part = a.topo.lb[l];
        const int nb = __ldg(base + pb_part + 1) - __ldg(base + pb_part);
        const int local = local0 - __ldg(pp + l);
        const int qa = local / nb;
        const int ia = __ldg(base + pa_part) + qa;
        const int ib = __ldg(base + pb_part) + (local - qa * nb);
        const uint32_t *cells = a.pk_cell + (size_t)b * a.cap_frame;
        double score;
        int ngood;
        const float *paf_f = a.paf + (size_t)b * (2 * L) * a.h * a.w;
        if (!score_pair(a, paf_f, l, __ldcg(cells + ia), __ldcg(cells + ib), s_t, max_fail, score, ngood)) continue;
        const int slot = atomicAdd(a.cand_n + b, 1);
        if (slot < a.cap_cands) {
            Cand c;
            c.score = score;
            c.ab = (uint32_t(ia) << 16) | uint32_t(ib);
            c.lg = (uint32_t(l) << 24) | uint32_t(ngood);
            a.cand_g[(size_t)b * a.cap_cands + slot] = c;
        }
    }
}

size_t parse_smem_bytes(int cap_frame, int cap_part, int cap_cands, int cap_humans, int K, int L, int n_warps,
                        bool split, bool crowd)
{
    (void)cap_cands;
    const int pm_words = (cap_part + 31) / 32;
    const int cs = crowd ? kCandSmemCrowd : (split ? kCandSmemSplit : kCandSmem);
    size_t s = (size_t)cs * sizeof(Cand);
    s += (size_t)cap_humans * sizeof(double);
    if (!split) s += (size_t)cap_frame * (sizeof(uint32_t) + sizeof(float));
    s += (size_t)cap_humans * (sizeof(uint32_t) + sizeof(int));
    s += (size_t)L * 2 * pm_words * sizeof(uint32_t);
    s += (size_t)cap_frame * sizeof(int16_t);
    s += (size_t)cap_humans * K * (sizeof(int16_t) + sizeof(int8_t));
    s += (size_t)cap_humans * 2;
    s = (s + 15) & ~size_t(15);
    s += (size_t)cs * sizeof(ConnRec);
    return (s + 15) & ~size_t(15);
}

size_t cand_record_bytes() { return sizeof(Cand); }

size_t cand_spill_bytes_per_frame(int cap_cands)
{
    return cap_cands > kCandSmem ? (size_t)(cap_cands - kCandSmem) * sizeof(Cand) : 0;
}

cudaError_t launch_parse_frames(const ParseArgs &a, int B, int threads, size_t smem, cudaStream_t s)
{
    if (B == 0) return cudaSuccess;
    if (a.split) {
        cudaError_t e = launch_pdl(kPdlParseFrames, k_parse_frames<true>, dim3(B), dim3(threads), smem, s, a);
        if (e != cudaSuccess || !a.crowd_frames) return e;
        // crowded frames (listed by k_parse_frames<true>): one CTA per SM
        int dev = 0, sms = 0;
        e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        const size_t smem_c = parse_smem_bytes(a.cap_frame, a.cap_part, a.cap_cands, a.cap_humans, a.topo.K,
                                               a.topo.L, kParseCrowdThreads / kWarp, true, true);
        k_parse_crowd<<<std::min(B, sms), kParseCrowdThreads, smem_c, s>>>(a);
        return cudaGetLastError();
    }
    if (a.paf_touch) k_parse_frames<false, true><<<B, threads, smem, s>>>(a);
    else if (threads == kParseWideThreads)
        return launch_pdl(kPdlParseWide, k_parse_frames_wide, dim3(B), dim3(threads), smem, s, a);
    else k_parse_frames<false><<<B, threads, smem, s>>>(a);
    return cudaGetLastError();
}

#ifndef PF_PEAK_WPF_FRAMES_PER_SM
#define PF_PEAK_WPF_FRAMES_PER_SM 4
#endif
constexpr int kPeakWpfMaxFramesPerSm = PF_PEAK_WPF_FRAMES_PER_SM;

cudaError_t launch_parse_peaks(const ParseArgs &a, int B, cudaStream_t s)
{
    if (B == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    // a CTA per frame while the batch leaves SMs short of warps (kPeakWpfMaxFramesPerSm)
    if (B <= kPeakWpfMaxFramesPerSm * sms)
        e = launch_pdl(kPdlParsePeaks, k_parse_peaks<kPeakWarps>, dim3(B), dim3(kPeakWarps * kWarp), 0, s, a, B);
    else
        e = launch_pdl(kPdlParsePeaks, k_parse_peaks<1>, dim3((B + kPeakWarps - 1) / kPeakWarps), dim3(kPeakWarps * kWarp), 0,
                       s, a, B);
    if (e != cudaSuccess) return e;
    return launch_pdl(kPdlPairScan, k_pair_scan, dim3(1), dim3(1024), 0, s, a, B);
}

cudaError_t launch_score_pairs(const ParseArgs &a, int B, cudaStream_t s)
{
    if (B == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    return launch_pdl(kPdlScorePairs, k_score_pairs, dim3(sms * 8), dim3(kScoreThreads), 0, s, a, B);
}

cudaError_t configure_parse_kernels(int max_smem)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k_parse_frames<false>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_parse_frames<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_parse_frames<false, true>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_parse_frames<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_parse_frames<true>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_parse_frames<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_parse_frames_wide);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_parse_frames_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k_parse_crowd);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_parse_crowd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - (int)fa.sharedSizeBytes);
    return e;
}

}  // namespace pf
