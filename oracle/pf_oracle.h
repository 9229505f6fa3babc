/* pf_oracle.h — CPU restatement of the reference pose-parsing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the CUDA path is
 * compared against (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline leg and `bench.py --impl reference`).  The product path in
 * paper_2108_11826_b200/ never links, loads or calls it.
 *
 * Every function restates one reference function (poseflow, pure
 * Python/numpy, /root/reference/pkg/src/poseflow/...) with the same
 * floating-point operation order, so results are bit-identical:
 *   - fp32 threshold compare (numpy >= 2 NEP-50 weak-scalar promotion),
 *   - fp64 arithmetic without FMA contraction (compile with
 *     -ffp-contract=off; x86-64 SSE2 has no extended precision),
 *   - CPython >= 3.12 `sum()` (Neumaier compensated) for the human
 *     keypoint-score sum,
 *   - every reference tie-break order.
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 */
#ifndef PF_ORACLE_H
#define PF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_params {          /* paf.py:34-42 ParserParams */
    double conf_threshold;
    int32_t nms_window;
    int32_t n_samples;
    double sample_dot_threshold;
    double good_fraction_min;
    int32_t min_parts;
    double min_human_score;
} orc_params;

/* Per-frame result slabs (caller-owned, capacities in the *_cap fields).
 * Every count is the TRUE count; when it exceeds the capacity only the
 * first `cap` entries are written and orc_parse returns 3 (capacity). */
typedef struct orc_result {
    /* peaks, in id order (part-major; score desc, row, col within part) */
    int32_t n_peaks, peaks_cap;
    int32_t *peak_part, *peak_i, *peak_j;
    float *peak_score;
    /* accepted connections in connect_limbs order (paf.py:185-199) */
    int32_t n_conns, conns_cap;
    int32_t *conn_limb, *conn_a, *conn_b;
    double *conn_score, *conn_good;
    /* humans after filtering and stable sort (paf.py:273-289) */
    int32_t n_humans, humans_cap;
    int32_t n_keypoints;            /* K, slab stride */
    double *human_score;            /* [humans_cap] */
    int32_t *human_n_parts;         /* [humans_cap] */
    double *kp_x, *kp_y;            /* [humans_cap * K] */
    float *kp_score;                /* [humans_cap * K] */
    int32_t *kp_peak;               /* [humans_cap * K], -1 = absent */
} orc_result;

/* formats.py:116-117: u8 / 255.0 in fp32 (IEEE division). */
void orc_u8_to_f32(const uint8_t *src, int64_t n, float *dst);

/* operators.py:79-107, 2-D branch applied per channel: [C,in_h,in_w] ->
 * [C,out_h,out_w]; equal sizes -> exact copy (operators.py:84-85). */
int orc_resize_chw(const float *src, int C, int in_h, int in_w,
                   float *dst, int out_h, int out_w);

/* operators.py:79-107, 3-D branch: [in_h,in_w,C] -> [out_h,out_w,C]. */
int orc_resize_hwc(const float *src, int in_h, int in_w, int C,
                   float *dst, int out_h, int out_w);

/* operators.py:114-131 after formats.read_ppm (formats.py:100-117):
 * u8 [h,w,3] -> f32 [3,out_h,out_w]. */
int orc_preprocess(const uint8_t *src, int h, int w,
                   float *dst, int out_h, int out_w);

/* paf.py:74-109 on one channel.  Writes up to `cap` peaks sorted by
 * (score desc, row asc, col asc); returns the true peak count. */
int orc_nms_peaks(const float *conf, int h, int w, double conf_threshold,
                  int nms_window, int32_t *out_i, int32_t *out_j,
                  float *out_score, int cap);

/* paf.py:112-146 on the two PAF channels of one limb. */
void orc_score_limb(const float *paf_x, const float *paf_y, int h, int w,
                    int ai, int aj, int bi, int bj, int n_samples,
                    double sample_dot_threshold, double *score, double *good);

/* paf.py:168-182 _greedy_select on one limb's candidates (score, id_a,
 * id_b); writes the accepted candidate indices in acceptance order and
 * returns their count. */
int orc_greedy_select(const double *score, const int32_t *id_a, const int32_t *id_b,
                      int n, int32_t *accepted);

/* CPython >= 3.12 builtin sum() of a float sequence starting from int 0. */
double orc_py_sum(const double *x, int n);

/* paf.py:292-305 parse(): conf [K+1,h,w], paf [2L,h,w] (row-major f32).
 * limbs/paf_ch are [L][2].  Returns 0 ok, 1 config error, 2 contract
 * error, 3 capacity exceeded in `res`. */
int orc_parse(const float *conf, const float *paf, int K, int L,
              const int32_t *limbs, const int32_t *paf_ch, int h, int w,
              int stride, const orc_params *p, orc_result *res);

/* Mode U oracle: every conf and paf channel resized with operators.py:79-107
 * (2-D branch) from [h,w] to [h*up,w*up], optional conf blur (below), then
 * parse() with stride/up.  Composition of reference functions; the blur
 * has no reference (parity unpinned for blur_sigma > 0). */
int orc_parse_upsampled(const float *conf, const float *paf, int K, int L,
                        const int32_t *limbs, const int32_t *paf_ch,
                        int h, int w, int stride, int up,
                        const double *blur_taps, int blur_radius,
                        const orc_params *p, orc_result *res);

/* Separable Gaussian smoothing (NO reference implementation, defined by
 * this repo): horizontal then vertical pass, taps
 * k=-r..r accumulated in fp64 in ascending k with clamped edges and no
 * FMA, each pass rounded to fp32.  In place on [C,h,w]. */
int orc_blur_chw(float *maps, int C, int h, int w, const double *taps, int r);

#ifdef __cplusplus
}
#endif
#endif
