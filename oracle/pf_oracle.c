/* pf_oracle.c — CPU restatement of the reference pose-parsing hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see pf_oracle.h).  Each function names the
 * reference lines it restates; /root/reference/pkg/src/poseflow/ is the
 * reference tree.  Build with -O2 -ffp-contract=off (oracle/Makefile):
 * contraction into FMA would change fp64 rounding.
 */
#include "pf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* formats.py:116-117  arr.astype(np.float32) / 255.0  (fp32 IEEE div) */
void orc_u8_to_f32(const uint8_t *src, int64_t n, float *dst)
{
    for (int64_t k = 0; k < n; ++k) dst[k] = (float)src[k] / 255.0f;
}

/* ------------------------------------------------------------------ */
/* operators.py:86-96 — per-axis source coordinates:
 *   s = (o + 0.5) * (in / out) - 0.5 ; i0 = floor(s) ; t = s - i0
 *   indices clipped to [0, in-1]; (1 - t) formed as its own fp64 op. */
static void resize_axis(int in_n, int out_n, int32_t *i0c, int32_t *i1c,
                        double *t, double *omt)
{
    double ratio = (double)in_n / (double)out_n;
    for (int o = 0; o < out_n; ++o) {
        double s = ((double)o + 0.5) * ratio - 0.5;
        int64_t i0 = (int64_t)floor(s);
        t[o] = s - (double)i0;
        omt[o] = 1.0 - t[o];
        int64_t a = i0 < 0 ? 0 : (i0 > in_n - 1 ? in_n - 1 : i0);
        int64_t b = i0 + 1 < 0 ? 0 : (i0 + 1 > in_n - 1 ? in_n - 1 : i0 + 1);
        i0c[o] = (int32_t)a;
        i1c[o] = (int32_t)b;
    }
}

typedef struct axis_tab {
    int32_t *i0, *i1;
    double *t, *omt;
} axis_tab;

static int axis_alloc(axis_tab *a, int in_n, int out_n)
{
    a->i0 = malloc(sizeof(int32_t) * (size_t)out_n);
    a->i1 = malloc(sizeof(int32_t) * (size_t)out_n);
    a->t = malloc(sizeof(double) * (size_t)out_n);
    a->omt = malloc(sizeof(double) * (size_t)out_n);
    if (!a->i0 || !a->i1 || !a->t || !a->omt) return -1;
    resize_axis(in_n, out_n, a->i0, a->i1, a->t, a->omt);
    return 0;
}

static void axis_free(axis_tab *a)
{
    free(a->i0); free(a->i1); free(a->t); free(a->omt);
}

/* operators.py:102-107: top = a*(1-tx) + b*tx ; bot likewise ;
 * out = top*(1-ty) + bot*ty ; cast to fp32.  Every product and sum is a
 * separately rounded fp64 operation (numpy elementwise, no FMA). */
static inline float bilerp(double a, double b, double c, double d,
                           double tx, double omtx, double ty, double omty)
{
    double top = a * omtx + b * tx;
    double bot = c * omtx + d * tx;
    return (float)(top * omty + bot * ty);
}

int orc_resize_chw(const float *src, int C, int in_h, int in_w,
                   float *dst, int out_h, int out_w)
{
    if (in_h < 1 || in_w < 1 || out_h < 1 || out_w < 1) return 2;
    if (in_h == out_h && in_w == out_w) {       /* operators.py:84-85 */
        memcpy(dst, src, sizeof(float) * (size_t)C * in_h * in_w);
        return 0;
    }
    axis_tab ay, ax;
    if (axis_alloc(&ay, in_h, out_h) || axis_alloc(&ax, in_w, out_w)) return 4;
    for (int c = 0; c < C; ++c) {
        const float *s = src + (size_t)c * in_h * in_w;
        float *o = dst + (size_t)c * out_h * out_w;
        for (int y = 0; y < out_h; ++y) {
            const float *r0 = s + (size_t)ay.i0[y] * in_w;
            const float *r1 = s + (size_t)ay.i1[y] * in_w;
            for (int x = 0; x < out_w; ++x) {
                o[(size_t)y * out_w + x] =
                    bilerp(r0[ax.i0[x]], r0[ax.i1[x]], r1[ax.i0[x]], r1[ax.i1[x]],
                           ax.t[x], ax.omt[x], ay.t[y], ay.omt[y]);
            }
        }
    }
    axis_free(&ay); axis_free(&ax);
    return 0;
}

int orc_resize_hwc(const float *src, int in_h, int in_w, int C,
                   float *dst, int out_h, int out_w)
{
    if (in_h < 1 || in_w < 1 || out_h < 1 || out_w < 1) return 2;
    if (in_h == out_h && in_w == out_w) {
        memcpy(dst, src, sizeof(float) * (size_t)C * in_h * in_w);
        return 0;
    }
    axis_tab ay, ax;
    if (axis_alloc(&ay, in_h, out_h) || axis_alloc(&ax, in_w, out_w)) return 4;
    for (int y = 0; y < out_h; ++y) {
        const float *r0 = src + (size_t)ay.i0[y] * in_w * C;
        const float *r1 = src + (size_t)ay.i1[y] * in_w * C;
        for (int x = 0; x < out_w; ++x) {
            for (int c = 0; c < C; ++c) {
                dst[((size_t)y * out_w + x) * C + c] =
                    bilerp(r0[(size_t)ax.i0[x] * C + c], r0[(size_t)ax.i1[x] * C + c],
                           r1[(size_t)ax.i0[x] * C + c], r1[(size_t)ax.i1[x] * C + c],
                           ax.t[x], ax.omt[x], ay.t[y], ay.omt[y]);
            }
        }
    }
    axis_free(&ay); axis_free(&ax);
    return 0;
}

/* operators.py:118-129 fn(): read_ppm normalisation, then either a pure
 * HWC->CHW permutation (same size) or bilinear_resize + HWC->CHW. */
int orc_preprocess(const uint8_t *src, int h, int w,
                   float *dst, int out_h, int out_w)
{
    if (h < 1 || w < 1 || out_h < 1 || out_w < 1) return 2;
    size_t n = (size_t)h * w * 3;
    float *img = malloc(sizeof(float) * n);
    if (!img) return 4;
    orc_u8_to_f32(src, (int64_t)n, img);
    const float *hwc = img;
    float *rs = NULL;
    if (h != out_h || w != out_w) {
        rs = malloc(sizeof(float) * (size_t)out_h * out_w * 3);
        if (!rs) { free(img); return 4; }
        orc_resize_hwc(img, h, w, 3, rs, out_h, out_w);
        hwc = rs;
    }
    for (int c = 0; c < 3; ++c)
        for (int y = 0; y < out_h; ++y)
            for (int x = 0; x < out_w; ++x)
                dst[((size_t)c * out_h + y) * out_w + x] =
                    hwc[((size_t)y * out_w + x) * 3 + c];
    free(rs);
    free(img);
    return 0;
}

/* ------------------------------------------------------------------ */
/* paf.py:74-109 nms_peaks */
typedef struct pk { int32_t i, j; float s; } pk;

static int pk_cmp(const void *pa, const void *pb)
{
    /* np.lexsort((jj, ii, -scores)): score desc, then row, then col */
    const pk *a = pa, *b = pb;
    if (a->s > b->s) return -1;
    if (a->s < b->s) return 1;
    if (a->i != b->i) return a->i < b->i ? -1 : 1;
    if (a->j != b->j) return a->j < b->j ? -1 : 1;
    return 0;
}

int orc_nms_peaks(const float *conf, int h, int w, double conf_threshold,
                  int nms_window, int32_t *out_i, int32_t *out_j,
                  float *out_score, int cap)
{
    /* numpy >= 2 (NEP 50): `conf >= 0.1` compares in float32 */
    const float thr = (float)conf_threshold;
    const int half = nms_window / 2;
    int n = 0, alloc = 64;
    pk *list = malloc(sizeof(pk) * (size_t)alloc);
    for (int i = 0; i < h; ++i) {
        for (int j = 0; j < w; ++j) {
            float v = conf[(size_t)i * w + j];
            if (!(v >= thr)) continue;
            int keep = 1;
            for (int di = -half; di <= half && keep; ++di) {
                int ni = i + di;
                for (int dj = -half; dj <= half; ++dj) {
                    if (di == 0 && dj == 0) continue;
                    int nj = j + dj;
                    /* -inf padding (paf.py:87-88): out-of-range never wins */
                    if (ni < 0 || ni >= h || nj < 0 || nj >= w) continue;
                    float nv = conf[(size_t)ni * w + nj];
                    int later = di > 0 || (di == 0 && dj > 0);  /* paf.py:95-99 */
                    if (later ? !(v >= nv) : !(v > nv)) { keep = 0; break; }
                }
            }
            if (!keep) continue;
            if (n == alloc) { alloc *= 2; list = realloc(list, sizeof(pk) * (size_t)alloc); }
            list[n].i = i; list[n].j = j; list[n].s = v;
            ++n;
        }
    }
    qsort(list, (size_t)n, sizeof(pk), pk_cmp);
    for (int k = 0; k < n && k < cap; ++k) {
        out_i[k] = list[k].i;
        out_j[k] = list[k].j;
        out_score[k] = list[k].s;
    }
    free(list);
    return n;
}

/* ------------------------------------------------------------------ */
/* paf.py:112-146 score_limb */
void orc_score_limb(const float *paf_x, const float *paf_y, int h, int w,
                    int ai, int aj, int bi, int bj, int n_samples,
                    double sample_dot_threshold, double *score, double *good)
{
    (void)h;
    if (ai == bi && aj == bj) { *score = 0.0; *good = 0.0; return; }
    int di = bi - ai, dj = bj - aj;
    double norm = sqrt((double)((long long)di * di + (long long)dj * dj));
    double vx = (double)dj / norm, vy = (double)di / norm;
    double total = 0.0;
    int ngood = 0;
    for (int u = 0; u < n_samples; ++u) {
        double t = (double)u / (double)(n_samples - 1);
        int ci = (int)floor((double)ai + t * (double)di + 0.5);
        int cj = (int)floor((double)aj + t * (double)dj + 0.5);
        double d = (double)paf_x[(size_t)ci * w + cj] * vx +
                   (double)paf_y[(size_t)ci * w + cj] * vy;
        total += d;
        if (d >= sample_dot_threshold) ++ngood;
    }
    *score = total / (double)n_samples;
    *good = (double)ngood / (double)n_samples;
}

/* CPython 3.12 Python/bltinmodule.c builtin_sum_impl: start int 0; the
 * first float goes through PyNumber_Add(0, x); later floats use the
 * Neumaier-compensated loop; the compensation is added once at the end. */
double orc_py_sum(const double *x, int n)
{
    if (n <= 0) return 0.0;
    double f = 0.0 + x[0];
    double c = 0.0;
    for (int k = 1; k < n; ++k) {
        double v = x[k];
        double t = f + v;
        if (fabs(f) >= fabs(v)) c += (f - t) + v;
        else c += (v - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

/* ------------------------------------------------------------------ */
/* paf.py:44-54 ParserParams.validate */
static int validate_params(const orc_params *p)
{
    if (p->nms_window < 3 || p->nms_window % 2 == 0) return 1;
    if (p->n_samples < 2) return 1;
    double v[3] = {p->conf_threshold, p->sample_dot_threshold, p->good_fraction_min};
    for (int k = 0; k < 3; ++k)
        if (!(0.0 <= v[k] && v[k] <= 1.0)) return 1;
    if (p->min_parts < 1) return 1;
    return 0;
}

typedef struct cand { double score, good; int32_t a, b; } cand;

static int cand_cmp(const void *pa, const void *pb)
{
    /* paf.py:173 key (-score, id_a, id_b) */
    const cand *x = pa, *y = pb;
    if (x->score > y->score) return -1;
    if (x->score < y->score) return 1;
    if (x->a != y->a) return x->a < y->a ? -1 : 1;
    if (x->b != y->b) return x->b < y->b ? -1 : 1;
    return 0;
}

static int cand_cmp_stable(const void *pa, const void *pb)
{
    int c = cand_cmp(pa, pb);
    if (c) return c;
    const cand *x = pa, *y = pb;          /* `good` carries the input position */
    return (x->good > y->good) - (x->good < y->good);
}

int orc_greedy_select(const double *score, const int32_t *id_a, const int32_t *id_b,
                      int n, int32_t *accepted)
{
    cand *cs = malloc(sizeof(cand) * ((size_t)n + 1));
    int32_t max_id = 0;
    for (int q = 0; q < n; ++q) {
        cs[q].score = score[q]; cs[q].good = (double)q; cs[q].a = id_a[q]; cs[q].b = id_b[q];
        if (id_a[q] > max_id) max_id = id_a[q];
        if (id_b[q] > max_id) max_id = id_b[q];
    }
    qsort(cs, (size_t)n, sizeof(cand), cand_cmp_stable);   /* paf.py:173, sorted() is stable */
    uint8_t *ua = calloc((size_t)max_id + 1, 1), *ub = calloc((size_t)max_id + 1, 1);
    int m = 0;
    for (int q = 0; q < n; ++q) {                        /* paf.py:176-181 */
        if (ua[cs[q].a] || ub[cs[q].b]) continue;
        ua[cs[q].a] = 1;
        ub[cs[q].b] = 1;
        accepted[m++] = (int32_t)cs[q].good;
    }
    free(ua); free(ub); free(cs);
    return m;
}

typedef struct builder {             /* paf.py:202-207 _Builder */
    int32_t *parts;                  /* [K] peak id or -1 */
    int32_t *order;                  /* dict insertion order of part keys */
    int32_t n;
    double conn_score;
    int alive;
} builder;

int orc_parse(const float *conf, const float *paf, int K, int L,
              const int32_t *limbs, const int32_t *paf_ch, int h, int w,
              int stride, const orc_params *p, orc_result *res)
{
    int rc = validate_params(p);                      /* paf.py:295 */
    if (rc) return rc;
    if (stride < 1 || K < 1 || L < 0 || h < 0 || w < 0) return 2;  /* types.py:185-205 */
    const size_t plane = (size_t)h * w;

    /* ---- peaks: paf.py:298-303 ---- */
    int32_t *part_base = calloc((size_t)K + 1, sizeof(int32_t));
    int n_alloc = 256, n_peaks = 0;
    int32_t *pi = malloc(sizeof(int32_t) * n_alloc), *pj = malloc(sizeof(int32_t) * n_alloc),
            *ppart = malloc(sizeof(int32_t) * n_alloc);
    float *ps = malloc(sizeof(float) * n_alloc);
    for (int k = 0; k < K; ++k) {
        part_base[k] = n_peaks;
        int cnt = orc_nms_peaks(conf + (size_t)k * plane, h, w, p->conf_threshold,
                                p->nms_window, NULL, NULL, NULL, 0);
        while (n_peaks + cnt > n_alloc) {
            n_alloc *= 2;
            pi = realloc(pi, sizeof(int32_t) * n_alloc);
            pj = realloc(pj, sizeof(int32_t) * n_alloc);
            ppart = realloc(ppart, sizeof(int32_t) * n_alloc);
            ps = realloc(ps, sizeof(float) * n_alloc);
        }
        orc_nms_peaks(conf + (size_t)k * plane, h, w, p->conf_threshold, p->nms_window,
                      pi + n_peaks, pj + n_peaks, ps + n_peaks, cnt);
        for (int q = 0; q < cnt; ++q) ppart[n_peaks + q] = k;
        n_peaks += cnt;
    }
    part_base[K] = n_peaks;

    /* ---- connect_limbs: paf.py:149-199 ---- */
    int c_alloc = 256, n_conns = 0;
    cand *conns = malloc(sizeof(cand) * c_alloc);
    int32_t *conn_limb = malloc(sizeof(int32_t) * c_alloc);
    uint8_t *used_a = calloc((size_t)n_peaks + 1, 1), *used_b = calloc((size_t)n_peaks + 1, 1);
    for (int l = 0; l < L; ++l) {
        int a_part = limbs[2 * l], b_part = limbs[2 * l + 1];
        const float *px = paf + (size_t)paf_ch[2 * l] * plane;
        const float *py = paf + (size_t)paf_ch[2 * l + 1] * plane;
        int na = part_base[a_part + 1] - part_base[a_part];
        int nb = part_base[b_part + 1] - part_base[b_part];
        cand *cs = malloc(sizeof(cand) * ((size_t)na * nb + 1));
        int nc = 0;
        for (int x = 0; x < na; ++x) {
            int ia = part_base[a_part] + x;
            for (int y = 0; y < nb; ++y) {
                int ib = part_base[b_part] + y;
                double s, g;
                orc_score_limb(px, py, h, w, pi[ia], pj[ia], pi[ib], pj[ib],
                               p->n_samples, p->sample_dot_threshold, &s, &g);
                if (g >= p->good_fraction_min && s > 0.0) {  /* paf.py:162 */
                    cs[nc].score = s; cs[nc].good = g; cs[nc].a = ia; cs[nc].b = ib;
                    ++nc;
                }
            }
        }
        qsort(cs, (size_t)nc, sizeof(cand), cand_cmp);
        memset(used_a, 0, (size_t)n_peaks + 1);
        memset(used_b, 0, (size_t)n_peaks + 1);
        for (int q = 0; q < nc; ++q) {                   /* paf.py:174-181 */
            if (used_a[cs[q].a] || used_b[cs[q].b]) continue;
            used_a[cs[q].a] = 1;
            used_b[cs[q].b] = 1;
            if (n_conns == c_alloc) {
                c_alloc *= 2;
                conns = realloc(conns, sizeof(cand) * c_alloc);
                conn_limb = realloc(conn_limb, sizeof(int32_t) * c_alloc);
            }
            conns[n_conns] = cs[q];
            conn_limb[n_conns] = l;
            ++n_conns;
        }
        free(cs);
    }
    free(used_a); free(used_b);

    /* ---- assemble_humans: paf.py:210-289 ---- */
    /* connections are limb-major already, which equals the by_limb walk */
    builder *hs = calloc((size_t)n_conns + 1, sizeof(builder));
    int32_t *hparts = malloc(sizeof(int32_t) * ((size_t)n_conns + 1) * K);
    int32_t *horder = malloc(sizeof(int32_t) * ((size_t)n_conns + 1) * K);
    int32_t *owner = malloc(sizeof(int32_t) * ((size_t)n_peaks + 1));
    for (int q = 0; q < n_peaks; ++q) owner[q] = -1;
    int n_h = 0;
    for (int q = 0; q < n_conns; ++q) {
        int l = conn_limb[q];
        int a_part = limbs[2 * l], b_part = limbs[2 * l + 1];
        int pa = conns[q].a, pb = conns[q].b;
        int ha = owner[pa], hb = owner[pb];
        if (ha < 0 && hb < 0) {                            /* paf.py:246-253 */
            builder *b = &hs[n_h];
            b->parts = hparts + (size_t)n_h * K;
            b->order = horder + (size_t)n_h * K;
            for (int k = 0; k < K; ++k) b->parts[k] = -1;
            b->parts[a_part] = pa; b->order[b->n++] = a_part;
            b->parts[b_part] = pb; b->order[b->n++] = b_part;
            b->conn_score = conns[q].score;
            b->alive = 1;
            owner[pa] = n_h; owner[pb] = n_h;
            ++n_h;
        } else if (ha >= 0 && hb >= 0) {
            if (ha == hb) {                                /* paf.py:255-256 */
                hs[ha].conn_score += conns[q].score;
            } else {
                builder *A = &hs[ha], *B = &hs[hb];
                int disjoint = 1;
                for (int k = 0; k < B->n; ++k)
                    if (A->parts[B->order[k]] >= 0) { disjoint = 0; break; }
                if (disjoint) {                             /* paf.py:257-262 */
                    for (int k = 0; k < B->n; ++k) {
                        int part = B->order[k];
                        A->parts[part] = B->parts[part];
                        A->order[A->n++] = part;
                        owner[B->parts[part]] = ha;
                    }
                    A->conn_score += B->conn_score + conns[q].score;
                    B->alive = 0;
                }
                /* else: paf.py:263 overlapping parts, leave both */
            }
        } else {                                           /* paf.py:264-271 */
            int hidx = ha >= 0 ? ha : hb;
            int part = ha >= 0 ? b_part : a_part;
            int pid = ha >= 0 ? pb : pa;
            builder *b = &hs[hidx];
            if (b->parts[part] < 0) {
                b->parts[part] = pid;
                b->order[b->n++] = part;
                b->conn_score += conns[q].score;
                owner[pid] = hidx;
            }
        }
    }

    /* filter + score: paf.py:273-287 */
    int32_t *keep = malloc(sizeof(int32_t) * ((size_t)n_h + 1));
    double *kscore = malloc(sizeof(double) * ((size_t)n_h + 1));
    double *tmp = malloc(sizeof(double) * ((size_t)K + 1));
    int n_keep = 0;
    for (int q = 0; q < n_h; ++q) {
        builder *b = &hs[q];
        if (!b->alive) continue;
        if (b->n < p->min_parts) continue;
        for (int k = 0; k < b->n; ++k) tmp[k] = (double)ps[b->parts[b->order[k]]];
        double kp_sum = orc_py_sum(tmp, b->n);
        double score = (kp_sum + b->conn_score) / (double)b->n;
        if (score < p->min_human_score) continue;
        keep[n_keep] = q;
        kscore[n_keep] = score;
        ++n_keep;
    }
    /* paf.py:288 stable sort by -score (insertion sort keeps ties in order) */
    for (int a = 1; a < n_keep; ++a) {
        int32_t kq = keep[a];
        double ks = kscore[a];
        int b = a - 1;
        while (b >= 0 && kscore[b] < ks) {
            keep[b + 1] = keep[b];
            kscore[b + 1] = kscore[b];
            --b;
        }
        keep[b + 1] = kq;
        kscore[b + 1] = ks;
    }

    /* ---- write results ---- */
    rc = 0;
    res->n_peaks = n_peaks;
    if (n_peaks > res->peaks_cap) rc = 3;
    for (int q = 0; q < n_peaks && q < res->peaks_cap; ++q) {
        if (res->peak_part) res->peak_part[q] = ppart[q];
        if (res->peak_i) res->peak_i[q] = pi[q];
        if (res->peak_j) res->peak_j[q] = pj[q];
        if (res->peak_score) res->peak_score[q] = ps[q];
    }
    res->n_conns = n_conns;
    if (n_conns > res->conns_cap) rc = 3;
    for (int q = 0; q < n_conns && q < res->conns_cap; ++q) {
        if (res->conn_limb) res->conn_limb[q] = conn_limb[q];
        if (res->conn_a) res->conn_a[q] = conns[q].a;
        if (res->conn_b) res->conn_b[q] = conns[q].b;
        if (res->conn_score) res->conn_score[q] = conns[q].score;
        if (res->conn_good) res->conn_good[q] = conns[q].good;
    }
    res->n_humans = n_keep;
    res->n_keypoints = K;
    if (n_keep > res->humans_cap) rc = 3;
    for (int q = 0; q < n_keep && q < res->humans_cap; ++q) {
        builder *b = &hs[keep[q]];
        res->human_score[q] = kscore[q];
        res->human_n_parts[q] = b->n;
        for (int k = 0; k < K; ++k) {
            size_t o = (size_t)q * K + k;
            int pid = b->parts[k];
            if (pid < 0) {
                res->kp_x[o] = 0.0; res->kp_y[o] = 0.0; res->kp_score[o] = 0.0f;
                res->kp_peak[o] = -1;
            } else {
                /* types.py:233-235 cell_to_pixel */
                res->kp_x[o] = ((double)pj[pid] + 0.5) * (double)stride - 0.5;
                res->kp_y[o] = ((double)pi[pid] + 0.5) * (double)stride - 0.5;
                res->kp_score[o] = ps[pid];
                res->kp_peak[o] = pid;
            }
        }
    }

    free(keep); free(kscore); free(tmp);
    free(hs); free(hparts); free(horder); free(owner);
    free(conns); free(conn_limb);
    free(pi); free(pj); free(ppart); free(ps); free(part_base);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Separable Gaussian (no reference; DESIGN.md §5 defines it): horizontal then
 * vertical, clamped edges, acc = fmaf(w_k, v, acc) in fp32 from 0.0f in
 * ascending k with w_k = (float)taps[k] (the fp64-normalised taps rounded to
 * nearest).  C99 fmaf() is correctly rounded. */
int orc_blur_chw(float *maps, int C, int h, int w, const double *taps, int r)
{
    if (r <= 0) return 0;
    float *tmp = malloc(sizeof(float) * (size_t)h * w);
    float *tf = malloc(sizeof(float) * (size_t)(2 * r + 1));
    if (!tmp || !tf) { free(tmp); free(tf); return 4; }
    for (int k = 0; k <= 2 * r; ++k) tf[k] = (float)taps[k];
    for (int c = 0; c < C; ++c) {
        float *m = maps + (size_t)c * h * w;
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                float acc = 0.0f;
                for (int k = -r; k <= r; ++k) {
                    int xx = x + k < 0 ? 0 : (x + k > w - 1 ? w - 1 : x + k);
                    acc = fmaf(tf[k + r], m[(size_t)y * w + xx], acc);
                }
                tmp[(size_t)y * w + x] = acc;
            }
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                float acc = 0.0f;
                for (int k = -r; k <= r; ++k) {
                    int yy = y + k < 0 ? 0 : (y + k > h - 1 ? h - 1 : y + k);
                    acc = fmaf(tf[k + r], tmp[(size_t)yy * w + x], acc);
                }
                m[(size_t)y * w + x] = acc;
            }
    }
    free(tf);
    free(tmp);
    return 0;
}

int orc_parse_upsampled(const float *conf, const float *paf, int K, int L,
                        const int32_t *limbs, const int32_t *paf_ch,
                        int h, int w, int stride, int up,
                        const double *blur_taps, int blur_radius,
                        const orc_params *p, orc_result *res)
{
    int rc = validate_params(p);
    if (rc) return rc;
    if (up < 1 || stride < 1 || stride % up != 0 || h < 1 || w < 1) return 2;
    int H = h * up, W = w * up;
    float *cu = malloc(sizeof(float) * (size_t)(K + 1) * H * W);
    float *pu = malloc(sizeof(float) * ((size_t)2 * L + 1) * H * W);
    if (!cu || !pu) { free(cu); free(pu); return 4; }
    orc_resize_chw(conf, K + 1, h, w, cu, H, W);
    if (L > 0) orc_resize_chw(paf, 2 * L, h, w, pu, H, W);
    if (blur_taps && blur_radius > 0) orc_blur_chw(cu, K, H, W, blur_taps, blur_radius);
    rc = orc_parse(cu, pu, K, L, limbs, paf_ch, H, W, stride / up, p, res);
    free(cu); free(pu);
    return rc;
}
