/*
 * oracle/ds_oracle.c -- TEST INFRASTRUCTURE: the parity checker, never the
 * product.  A plain-C FP64 restatement of the reference's dual-scale cascade,
 * written from the reference's algorithm (paths relative to the reference
 * repo).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load
 * liboracle.so.  Pinned against the reference itself (oracle/_ref) and the
 * committed golden vectors by tests/test_oracle.py.
 *
 *   fft_plus           Fft::dft_plus, radix-2 DIT, unnormalised   proj/src/fft.cpp:10-51
 *   mgift_cell         build_mf(RM|KtRm) + compensated_ifft + PreDfm
 *                                                   proj/src/transforms.cpp:32-94,134-173
 *   gft_row            build_mf(DFM) x row, dft_plus(M), recentre, twiddle
 *                                                   proj/src/transforms.cpp:180-214
 *   oracle_keystone    keystone                     proj/src/transforms.cpp:96-130
 *   oracle_range_fft   range_fft (Fft::dft_minus per pulse)
 *                                                   proj/src/signal_model.cpp:97-107, proj/src/fft.cpp:30-51
 *   oracle_ds          ds_grft / ds_kt_mfp -> run_dual_scale + UnitScan + merge_units
 *                                                   proj/src/detectors.cpp:16-50,337-481
 *   oracle_td_grft     td_grft (rounded-trajectory sums)   proj/src/detectors.cpp:199-264
 *   oracle_kt_mfp      kt_mfp (keystone, gift(KtRm), gft)  proj/src/detectors.cpp:266-326
 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ltci_cuda.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#define C_LIGHT 3.0e8

typedef double complex cplx;

/* ---------------------------------------------------------------- FFT --- */
/* Radix-2 DIT with bit reversal and e^{+j2pi k/N} twiddles (proj/src/fft.cpp). */
static void fft_plus(cplx *x, int n, const cplx *tw /* n/2 */) {
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    for (int i = 0; i < n; ++i) {
        int r = 0;
        for (int b = 0; b < lg; ++b)
            if (i & (1 << b)) r |= 1 << (lg - 1 - b);
        if (r > i) {
            cplx t = x[i];
            x[i] = x[r];
            x[r] = t;
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        int half = len >> 1, step = n / len;
        for (int base = 0; base < n; base += len)
            for (int k = 0; k < half; ++k) {
                cplx w = tw[k * step];
                cplx u = x[base + k], v = x[base + k + half] * w;
                x[base + k] = u + v;
                x[base + k + half] = u - v;
            }
    }
}

static cplx *twiddles(int n) {
    cplx *tw = malloc(sizeof(cplx) * (n / 2 > 0 ? n / 2 : 1));
    for (int k = 0; k < n / 2; ++k) {
        double a = 2.0 * M_PI * k / n;
        tw[k] = cos(a) + I * sin(a);
    }
    return tw;
}

static cplx polar1(double ph) { return cos(ph) + I * sin(ph); }

/* ------------------------------------------------------- radar helpers --- */
static double lambda_of(const ltci_radar *p) { return C_LIGHT / p->fc; }
static double va_of(const ltci_radar *p) { return lambda_of(p) * p->PRF / 2.0; }
static double slow_time(const ltci_radar *p, int m) { return (double)(m + 1) / p->PRF; }
static double freq_of_row(const ltci_radar *p, int r) { return p->delta_f * (double)(r < p->K / 2 ? r : r - p->K); }

/* sum_{i} c[i] t^{i+first} (poly_from, proj/src/transforms.cpp:12-22) */
static double poly_from(const double *c, int n, double t, int first) {
    double tp = 1.0, acc = 0.0;
    for (int p = 1; p < first; ++p) tp *= t;
    for (int i = 0; i < n; ++i) {
        tp *= t;
        acc += c[i] * tp;
    }
    return acc;
}

/* mgift for one coarse cell: out is K x M complex, [n + K*m].
 * variant 0: c = c1..cP ; variant 1: c = (q, c2). */
static void mgift_cell(const cplx *cube, const ltci_radar *p, const double *c, int nc, int variant, cplx *out,
                       const cplx *twK) {
    const int K = p->K, M = p->M;
    const double s4 = 4.0 * M_PI / C_LIGHT, sl = 4.0 * M_PI / lambda_of(p);
    for (int m = 0; m < M; ++m) {
        const double tm = slow_time(p, m);
        cplx *dst = out + (size_t)K * m;
        const cplx *src = cube + (size_t)K * m;
        double pre;
        if (variant == 0) {
            double s = poly_from(c, nc, tm, 1);
            for (int k = 0; k < K; ++k) dst[k] = src[k] * polar1(s4 * freq_of_row(p, k) * s);
            pre = sl * s;
        } else {
            double qva = c[0] * va_of(p), c2 = c[1];
            for (int k = 0; k < K; ++k) {
                double fk = freq_of_row(p, k), fbar = 1.0 - fk / p->fc;
                dst[k] = src[k] * polar1(s4 * fk * (fbar * qva * tm - c2 * tm * tm));
            }
            pre = sl * c2 * tm * tm;
        }
        fft_plus(dst, K, twK);
        cplx w = polar1(pre);
        for (int n = 0; n < K; ++n) dst[n] *= w;
    }
}

/* DFM chirp of one fine cell: H(m) = exp(+j 4pi/lambda sum_{p>=2} c_p t^p) */
static void dfm_chirp(const ltci_radar *p, const double *fine_higher, int nf, cplx *h) {
    const double sl = 4.0 * M_PI / lambda_of(p);
    for (int m = 0; m < p->M; ++m) h[m] = polar1(sl * poly_from(fine_higher, nf, slow_time(p, m), 2));
}

/* gft for one row n of a range-pulse cube: y[j], j = 0..M-1 (full axis). */
static void gft_row(const cplx *rows, const ltci_radar *p, int n, const cplx *h, cplx *y, cplx *scratch,
                    const cplx *twM) {
    const int K = p->K, M = p->M;
    for (int m = 0; m < M; ++m) scratch[m] = rows[n + (size_t)K * m] * h[m];
    fft_plus(scratch, M, twM);
    for (int j = 0; j < M; ++j) {
        int wrapped = (j - M / 2 + M) % M;
        double dt = (double)j - M / 2.0;
        y[j] = scratch[wrapped] * polar1(2.0 * M_PI * dt / M);
    }
}

/* ------------------------------------------------------------ keystone --- */
static double sinc(double u) { return u == 0.0 ? 1.0 : sin(M_PI * u) / (M_PI * u); }
static int clampi(long v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : (int)v); }

static void keystone_impl(const cplx *cube, const ltci_radar *p, int taps, cplx *out) {
    const int K = p->K, M = p->M, half = taps / 2;
    for (int k = 0; k < K; ++k) {
        double fk = freq_of_row(p, k), fbar = p->fc / (fk + p->fc);
        for (int m = 0; m < M; ++m) {
            double x = fbar * (double)(m + 1);
            long j0 = lround(x);
            if (x == (double)j0) {
                out[k + (size_t)K * m] = cube[k + (size_t)K * clampi(j0 - 1, 0, M - 1)];
                continue;
            }
            cplx acc = 0;
            double wsum = 0;
            for (long j = j0 - half + 1; j <= j0 + half; ++j) {
                double u = x - (double)j;
                double w = sinc(u) * (0.54 + 0.46 * cos(M_PI * u / half));
                wsum += w;
                acc += w * cube[k + (size_t)K * clampi(j - 1, 0, M - 1)];
            }
            out[k + (size_t)K * m] = acc / wsum;
        }
    }
}

/* -------------------------------------------------------- dual scale ----- */
typedef struct {
    uint64_t idx;
    cplx v;
} cand_t;

typedef struct {
    /* plan */
    const cplx *input;
    const ltci_radar *p;
    int variant, P, R, roi_first, dop_first, D;
    int n_coarse_axes;
    ltci_grid coarse_axes[LTCI_MAX_ORDER];
    int n_fine_axes;
    ltci_grid fine_axes[LTCI_MAX_ORDER];
    int q_min;
    uint64_t coarse_cells, fine_cells;
    double kappa, retain;
    int keep_dense;
    cplx *dense;
    /* per coarse cell outputs */
    cand_t **cand;
    uint64_t *ncand, *capcand;
    double *row_mag;   /* [coarse][R] */
    uint64_t *row_idx; /* [coarse][R] */
    cplx *row_val;     /* [coarse][R] */
    /* work distribution */
    pthread_mutex_t mu;
    uint64_t next;
} ds_job;

static void consider(ds_job *jb, uint64_t cidx, int r, uint64_t idx, cplx v) {
    double m = cabs(v);
    if (m > jb->retain) {
        if (jb->ncand[cidx] == jb->capcand[cidx]) {
            jb->capcand[cidx] = jb->capcand[cidx] ? 2 * jb->capcand[cidx] : 64;
            jb->cand[cidx] = realloc(jb->cand[cidx], sizeof(cand_t) * jb->capcand[cidx]);
        }
        jb->cand[cidx][jb->ncand[cidx]++] = (cand_t){idx, v};
    }
    size_t s = cidx * (size_t)jb->R + r;
    if (m > jb->row_mag[s] || (m == jb->row_mag[s] && idx < jb->row_idx[s])) {
        jb->row_mag[s] = m;
        jb->row_idx[s] = idx;
        jb->row_val[s] = v;
    }
    if (jb->keep_dense) jb->dense[idx] = v;
}

static void run_coarse_cell(ds_job *jb, uint64_t cidx, cplx *mg, cplx *y, cplx *scratch, const cplx *twK,
                            const cplx *twM) {
    const ltci_radar *p = jb->p;
    uint64_t rem = cidx;
    int ci[LTCI_MAX_ORDER];
    for (int i = jb->n_coarse_axes - 1; i >= 0; --i) {
        ci[i] = (int)(rem % (uint64_t)jb->coarse_axes[i].count);
        rem /= (uint64_t)jb->coarse_axes[i].count;
    }
    double cv[LTCI_MAX_ORDER];
    int nc;
    if (jb->variant == 1) {
        cv[0] = (double)(jb->q_min + (int)rem);
        cv[1] = jb->coarse_axes[0].start + jb->coarse_axes[0].step * ci[0];
        nc = 2;
    } else {
        for (int i = 0; i < jb->n_coarse_axes; ++i) cv[i] = jb->coarse_axes[i].start + jb->coarse_axes[i].step * ci[i];
        nc = jb->n_coarse_axes;
    }
    mgift_cell(jb->input, p, cv, nc, jb->variant, mg, twK);
    for (uint64_t fidx = 0; fidx < jb->fine_cells; ++fidx) {
        uint64_t frem = fidx;
        double fs[LTCI_MAX_ORDER];
        int fi[LTCI_MAX_ORDER];
        for (int i = jb->n_fine_axes - 1; i >= 0; --i) {
            fi[i] = (int)(frem % (uint64_t)jb->fine_axes[i].count);
            frem /= (uint64_t)jb->fine_axes[i].count;
        }
        for (int i = 0; i < jb->n_fine_axes; ++i)
            fs[i] = jb->kappa * (jb->fine_axes[i].start + jb->fine_axes[i].step * fi[i]);
        uint64_t base = (cidx * jb->fine_cells + fidx) * (uint64_t)jb->R * (uint64_t)jb->D;
        cplx *h = scratch + p->M;
        dfm_chirp(p, fs, jb->n_fine_axes, h);
        for (int r = 0; r < jb->R; ++r) {
            gft_row(mg, p, jb->roi_first + r, h, y, scratch, twM);
            for (int j = 0; j < jb->D; ++j)
                consider(jb, cidx, r, base + (uint64_t)r * jb->D + (uint64_t)j, y[jb->dop_first + j]);
        }
    }
}

static void *worker(void *arg) {
    ds_job *jb = arg;
    const ltci_radar *p = jb->p;
    cplx *mg = malloc(sizeof(cplx) * (size_t)p->K * p->M);
    cplx *y = malloc(sizeof(cplx) * p->M), *scratch = malloc(sizeof(cplx) * 2 * p->M);
    cplx *twK = twiddles(p->K), *twM = twiddles(p->M);
    for (;;) {
        pthread_mutex_lock(&jb->mu);
        uint64_t c = jb->next++;
        pthread_mutex_unlock(&jb->mu);
        if (c >= jb->coarse_cells) break;
        run_coarse_cell(jb, c, mg, y, scratch, twK, twM);
    }
    free(mg);
    free(y);
    free(scratch);
    free(twK);
    free(twM);
    return NULL;
}

static int cmp_cand(const void *a, const void *b) {
    uint64_t x = ((const cand_t *)a)->idx, y = ((const cand_t *)b)->idx;
    return x < y ? -1 : (x > y ? 1 : 0);
}

static cplx *to_cplx(const double *d, size_t n) {
    cplx *c = malloc(sizeof(cplx) * (n ? n : 1));
    for (size_t i = 0; i < n; ++i) c[i] = d[2 * i] + I * d[2 * i + 1];
    return c;
}

/* ds_grft (variant 0) / ds_kt_mfp (variant 1) including the per-row peak map. */
int oracle_ds(const double *cube_d, const ltci_radar *p, const ltci_ambiguity *amb, const ltci_dual_space *s,
              const ltci_options *opt, int variant, int threads, ltci_detection_map **out) {
    const int K = p->K, M = p->M;
    if (p->K != s->radar.K || p->M != s->radar.M || p->fc != s->radar.fc || p->fs != s->radar.fs ||
        p->PRF != s->radar.PRF)
        return LTCI_INVALID_ARGUMENT;
    if (variant == 1 && s->order != 2) return LTCI_INVALID_ARGUMENT;
    int R = s->roi_last - s->roi_first + 1;
    if (R <= 0 || s->roi_first < 0 || s->roi_last >= K) return LTCI_INVALID_ARGUMENT;
    ds_job jb;
    memset(&jb, 0, sizeof(jb));
    jb.p = p;
    jb.variant = variant;
    jb.P = s->order;
    jb.R = R;
    jb.roi_first = s->roi_first;
    jb.kappa = s->kappa;
    jb.retain = opt ? opt->retain_threshold : 0.0;
    jb.keep_dense = opt ? opt->keep_dense : 0;
    cplx *cube = to_cplx(cube_d, (size_t)K * M), *kt = NULL;
    jb.input = cube;
    ltci_detection_map *mp = calloc(1, sizeof(*mp));
    if (variant == 0) {
        /* Doppler window (proj/src/detectors.cpp:420-432) */
        double dop_bin = va_of(p) / M;
        int keep = (int)ceil(s->kappa * s->rm_step[0] / 2.0 / dop_bin - 1e-9);
        if (keep > M / 2 - 1) keep = M / 2 - 1;
        jb.dop_first = M / 2 - keep;
        jb.D = 2 * keep + 1;
        jb.n_coarse_axes = s->order;
        for (int i = 0; i < s->order; ++i) jb.coarse_axes[i] = s->coarse[i];
        jb.n_fine_axes = s->order - 1;
        for (int i = 1; i < s->order; ++i) jb.fine_axes[i - 1] = s->fine[i];
        jb.coarse_cells = 1;
        mp->kind = LTCI_DS_GRFT;
        int a = 0;
        for (int i = 1; i <= s->order; ++i) mp->axes[a++] = (ltci_axis){LTCI_AXIS_COARSE, i, s->coarse[i - 1].count};
        for (int i = 2; i <= s->order; ++i) mp->axes[a++] = (ltci_axis){LTCI_AXIS_FINE, i, s->fine[i - 1].count};
        mp->axes[a++] = (ltci_axis){LTCI_AXIS_RANGE, 0, R};
        mp->axes[a++] = (ltci_axis){LTCI_AXIS_DOPPLER, 0, jb.D};
        mp->n_axes = a;
    } else {
        kt = malloc(sizeof(cplx) * (size_t)K * M);
        keystone_impl(cube, p, opt && opt->keystone_taps > 0 ? opt->keystone_taps : 8, kt);
        jb.input = kt;
        jb.dop_first = 0;
        jb.D = M;
        jb.n_coarse_axes = 1;
        jb.coarse_axes[0] = s->coarse[1];
        jb.n_fine_axes = 1;
        jb.fine_axes[0] = s->fine[1];
        jb.q_min = amb->q_min;
        mp->kind = LTCI_DS_KT_MFP;
        mp->axes[0] = (ltci_axis){LTCI_AXIS_FOLDING, 0, amb->q_max - amb->q_min + 1};
        mp->axes[1] = (ltci_axis){LTCI_AXIS_COARSE, 2, s->coarse[1].count};
        mp->axes[2] = (ltci_axis){LTCI_AXIS_FINE, 2, s->fine[1].count};
        mp->axes[3] = (ltci_axis){LTCI_AXIS_RANGE, 0, R};
        mp->axes[4] = (ltci_axis){LTCI_AXIS_DOPPLER, 0, M};
        mp->n_axes = 5;
    }
    jb.coarse_cells = 1;
    for (int i = 0; i < jb.n_coarse_axes; ++i) jb.coarse_cells *= (uint64_t)jb.coarse_axes[i].count;
    if (variant == 1) jb.coarse_cells *= (uint64_t)(amb->q_max - amb->q_min + 1);
    jb.fine_cells = 1;
    for (int i = 0; i < jb.n_fine_axes; ++i) jb.fine_cells *= (uint64_t)jb.fine_axes[i].count;
    uint64_t cells = jb.coarse_cells * jb.fine_cells * (uint64_t)R * (uint64_t)jb.D;
    if (jb.keep_dense) jb.dense = calloc(cells, sizeof(cplx));
    jb.cand = calloc(jb.coarse_cells, sizeof(cand_t *));
    jb.ncand = calloc(jb.coarse_cells, sizeof(uint64_t));
    jb.capcand = calloc(jb.coarse_cells, sizeof(uint64_t));
    size_t nrow = jb.coarse_cells * (size_t)R;
    jb.row_mag = malloc(sizeof(double) * nrow);
    jb.row_idx = malloc(sizeof(uint64_t) * nrow);
    jb.row_val = calloc(nrow, sizeof(cplx));
    for (size_t i = 0; i < nrow; ++i) {
        jb.row_mag[i] = -1.0;
        jb.row_idx[i] = UINT64_MAX;
    }
    pthread_mutex_init(&jb.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t th[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &jb);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&jb.mu);

    /* merge_units: concatenate in unit order, sort by index; argmax total order */
    uint64_t total = 0;
    for (uint64_t c = 0; c < jb.coarse_cells; ++c) total += jb.ncand[c];
    cand_t *all = malloc(sizeof(cand_t) * (total ? total : 1));
    uint64_t pos = 0;
    for (uint64_t c = 0; c < jb.coarse_cells; ++c) {
        if (jb.ncand[c]) memcpy(all + pos, jb.cand[c], sizeof(cand_t) * jb.ncand[c]);
        pos += jb.ncand[c];
        free(jb.cand[c]);
    }
    qsort(all, total, sizeof(cand_t), cmp_cand);
    mp->n_candidates = total;
    mp->cand_index = malloc(sizeof(uint64_t) * (total ? total : 1));
    mp->cand_value = malloc(sizeof(double) * 2 * (total ? total : 1));
    for (uint64_t i = 0; i < total; ++i) {
        mp->cand_index[i] = all[i].idx;
        mp->cand_value[2 * i] = creal(all[i].v);
        mp->cand_value[2 * i + 1] = cimag(all[i].v);
    }
    free(all);
    mp->n_rows = R;
    mp->peak_index = malloc(sizeof(uint64_t) * R);
    mp->peak_value = malloc(sizeof(double) * 2 * R);
    double best_m = -1.0;
    uint64_t best_i = 0;
    cplx best_v = 0;
    for (int r = 0; r < R; ++r) {
        double bm = -1.0;
        uint64_t bi = UINT64_MAX;
        cplx bv = 0;
        for (uint64_t c = 0; c < jb.coarse_cells; ++c) {
            size_t s2 = c * (size_t)R + r;
            if (jb.row_mag[s2] > bm || (jb.row_mag[s2] == bm && jb.row_idx[s2] < bi)) {
                bm = jb.row_mag[s2];
                bi = jb.row_idx[s2];
                bv = jb.row_val[s2];
            }
        }
        mp->peak_index[r] = bi;
        mp->peak_value[2 * r] = creal(bv);
        mp->peak_value[2 * r + 1] = cimag(bv);
        if (bm > best_m || (bm == best_m && bi < best_i)) {
            best_m = bm;
            best_i = bi;
            best_v = bv;
        }
    }
    mp->argmax = best_i;
    mp->argmax_value[0] = creal(best_v);
    mp->argmax_value[1] = cimag(best_v);
    mp->retain_threshold = jb.retain;
    mp->doppler_first = jb.dop_first;
    uint64_t Mu = (uint64_t)M, Nt = (uint64_t)R;
    mp->counters[0] = variant == 1 ? 1 : 0;
    mp->counters[2] = jb.coarse_cells * Mu;
    mp->counters[1] = jb.coarse_cells * jb.fine_cells * Nt;
    mp->counters[3] = jb.coarse_cells * jb.fine_cells * Nt;
    if (jb.keep_dense) {
        mp->dense_stored = 1;
        mp->dense_count = cells;
        mp->dense = malloc(sizeof(double) * 2 * cells);
        for (uint64_t i = 0; i < cells; ++i) {
            mp->dense[2 * i] = creal(jb.dense[i]);
            mp->dense[2 * i + 1] = cimag(jb.dense[i]);
        }
        free(jb.dense);
    }
    free(jb.cand);
    free(jb.ncand);
    free(jb.capcand);
    free(jb.row_mag);
    free(jb.row_idx);
    free(jb.row_val);
    free(cube);
    free(kt);
    *out = mp;
    return LTCI_OK;
}

void oracle_free_map(ltci_detection_map *m) {
    if (!m) return;
    free(m->cand_index);
    free(m->cand_value);
    free(m->dense);
    free(m->peak_index);
    free(m->peak_value);
    free(m);
}

int oracle_mgift(const double *cube_d, const ltci_radar *p, const double *c, int nc, int variant, double *out) {
    size_t n = (size_t)p->K * p->M;
    cplx *cube = to_cplx(cube_d, n), *o = malloc(sizeof(cplx) * n), *tw = twiddles(p->K);
    mgift_cell(cube, p, c, nc, variant, o, tw);
    for (size_t i = 0; i < n; ++i) {
        out[2 * i] = creal(o[i]);
        out[2 * i + 1] = cimag(o[i]);
    }
    free(cube);
    free(o);
    free(tw);
    return LTCI_OK;
}

int oracle_gft(const double *rows_d, const ltci_radar *p, const double *fine, int nf, int roi_first, int roi_last,
               double *out) {
    size_t n = (size_t)p->K * p->M;
    int R = roi_last - roi_first + 1, M = p->M;
    if (R <= 0 || roi_first < 0 || roi_last >= p->K) return LTCI_INVALID_ARGUMENT;
    cplx *rows = to_cplx(rows_d, n), *y = malloc(sizeof(cplx) * M), *sc = malloc(sizeof(cplx) * 2 * M);
    cplx *tw = twiddles(M);
    dfm_chirp(p, fine, nf, sc + M);
    for (int r = 0; r < R; ++r) {
        gft_row(rows, p, roi_first + r, sc + M, y, sc, tw);
        for (int j = 0; j < M; ++j) {
            out[2 * (r + (size_t)R * j)] = creal(y[j]);
            out[2 * (r + (size_t)R * j) + 1] = cimag(y[j]);
        }
    }
    free(rows);
    free(y);
    free(sc);
    free(tw);
    return LTCI_OK;
}

int oracle_keystone(const double *cube_d, const ltci_radar *p, int taps, double *out) {
    if (taps < 2) return LTCI_INVALID_ARGUMENT;
    size_t n = (size_t)p->K * p->M;
    cplx *cube = to_cplx(cube_d, n), *o = malloc(sizeof(cplx) * n);
    keystone_impl(cube, p, taps, o);
    for (size_t i = 0; i < n; ++i) {
        out[2 * i] = creal(o[i]);
        out[2 * i + 1] = cimag(o[i]);
    }
    free(cube);
    free(o);
    return LTCI_OK;
}

/* range_fft (proj/src/signal_model.cpp:97-107): per pulse, Fft::dft_minus --
 * the same radix-2 DIT as fft_plus with conjugated twiddles (proj/src/fft.cpp:30-51). */
int oracle_range_fft(const double *cube_d, const ltci_radar *p, double *out) {
    const int K = p->K;
    if (K < 1 || (K & (K - 1))) return LTCI_INVALID_ARGUMENT;
    size_t n = (size_t)K * p->M;
    cplx *x = to_cplx(cube_d, n);
    cplx *tw = twiddles(K);
    for (int k = 0; k < K / 2; ++k) tw[k] = conj(tw[k]);
    for (int m = 0; m < p->M; ++m) fft_plus(x + (size_t)m * K, K, tw);
    for (size_t i = 0; i < n; ++i) {
        out[2 * i] = creal(x[i]);
        out[2 * i + 1] = cimag(x[i]);
    }
    free(tw);
    free(x);
    return LTCI_OK;
}

/* ------------------------------------------- single-scale td_grft / kt_mfp --- */
/* One scan over cells in index order: UnitScan::consider + merge_units
 * (proj/src/detectors.cpp:16-50) collapse to this when units are visited in order. */
typedef struct {
    double retain;
    int keep_dense;
    cand_t *cand;
    uint64_t ncand, cap;
    double best_m;
    uint64_t best_i;
    cplx best_v;
    cplx *dense;
} scan_t;

static void scan_consider(scan_t *sc, uint64_t idx, cplx v) {
    double m = cabs(v);
    if (m > sc->retain) {
        if (sc->ncand == sc->cap) {
            sc->cap = sc->cap ? 2 * sc->cap : 256;
            sc->cand = realloc(sc->cand, sizeof(cand_t) * sc->cap);
        }
        sc->cand[sc->ncand++] = (cand_t){idx, v};
    }
    if (m > sc->best_m || (m == sc->best_m && idx < sc->best_i)) {
        sc->best_m = m;
        sc->best_i = idx;
        sc->best_v = v;
    }
    if (sc->keep_dense) sc->dense[idx] = v;
}

static void scan_finish(scan_t *sc, ltci_detection_map *mp, uint64_t cells) {
    qsort(sc->cand, sc->ncand, sizeof(cand_t), cmp_cand);
    mp->n_candidates = sc->ncand;
    mp->cand_index = malloc(sizeof(uint64_t) * (sc->ncand ? sc->ncand : 1));
    mp->cand_value = malloc(sizeof(double) * 2 * (sc->ncand ? sc->ncand : 1));
    for (uint64_t i = 0; i < sc->ncand; ++i) {
        mp->cand_index[i] = sc->cand[i].idx;
        mp->cand_value[2 * i] = creal(sc->cand[i].v);
        mp->cand_value[2 * i + 1] = cimag(sc->cand[i].v);
    }
    mp->argmax = sc->best_i;
    mp->argmax_value[0] = creal(sc->best_v);
    mp->argmax_value[1] = cimag(sc->best_v);
    mp->retain_threshold = sc->retain;
    if (sc->keep_dense) {
        mp->dense_stored = 1;
        mp->dense_count = cells;
        mp->dense = malloc(sizeof(double) * 2 * (cells ? cells : 1));
        for (uint64_t i = 0; i < cells; ++i) {
            mp->dense[2 * i] = creal(sc->dense[i]);
            mp->dense[2 * i + 1] = cimag(sc->dense[i]);
        }
    }
    free(sc->cand);
    free(sc->dense);
}

static int same_radar(const ltci_radar *a, const ltci_radar *b) {
    return a->K == b->K && a->M == b->M && a->fc == b->fc && a->fs == b->fs && a->PRF == b->PRF;
}

/* td_grft (proj/src/detectors.cpp:199-264) on a range-pulse cube [n + K*m].
 * opt->trajectory: 0 ZeroOutside, 1 Wrap, 2 Error (returns LTCI_OUT_OF_RANGE). */
int oracle_td_grft(const double *cube_d, const ltci_radar *p, const ltci_single_space *s, const ltci_options *opt,
                   ltci_detection_map **out) {
    const int K = p->K, M = p->M, P = s->order;
    if (!same_radar(p, &s->radar)) return LTCI_INVALID_ARGUMENT;
    const int R = s->roi_last - s->roi_first + 1;
    uint64_t cells = 1;
    for (int q = 0; q < P; ++q) cells *= (uint64_t)s->c[q].count;
    const int policy = opt ? opt->trajectory : 0;
    scan_t sc;
    memset(&sc, 0, sizeof(sc));
    sc.retain = opt ? opt->retain_threshold : 0.0;
    sc.keep_dense = opt ? opt->keep_dense : 0;
    sc.best_m = -1.0;
    if (sc.keep_dense) sc.dense = calloc(cells * (uint64_t)R ? cells * (uint64_t)R : 1, sizeof(cplx));
    cplx *cube = to_cplx(cube_d, (size_t)K * M);
    const double dop_scale = 4.0 * M_PI / lambda_of(p), bin_scale = 2.0 * p->fs / C_LIGHT;
    double *offset = malloc(sizeof(double) * M);
    cplx *phase = malloc(sizeof(cplx) * M);
    int rc = LTCI_OK;
    for (uint64_t cidx = 0; cidx < cells && rc == LTCI_OK; ++cidx) {
        /* decode_motion (proj/src/detectors.cpp:84-92): c_1 fastest */
        double cv[LTCI_MAX_ORDER];
        uint64_t rem = cidx;
        for (int q = 0; q < P; ++q) {
            int ip = (int)(rem % (uint64_t)s->c[q].count);
            rem /= (uint64_t)s->c[q].count;
            cv[q] = s->c[q].start + s->c[q].step * ip;
        }
        for (int m = 0; m < M; ++m) {
            double sv = poly_from(cv, P, slow_time(p, m), 1);
            offset[m] = bin_scale * sv;
            phase[m] = polar1(dop_scale * sv);
        }
        for (int r = 0; r < R && rc == LTCI_OK; ++r) {
            int n0 = s->roi_first + r;
            cplx acc = 0;
            for (int m = 0; m < M; ++m) {
                long n = lround((double)n0 + offset[m]);
                if (n < 0 || n >= K) {
                    if (policy == 0) continue;
                    if (policy == 1) {
                        n = ((n % K) + K) % K;
                    } else {
                        rc = LTCI_OUT_OF_RANGE;
                        break;
                    }
                }
                acc += cube[n + (size_t)K * m] * phase[m];
            }
            if (rc == LTCI_OK) scan_consider(&sc, cidx * (uint64_t)R + (uint64_t)r, acc);
        }
    }
    free(offset);
    free(phase);
    free(cube);
    if (rc != LTCI_OK) {
        free(sc.cand);
        free(sc.dense);
        return rc;
    }
    ltci_detection_map *mp = calloc(1, sizeof(*mp));
    mp->kind = LTCI_TD_GRFT;
    int a = 0; /* single_scale_axes (proj/src/detectors.cpp:94-101) */
    for (int q = P; q >= 2; --q) mp->axes[a++] = (ltci_axis){LTCI_AXIS_HIGHER, q, s->c[q - 1].count};
    mp->axes[a++] = (ltci_axis){LTCI_AXIS_VELOCITY, 1, s->c[0].count};
    mp->axes[a++] = (ltci_axis){LTCI_AXIS_RANGE, 0, R};
    mp->n_axes = a;
    mp->counters[1] = cells * (uint64_t)R;
    scan_finish(&sc, mp, cells * (uint64_t)R);
    *out = mp;
    return LTCI_OK;
}

/* kt_mfp (proj/src/detectors.cpp:266-326): keystone once; per (q, c2) cell
 * gift(KtRm) -- y .* H_KtRm, dft_plus(K) per pulse, no preDFM -- then gft({c2}). */
int oracle_kt_mfp(const double *cube_d, const ltci_radar *p, const ltci_ambiguity *amb, const ltci_single_space *s,
                  const ltci_options *opt, ltci_detection_map **out) {
    const int K = p->K, M = p->M;
    if (!same_radar(p, &s->radar) || s->order != 2) return LTCI_INVALID_ARGUMENT;
    const int R = s->roi_last - s->roi_first + 1;
    if (R <= 0 || s->roi_first < 0 || s->roi_last >= K) return LTCI_INVALID_ARGUMENT;
    const int nq = amb->q_max - amb->q_min + 1, n2 = s->c[1].count;
    const uint64_t cells = (uint64_t)nq * (uint64_t)n2, total = cells * (uint64_t)R * (uint64_t)M;
    scan_t sc;
    memset(&sc, 0, sizeof(sc));
    sc.retain = opt ? opt->retain_threshold : 0.0;
    sc.keep_dense = opt ? opt->keep_dense : 0;
    sc.best_m = -1.0;
    if (sc.keep_dense) sc.dense = calloc(total ? total : 1, sizeof(cplx));
    cplx *cube = to_cplx(cube_d, (size_t)K * M), *kt = malloc(sizeof(cplx) * (size_t)K * M);
    keystone_impl(cube, p, opt && opt->keystone_taps > 0 ? opt->keystone_taps : 8, kt);
    cplx *comp = malloc(sizeof(cplx) * (size_t)K * M), *h = malloc(sizeof(cplx) * M);
    cplx *y = malloc(sizeof(cplx) * M), *scratch = malloc(sizeof(cplx) * 2 * M);
    cplx *twK = twiddles(K), *twM = twiddles(M);
    const double s4 = 4.0 * M_PI / C_LIGHT;
    for (uint64_t cidx = 0; cidx < cells; ++cidx) {
        const int i2 = (int)(cidx % (uint64_t)n2), iq = (int)(cidx / (uint64_t)n2);
        const double c2 = s->c[1].start + s->c[1].step * i2, qva = (double)(amb->q_min + iq) * va_of(p);
        for (int m = 0; m < M; ++m) { /* build_mf(KtRm) + compensated_ifft (transforms.cpp:53-70,134-147) */
            const double tm = slow_time(p, m);
            cplx *dst = comp + (size_t)K * m;
            const cplx *src = kt + (size_t)K * m;
            for (int k = 0; k < K; ++k) {
                double fk = freq_of_row(p, k), fbar = 1.0 - fk / p->fc;
                dst[k] = src[k] * polar1(s4 * fk * (fbar * qva * tm - c2 * tm * tm));
            }
            fft_plus(dst, K, twK);
        }
        dfm_chirp(p, &c2, 1, h);
        const uint64_t base = cidx * (uint64_t)R * (uint64_t)M;
        for (int r = 0; r < R; ++r) {
            gft_row(comp, p, s->roi_first + r, h, y, scratch, twM);
            for (int j = 0; j < M; ++j) scan_consider(&sc, base + (uint64_t)r * M + (uint64_t)j, y[j]);
        }
    }
    free(cube);
    free(kt);
    free(comp);
    free(h);
    free(y);
    free(scratch);
    free(twK);
    free(twM);
    ltci_detection_map *mp = calloc(1, sizeof(*mp));
    mp->kind = LTCI_KT_MFP;
    mp->axes[0] = (ltci_axis){LTCI_AXIS_FOLDING, 0, nq};
    mp->axes[1] = (ltci_axis){LTCI_AXIS_HIGHER, 2, n2};
    mp->axes[2] = (ltci_axis){LTCI_AXIS_RANGE, 0, R};
    mp->axes[3] = (ltci_axis){LTCI_AXIS_DOPPLER, 0, M};
    mp->n_axes = 4;
    mp->counters[0] = 1;
    mp->counters[1] = cells * (uint64_t)K;
    mp->counters[2] = cells * (uint64_t)M;
    mp->counters[3] = cells * (uint64_t)R;
    scan_finish(&sc, mp, total);
    *out = mp;
    return LTCI_OK;
}
