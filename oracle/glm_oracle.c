/*
 * glm_oracle.c — CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity oracle for the B200 kernels.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It is never on the product path.
 *
 * Every function restates a reference function (paths relative to
 * /root/reference/pkg/src/hierglm/) and is pinned by the golden fixtures in
 * tests/golden/ that were produced by running the reference itself
 * (tests/golden/make_golden.py).
 *
 * Objective kinds (objectives.py:22 for 0..3; 4..7 are restated kinds with
 * parity UNPINNED by the reference):
 *   0 dual_l2_logistic  1 dual_l2_svm  2 ridge_primal  3 lasso_primal
 *   4 dual_ridge        5 elastic_net_primal  6 logistic_primal
 *   7 squared_hinge_primal  8 hinge_primal (smoothed hinge: target[r] = y_r / mu)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_SOLVER_ERROR 1
#define OR_DIVERGENCE 2
#define OR_USAGE 3

static const double BOUNDARY_EPS = 1e-12;      /* objectives.py:26 */
static const double DAMPING_FLOOR = 9.5367431640625e-07; /* 2^-20, solver.py:28 */
static const double PLATEAU_REL = 1e-12;       /* solver.py:247 */
static const uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;

/* ---------------------------------------------------------------- PRNG */

/* solver.py:41-46 */
uint64_t or_xorshift64_step(uint64_t s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

/* solver.py:49-54 */
uint64_t or_splitmix64(uint64_t x) {
    x += GOLDEN;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

/* solver.py:57-61 */
uint64_t or_derive_seed(uint64_t base, const uint64_t *idx, int n_idx) {
    uint64_t s = or_splitmix64(base);
    for (int i = 0; i < n_idx; ++i) s = or_splitmix64(s ^ (idx[i] + 0x632BE59BD9B4E019ULL));
    return s ? s : GOLDEN;
}

/* PermutationGenerator.keys (solver.py:77-84); state advanced in place. */
void or_perm_keys(uint64_t *state, int64_t n, uint32_t *keys) {
    uint64_t s = *state;
    for (int64_t i = 0; i < n; ++i) {
        s = or_xorshift64_step(s);
        keys[i] = (uint32_t)s;
    }
    *state = s;
}

/* np.argsort(keys, kind="stable") (solver.py:89, pipeline.py:78): LSD radix
 * sort of (key, index) pairs, 4 passes of 8 bits; LSD radix is stable. */
void or_stable_argsort_u32(const uint32_t *keys, int64_t n, int64_t *perm) {
    if (n <= 0) return;
    uint32_t *ka = malloc(sizeof(uint32_t) * n), *kb = malloc(sizeof(uint32_t) * n);
    int64_t *ib = malloc(sizeof(int64_t) * n);
    memcpy(ka, keys, sizeof(uint32_t) * n);
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    uint32_t *ksrc = ka, *kdst = kb;
    int64_t *isrc = perm, *idst = ib;
    for (int pass = 0; pass < 4; ++pass) {
        int shift = 8 * pass;
        int64_t count[257] = {0};
        for (int64_t i = 0; i < n; ++i) count[((ksrc[i] >> shift) & 0xFF) + 1]++;
        for (int b = 0; b < 256; ++b) count[b + 1] += count[b];
        for (int64_t i = 0; i < n; ++i) {
            int64_t pos = count[(ksrc[i] >> shift) & 0xFF]++;
            kdst[pos] = ksrc[i];
            idst[pos] = isrc[i];
        }
        uint32_t *kt = ksrc; ksrc = kdst; kdst = kt;
        int64_t *it = isrc; isrc = idst; idst = it;
    }
    /* 4 passes: data ends in the original buffers (perm / ka). */
    free(ka); free(kb); free(ib);
}

/* PermutationGenerator.permute (solver.py:86-89). */
void or_permute(uint64_t *state, int64_t n, int64_t *perm) {
    if (n <= 0) return;
    uint32_t *keys = malloc(sizeof(uint32_t) * n);
    or_perm_keys(state, n, keys);
    or_stable_argsort_u32(keys, n, perm);
    free(keys);
}

/* pipeline.generate_keys (pipeline.py:29-73): KEY_BLOCK=4096 blocks, block b
 * seeded by derive_seed(seed, b). */
void or_generate_keys(uint64_t seed, int64_t n, uint32_t *keys) {
    const int64_t KB = 4096;
    for (int64_t lo = 0, b = 0; lo < n; lo += KB, ++b) {
        uint64_t bi = (uint64_t)b;
        uint64_t s = or_derive_seed(seed, &bi, 1);
        int64_t hi = lo + KB < n ? lo + KB : n;
        for (int64_t i = lo; i < hi; ++i) {
            s = or_xorshift64_step(s);
            keys[i] = (uint32_t)s;
        }
    }
}

/* ------------------------------------------------------- objectives */

static int is_dual(int kind) { return kind == 0 || kind == 1 || kind == 4; }

/* binary entropy, objectives.py:142-147 */
static double entropy(double a) {
    double t1 = a > 0.0 ? a * log(a > 1e-320 ? a : 1e-320) : 0.0;
    double b = 1.0 - a;
    double t2 = a < 1.0 ? b * log(b > 1e-320 ? b : 1e-320) : 0.0;
    return t1 + t2;
}

static double softplus(double s) { /* np.logaddexp(0, s) */
    return s > 0 ? s + log1p(exp(-s)) : log1p(exp(s));
}

/* g_i(a) for one coordinate; y = per-coordinate target (dual_ridge) */
static double g_one(int kind, double lam, double rho, double y, double a) {
    switch (kind) {
    case 0: return entropy(a);                         /* objectives.py:167-168 */
    case 1: return -a;                                 /* objectives.py:169-170 */
    case 2: case 6: case 7: case 8: return 0.5 * lam * a * a;  /* objectives.py:171-172 */
    case 3: return lam * fabs(a);                      /* objectives.py:173 */
    case 4: return 0.5 * a * a - y * a;                /* restated */
    case 5: return lam * (rho * fabs(a) + 0.5 * (1.0 - rho) * a * a); /* restated */
    }
    return NAN;
}

/* g_sum (objectives.py:165-173) over alpha; y may be NULL unless kind 4 */
double or_g_sum(int kind, double lam, double rho, const double *y, const double *alpha,
                int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += g_one(kind, lam, rho, y ? y[i] : 0.0, alpha[i]);
    return s;
}

/* g_conjugate_sum (objectives.py:211-220) of s[i]; returns NAN when absent */
double or_g_conj_sum(int kind, double lam, double rho, const double *y, const double *s,
                     int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double x = s[i];
        switch (kind) {
        case 0: acc += softplus(x); break;
        case 1: acc += x + 1.0 > 0.0 ? x + 1.0 : 0.0; break;
        case 2: case 6: case 7: case 8: acc += x * x / (2.0 * lam); break;
        case 4: { double u = x + y[i]; acc += 0.5 * u * u; } break;
        case 5: {
            if (rho >= 1.0) return NAN;
            double u = fabs(x) - lam * rho;
            if (u > 0) acc += u * u / (2.0 * lam * (1.0 - rho));
        } break;
        default: return NAN;
        }
    }
    return acc;
}

/* Smoothed hinge (restated kind 8), target t = y / mu: h(z) = 0 for z >= 1,
 * (1 - z)^2 / (2 mu) for 1 - mu < z < 1, 1 - z - mu / 2 below; z = y v.
 * Returns h and its derivative in v; mu -> 0 gives the hinge max(0, 1 - z). */
static double smooth_hinge(double t, double v, double *dv) {
    const double y = t > 0.0 ? 1.0 : -1.0, mu = 1.0 / fabs(t), z = y * v;
    if (z >= 1.0) { *dv = 0.0; return 0.0; }
    if (z > 1.0 - mu) { const double m = 1.0 - z; *dv = -y * m / mu; return m * m / (2.0 * mu); }
    *dv = -y;
    return 1.0 - z - 0.5 * mu;
}

/* f_eval (objectives.py:129-133); target = b (primal) */
double or_f_eval(int kind, double lam, const double *target, const double *v, int64_t d) {
    double acc = 0.0;
    if (is_dual(kind)) {
        for (int64_t r = 0; r < d; ++r) acc += v[r] * v[r];
        return acc / (2.0 * lam);
    }
    if (kind == 6) {            /* restated: sum softplus(-y v) */
        for (int64_t r = 0; r < d; ++r) acc += softplus(-target[r] * v[r]);
        return acc;
    }
    if (kind == 7) {            /* restated: 1/2 sum max(0, 1 - y v)^2 */
        for (int64_t r = 0; r < d; ++r) {
            double m = 1.0 - target[r] * v[r];
            if (m > 0) acc += m * m;
        }
        return 0.5 * acc;
    }
    if (kind == 8) {            /* restated: sum smoothed hinge */
        double g;
        for (int64_t r = 0; r < d; ++r) acc += smooth_hinge(target[r], v[r], &g);
        return acc;
    }
    for (int64_t r = 0; r < d; ++r) {
        double e = v[r] - target[r];
        acc += e * e;
    }
    return 0.5 * acc;
}

static double sigm(double z) { return 0.5 * (1.0 + tanh(0.5 * z)); }

/* f_grad (objectives.py:136-139) */
void or_f_grad(int kind, double lam, const double *target, const double *v, int64_t d,
               double *grad) {
    for (int64_t r = 0; r < d; ++r) {
        if (is_dual(kind)) grad[r] = v[r] / lam;
        else if (kind == 6) grad[r] = -target[r] * sigm(-target[r] * v[r]);
        else if (kind == 7) {
            double m = 1.0 - target[r] * v[r];
            grad[r] = m > 0 ? -target[r] * m : 0.0;
        } else if (kind == 8) smooth_hinge(target[r], v[r], &grad[r]);
        else grad[r] = v[r] - target[r];
    }
}

/* f_conjugate (objectives.py:205-208) at w */
double or_f_conj(int kind, double lam, const double *target, const double *w, int64_t d) {
    double acc = 0.0, acc2 = 0.0;
    if (is_dual(kind)) {
        for (int64_t r = 0; r < d; ++r) acc += w[r] * w[r];
        return 0.5 * lam * acc;
    }
    if (kind == 6) {
        for (int64_t r = 0; r < d; ++r) {
            double p = -w[r] * target[r];
            acc += entropy(p);
        }
        return acc;
    }
    if (kind == 7) {
        for (int64_t r = 0; r < d; ++r) {
            double q = -w[r] * target[r];
            acc += 0.5 * q * q - q;
        }
        return acc;
    }
    if (kind == 8) {            /* h*(u) = u + mu u^2 / 2 on [-1, 0], u = y w */
        for (int64_t r = 0; r < d; ++r) {
            const double y = target[r] > 0.0 ? 1.0 : -1.0, mu = 1.0 / fabs(target[r]);
            const double u = y * w[r];
            acc += u + 0.5 * mu * u * u;
        }
        return acc;
    }
    for (int64_t r = 0; r < d; ++r) {
        acc += w[r] * w[r];
        acc2 += w[r] * target[r];
    }
    return 0.5 * acc + acc2;
}

/* --------------------------------------------------------- matrix ops */

/* SparseColumnMatrix.matvec (data.py:109-114) */
void or_matvec(int64_t n_rows, int64_t n_cols, const int64_t *indptr, const int32_t *rows,
               const double *vals, const double *x, double *out) {
    for (int64_t r = 0; r < n_rows; ++r) out[r] = 0.0;
    for (int64_t j = 0; j < n_cols; ++j)
        for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) out[rows[p]] += vals[p] * x[j];
}

/* SparseColumnMatrix.rmatvec (data.py:116-123) */
void or_rmatvec(int64_t n_cols, const int64_t *indptr, const int32_t *rows,
                const double *vals, const double *w, double *out) {
    for (int64_t j = 0; j < n_cols; ++j) {
        double acc = 0.0;
        for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) acc += vals[p] * w[rows[p]];
        out[j] = acc;
    }
}

/* col_sqnorms (data.py:98-107) */
void or_col_sqnorms(int64_t n_cols, const int64_t *indptr, const double *vals, double *out) {
    for (int64_t j = 0; j < n_cols; ++j) {
        double acc = 0.0;
        for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) acc += vals[p] * vals[p];
        out[j] = acc;
    }
}

/* ------------------------------------------------------ local solver */

/* coordinate_update (solver.py:152-187) from a precomputed ga; restated kinds
 * 4..7 follow DESIGN.md Appendix (parity unpinned). */
int or_step_from_ga(int kind, double lam, double rho, double y, double ga, double c,
                    double t, double *step) {
    if (!isfinite(ga)) return OR_SOLVER_ERROR;
    switch (kind) {
    case 2: case 6: case 7: case 8:   /* ridge-type g = lam a^2/2 */
        *step = -(ga + lam * t) / (c + lam);
        return OR_OK;
    case 3:
    lasso:
        if (c == 0.0) { *step = -t; return OR_OK; }
        {
            double u = t - ga / c, thr = lam / c;
            double m = fabs(u) - thr;
            *step = copysign(m > 0.0 ? m : 0.0, u) - t;
        }
        return OR_OK;
    case 1: {
        double tn;
        if (c == 0.0) tn = ga < 1.0 ? 1.0 : 0.0;
        else {
            tn = t + (1.0 - ga) / c;
            tn = tn > 1.0 ? 1.0 : (tn < 0.0 ? 0.0 : tn);   /* min(1, max(0, .)) */
        }
        *step = tn - t;
        return OR_OK;
    }
    case 4:
        *step = -(ga + t - y) / (c + 1.0);
        return OR_OK;
    case 5: {
        if (rho >= 1.0) goto lasso;
        double den = c + lam * (1.0 - rho);
        double z = c * t - ga, thr = lam * rho;
        double m = fabs(z) - thr;
        double tn = copysign(m > 0.0 ? m : 0.0, z) / den;
        *step = tn - t;
        return OR_OK;
    }
    case 0: {
        /* math.log(t / (1 - t)) raises outside (0, 1) (solver.py:181) */
        if (!(t > 0.0 && t < 1.0)) return OR_SOLVER_ERROR;
        double grad = ga + log(t / (1.0 - t));
        double curv = c + 1.0 / (t * (1.0 - t));
        double tn = t - grad / curv;
        tn = tn < BOUNDARY_EPS ? BOUNDARY_EPS : tn;            /* max(eps, .) */
        tn = (1.0 - BOUNDARY_EPS) < tn ? (1.0 - BOUNDARY_EPS) : tn; /* min(1-eps, .) */
        if (!isfinite(tn)) return OR_SOLVER_ERROR;
        *step = tn - t;
        return OR_OK;
    }
    }
    return OR_USAGE;
}

int or_coordinate_update(int kind, double lam, double rho, double y, const int32_t *rows,
                         const double *vals, int64_t nnz, double sqnorm, double t,
                         const double *view, double quad, double *step) {
    double ga = 0.0;
    for (int64_t p = 0; p < nnz; ++p) ga += vals[p] * view[rows[p]];
    return or_step_from_ga(kind, lam, rho, y, ga, quad * sqnorm, t, step);
}

typedef struct {
    int kind;
    double lam, rho;
    const double *y;        /* per-coordinate target (dual_ridge) or NULL */
    int64_t d, m;           /* rows (len of v), local coordinates */
    const int64_t *indptr;
    const int32_t *rows;
    const double *vals;
    const double *lin;
    double quad, cnst;
    const double *base;
} or_sub;

/* LocalSubproblem.value (solver.py:127-135): exact w = B delta */
static double sub_value(const or_sub *s, const double *delta, double *w, double *tmp) {
    or_matvec(s->d, s->m, s->indptr, s->rows, s->vals, delta, w);
    double lw = 0.0, ww = 0.0;
    for (int64_t r = 0; r < s->d; ++r) {
        lw += s->lin[r] * w[r];
        ww += w[r] * w[r];
    }
    for (int64_t i = 0; i < s->m; ++i) tmp[i] = s->base[i] + delta[i];
    return s->cnst + lw + 0.5 * s->quad * ww + or_g_sum(s->kind, s->lam, s->rho, s->y, tmp, s->m);
}

/* run_pass with n_threads=1 (solver.py:202-211) */
static int run_pass(const or_sub *s, double *delta, double *view, const int64_t *order,
                    const double *sq, double damping) {
    for (int64_t k = 0; k < s->m; ++k) {
        int64_t i = order[k];
        int64_t lo = s->indptr[i], hi = s->indptr[i + 1];
        double raw;
        int st = or_coordinate_update(s->kind, s->lam, s->rho, s->y ? s->y[i] : 0.0,
                                      s->rows + lo, s->vals + lo, hi - lo, sq[i],
                                      s->base[i] + delta[i], view, s->quad, &raw);
        if (st) return st;
        double step = damping * raw;
        if (step != 0.0) {
            delta[i] += step;
            double f = s->quad * step;
            for (int64_t p = lo; p < hi; ++p) view[s->rows[p]] += f * s->vals[p];
        }
    }
    return OR_OK;
}

/* damped_solve (solver.py:250-305), sequential.  Outputs:
 *   delta_out[m], dv_out[d], values_out[t_epochs] (accepted G per epoch),
 *   info: epochs_run, retries, plateaued
 *   vals_io: [0] damping (in/out), [1] initial G (out), [2] final G (out)
 *   gen_state: PermutationGenerator.state (in/out) */
int or_damped_solve(int kind, double lam, double rho, const double *y, int64_t d, int64_t m,
                    const int64_t *indptr, const int32_t *rows, const double *vals,
                    const double *lin, double quad, double cnst, const double *base,
                    uint64_t *gen_state, int t_epochs, double *delta_out, double *dv_out,
                    double *values_out, int32_t *info, double *vals_io) {
    if (t_epochs < 1) return OR_USAGE;
    or_sub s = {kind, lam, rho, y, d, m, indptr, rows, vals, lin, quad, cnst, base};
    double *sq = malloc(sizeof(double) * (m + 1));
    double *view = malloc(sizeof(double) * (d + 1));
    double *snap_v = malloc(sizeof(double) * (d + 1));
    double *snap_d = malloc(sizeof(double) * (m + 1));
    double *w = malloc(sizeof(double) * (d + 1));
    double *tmp = malloc(sizeof(double) * (m + 1));
    int64_t *order = malloc(sizeof(int64_t) * (m + 1));
    int status = OR_OK;
    or_col_sqnorms(m, indptr, vals, sq);
    double *delta = delta_out;
    for (int64_t i = 0; i < m; ++i) delta[i] = 0.0;
    memcpy(view, lin, sizeof(double) * d);
    double value = sub_value(&s, delta, w, tmp);
    double initial = value;
    double damping = vals_io[0];
    int epochs_run = 0, retries = 0, plateaued = 0;
    for (int e = 0; e < t_epochs && !plateaued; ++e) {
        for (;;) {
            memcpy(snap_d, delta, sizeof(double) * m);
            memcpy(snap_v, view, sizeof(double) * d);
            or_permute(gen_state, m, order);
            status = run_pass(&s, delta, view, order, sq, damping);
            if (status) goto done;
            for (int64_t r = 0; r < d; ++r)
                if (!isfinite(view[r])) { status = OR_SOLVER_ERROR; goto done; }
            double nv = sub_value(&s, delta, w, tmp);
            if (nv > value) {
                memcpy(delta, snap_d, sizeof(double) * m);
                memcpy(view, snap_v, sizeof(double) * d);
                if (nv - value <= PLATEAU_REL * (1.0 + fabs(value))) { plateaued = 1; break; }
                retries++;
                damping *= 0.5;
                if (damping < DAMPING_FLOOR) { status = OR_DIVERGENCE; goto done; }
                continue;
            }
            value = nv;
            values_out[epochs_run++] = value;
            break;
        }
    }
    or_matvec(d, m, indptr, rows, vals, delta, dv_out);   /* solver.py:300 */
done:
    info[0] = epochs_run;
    info[1] = retries;
    info[2] = plateaued;
    vals_io[0] = damping;
    vals_io[1] = initial;
    vals_io[2] = value;
    free(sq); free(view); free(snap_v); free(snap_d); free(w); free(tmp); free(order);
    return status;
}

/* Chunked epoch (pipeline.py:158-197, 200-242 sequential): one pass over the
 * chunks [offsets[c], offsets[c+1]) of the device's coordinates, keys from
 * generate_keys(derive_seed(seed, epoch_index, c)), chunk-granular damping.
 * delta/view in-out; returns the device value after the epoch in *value_out. */
int or_chunked_epoch(int kind, double lam, double rho, const double *y, int64_t d, int64_t m,
                     const int64_t *indptr, const int32_t *rows, const double *vals,
                     const double *lin, double quad, double cnst, const double *base,
                     int n_chunks, const int64_t *offsets, uint64_t seed, uint64_t epoch_index,
                     double *damping_io, double *delta, double *view, double *value_out) {
    or_sub s = {kind, lam, rho, y, d, m, indptr, rows, vals, lin, quad, cnst, base};
    double *sq = malloc(sizeof(double) * (m + 1));
    double *w = malloc(sizeof(double) * (d + 1));
    double *tmp = malloc(sizeof(double) * (m + 1));
    double *snap_v = malloc(sizeof(double) * (d + 1));
    double *snap_d = malloc(sizeof(double) * (m + 1));
    int status = OR_OK;
    or_col_sqnorms(m, indptr, vals, sq);
    double value = sub_value(&s, delta, w, tmp);
    for (int c = 0; c < n_chunks; ++c) {
        int64_t lo = offsets[c], hi = offsets[c + 1], nc = hi - lo;
        uint64_t ix[2] = {epoch_index, (uint64_t)c};
        uint64_t cs = or_derive_seed(seed, ix, 2);
        uint32_t *keys = malloc(sizeof(uint32_t) * (nc + 1));
        int64_t *order = malloc(sizeof(int64_t) * (nc + 1));
        or_generate_keys(cs, nc, keys);
        or_stable_argsort_u32(keys, nc, order);
        for (int64_t k = 0; k < nc; ++k) order[k] += lo;
        double value0 = sub_value(&s, delta, w, tmp);
        for (;;) {
            memcpy(snap_d, delta + lo, sizeof(double) * nc);
            memcpy(snap_v, view, sizeof(double) * d);
            /* run_pass over the chunk's order (device-local coordinates) */
            for (int64_t k = 0; k < nc && !status; ++k) {
                int64_t i = order[k];
                double raw;
                int64_t a = indptr[i], b = indptr[i + 1];
                status = or_coordinate_update(kind, lam, rho, y ? y[i] : 0.0, rows + a, vals + a,
                                              b - a, sq[i], base[i] + delta[i], view, quad, &raw);
                if (status) break;
                double step = *damping_io * raw;
                if (step != 0.0) {
                    delta[i] += step;
                    double f = quad * step;
                    for (int64_t p = a; p < b; ++p) view[rows[p]] += f * vals[p];
                }
            }
            if (status) { free(keys); free(order); goto done; }
            double nv = sub_value(&s, delta, w, tmp);
            if (nv > value0) {
                memcpy(delta + lo, snap_d, sizeof(double) * nc);
                memcpy(view, snap_v, sizeof(double) * d);
                if (nv - value0 <= PLATEAU_REL * (1.0 + fabs(value0))) { value = value0; break; }
                *damping_io *= 0.5;
                if (*damping_io < DAMPING_FLOOR) { status = OR_DIVERGENCE; free(keys); free(order); goto done; }
                continue;
            }
            value = nv;
            break;
        }
        free(keys);
        free(order);
    }
done:
    *value_out = value;
    free(sq); free(w); free(tmp); free(snap_v); free(snap_d);
    return status;
}
