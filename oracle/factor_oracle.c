/*
 * factor_oracle.c -- CPU restatement of the reference's test-matrix factory
 * front end: the complete-pivoting Bunch-Parlett factorization in
 * double-double (hjsvd.factory.bunch_parlett_factor) and Householder QR
 * shortening (hjsvd.factory.qr_shorten).
 *
 *   TEST INFRASTRUCTURE, NOT PRODUCT.  Only tests/ and bench-side CPU legs
 *   load this code, as the checker or the timed CPU baseline.  The product
 *   (paper_1008_1371_b200.factory over csrc/hsvd_factor.cu) never calls it.
 *
 * Same IEEE operation sequence as the reference (numpy evaluates every
 * expression with one rounding per operation and no contraction; built with
 * -ffp-contract=off), so the factor G, the signs and the permutation are
 * bit-identical to bunch_parlett_factor (pinned by tests/golden/factor_*.npz,
 * made by tests/golden/make_golden_factor.py from the real reference).
 *
 * Reference anchors (under /root/reference/pkg/src/hjsvd/):
 *   _two_sum .. sqrt       _dd.py:25-93
 *   _swap_sym              factory.py:117-121
 *   _symmetrize            factory.py:124-128
 *   _abs_dd                factory.py:131-133
 *   _bunch_parlett_dd      factory.py:136-255
 *   _assemble_factor       factory.py:258-267
 *   bunch_parlett_factor   factory.py:270-282
 *   qr_shorten             factory.py:300-334 (not bit-exact: numpy's norm and
 *                          dot use BLAS reduction orders; tolerance-checked)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

typedef struct { double h, l; } dd_t;

/* ---- _dd.py:25-93 --------------------------------------------------------- */
static inline dd_t two_sum(double a, double b)
{
    double s = a + b, bb = s - a;
    dd_t r = {s, (a - (s - bb)) + (b - bb)};
    return r;
}
static inline dd_t quick_two_sum(double a, double b)
{
    double s = a + b;
    dd_t r = {s, b - (s - a)};
    return r;
}
static inline void split(double a, double *hi, double *lo)
{
    double t = 134217729.0 * a;
    *hi = t - (t - a);
    *lo = a - *hi;
}
static inline dd_t two_prod(double a, double b)
{
    double p = a * b, ah, al, bh, bl;
    split(a, &ah, &al);
    split(b, &bh, &bl);
    dd_t r = {p, ((ah * bh - p) + ah * bl + al * bh) + al * bl};
    return r;
}
static inline dd_t dd_add(dd_t x, dd_t y)
{
    dd_t s = two_sum(x.h, y.h);
    double e = s.l + (x.l + y.l);
    return quick_two_sum(s.h, e);
}
static inline dd_t dd_neg(dd_t x)
{
    dd_t r = {-x.h, -x.l};
    return r;
}
static inline dd_t dd_sub(dd_t x, dd_t y) { return dd_add(x, dd_neg(y)); }
static inline dd_t dd_mul(dd_t x, dd_t y)
{
    dd_t p = two_prod(x.h, y.h);
    double e = p.l + (x.h * y.l + x.l * y.h);
    return quick_two_sum(p.h, e);
}
static inline dd_t dd_mul_f(dd_t x, double f)
{
    dd_t p = two_prod(x.h, f);
    double e = p.l + x.l * f;
    return quick_two_sum(p.h, e);
}
static inline dd_t dd_div(dd_t x, dd_t y)
{
    double q1 = x.h / y.h;
    dd_t r = dd_sub(x, dd_mul_f(y, q1));
    double q2 = (r.h + r.l) / y.h;
    return quick_two_sum(q1, q2);
}
static inline dd_t dd_sqrt(dd_t x)
{
    double r = sqrt(x.h);
    dd_t rr = two_prod(r, r);
    dd_t diff = dd_sub(x, rr);
    double corr = r > 0.0 ? (diff.h + diff.l) / (2.0 * r) : 0.0;
    return quick_two_sum(r, corr);
}
static inline dd_t dd_abs(dd_t x) { return x.h < 0.0 ? dd_neg(x) : x; }
static inline dd_t dd_c(double a)
{
    dd_t r = {a, 0.0};
    return r;
}

#define ALPHA ((1.0 + sqrt(17.0)) / 8.0)

/* ---- factory.py:136-255 (+ _assemble_factor 258-267) ---------------------
 * M: n x n, exactly symmetric (either storage order).  Outputs: G (n x n,
 * column-major, rows un-permuted, +1 columns first), signs (+1 first), perm,
 * *p_out.  Returns 0, or 3 = numerical singularity (stage in *stage_out). */
ORC_API int orc_bp_factor(const double *M, int64_t n, double thresh, double *G, int8_t *signs_out,
                          int64_t *perm, int64_t *p_out, int64_t *stage_out)
{
    const double alpha = ALPHA;
    double *Ah = malloc(sizeof(double) * n * n), *Al = calloc(n * n, sizeof(double));
    double *Lh = calloc(n * n, sizeof(double)), *Ll = calloc(n * n, sizeof(double));
    double *Xh = malloc(sizeof(double) * n * n), *Xl = malloc(sizeof(double) * n * n);
    int64_t *bcol = malloc(sizeof(int64_t) * n), *bsz = malloc(sizeof(int64_t) * n);
    dd_t *bd = malloc(sizeof(dd_t) * 3 * n);
    double *w0h = malloc(sizeof(double) * n), *w0l = malloc(sizeof(double) * n);
    double *w1h = malloc(sizeof(double) * n), *w1l = malloc(sizeof(double) * n);
    double *l0h = malloc(sizeof(double) * n), *l0l = malloc(sizeof(double) * n);
    double *l1h = malloc(sizeof(double) * n), *l1l = malloc(sizeof(double) * n);
    int status = 0;
    int64_t nb = 0;
#define A_H(i, j) Ah[(i) * n + (j)]
#define A_L(i, j) Al[(i) * n + (j)]
#define L_H(i, j) Lh[(i) * n + (j)]
#define L_L(i, j) Ll[(i) * n + (j)]
    memcpy(Ah, M, sizeof(double) * n * n);
    for (int64_t i = 0; i < n; ++i) {
        L_H(i, i) = 1.0;
        perm[i] = i;
    }
    int64_t k = 0;
    while (k < n) {
        const int64_t m = n - k;
        /* pivot search on |Ah[k:, k:]| (hi parts): first max of the diagonal,
         * first max in row-major order with the diagonal zeroed */
        int64_t i0 = 0;
        double mu0 = fabs(A_H(k, k));
        for (int64_t t = 1; t < m; ++t) {
            double v = fabs(A_H(k + t, k + t));
            if (v > mu0) { mu0 = v; i0 = t; }
        }
        int64_t i1 = 0, j1 = 0;
        double mu1 = 0.0;  /* off[0][0] = 0 */
        for (int64_t a = 0; a < m; ++a)
            for (int64_t b = 0; b < m; ++b) {
                double v = a == b ? 0.0 : fabs(A_H(k + a, k + b));
                if (v > mu1) { mu1 = v; i1 = a; j1 = b; }
            }
        if (i1 < j1) { int64_t t = i1; i1 = j1; j1 = t; }
        if (fmax(mu0, mu1) <= thresh) {  /* max() of two floats */
            status = 3;
            *stage_out = k;
            goto done;
        }
        if (m == 1 || mu0 >= alpha * mu1) {
            if (i0 != 0) {
                const int64_t a = k, b = k + i0;
                for (int64_t c = k; c < n; ++c) {  /* rows a, b over columns k: */
                    double t = A_H(a, c); A_H(a, c) = A_H(b, c); A_H(b, c) = t;
                    t = A_L(a, c); A_L(a, c) = A_L(b, c); A_L(b, c) = t;
                }
                for (int64_t r = k; r < n; ++r) {  /* columns a, b over rows k: */
                    double t = A_H(r, a); A_H(r, a) = A_H(r, b); A_H(r, b) = t;
                    t = A_L(r, a); A_L(r, a) = A_L(r, b); A_L(r, b) = t;
                }
                for (int64_t c = 0; c < k; ++c) {
                    double t = L_H(a, c); L_H(a, c) = L_H(b, c); L_H(b, c) = t;
                    t = L_L(a, c); L_L(a, c) = L_L(b, c); L_L(b, c) = t;
                }
                int64_t t = perm[a]; perm[a] = perm[b]; perm[b] = t;
            }
            const dd_t d = {A_H(k, k), A_L(k, k)};
            for (int64_t i = k + 1; i < n; ++i) {
                w0h[i] = A_H(i, k);
                w0l[i] = A_L(i, k);
                dd_t col = {w0h[i], w0l[i]};
                dd_t l = dd_div(col, d);
                l0h[i] = l.h;
                l0l[i] = l.l;
                L_H(i, k) = l.h;
                L_L(i, k) = l.l;
            }
            for (int64_t i = k + 1; i < n; ++i)
                for (int64_t j = k + 1; j < n; ++j) {
                    dd_t li = {l0h[i], l0l[i]}, cj = {w0h[j], w0l[j]};
                    dd_t aij = {A_H(i, j), A_L(i, j)};
                    dd_t x = dd_sub(aij, dd_mul(li, cj));
                    Xh[i * n + j] = x.h;
                    Xl[i * n + j] = x.l;
                }
            for (int64_t i = k + 1; i < n; ++i)
                for (int64_t j = k + 1; j < n; ++j) {
                    dd_t a = {Xh[i * n + j], Xl[i * n + j]}, b = {Xh[j * n + i], Xl[j * n + i]};
                    dd_t s = dd_mul_f(dd_add(a, b), 0.5);
                    A_H(i, j) = s.h;
                    A_L(i, j) = s.l;
                }
            bcol[nb] = k;
            bsz[nb] = 1;
            bd[3 * nb] = d;
            ++nb;
            k += 1;
        } else {
            const int64_t pr[2][2] = {{k, k + j1}, {k + 1, k + i1}};
            for (int q = 0; q < 2; ++q) {
                const int64_t a = pr[q][0], b = pr[q][1];
                if (a == b) continue;
                for (int64_t c = k; c < n; ++c) {
                    double t = A_H(a, c); A_H(a, c) = A_H(b, c); A_H(b, c) = t;
                    t = A_L(a, c); A_L(a, c) = A_L(b, c); A_L(b, c) = t;
                }
                for (int64_t r = k; r < n; ++r) {
                    double t = A_H(r, a); A_H(r, a) = A_H(r, b); A_H(r, b) = t;
                    t = A_L(r, a); A_L(r, a) = A_L(r, b); A_L(r, b) = t;
                }
                for (int64_t c = 0; c < k; ++c) {
                    double t = L_H(a, c); L_H(a, c) = L_H(b, c); L_H(b, c) = t;
                    t = L_L(a, c); L_L(a, c) = L_L(b, c); L_L(b, c) = t;
                }
                int64_t t = perm[a]; perm[a] = perm[b]; perm[b] = t;
            }
            const dd_t ea = {A_H(k, k), A_L(k, k)}, eb = {A_H(k + 1, k), A_L(k + 1, k)},
                       ec = {A_H(k + 1, k + 1), A_L(k + 1, k + 1)};
            const dd_t det = dd_sub(dd_mul(ea, ec), dd_mul(eb, eb));
            for (int64_t i = k + 2; i < n; ++i) {
                dd_t W0 = {A_H(i, k), A_L(i, k)}, W1 = {A_H(i, k + 1), A_L(i, k + 1)};
                w0h[i] = W0.h; w0l[i] = W0.l;
                w1h[i] = W1.h; w1l[i] = W1.l;
                dd_t l0 = dd_div(dd_sub(dd_mul(W0, ec), dd_mul(W1, eb)), det);
                dd_t l1 = dd_div(dd_sub(dd_mul(W1, ea), dd_mul(W0, eb)), det);
                l0h[i] = l0.h; l0l[i] = l0.l;
                l1h[i] = l1.h; l1l[i] = l1.l;
                L_H(i, k) = l0.h; L_L(i, k) = l0.l;
                L_H(i, k + 1) = l1.h; L_L(i, k + 1) = l1.l;
            }
            for (int64_t i = k + 2; i < n; ++i)
                for (int64_t j = k + 2; j < n; ++j) {
                    dd_t l0 = {l0h[i], l0l[i]}, l1 = {l1h[i], l1l[i]};
                    dd_t W0 = {w0h[j], w0l[j]}, W1 = {w1h[j], w1l[j]};
                    dd_t upd = dd_add(dd_mul(l0, W0), dd_mul(l1, W1));
                    dd_t aij = {A_H(i, j), A_L(i, j)};
                    dd_t x = dd_sub(aij, upd);
                    Xh[i * n + j] = x.h;
                    Xl[i * n + j] = x.l;
                }
            for (int64_t i = k + 2; i < n; ++i)
                for (int64_t j = k + 2; j < n; ++j) {
                    dd_t a = {Xh[i * n + j], Xl[i * n + j]}, b = {Xh[j * n + i], Xl[j * n + i]};
                    dd_t s = dd_mul_f(dd_add(a, b), 0.5);
                    A_H(i, j) = s.h;
                    A_L(i, j) = s.l;
                }
            bcol[nb] = k;
            bsz[nb] = 2;
            bd[3 * nb] = ea;
            bd[3 * nb + 1] = eb;
            bd[3 * nb + 2] = ec;
            ++nb;
            k += 2;
        }
    }
    {
        /* post-processing: G = P L Q_D |Lambda_D|^{1/2} (rows still pivoted) */
        double *Gh = calloc(n * n, sizeof(double)), *Gl = calloc(n * n, sizeof(double));
        int8_t *sg = malloc(n);
        const dd_t one = dd_c(1.0);
        for (int64_t q = 0; q < nb; ++q) {
            const int64_t col = bcol[q];
            if (bsz[q] == 1) {
                const dd_t d = bd[3 * q];
                const dd_t s = dd_sqrt(dd_abs(d));
                for (int64_t i = 0; i < n; ++i) {
                    dd_t g = dd_mul((dd_t){L_H(i, col), L_L(i, col)}, s);
                    Gh[i * n + col] = g.h;
                    Gl[i * n + col] = g.l;
                }
                sg[col] = d.h > 0.0 ? 1 : -1;
            } else {
                const dd_t ea = bd[3 * q], eb = bd[3 * q + 1], ec = bd[3 * q + 2];
                const dd_t zeta = dd_div(dd_sub(ec, ea), dd_mul_f(eb, 2.0));
                const double sgn = zeta.h >= 0.0 ? 1.0 : -1.0;
                const dd_t root = dd_sqrt(dd_add(one, dd_mul(zeta, zeta)));
                const dd_t t = dd_div(dd_c(sgn), dd_add(dd_abs(zeta), root));
                const dd_t cs = dd_div(one, dd_sqrt(dd_add(one, dd_mul(t, t))));
                const dd_t sn = dd_mul(t, cs);
                const dd_t lam1 = dd_sub(ea, dd_mul(t, eb));
                const dd_t lam2 = dd_add(ec, dd_mul(t, eb));
                const dd_t s1 = dd_sqrt(dd_abs(lam1)), s2 = dd_sqrt(dd_abs(lam2));
                for (int64_t i = 0; i < n; ++i) {
                    const dd_t L0 = {L_H(i, col), L_L(i, col)};
                    const dd_t L1 = {L_H(i, col + 1), L_L(i, col + 1)};
                    const dd_t u1 = dd_sub(dd_mul(L0, cs), dd_mul(L1, sn));
                    const dd_t u2 = dd_add(dd_mul(L0, sn), dd_mul(L1, cs));
                    const dd_t g1 = dd_mul(u1, s1), g2 = dd_mul(u2, s2);
                    Gh[i * n + col] = g1.h;
                    Gl[i * n + col] = g1.l;
                    Gh[i * n + col + 1] = g2.h;
                    Gl[i * n + col + 1] = g2.l;
                }
                sg[col] = lam1.h > 0.0 ? 1 : -1;
                sg[col + 1] = lam2.h > 0.0 ? 1 : -1;
            }
        }
        /* _assemble_factor: G[perm, :] = hi + lo; +1 columns first */
        int64_t p = 0;
        for (int64_t c = 0; c < n; ++c) p += sg[c] == 1;
        int64_t oc = 0;
        for (int pass = 0; pass < 2; ++pass)
            for (int64_t c = 0; c < n; ++c) {
                if ((pass == 0) != (sg[c] == 1)) continue;
                for (int64_t i = 0; i < n; ++i) G[oc * n + perm[i]] = Gh[i * n + c] + Gl[i * n + c];
                signs_out[oc] = sg[c];
                ++oc;
            }
        *p_out = p;
        free(Gh);
        free(Gl);
        free(sg);
    }
done:
    free(Ah); free(Al); free(Lh); free(Ll); free(Xh); free(Xl);
    free(bcol); free(bsz); free(bd);
    free(w0h); free(w0l); free(w1h); free(w1l); free(l0h); free(l0l); free(l1h); free(l1l);
#undef A_H
#undef A_L
#undef L_H
#undef L_L
    return status;
}
