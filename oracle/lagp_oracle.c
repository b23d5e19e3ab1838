/*
 * lagp_oracle.c — plain, slow, obviously-correct CPU oracle for the hot path of
 * Gramacy, Niemi & Weiss, "Massively parallel approximate Gaussian process
 * regression" (arXiv 1310.5182).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code,
 * header, table or constant with the CUDA path (paper_1310_5182_b200/csrc).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (with section / equation /
 * figure); readings Rk = DESIGN.md §3 reading k (where the paper is silent,
 * garbled or inconsistent).
 *
 * Everything is IEEE FP64 (the paper's kernel is double precision, P:525,
 * P:539), compiled without -ffast-math and with -ffp-contract=off so
 * that the only fused multiply-adds are the explicit fma() calls below.
 *
 * Pins (tests/test_oracle_pins.py): every function here is checked against
 * something other than itself — brute-force variance differences, direct
 * inversion, exhaustive sorting, the full-GP special case, closed forms and the
 * worked examples of tests/golden/. See DESIGN.md §4 for the pin table.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* per-location flag bits (reading R12 / SPEC S:171) */
#define OR_FLAG_NEAR_TIE 1u
#define OR_FLAG_SENTINEL 2u
#define OR_FLAG_EXHAUSTED 4u
#define OR_FLAG_NONFINITE 8u

#define OR_S_MIN 1e-12  /* candidates with m_j^{-1}(x') <= 1e-12 are excluded (R12) */
#define OR_TIE_GAP 1e-12 /* near-tie threshold on the top-2 relative gap (north_star) */

/* ------------------------------------------------------------------------- */
/* Squared Euclidean distance, accumulated with fma in the fixed order
 * k = 0..p-1 starting from 0 (reading R8: NN distances "relative to the chosen
 * correlation function", i.e. Euclidean for the isotropic Gaussian). */
static double sqdist(const double *a, const double *b, int p) {
    double acc = 0.0;
    for (int k = 0; k < p; k++) {
        double diff = a[k] - b[k];
        acc = fma(diff, diff, acc);
    }
    return acc;
}

/* Isotropic Gaussian correlation K(x,x') = exp(-||x-x'||^2 / theta).
 * No nugget here: eta enters only the diagonal of K_j (Fig 3 step 5; R5). */
static double corr(const double *a, const double *b, int p, double theta) {
    return exp(-sqdist(a, b, p) / theta);
}

/* ------------------------------------------------------------------------- */
/* a1 — nearest-neighbour pool, P:250-253 (NN sub-design), Fig 1 step 2(a)
 * P:365, and the N' NN candidate restriction P:484-487.
 * Exhaustive: all N distances, stable ordering by the key (d^2, index)
 * (ties -> lowest index, R8 / SPEC S:258), first m rows. */
typedef struct { double d2; int64_t i; } or_key;

static int key_cmp(const void *pa, const void *pb) {
    const or_key *a = (const or_key *)pa, *b = (const or_key *)pb;
    if (a->d2 < b->d2) return -1;
    if (a->d2 > b->d2) return 1;
    return (a->i < b->i) ? -1 : (a->i > b->i);
}

int oracle_nn(const double *X, int64_t N, int p, const double *x, int32_t m,
              int32_t *idx_out, double *d2_out) {
    if (m < 0 || m > N) return 2;
    or_key *keys = (or_key *)malloc(sizeof(or_key) * (size_t)(N > 0 ? N : 1));
    if (!keys) return 4;
    for (int64_t i = 0; i < N; i++) {
        keys[i].d2 = sqdist(x, X + i * p, p);
        keys[i].i = i;
    }
    qsort(keys, (size_t)N, sizeof(or_key), key_cmp);
    for (int32_t r = 0; r < m; r++) {
        idx_out[r] = (int32_t)keys[r].i;
        if (d2_out) d2_out[r] = keys[r].d2;
    }
    free(keys);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Dense SPD helpers: textbook Cholesky K = L L^T (lower, row-major). */
static int cholesky(int n, const double *A, double *L) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; i++) {
        for (int k = 0; k <= i; k++) {
            double s = A[i * n + k];
            for (int t = 0; t < k; t++) s -= L[i * n + t] * L[k * n + t];
            if (i == k) {
                if (!(s > 0.0)) return 1;
                L[i * n + i] = sqrt(s);
            } else {
                L[i * n + k] = s / L[k * n + k];
            }
        }
    }
    return 0;
}

/* solve L L^T y = b in place */
static void chol_solve(int n, const double *L, double *y) {
    for (int i = 0; i < n; i++) {
        double s = y[i];
        for (int t = 0; t < i; t++) s -= L[i * n + t] * y[t];
        y[i] = s / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; i--) {
        double s = y[i];
        for (int t = i + 1; t < n; t++) s -= L[t * n + i] * y[t];
        y[i] = s / L[i * n + i];
    }
}

/* Explicit inverse of an SPD matrix via Cholesky: column-by-column solves.
 * The paper keeps an explicit K_j^{-1} (Fig 2). Symmetrised by averaging
 * is NOT done; instead entry (a,b) is taken from solve b for a >= b and mirrored. */
int oracle_invert_spd(int n, const double *A, double *Ainv) {
    double *L = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *e = (double *)malloc(sizeof(double) * (size_t)n + 8);
    if (!L || !e) { free(L); free(e); return 4; }
    if (cholesky(n, A, L)) { free(L); free(e); return 1; }
    for (int b = 0; b < n; b++) {
        for (int i = 0; i < n; i++) e[i] = (i == b) ? 1.0 : 0.0;
        chol_solve(n, L, e);
        for (int a = b; a < n; a++) { Ainv[a * n + b] = e[a]; Ainv[b * n + a] = e[a]; }
    }
    free(L); free(e);
    return 0;
}

/* K_j = C(X_j) + eta I  (A3 correlation + nugget on the diagonal) */
static void build_K(int j, int p, const double *Xj, double theta, double eta, double *K) {
    for (int a = 0; a < j; a++)
        for (int b = 0; b < j; b++)
            K[a * j + b] = corr(Xj + a * p, Xj + b * p, p, theta) + (a == b ? eta : 0.0);
}

/* ------------------------------------------------------------------------- */
/* a3 — ALC reduction in variance for one candidate x' given the explicit
 * K_j^{-1} and h = k_j(x), following Eq (5)-(6):
 *   u      = K_j^{-1} k_j(x')                       (Fig 3 step 3)
 *   m^{-1} = K_j(x',x') - k_j(x')^T u = 1 + eta - k^T u   (Eq 6; Fig 3 step 5)
 *   g      = -m K_j^{-1} k_j(x') = -u / m^{-1}      (Eq 6; sign per Eq 6, R1)
 *   kap    = K(x', x)                               (Fig 3 step 5, no nugget, R5)
 *   Eq (5) literal: Delta = h^T G m^{-1} h + 2 h^T g kap + kap^2 m,  G = g g^T (R3)
 *   closed form    : Delta = (kap - h^T u)^2 / m^{-1}   (algebra on Eq 5, R1)
 * Returns m^{-1}; writes both forms. */
static double alc_one(int j, int p, const double *Xj, const double *Kinv, const double *h,
                      const double *xc, const double *x, double theta, double eta,
                      double *u /* scratch j */, double *kc /* scratch j */,
                      double *delta_cf, double *delta_lit) {
    for (int a = 0; a < j; a++) kc[a] = corr(Xj + a * p, xc, p, theta);
    for (int a = 0; a < j; a++) {
        double s = 0.0;
        for (int b = 0; b < j; b++) s += Kinv[a * j + b] * kc[b];
        u[a] = s;
    }
    double ku = 0.0;
    for (int a = 0; a < j; a++) ku += kc[a] * u[a];
    double minv = 1.0 + eta - ku;
    double kap = corr(xc, x, p, theta);
    double hu = 0.0;
    for (int a = 0; a < j; a++) hu += h[a] * u[a];
    if (delta_cf) { double c = kap - hu; *delta_cf = c * c / minv; }
    if (delta_lit) {
        /* h^T g with g = -u/minv */
        double hg = 0.0;
        for (int a = 0; a < j; a++) hg += h[a] * (-u[a] / minv);
        *delta_lit = hg * hg * minv + 2.0 * hg * kap + kap * kap / minv;
    }
    return minv;
}

/* Diagnostic entry (Fig 2 I/O for one location): scores of nc candidates. */
int oracle_alc_scores(int j, int p, int nc, const double *Xj, const double *Kinv,
                      const double *cands, const double *x, double theta, double eta,
                      double *delta_cf, double *delta_lit, double *minv_out) {
    double *h = (double *)malloc(sizeof(double) * (size_t)(j + 1));
    double *u = (double *)malloc(sizeof(double) * (size_t)(j + 1));
    double *kc = (double *)malloc(sizeof(double) * (size_t)(j + 1));
    if (!h || !u || !kc) { free(h); free(u); free(kc); return 4; }
    for (int a = 0; a < j; a++) h[a] = corr(Xj + a * p, x, p, theta);
    for (int c = 0; c < nc; c++) {
        double dc, dl;
        double m = alc_one(j, p, Xj, Kinv, h, cands + (size_t)c * p, x, theta, eta, u, kc, &dc, &dl);
        if (delta_cf) delta_cf[c] = dc;
        if (delta_lit) delta_lit[c] = dl;
        if (minv_out) minv_out[c] = m;
    }
    free(h); free(u); free(kc);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* a4 — partitioned-inverse update (Barnett 1979,
 * Gramacy & Polson 2011): with u = K_j^{-1} k, m^{-1} = kdiag - k^T u,
 * g = -u / m^{-1}, m = 1/m^{-1}:
 *   K_{j+1}^{-1} = [[ K_j^{-1} + g g^T m^{-1} , g ],
 *                   [ g^T                     , m ]]                    */
int oracle_pinv_update(int j, const double *Kinv, const double *k, double kdiag, double *Kout) {
    int J = j + 1;
    double *u = (double *)malloc(sizeof(double) * (size_t)J);
    double *g = (double *)malloc(sizeof(double) * (size_t)J);
    if (!u || !g) { free(u); free(g); return 4; }
    for (int a = 0; a < j; a++) {
        double s = 0.0;
        for (int b = 0; b < j; b++) s += Kinv[a * j + b] * k[b];
        u[a] = s;
    }
    double ku = 0.0;
    for (int a = 0; a < j; a++) ku += k[a] * u[a];
    double minv = kdiag - ku;
    for (int a = 0; a < j; a++) g[a] = -u[a] / minv;
    for (int a = 0; a < j; a++)
        for (int b = 0; b < j; b++) Kout[a * J + b] = Kinv[a * j + b] + g[a] * g[b] * minv;
    for (int a = 0; a < j; a++) { Kout[a * J + j] = g[a]; Kout[j * J + a] = g[a]; }
    Kout[j * J + j] = 1.0 / minv;
    free(u); free(g);
    return (minv > 0.0) ? 0 : 1;
}

/* ------------------------------------------------------------------------- */
/* a5 — local GP prediction, Eq (1)-(2) with N -> n on D_n(x)
 * (Fig 1 step 5): fresh Cholesky of K_n = C(X_n) + eta I;
 *   mu = h^T K^{-1} Y ; psi = Y^T K^{-1} Y ; s2 = psi (K(x,x) - h^T K^{-1} h) / n
 * with K(x,x) = 1 + eta (R4);  var = s2 n / (n - 2), NaN if n <= 2. */
int oracle_predict(int n, int p, const double *Xn, const double *Yn, const double *x,
                   double theta, double eta, double *mean, double *s2, double *var) {
    double *K = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *L = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *h = (double *)malloc(sizeof(double) * (size_t)n + 8);
    double *a = (double *)malloc(sizeof(double) * (size_t)n + 8);
    double *b = (double *)malloc(sizeof(double) * (size_t)n + 8);
    int rc = 0;
    if (!K || !L || !h || !a || !b) { rc = 4; goto out; }
    build_K(n, p, Xn, theta, eta, K);
    if (cholesky(n, K, L)) { rc = 1; goto out; }
    for (int i = 0; i < n; i++) { h[i] = corr(Xn + i * p, x, p, theta); a[i] = h[i]; b[i] = Yn[i]; }
    chol_solve(n, L, a);
    chol_solve(n, L, b);
    double mu = 0.0, psi = 0.0, hKh = 0.0;
    for (int i = 0; i < n; i++) { mu += h[i] * b[i]; psi += Yn[i] * b[i]; hKh += h[i] * a[i]; }
    double sc = psi * (1.0 + eta - hKh) / n;
    *mean = mu;
    *s2 = sc;
    *var = (n > 2) ? sc * n / (n - 2) : NAN;
out:
    free(K); free(L); free(h); free(a); free(b);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Fig 1 step 2 for ONE predictive location x:
 *   (a) NN design X_{n0}(x) = first n0 rows of the N' NN pool (a1, a2);
 *   (b) for j = n0 .. n-1 (R9): x_{j+1} = argmax over pool \ X_j of
 *       v_j(x) - v_{j+1}(x)  [Eq (5)], ties -> lowest global row index (R7),
 *       then the partitioned-inverse update (a4);
 *   step 5: predict on D_n(x) (a5).
 * Outputs: idx[n] (first n0 = NN order, then greedy order; -1 tail when
 * exhausted), mean/s2/var, flags, gaps[n-n0] = (D1-D2)/D1 per step,
 * best[n-n0] = D1 per step (telescoping pin P7), s2_acc = s2 read off the
 * accumulated K_n^{-1} (diagnostic only). */
int oracle_local_design(const double *X, int64_t N, int p, const double *Z, const double *x,
                        double theta, double eta, int n0, int n, int Nprime,
                        int32_t *idx, double *mean, double *s2, double *var, uint32_t *flags,
                        double *gaps, double *best, double *s2_acc) {
    uint32_t fl = 0;
    int rc = 0;
    int32_t *pool = (int32_t *)malloc(sizeof(int32_t) * (size_t)Nprime);
    char *chosen = (char *)calloc((size_t)Nprime, 1);
    double *Xj = (double *)malloc(sizeof(double) * (size_t)n * p);
    double *Yj = (double *)malloc(sizeof(double) * (size_t)n);
    double *Kinv = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *Knew = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *K0 = (double *)malloc(sizeof(double) * (size_t)n0 * n0);
    double *h = (double *)malloc(sizeof(double) * (size_t)n);
    double *u = (double *)malloc(sizeof(double) * (size_t)n);
    double *kc = (double *)malloc(sizeof(double) * (size_t)n);
    if (!pool || !chosen || !Xj || !Yj || !Kinv || !Knew || !K0 || !h || !u || !kc) { rc = 4; goto out; }

    for (int t = 0; t < n; t++) idx[t] = -1;
    for (int t = 0; t < n - n0; t++) { gaps[t] = NAN; best[t] = NAN; }

    /* (a) NN pool and initial design */
    rc = oracle_nn(X, N, p, x, Nprime, pool, NULL);
    if (rc) goto out;
    int j = n0;
    for (int t = 0; t < n0; t++) {
        idx[t] = pool[t];
        chosen[t] = 1;
        memcpy(Xj + t * p, X + (size_t)pool[t] * p, sizeof(double) * p);
        Yj[t] = Z[pool[t]];
    }
    build_K(n0, p, Xj, theta, eta, K0);
    if (oracle_invert_spd(n0, K0, Kinv)) { fl |= OR_FLAG_NONFINITE; rc = 0; goto predict; }
    for (int a = 0; a < n0; a++) h[a] = corr(Xj + a * p, x, p, theta);

    /* (b) greedy ALC loop */
    for (j = n0; j < n; j++) {
        int bpos = -1;
        int32_t bidx = -1;
        double d1 = -INFINITY, d2 = -INFINITY;
        for (int c = 0; c < Nprime; c++) {
            if (chosen[c]) continue;
            const double *xc = X + (size_t)pool[c] * p;
            double dcf;
            double minv = alc_one(j, p, Xj, Kinv, h, xc, x, theta, eta, u, kc, &dcf, NULL);
            if (!(minv > OR_S_MIN)) { fl |= OR_FLAG_SENTINEL; continue; }
            if (!isfinite(dcf)) { fl |= OR_FLAG_NONFINITE; continue; }
            if (dcf > d1 || (dcf == d1 && pool[c] < bidx)) {
                d2 = d1;
                d1 = dcf;
                bpos = c;
                bidx = pool[c];
            } else if (dcf > d2) {
                d2 = dcf;
            }
        }
        if (bpos < 0) { fl |= OR_FLAG_EXHAUSTED; break; }
        double gap = (d2 > 0.0) ? (d1 - d2) / d1 : ((d1 > 0.0) ? 1.0 : 0.0);
        if (!(d1 > 0.0) || gap < OR_TIE_GAP) fl |= OR_FLAG_NEAR_TIE;
        gaps[j - n0] = gap;
        best[j - n0] = d1;

        /* a4: partitioned inverse with the chosen x_{j+1} */
        const double *xs = X + (size_t)bidx * p;
        for (int a = 0; a < j; a++) kc[a] = corr(Xj + a * p, xs, p, theta);
        if (oracle_pinv_update(j, Kinv, kc, 1.0 + eta, Knew)) { fl |= OR_FLAG_NONFINITE; }
        memcpy(Kinv, Knew, sizeof(double) * (size_t)(j + 1) * (j + 1));
        chosen[bpos] = 1;
        idx[j] = bidx;
        memcpy(Xj + j * p, xs, sizeof(double) * p);
        Yj[j] = Z[bidx];
        h[j] = corr(xs, x, p, theta);
    }

predict:
    /* diagnostic: s2 from the accumulated inverse (not the output) */
    if (s2_acc) {
        double psi = 0.0, hKh = 0.0;
        for (int a = 0; a < j; a++)
            for (int b = 0; b < j; b++) {
                psi += Yj[a] * Kinv[a * j + b] * Yj[b];
                hKh += h[a] * Kinv[a * j + b] * h[b];
            }
        *s2_acc = psi * (1.0 + eta - hKh) / j;
    }
    if (oracle_predict(j, p, Xj, Yj, x, theta, eta, mean, s2, var)) {
        fl |= OR_FLAG_NONFINITE;
        *mean = NAN; *s2 = NAN; *var = NAN;
    }
    if (!isfinite(*mean) || !isfinite(*s2)) fl |= OR_FLAG_NONFINITE;
out:
    if (flags) *flags = fl;
    free(pool); free(chosen); free(Xj); free(Yj); free(Kinv); free(Knew); free(K0);
    free(h); free(u); free(kc);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Score noise of this oracle (reading R18: tau_cfg). Along the trajectory idx[n]
 * that oracle_local_design chose for x, recompute at every greedy step j the
 * oracle's own explicit-K_j^{-1} scores (the same oracle_invert_spd /
 * oracle_pinv_update / alc_one calls in the same order, so bit-identical to the
 * run) and reference scores by a FRESH long-double solve of the same Eq (5)
 * closed form (App A.1): with K_j = L L^T (long-double Cholesky of the long-
 * double kernel matrix), v = L^{-1} k_j(x'), z = L^{-1} h,
 *   Delta_ref = (kappa - z^T v)^2 / (1 + eta - v^T v).
 * noise[j - n0] = max_c |Delta_explicit - Delta_ref| / max_c Delta_ref over the
 * candidates both sides keep (s > 1e-12); ref_gap[j - n0] = the reference top-2
 * relative gap (R19). Steps after an exhaustion (-1 in idx) get NaN.
 * Measurement only: nothing here changes what the oracle selects. */
static long double corr_ld(const double *a, const double *b, int p, double theta) {
    long double acc = 0.0L;
    for (int k = 0; k < p; k++) {
        long double diff = (long double)a[k] - (long double)b[k];
        acc += diff * diff;
    }
    return expl(-acc / (long double)theta);
}

int oracle_score_noise(const double *X, int64_t N, int p, const double *x, double theta, double eta,
                       int n0, int n, int Nprime, const int32_t *idx, double *noise, double *ref_gap) {
    int rc = 0;
    int32_t *pool = (int32_t *)malloc(sizeof(int32_t) * (size_t)Nprime);
    char *chosen = (char *)calloc((size_t)Nprime, 1);
    double *Xj = (double *)malloc(sizeof(double) * (size_t)n * p);
    double *Kinv = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *Knew = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *K0 = (double *)malloc(sizeof(double) * (size_t)n0 * n0);
    double *h = (double *)malloc(sizeof(double) * (size_t)n);
    double *u = (double *)malloc(sizeof(double) * (size_t)n);
    double *kc = (double *)malloc(sizeof(double) * (size_t)n);
    double *dexp = (double *)malloc(sizeof(double) * (size_t)Nprime);
    long double *dref = (long double *)malloc(sizeof(long double) * (size_t)Nprime);
    long double *L = (long double *)malloc(sizeof(long double) * (size_t)n * n);
    long double *v = (long double *)malloc(sizeof(long double) * (size_t)n);
    long double *z = (long double *)malloc(sizeof(long double) * (size_t)n);
    if (!pool || !chosen || !Xj || !Kinv || !Knew || !K0 || !h || !u || !kc || !dexp || !dref || !L || !v || !z) {
        rc = 4;
        goto out;
    }
    for (int t = 0; t < n - n0; t++) { noise[t] = NAN; ref_gap[t] = NAN; }
    rc = oracle_nn(X, N, p, x, Nprime, pool, NULL);
    if (rc) goto out;
    for (int t = 0; t < n0; t++) {
        chosen[t] = 1;
        memcpy(Xj + t * p, X + (size_t)pool[t] * p, sizeof(double) * p);
    }
    build_K(n0, p, Xj, theta, eta, K0);
    if (oracle_invert_spd(n0, K0, Kinv)) goto out;
    for (int a = 0; a < n0; a++) h[a] = corr(Xj + a * p, x, p, theta);
    for (int j = n0; j < n && idx[j] >= 0; j++) {
        /* explicit scores, exactly as oracle_local_design forms them */
        for (int c = 0; c < Nprime; c++) {
            dexp[c] = NAN;
            if (chosen[c]) continue;
            double dcf;
            double minv = alc_one(j, p, Xj, Kinv, h, X + (size_t)pool[c] * p, x, theta, eta, u, kc, &dcf, NULL);
            if (minv > OR_S_MIN && isfinite(dcf)) dexp[c] = dcf;
        }
        /* fresh long-double factorisation of K_j = C(X_j) + eta I */
        for (int a = 0; a < j; a++)
            for (int b = 0; b <= a; b++)
                L[a * j + b] = corr_ld(Xj + a * p, Xj + b * p, p, theta) + (a == b ? (long double)eta : 0.0L);
        for (int k = 0; k < j; k++) {
            long double dkk = L[k * j + k];
            for (int t = 0; t < k; t++) dkk -= L[k * j + t] * L[k * j + t];
            if (!(dkk > 0.0L)) { rc = 1; goto out; }
            L[k * j + k] = sqrtl(dkk);
            for (int i = k + 1; i < j; i++) {
                long double sik = L[i * j + k];
                for (int t = 0; t < k; t++) sik -= L[i * j + t] * L[k * j + t];
                L[i * j + k] = sik / L[k * j + k];
            }
        }
        for (int a = 0; a < j; a++) {
            long double sa = corr_ld(Xj + a * p, x, p, theta);
            for (int t = 0; t < a; t++) sa -= L[a * j + t] * z[t];
            z[a] = sa / L[a * j + a];
        }
        long double m1 = -1.0L, m2 = -1.0L;
        for (int c = 0; c < Nprime; c++) {
            dref[c] = -1.0L;
            if (chosen[c]) continue;
            const double *xc = X + (size_t)pool[c] * p;
            long double vv = 0.0L, zv = 0.0L;
            for (int a = 0; a < j; a++) {
                long double sa = corr_ld(Xj + a * p, xc, p, theta);
                for (int t = 0; t < a; t++) sa -= L[a * j + t] * v[t];
                v[a] = sa / L[a * j + a];
                vv += v[a] * v[a];
                zv += z[a] * v[a];
            }
            long double s_ref = 1.0L + (long double)eta - vv;
            if (!(s_ref > (long double)OR_S_MIN)) continue;
            long double cv = corr_ld(xc, x, p, theta) - zv;
            dref[c] = cv * cv / s_ref;
            if (dref[c] > m1) { m2 = m1; m1 = dref[c]; } else if (dref[c] > m2) { m2 = dref[c]; }
        }
        long double worst = 0.0L;
        for (int c = 0; c < Nprime; c++)
            if (dref[c] >= 0.0L && !isnan(dexp[c])) {
                long double e = fabsl((long double)dexp[c] - dref[c]);
                if (e > worst) worst = e;
            }
        noise[j - n0] = m1 > 0.0L ? (double)(worst / m1) : 0.0;
        ref_gap[j - n0] = m1 > 0.0L ? (double)((m1 - (m2 > 0.0L ? m2 : 0.0L)) / m1) : 0.0;
        /* advance along the oracle's own trajectory (a4, the same calls as the run) */
        int bpos = -1;
        for (int c = 0; c < Nprime; c++)
            if (pool[c] == idx[j]) bpos = c;
        if (bpos < 0 || chosen[bpos]) { rc = 2; goto out; }
        const double *xs = X + (size_t)idx[j] * p;
        for (int a = 0; a < j; a++) kc[a] = corr(Xj + a * p, xs, p, theta);
        oracle_pinv_update(j, Kinv, kc, 1.0 + eta, Knew);
        memcpy(Kinv, Knew, sizeof(double) * (size_t)(j + 1) * (j + 1));
        chosen[bpos] = 1;
        memcpy(Xj + j * p, xs, sizeof(double) * p);
        h[j] = corr(xs, x, p, theta);
    }
out:
    free(pool); free(chosen); free(Xj); free(Kinv); free(Knew); free(K0); free(h); free(u); free(kc);
    free(dexp); free(dref); free(L); free(v); free(z);
    return rc;
}

/* All M locations, OpenMP over locations ("embarrassingly parallel").
 * Output layouts: idx M×n, gaps/best M×(n-n0). Returns the number of threads used. */
int oracle_alc_batch(const double *X, int64_t N, int p, const double *Z, const double *XX, int64_t M,
                     double theta, double eta, int n0, int n, int Nprime, int nthreads,
                     int32_t *idx, double *mean, double *s2, double *var, uint32_t *flags,
                     double *gaps, double *best, double *s2_acc) {
    int used = 1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    used = nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < M; i++) {
        int G = n - n0;
        oracle_local_design(X, N, p, Z, XX + i * p, theta, eta, n0, n, Nprime, idx + i * n, mean + i,
                            s2 + i, var + i, flags + i, gaps + i * G, best + i * G,
                            s2_acc ? s2_acc + i : NULL);
    }
    return used;
}

/* ========================================================================= */
/* Row f2: local MLE of the lengthscale and the multi-stage scheme
 * of Fig 1 steps 1-5 ("two-stage scheme").
 *
 * Concentrated log likelihood, Eq (3) on D_n(x):
 *   l(theta) = lgamma(n/2) - (n/2) log(2 pi) - (1/2) log|K| - (n/2) log(psi/2),
 *   K = C + eta I, C_ab = exp(-D_ab/theta), psi = Y^T K^{-1} Y.
 * The paper only says its derivatives "are also available analytically"
 * (P:201-203); reading R20 writes them out in tau = log(theta):
 *   P = dK/dtau,    P_ab = C_ab (D_ab/theta)
 *   Q = d2K/dtau2,  Q_ab = C_ab (D_ab/theta) (D_ab/theta - 1)
 *   alpha = K^{-1} Y
 *   dl/dtau   = -1/2 tr(K^{-1}P) + (n/2) alpha^T P alpha / psi
 *   d2l/dtau2 = -1/2 tr(K^{-1}Q) + 1/2 tr(K^{-1}P K^{-1}P)
 *               - (n/2) (2 alpha^T P K^{-1} P alpha - alpha^T Q alpha) / psi
 *               + (n/2) (alpha^T P alpha / psi)^2
 * Plain dense linear algebra: textbook Cholesky, explicit inverse by solves. */
#define OR_MLE_MAXIT 64
#define OR_MLE_BOUND 16u   /* theta-hat at a bound            */
#define OR_MLE_MAXITS 32u  /* iteration limit reached         */
#define OR_MLE_FAIL 64u    /* non-finite likelihood at start  */

typedef struct { double l, g, h; } or_lik;

/* Returns 0 and fills out (l, dl/dtau, d2l/dtau2) at theta; 1 if K is not SPD
 * or psi <= 0 (l = -inf). want_deriv = 0 skips the derivatives. */
int oracle_loglik(int n, int p, const double *Xn, const double *Yn, double theta, double eta,
                  int want_deriv, double *l, double *g, double *h) {
    double *D = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *C = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *K = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *L = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *A = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *T = (double *)malloc(sizeof(double) * (size_t)n * n + 8);
    double *al = (double *)malloc(sizeof(double) * (size_t)n + 8);
    double *v = (double *)malloc(sizeof(double) * (size_t)n + 8);
    double *e = (double *)malloc(sizeof(double) * (size_t)n + 8);
    int rc = 0;
    *l = -INFINITY;
    if (g) *g = NAN;
    if (h) *h = NAN;
    if (!D || !C || !K || !L || !A || !T || !al || !v || !e) { rc = 4; goto out; }
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) {
            D[a * n + b] = sqdist(Xn + a * p, Xn + b * p, p);
            C[a * n + b] = exp(-D[a * n + b] / theta);
            K[a * n + b] = C[a * n + b] + (a == b ? eta : 0.0);
        }
    if (cholesky(n, K, L)) { rc = 1; goto out; }
    double logdet = 0.0;
    for (int a = 0; a < n; a++) logdet += 2.0 * log(L[a * n + a]);
    for (int a = 0; a < n; a++) al[a] = Yn[a];
    chol_solve(n, L, al);
    double psi = 0.0;
    for (int a = 0; a < n; a++) psi += Yn[a] * al[a];
    if (!(psi > 0.0)) { rc = 1; goto out; }
    *l = lgamma(0.5 * n) - 0.5 * n * log(2.0 * M_PI) - 0.5 * logdet - 0.5 * n * log(0.5 * psi);
    if (!want_deriv) goto out;
    /* explicit K^{-1} */
    for (int b = 0; b < n; b++) {
        for (int i = 0; i < n; i++) e[i] = (i == b) ? 1.0 : 0.0;
        chol_solve(n, L, e);
        for (int a = 0; a < n; a++) A[a * n + b] = e[a];
    }
    /* P (into K's storage) and T = K^{-1} P */
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) K[a * n + b] = C[a * n + b] * (D[a * n + b] / theta);
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) {
            double s = 0.0;
            for (int t = 0; t < n; t++) s += A[a * n + t] * K[t * n + b];
            T[a * n + b] = s;
        }
    double trAP = 0.0, trAQ = 0.0, trTT = 0.0, aPa = 0.0, aQa = 0.0;
    for (int a = 0; a < n; a++) {
        double pv = 0.0;
        for (int b = 0; b < n; b++) {
            const double r = D[a * n + b] / theta;
            const double Pab = K[a * n + b];
            const double Qab = C[a * n + b] * r * (r - 1.0);
            trAP += A[a * n + b] * Pab;
            trAQ += A[a * n + b] * Qab;
            trTT += T[a * n + b] * T[b * n + a];
            aQa += al[a] * Qab * al[b];
            pv += Pab * al[b];
        }
        v[a] = pv;  /* v = P alpha */
        aPa += al[a] * pv;
    }
    double vAv = 0.0;
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) vAv += v[a] * A[a * n + b] * v[b];
    const double q = aPa / psi;
    *g = -0.5 * trAP + 0.5 * n * q;
    *h = -0.5 * trAQ + 0.5 * trTT - 0.5 * n * (2.0 * vAv - aQa) / psi + 0.5 * n * q * q;
out:
    free(D); free(C); free(K); free(L); free(A); free(T); free(al); free(v); free(e);
    return rc;
}

/* Local MLE theta-hat_n(x) | D_n(x), Fig 1 step 3: safeguarded
 * Newton on tau = log(theta) inside [log lo, log hi] (reading R21):
 *   evaluate (l, g, h) at tau; stop at a bound whose outward side the gradient
 *   points to; step = -g/h when h < 0, else sign(g); |step| <= 1; clamp into the
 *   bounds; steps longer than 1/4 (or non-Newton steps) are halved until l does
 *   not decrease (<= 40 halvings); stop when |tau_new - tau| <= 1e-10 max(1,|tau|)
 *   or after OR_MLE_MAXIT iterations. A start with non-finite l returns theta0
 *   (flag OR_MLE_FAIL; the incoming theta is kept, SPEC S:279 reading). */
int oracle_mle(int n, int p, const double *Xn, const double *Yn, double theta0, double lo, double hi,
               double eta, double *theta_hat, double *lhat, int *iters, uint32_t *flags) {
    const double tlo = log(lo), thi = log(hi);
    double tau = log(theta0);
    if (tau < tlo) tau = tlo;
    if (tau > thi) tau = thi;
    uint32_t fl = 0;
    double l, g, h;
    int it = 0;
    if (oracle_loglik(n, p, Xn, Yn, exp(tau), eta, 1, &l, &g, &h) || !isfinite(g) || !isfinite(h)) {
        *theta_hat = theta0; *lhat = l; *iters = 0; *flags = OR_MLE_FAIL;
        return 0;
    }
    for (it = 1; it <= OR_MLE_MAXIT; it++) {
        if ((tau <= tlo && g <= 0.0) || (tau >= thi && g >= 0.0)) { fl |= OR_MLE_BOUND; break; }
        if (g == 0.0 && !(h < 0.0)) break;
        double step = (h < 0.0) ? -g / h : (g > 0.0 ? 1.0 : -1.0);
        if (step > 1.0) step = 1.0;
        if (step < -1.0) step = -1.0;
        double tn = tau + step;
        if (tn < tlo) tn = tlo;
        if (tn > thi) tn = thi;
        double ln, gn, hn;
        int bad = oracle_loglik(n, p, Xn, Yn, exp(tn), eta, 1, &ln, &gn, &hn) || !isfinite(gn) || !isfinite(hn);
        if (fabs(step) > 0.25 || !(h < 0.0)) {
            for (int t = 0; t < 40 && (bad || ln < l); t++) {
                tn = 0.5 * (tau + tn);
                bad = oracle_loglik(n, p, Xn, Yn, exp(tn), eta, 1, &ln, &gn, &hn) || !isfinite(gn) || !isfinite(hn);
            }
            if (bad || ln < l) break;  /* no ascent along the step: stay at tau */
        } else if (bad) {
            break;
        }
        const double dt = fabs(tn - tau);
        tau = tn; l = ln; g = gn; h = hn;
        if (dt <= 1e-10 * (fabs(tau) > 1.0 ? fabs(tau) : 1.0)) break;
    }
    if (it > OR_MLE_MAXIT) fl |= OR_MLE_MAXITS;
    if (tau <= tlo || tau >= thi) fl |= OR_MLE_BOUND;
    *theta_hat = exp(tau);
    *lhat = l;
    *iters = it > OR_MLE_MAXIT ? OR_MLE_MAXIT : it;
    *flags = fl;
    return 0;
}

/* Multi-stage scheme, Fig 1 for ONE location x:
 *   1. theta_x = theta0;
 *   2. local design X_n(x, theta_x) (oracle_local_design: NN start + greedy ALC);
 *   3. theta_x = theta-hat_n(x) | D_n(x, theta_x)  (oracle_mle, started at theta_x);
 *   4. repeat 2-3 `stages` times in all;
 *   5. predict with theta_x on the last D_n(x) (oracle_predict, fresh Cholesky).
 * theta_out[s] = theta_x after stage s; flags = last design's flags | last MLE's. */
int oracle_local_fit(const double *X, int64_t N, int p, const double *Z, const double *x,
                     double theta0, double lo, double hi, double eta, int n0, int n, int Nprime, int stages,
                     int32_t *idx, double *theta_out, double *mean, double *s2, double *var, uint32_t *flags) {
    double th = theta0;
    uint32_t fl = 0;
    int G = n - n0;
    double *gaps = (double *)malloc(sizeof(double) * (size_t)(G > 0 ? G : 1));
    double *best = (double *)malloc(sizeof(double) * (size_t)(G > 0 ? G : 1));
    double *Xn = (double *)malloc(sizeof(double) * (size_t)n * p);
    double *Yn = (double *)malloc(sizeof(double) * (size_t)n);
    if (!gaps || !best || !Xn || !Yn) { free(gaps); free(best); free(Xn); free(Yn); return 4; }
    int j = n;
    for (int s = 0; s < stages; s++) {
        double mu, sc, vr;
        uint32_t dfl = 0;
        int rc = oracle_local_design(X, N, p, Z, x, th, eta, n0, n, Nprime, idx, &mu, &sc, &vr, &dfl, gaps, best, NULL);
        if (rc) { free(gaps); free(best); free(Xn); free(Yn); return rc; }
        for (j = 0; j < n && idx[j] >= 0; j++) {
            memcpy(Xn + j * p, X + (size_t)idx[j] * p, sizeof(double) * p);
            Yn[j] = Z[idx[j]];
        }
        double lh;
        int its;
        uint32_t mfl = 0;
        oracle_mle(j, p, Xn, Yn, th, lo, hi, eta, &th, &lh, &its, &mfl);
        theta_out[s] = th;
        fl = dfl | mfl;
    }
    if (oracle_predict(j, p, Xn, Yn, x, th, eta, mean, s2, var)) {
        fl |= OR_FLAG_NONFINITE;
        *mean = NAN; *s2 = NAN; *var = NAN;
    }
    if (!isfinite(*mean) || !isfinite(*s2)) fl |= OR_FLAG_NONFINITE;
    *flags = fl;
    free(gaps); free(best); free(Xn); free(Yn);
    return 0;
}

/* All M locations (OpenMP over locations). theta_out is stages x M. */
int oracle_local_fit_batch(const double *X, int64_t N, int p, const double *Z, const double *XX, int64_t M,
                           double theta0, double lo, double hi, double eta, int n0, int n, int Nprime,
                           int stages, int nthreads, int32_t *idx, double *theta_out, double *mean, double *s2,
                           double *var, uint32_t *flags) {
    int used = 1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    used = nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < M; i++) {
        double th[16];
        oracle_local_fit(X, N, p, Z, XX + i * p, theta0, lo, hi, eta, n0, n, Nprime, stages, idx + i * n, th,
                         mean + i, s2 + i, var + i, flags + i);
        for (int s = 0; s < stages && s < 16; s++) theta_out[(size_t)s * M + i] = th[s];
    }
    return used;
}

/* ========================================================================= */
/* Row f3: separable lengthscales. P:667-670: Steps 2 & 6 of Fig 3
 * assume the isotropic Gaussian correlation; "simple modification would
 * accommodate ... a separable version via a vectorized theta parameter":
 *   K(x, x') = exp(-sum_k (x_k - x'_k)^2 / theta_k)                      (*)
 * (η on the diagonal as before). Writing s_k = 1/sqrt(theta_k) and
 * x~_k = s_k x_k, (*) is exp(-||x~ - x~'||^2): the isotropic correlation of
 * P:213-215 with theta = 1 on the rescaled inputs, and the NN ordering
 * "relative to the chosen correlation function" is the Euclidean
 * order of the rescaled inputs (reading R23). This function forms x~ (one
 * correctly rounded sqrt, one division and one product per entry); the
 * separable path is then the isotropic path with d = 1 on (X~, XX~). */
void oracle_sep_scale(const double *X, int64_t N, int p, const double *theta, double *Xs) {
    for (int k = 0; k < p; k++) {
        const double s = 1.0 / sqrt(theta[k]);
        for (int64_t i = 0; i < N; i++) Xs[i * p + k] = X[i * p + k] * s;
    }
}
