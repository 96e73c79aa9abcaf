/*
 * TRPL+K CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain fp64 C + OpenMP, no BLAS, no code shared with the CUDA path.
 * Every function cites the passage it follows.  "P:n" = PAPER.md line n,
 * "S:n" = SPEC.md line n, "Rn" = reading n of SURVEY.md 8(c.3) / DESIGN.md.
 *
 * Determinism: every dot product uses 4096-row blocks summed sequentially and
 * combined pairwise in a fixed order, so results do not depend on the number
 * of OpenMP threads.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_BLK 4096

/* ---------------------------------------------------------------- RNG (R13) */
double orc_u01(uint64_t seed, uint64_t stream, uint64_t index) {
    /* splitmix64 finaliser over (seed, stream, index); identical formula is stated in
     * written out again here, not shared. */
    uint64_t key = (seed * 0xD1B54A32D192ED03ULL) ^ (stream * 0xABC98388FB8FAC03ULL);
    uint64_t z = key + (index + 1ULL) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------- sparse / BLAS-1 */
void orc_spmv(int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
              const double* x, double* y) {
    /* y = A x, row by row (eq 3.1 "z = A G(:,j)"). */
#pragma omp parallel for schedule(static) if (n > 32768)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s += val[p] * x[col[p]];
        y[i] = s;
    }
}

static double pairwise_sum(const double* s, int64_t nb) {
    if (nb == 1) return s[0];
    int64_t h = nb / 2;
    return pairwise_sum(s, h) + pairwise_sum(s + h, nb - h);
}

double orc_dot(int64_t n, const double* x, const double* y) {
    if (n <= 0) return 0.0;
    int64_t nb = (n + ORC_BLK - 1) / ORC_BLK;
    double* s = (double*)malloc((size_t)nb * sizeof(double));
#pragma omp parallel for schedule(static) if (n > 32768)
    for (int64_t b = 0; b < nb; ++b) {
        int64_t e = (b + 1) * ORC_BLK < n ? (b + 1) * ORC_BLK : n;
        double a = 0.0;
        for (int64_t i = b * ORC_BLK; i < e; ++i) a += x[i] * y[i];
        s[b] = a;
    }
    double r = pairwise_sum(s, nb);
    free(s);
    return r;
}

double orc_frobenius(int64_t nnz, const double* val) {
    /* eq 5.1: ||A||_F over all stored entries (both triangles) */
    return sqrt(orc_dot(nnz, val, val));
}

static void axpy(int64_t n, double a, const double* x, double* y) {
#pragma omp parallel for schedule(static) if (n > 32768)
    for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}

static void scal_copy(int64_t n, double a, const double* x, double* y) {
#pragma omp parallel for schedule(static) if (n > 32768)
    for (int64_t i = 0; i < n; ++i) y[i] = a * x[i];
}

void orc_jacobi_diag(int64_t n, const int64_t* a_rowptr, const int64_t* a_col, const double* a_val,
                     const int64_t* b_rowptr, const int64_t* b_col, const double* b_val,
                     double sigma, double floor_rel, double* M) {
    /* d_i = max(|A_ii - sigma B_ii|, eps_d * max_j |A_jj|), M = diag(d)^-1 (R12). */
    double* ad = (double*)calloc((size_t)n, sizeof(double));
    double amax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t p = a_rowptr[i]; p < a_rowptr[i + 1]; ++p)
            if (a_col[p] == i) ad[i] += a_val[p];
        if (fabs(ad[i]) > amax) amax = fabs(ad[i]);
    }
    for (int64_t i = 0; i < n; ++i) {
        double bd = 1.0;
        if (b_rowptr) {
            bd = 0.0;
            for (int64_t p = b_rowptr[i]; p < b_rowptr[i + 1]; ++p)
                if (b_col[p] == i) bd += b_val[p];
        }
        double d = fabs(ad[i] - sigma * bd);
        double fl = floor_rel * amax;
        M[i] = 1.0 / (d > fl ? d : fl);
    }
    free(ad);
}

/* ------------------------------------------------------------ small eig */
int orc_sym_eig(int k, const double* T, double* theta, double* Y) {
    /* Cyclic-by-row Jacobi (Golub & Van Loan Alg. 8.5.2/8.5.3) on sym(T).
     * A rotation (p,q) is skipped when |a_pq| <= eps*sqrt(|a_pp a_qq|) or |a_pq| <= 1e-30||T||_F;
     * a sweep without rotations ends the iteration. */
    double* A = (double*)malloc((size_t)k * k * sizeof(double));
    double* V = (double*)malloc((size_t)k * k * sizeof(double));
    double fro = 0.0;
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < k; ++i) {
            A[i + (size_t)k * j] = 0.5 * (T[i + (size_t)k * j] + T[j + (size_t)k * i]);
            V[i + (size_t)k * j] = (i == j) ? 1.0 : 0.0;
            fro += A[i + (size_t)k * j] * A[i + (size_t)k * j];
        }
    fro = sqrt(fro);
    const double eps = 2.220446049250313e-16;
    int sweep, rotated = 1;
    for (sweep = 0; sweep < 100 && rotated; ++sweep) {
        rotated = 0;
        for (int p = 0; p < k - 1; ++p)
            for (int q = p + 1; q < k; ++q) {
                double apq = A[p + (size_t)k * q];
                double app = A[p + (size_t)k * p], aqq = A[q + (size_t)k * q];
                if (fabs(apq) <= eps * sqrt(fabs(app * aqq)) || fabs(apq) <= 1e-30 * fro) continue;
                rotated = 1;
                double tau = (aqq - app) / (2.0 * apq);
                double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int i = 0; i < k; ++i) { /* A <- A J */
                    double aip = A[i + (size_t)k * p], aiq = A[i + (size_t)k * q];
                    A[i + (size_t)k * p] = c * aip - s * aiq;
                    A[i + (size_t)k * q] = s * aip + c * aiq;
                }
                for (int j = 0; j < k; ++j) { /* A <- J^T A */
                    double apj = A[p + (size_t)k * j], aqj = A[q + (size_t)k * j];
                    A[p + (size_t)k * j] = c * apj - s * aqj;
                    A[q + (size_t)k * j] = s * apj + c * aqj;
                }
                A[p + (size_t)k * q] = 0.0;
                A[q + (size_t)k * p] = 0.0;
                for (int i = 0; i < k; ++i) { /* V <- V J */
                    double vip = V[i + (size_t)k * p], viq = V[i + (size_t)k * q];
                    V[i + (size_t)k * p] = c * vip - s * viq;
                    V[i + (size_t)k * q] = s * vip + c * viq;
                }
            }
    }
    /* ascending, stable on ties (R11): insertion sort of indices */
    int* idx = (int*)malloc((size_t)k * sizeof(int));
    for (int i = 0; i < k; ++i) idx[i] = i;
    for (int i = 1; i < k; ++i) {
        int v = idx[i], j = i - 1;
        while (j >= 0 && A[idx[j] + (size_t)k * idx[j]] > A[v + (size_t)k * v]) { idx[j + 1] = idx[j]; --j; }
        idx[j + 1] = v;
    }
    for (int c = 0; c < k; ++c) {
        int src = idx[c];
        theta[c] = A[src + (size_t)k * src];
        int imax = 0;
        double vmax = -1.0;
        for (int i = 0; i < k; ++i)
            if (fabs(V[i + (size_t)k * src]) > vmax) { vmax = fabs(V[i + (size_t)k * src]); imax = i; }
        double sg = V[imax + (size_t)k * src] < 0.0 ? -1.0 : 1.0; /* sign rule (R11) */
        for (int i = 0; i < k; ++i) Y[i + (size_t)k * c] = sg * V[i + (size_t)k * src];
    }
    free(idx);
    free(A);
    free(V);
    return rotated ? -1 : sweep;
}

/* ------------------------------------------------------------ solver ctx */
typedef struct {
    const orc_problem* P;
    int64_t n;
    int64_t a_mv, b_mv, prec;
} ctx_t;

static void applyA(ctx_t* c, const double* x, double* y) {
    orc_spmv(c->n, c->P->a_rowptr, c->P->a_col, c->P->a_val, x, y);
    c->a_mv++;
}

static void applyB(ctx_t* c, const double* x, double* y) {
    if (c->P->b_rowptr) {
        orc_spmv(c->n, c->P->b_rowptr, c->P->b_col, c->P->b_val, x, y);
        c->b_mv++;
    } else {
        memcpy(y, x, (size_t)c->n * sizeof(double));
    }
}

/* CGS2 in the B-inner product (R3; "orthonormal basis" P:184). */
static int cgs2_ctx(ctx_t* c, int k, const double* V, double* w, double* Bw, double* h,
                    double* beta, int* passes) {
    int64_t n = c->n;
    applyB(c, w, Bw);
    double nin = sqrt(orc_dot(n, w, Bw));
    double* coef = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
    if (h) for (int j = 0; j < k; ++j) h[j] = 0.0;
    double nprev = nin, nrm = nin;
    int np = 0;
    for (int pass = 1; pass <= 3; ++pass) {
        /* classical GS: all coefficients from the same w, then the update */
        for (int j = 0; j < k; ++j) coef[j] = orc_dot(n, V + (size_t)n * j, Bw);
        for (int j = 0; j < k; ++j) axpy(n, -coef[j], V + (size_t)n * j, w);
        if (h) for (int j = 0; j < k; ++j) h[j] += coef[j];
        applyB(c, w, Bw);
        nprev = nrm;
        nrm = sqrt(orc_dot(n, w, Bw));
        np = pass;
        if (pass >= 2 && !(nrm < nprev / sqrt(2.0))) break; /* 3rd pass only if pass 2 dropped >1/sqrt2 */
    }
    free(coef);
    *beta = nrm;
    if (passes) *passes = np;
    return (nrm < 1e-14 * nin || nin == 0.0) ? 1 : 0;
}

int orc_cgs2(int64_t n, int k, const double* V, double* w, const int64_t* b_rowptr,
             const int64_t* b_col, const double* b_val, double* h, double* beta, int* passes) {
    orc_problem P;
    memset(&P, 0, sizeof(P));
    P.n = n;
    P.b_rowptr = b_rowptr; P.b_col = b_col; P.b_val = b_val;
    ctx_t c = {&P, n, 0, 0, 0};
    double* Bw = (double*)malloc((size_t)n * sizeof(double));
    int r = cgs2_ctx(&c, k, V, w, Bw, h, beta, passes);
    free(Bw);
    return r;
}

/* random replacement for a dependent vector (R16): stream 2, draw counter d */
static void draw_random(ctx_t* c, int64_t draw, double* w) {
    int64_t n = c->n;
#pragma omp parallel for schedule(static) if (n > 32768)
    for (int64_t i = 0; i < n; ++i) w[i] = orc_u01(c->P->seed, 2, (uint64_t)draw * (uint64_t)n + (uint64_t)i);
}

/* r = A x - theta B x ; returns ||r||_2  (Alg. 1 step 12; R15) */
static double residual(ctx_t* c, const double* x, double theta, double* r, double* tmp) {
    applyA(c, x, r);
    applyB(c, x, tmp);
    axpy(c->n, -theta, tmp, r);
    return sqrt(orc_dot(c->n, r, r));
}

/* Xn(:,0:ncol) = U(:,0:k) Y(0:k, 0:ncol)   ("x_i = U Y(:,i)") */
void orc_rotate(int64_t n, int k, const double* U, const double* Y, int ldy, int ncol, double* Xn) {
#pragma omp parallel for schedule(static) if (n > 32768)
    for (int64_t i = 0; i < n; ++i)
        for (int cc = 0; cc < ncol; ++cc) {
            double s = 0.0;
            for (int j = 0; j < k; ++j) s += U[i + (size_t)n * j] * Y[j + (size_t)ldy * cc];
            Xn[i + (size_t)n * cc] = s;
        }
}

/* The same sums as orc_rotate, written back into U(:,0:ncol) row by row (each row's k inputs are
 * read before any of its outputs is stored; ncol <= k). */
static void rotate_rows_inplace(int64_t n, int k, double* U, const double* Y, int ldy, int ncol) {
#pragma omp parallel if (n > 32768)
    {
        double* row = (double*)malloc((size_t)ncol * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            for (int cc = 0; cc < ncol; ++cc) {
                double s = 0.0;
                for (int j = 0; j < k; ++j) s += U[i + (size_t)n * j] * Y[j + (size_t)ldy * cc];
                row[cc] = s;
            }
            for (int cc = 0; cc < ncol; ++cc) U[i + (size_t)n * cc] = row[cc];
        }
        free(row);
    }
}

/* One inner step of eq 3.1 on the basis U(:,0:k), g_j = U(:,k-1):
 *   z = A g_j;  T(1:k,k) = U^T z (mirrored);  if `next`: w = M(z - rho B g_j) (R1), CGS2_B of w
 *   against U(:,0:k) (R2, R3) and g_{j+1} = w/beta into U(:,k).  Returns 1 on a breakdown (R16). */
/* ------------------------------------------------ preconditioner M (R12; P2c; NEXT-2 IC(0))
 * Either the diagonal M (Jacobi, R12 / P2c) or M = (L L^T)^-1 with L the IC(0) factor of
 * K = A - sigma B (reading P2a): L has the sparsity of K's lower triangle (no fill);
 *   L_ij = (K_ij - sum_{k<j} L_ik L_jk) / L_jj  (j < i, k over the common lower pattern),
 *   L_ii = sqrt(K_ii - sum_{j<i} L_ij^2),  a pivot <= 0 replaced by eps_d max_j|K_jj| (R12 floor);
 * applied by a forward solve L y = v and a backward solve L^T w = y, in row order. */
typedef struct {
    const double* M;         /* diagonal, or NULL */
    int64_t n;
    int64_t *rp, *ci;        /* IC(0) factor (CSR, columns ascending, diagonal last) */
    double* val;
    double* tmp;
} prec_t;

static void prec_apply(const prec_t* pc, double* v) {
    const int64_t n = pc->n;
    if (pc->M) {
        for (int64_t i = 0; i < n; ++i) v[i] = pc->M[i] * v[i];
        return;
    }
    for (int64_t i = 0; i < n; ++i) { /* L y = v */
        double s = v[i];
        const int64_t e = pc->rp[i + 1] - 1; /* diagonal */
        for (int64_t p = pc->rp[i]; p < e; ++p) s -= pc->val[p] * v[pc->ci[p]];
        v[i] = s / pc->val[e];
    }
    for (int64_t i = n - 1; i >= 0; --i) { /* L^T w = y, column-oriented */
        const int64_t e = pc->rp[i + 1] - 1;
        v[i] /= pc->val[e];
        for (int64_t p = pc->rp[i]; p < e; ++p) v[pc->ci[p]] -= pc->val[p] * v[i];
    }
}

/* IC(0) of K = A - sigma B on A's lower pattern (B's entries outside it are ignored). */
static int ic0_build(const orc_problem* P, double sigma, prec_t* pc) {
    const int64_t n = P->n;
    int64_t* rp = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    rp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t cnt = 0;
        for (int64_t p = P->a_rowptr[i]; p < P->a_rowptr[i + 1]; ++p)
            if (P->a_col[p] < i) ++cnt;
        rp[i + 1] = rp[i] + cnt + 1;
    }
    int64_t* ci = (int64_t*)malloc((size_t)rp[n] * sizeof(int64_t));
    double* val = (double*)malloc((size_t)rp[n] * sizeof(double));
    double amax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t q = rp[i];
        double kd = 0.0;
        for (int64_t p = P->a_rowptr[i]; p < P->a_rowptr[i + 1]; ++p) {
            const int64_t j = P->a_col[p];
            double kij = P->a_val[p];
            if (P->b_rowptr)
                for (int64_t t = P->b_rowptr[i]; t < P->b_rowptr[i + 1]; ++t)
                    if (P->b_col[t] == j) kij -= sigma * P->b_val[t];
            if (!P->b_rowptr && j == i) kij -= sigma;
            if (j < i) { ci[q] = j; val[q] = kij; ++q; }
            if (j == i) kd = kij;
        }
        ci[q] = i;
        val[q] = kd;
        if (fabs(kd) > amax) amax = fabs(kd);
    }
    for (int64_t i = 0; i < n; ++i) {
        const int64_t e = rp[i + 1] - 1;
        for (int64_t p = rp[i]; p < e; ++p) {
            const int64_t j = ci[p];
            /* s = K_ij - sum_{k < j} L_ik L_jk over the common pattern (both rows ascending) */
            double s = val[p];
            int64_t a = rp[i], b = rp[j];
            const int64_t be = rp[j + 1] - 1;
            while (a < p && b < be) {
                if (ci[a] == ci[b]) { s -= val[a] * val[b]; ++a; ++b; }
                else if (ci[a] < ci[b]) ++a;
                else ++b;
            }
            val[p] = s / val[rp[j + 1] - 1];
        }
        double d = val[e];
        for (int64_t p = rp[i]; p < e; ++p) d -= val[p] * val[p];
        if (!(d > 1e-8 * amax)) d = 1e-8 * amax;
        val[e] = sqrt(d);
    }
    pc->M = NULL;
    pc->n = n;
    pc->rp = rp;
    pc->ci = ci;
    pc->val = val;
    return 0;
}

int64_t orc_ic0(const orc_problem* P, double sigma, int64_t* rp_out, int64_t* ci_out, double* val_out, int64_t cap) {
    prec_t pc;
    ic0_build(P, sigma, &pc);
    const int64_t nnz = pc.rp[P->n];
    if (rp_out && ci_out && val_out && cap >= nnz) {
        memcpy(rp_out, pc.rp, (size_t)(P->n + 1) * sizeof(int64_t));
        memcpy(ci_out, pc.ci, (size_t)nnz * sizeof(int64_t));
        memcpy(val_out, pc.val, (size_t)nnz * sizeof(double));
    }
    free(pc.rp); free(pc.ci); free(pc.val);
    return nnz;
}

static int inner_step_at(ctx_t* c, const prec_t* pc, double rho, int next, double* U, int k, int gpos, double* T,
                         int q, double* z, double* s, double* w, double* Bw) {
    /* g = U(:, gpos) of a basis of width k; its T column covers rows 0..k-1 (mirrored), its
     * preconditioned image is CGS2-orthogonalised against all k columns and appended at k */
    const int64_t n = c->n;
    double* g = U + (size_t)n * gpos;
    double beta;
    applyA(c, g, z);
    for (int i = 0; i < k; ++i) {
        double v = orc_dot(n, U + (size_t)n * i, z);
        T[i + (size_t)q * gpos] = v;
        T[gpos + (size_t)q * i] = v;
    }
    if (!next) return 0;
    applyB(c, g, s);
    for (int64_t i = 0; i < n; ++i) w[i] = z[i] - rho * s[i];
    prec_apply(pc, w); /* w = M (z - rho B g), R1 */
    c->prec++;
    if (cgs2_ctx(c, k, U, w, Bw, NULL, &beta, NULL)) return 1;
    scal_copy(n, 1.0 / beta, w, U + (size_t)n * k);
    return 0;
}

static int inner_step(ctx_t* c, const prec_t* pc, double rho, int next, double* U, int k, double* T, int q,
                      double* z, double* s, double* w, double* Bw) {
    return inner_step_at(c, pc, rho, next, U, k, k - 1, T, q, z, s, w, Bw);
}

int orc_inner_steps(const orc_problem* P, const double* M, double rho, double* U, int k0, int nsteps,
                    double* T, int ldT, double* work) {
    const int64_t n = P->n;
    ctx_t c = {P, n, 0, 0, 0};
    double* wk = work ? work : (double*)malloc((size_t)4 * n * sizeof(double));
    double *z = wk, *s = wk + n, *w = wk + 2 * n, *Bw = wk + 3 * n;
    int done = 0;
    for (int j = 0; j < nsteps; ++j) {
        ++done;
        prec_t pc = {M, n, NULL, NULL, NULL, NULL};
        if (inner_step(&c, &pc, rho, 1, U, k0 + j, T, ldT, z, s, w, Bw)) break;
    }
    if (!work) free(wk);
    return done;
}

int orc_trplk_solve(const orc_problem* P, double* evals, double* evecs, double* resid, orc_report* rep) {
    const int64_t n = P->n;
    const int p = P->p, q = P->q, l = P->l;
    const int ph = P->restart_size > 0 ? P->restart_size : p; /* R5: p^ = p by default */
    if (rep) { rep->status = 1; rep->cycles = 0; rep->log_len = 0; }
    if (n < 1 || p < 1 || l < 0 || ph < p || q - ph - l < 1 || !(P->tol > 0.0) || ph + 1 > n ||
        P->max_cycles < 1 || P->block > 8 || q > 64 || P->precond < 0 || P->precond > 3 ||
        (P->precond == 2 && P->block > 1))
        return 1; /* EINVAL */
    const int m = q - ph - l; /* inner steps per cycle (R5) */

    ctx_t c = {P, n, 0, 0, 0};
    int64_t verify_mv = 0, inner_steps = 0, draws = 0;

    double* M = (double*)malloc((size_t)n * sizeof(double));
    orc_jacobi_diag(n, P->a_rowptr, P->a_col, P->a_val, P->b_rowptr, P->b_col, P->b_val, P->sigma,
                    1e-8, M);
    if (P->precond == 1) /* no preconditioning: the TRLan / LOPCG baselines of PAPER.md:77-95 */
        for (int64_t i = 0; i < n; ++i) M[i] = 1.0;
    prec_t pc = {M, n, NULL, NULL, NULL, NULL};
    if (P->precond == 3) ic0_build(P, P->sigma, &pc); /* IC(0) of A - sigma B (P2a) */
    double tau = P->tol;
    if (P->tol_mode == 1) tau = P->tol * orc_frobenius(P->a_rowptr[n], P->a_val); /* eq 5.1 */

    /* Storage (no arithmetic depends on it): the rotation X = U Y(:,1:p^) is written row by row
     * into U's first p^ columns (rotate_rows_inplace, same sums as orc_rotate), so X lives in
     * U(:,1:p^) and no separate n x p^ block is kept; W = AX exists only during start-up; X^prev
     * is captured straight into Xp, whose previous contents were consumed by this cycle's +K
     * step.  This keeps the 512^3 config (C5) within a 62 GB host. */
    double* U = (double*)calloc((size_t)n * q, sizeof(double));
    double* W = NULL;
    double* Xp = NULL;
    double* w = (double*)malloc((size_t)n * sizeof(double));
    double* Bw = (double*)malloc((size_t)n * sizeof(double));
    double* z = (double*)malloc((size_t)n * sizeof(double));
    double* s = (double*)malloc((size_t)n * sizeof(double));
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* u = (double*)malloc((size_t)n * sizeof(double));
    double* T = (double*)calloc((size_t)q * q, sizeof(double));
    double* Tk = (double*)malloc((size_t)q * q * sizeof(double));
    double* Y = (double*)malloc((size_t)q * q * sizeof(double));
    double* th = (double*)malloc((size_t)q * sizeof(double));
    int status = 2, brk;
    double beta;

    /* ---- Alg. 1 steps 1-2: X = B-orthonormalised rand(n,p^), seed stream 0 (R13) */
    for (int cc = 0; cc < ph; ++cc) {
        double* x = U + (size_t)n * cc;
#pragma omp parallel for schedule(static) if (n > 32768)
        for (int64_t i = 0; i < n; ++i) x[i] = orc_u01(P->seed, 0, (uint64_t)cc * (uint64_t)n + (uint64_t)i);
        int tries = 0;
        while ((brk = cgs2_ctx(&c, cc, U, x, Bw, NULL, &beta, NULL)) && tries < 3) {
            draw_random(&c, draws++, x);
            ++tries;
        }
        if (brk) { status = 3; goto done_init_fail; }
        scal_copy(n, 1.0 / beta, x, x);
    }
    W = (double*)malloc((size_t)n * ph * sizeof(double));
    for (int cc = 0; cc < ph; ++cc) applyA(&c, U + (size_t)n * cc, W + (size_t)n * cc);
    for (int j = 0; j < ph; ++j)
        for (int i = 0; i < ph; ++i) Tk[i + (size_t)ph * j] = orc_dot(n, U + (size_t)n * i, W + (size_t)n * j);
    if (orc_sym_eig(ph, Tk, th, Y) < 0) { status = 3; goto done_init_fail; }
    rotate_rows_inplace(n, ph, U, Y, ph, ph); /* X <- X Y */
    rotate_rows_inplace(n, ph, W, Y, ph, ph); /* W <- W Y (AX of the rotated X) */
    memset(T, 0, (size_t)q * q * sizeof(double));
    for (int i = 0; i < ph; ++i) T[i + (size_t)q * i] = th[i];
    int t = 1; /* target, 1-based */
    double rho = th[0];
    if (P->precond == 2) /* M ~ (A - rho_i B)^-1 re-formed for every cycle's shift */
        orc_jacobi_diag(n, P->a_rowptr, P->a_col, P->a_val, P->b_rowptr, P->b_col, P->b_val, rho, 1e-8, M);
    applyB(&c, U, s);
    for (int64_t i = 0; i < n; ++i) r[i] = W[i] - rho * s[i];
    for (int64_t i = 0; i < n; ++i) u[i] = r[i];
    prec_apply(&pc, u);
    c.prec++;
    /* block TRPL+K (NEXT-3; reading B1): seeds M r_{t+i} of the next b-1 targets too */
    const int b = P->block > 1 ? P->block : 1;
    double* ub = b > 1 ? (double*)malloc((size_t)n * (b - 1) * sizeof(double)) : NULL;
    int nub = 0;
    if (b > 1) {
        nub = b - 1 < ph - 1 ? b - 1 : ph - 1;
        if (nub > m - 1) nub = m - 1 > 0 ? m - 1 : 0;
        for (int i = 1; i <= nub; ++i) { /* r_i = A x_i - theta_i B x_i from W (no matvec) */
            double* ui = ub + (size_t)n * (i - 1);
            applyB(&c, U + (size_t)n * i, s);
            for (int64_t j = 0; j < n; ++j) ui[j] = W[j + (size_t)n * i] - th[i] * s[j];
            prec_apply(&pc, ui);
            c.prec++;
        }
    }
    free(W);
    W = NULL;
    Xp = (double*)malloc((size_t)n * (l > 0 ? l : 1) * sizeof(double));
    int nprev = 0;
    int cyc;
    int all_conv = 0;

    for (cyc = 1; cyc <= P->max_cycles; ++cyc) {
        if (rep && rep->dump_cycles > cyc - 1 && rep->dump_X) {
            memcpy(rep->dump_X + (size_t)(cyc - 1) * n * ph, U, (size_t)n * ph * sizeof(double));
            if (rep->dump_rho) rep->dump_rho[cyc - 1] = rho;
            if (rep->dump_t) rep->dump_t[cyc - 1] = t;
        }
        /* ---- seed u1 = (I - X X^T B) M r_t, normalised (eq 3.2 u1 = C x_t, R4) */
        memcpy(w, u, (size_t)n * sizeof(double));
        {
            int tries = 0;
            while ((brk = cgs2_ctx(&c, ph, U, w, Bw, NULL, &beta, NULL)) && tries < 3) {
                draw_random(&c, draws++, w);
                ++tries;
            }
            if (brk) { status = 3; break; }
        }
        int k = ph;
        scal_copy(n, 1.0 / beta, w, U + (size_t)n * k);
        if (b == 1) {
            /* ---- inner projected Lanczos, eq 3.1, R1/R2 */
            for (int j = 1; j <= m; ++j) {
                k += 1; /* k = p^ + j */
                ++inner_steps;
                if (inner_step(&c, &pc, rho, j < m, U, k, T, q, z, s, w, Bw)) break; /* R16: basis ends early */
            }
        } else {
            /* ---- block version (B1): seeds M r_{t+i}, i < b_e, CGS2_B against [X, earlier seeds]
             * (a dependent one is dropped), then every column's image M (A - rho B) g under the
             * cycle's ONE shift rho = theta_t (eq 3.2's operator C), CGS2_B against the whole basis
             * and appended, in column order, until the basis has p^ + m columns: span{X} plus the
             * block Krylov space of C from the seed block, independent of the Gram-Schmidt order */
            int width = ph + 1;
            for (int i = 1; i <= nub && width < ph + m; ++i) {
                memcpy(w, ub + (size_t)n * (i - 1), (size_t)n * sizeof(double));
                if (cgs2_ctx(&c, width, U, w, Bw, NULL, &beta, NULL)) continue;
                scal_copy(n, 1.0 / beta, w, U + (size_t)n * width);
                ++width;
            }
            for (int next = ph; next < width; ++next) {
                ++inner_steps;
                const int produce = width < ph + m;
                if (!inner_step_at(&c, &pc, rho, produce, U, width, next, T, q, z, s, w, Bw) && produce) ++width;
            }
            k = width;
        }
        /* ---- +K: X^prev appended after G, explicitly orthogonalised, l matvecs (Alg.1 7-8) */
        int appended = 0;
        for (int cc = 0; cc < nprev; ++cc) {
            memcpy(w, Xp + (size_t)n * cc, (size_t)n * sizeof(double));
            brk = cgs2_ctx(&c, k, U, w, Bw, NULL, &beta, NULL);
            if (brk) continue; /* dependent: drop (R16) */
            double* xt = U + (size_t)n * k;
            scal_copy(n, 1.0 / beta, w, xt);
            k += 1;
            applyA(&c, xt, z);
            for (int i = 0; i < k; ++i) {
                double v = orc_dot(n, U + (size_t)n * i, z);
                T[i + (size_t)q * (k - 1)] = v;
                T[(k - 1) + (size_t)q * i] = v;
            }
            ++appended;
        }
        /* ---- Alg. 1 step 10: X^prev <- X(:, t : min(t+l-1, p)) before the RR (R6) */
        int last = t + l - 1 < p ? t + l - 1 : p;
        int nnew = last - t + 1;
        if (nnew < 0) nnew = 0;
        for (int cc = 0; cc < nnew; ++cc) /* Xp was consumed by the +K step above */
            memcpy(Xp + (size_t)n * cc, U + (size_t)n * (t - 1 + cc), (size_t)n * sizeof(double));
        /* ---- debug bookkeeping checks: T vs U^T A U, U^T B U - I */
        if (rep && P->debug && rep->log_cap >= cyc) {
            double terr = 0.0, oerr = 0.0;
            for (int jj = 0; jj < k; ++jj) {
                orc_spmv(n, P->a_rowptr, P->a_col, P->a_val, U + (size_t)n * jj, z);
                if (P->b_rowptr) orc_spmv(n, P->b_rowptr, P->b_col, P->b_val, U + (size_t)n * jj, s);
                else memcpy(s, U + (size_t)n * jj, (size_t)n * sizeof(double));
                for (int ii = 0; ii < k; ++ii) {
                    double e1 = fabs(orc_dot(n, U + (size_t)n * ii, z) - T[ii + (size_t)q * jj]);
                    double e2 = fabs(orc_dot(n, U + (size_t)n * ii, s) - (ii == jj ? 1.0 : 0.0));
                    if (e1 > terr) terr = e1;
                    if (e2 > oerr) oerr = e2;
                }
            }
            if (rep->log_terr) rep->log_terr[cyc - 1] = terr;
            if (rep->log_orth) rep->log_orth[cyc - 1] = oerr;
        }
        /* ---- Alg. 1 step 11: T = Y Theta Y^T, x_i = U Y(:,i) */
        for (int jj = 0; jj < k; ++jj)
            for (int ii = 0; ii < k; ++ii) Tk[ii + (size_t)k * jj] = T[ii + (size_t)q * jj];
        if (orc_sym_eig(k, Tk, th, Y) < 0) { status = 3; break; }
        rotate_rows_inplace(n, k, U, Y, k, ph); /* U(:,1:p^) <- X_new = U Y(:,1:p^) */
        /* ---- Alg. 1 steps 12-14: soft lock (R7 literal IF) */
        double res = residual(&c, U + (size_t)n * (t - 1), th[t - 1], r, s);
        if (rep && rep->log_cap >= cyc) {
            if (rep->log_t) rep->log_t[cyc - 1] = t;
            if (rep->log_theta_t) rep->log_theta_t[cyc - 1] = th[t - 1];
            if (rep->log_res) rep->log_res[cyc - 1] = res;
            if (rep->log_k) rep->log_k[cyc - 1] = k;
            if (rep->log_nprev) rep->log_nprev[cyc - 1] = appended;
            if (rep->log_thetas) for (int i = 0; i < ph; ++i) rep->log_thetas[(size_t)(cyc - 1) * ph + i] = th[i];
        }
        while (res <= tau) {
            t += 1;
            if (nnew > 0) { /* remove x1^prev (step 13) */
                for (int cc = 1; cc < nnew; ++cc)
                    memcpy(Xp + (size_t)n * (cc - 1), Xp + (size_t)n * cc, (size_t)n * sizeof(double));
                nnew -= 1;
            }
            if (t > p) { all_conv = 1; break; }
            res = residual(&c, U + (size_t)n * (t - 1), th[t - 1], r, s);
            if (P->lock_mode == 0) break;
        }
        /* ---- Alg. 1 step 15: restart.  X = U Y(:,1:p^) (already in U), T = diag(Theta)
         * (R10), X^prev = Xp(:,1:nnew) */
        memset(T, 0, (size_t)q * q * sizeof(double));
        for (int i = 0; i < ph; ++i) T[i + (size_t)q * i] = th[i];
        nprev = nnew;
        if (rep && rep->log_cap >= cyc) {
            if (rep->log_mv) rep->log_mv[cyc - 1] = c.a_mv;
            rep->log_len = cyc;
        }
        if (rep && rep->verbose)
            fprintf(stderr, "oracle cycle %d t=%d k=%d mv=%lld theta=%.16e\n", cyc, t, k, (long long)c.a_mv,
                    th[t - 1 <= ph - 1 ? t - 1 : ph - 1]);
        if (all_conv) {
            /* final verification of all p pairs (R9) */
            int first_fail = -1;
            for (int i = 0; i < p; ++i) {
                double ri = residual(&c, U + (size_t)n * i, th[i], w, s);
                verify_mv++;
                resid[i] = ri;
                if (ri > tau && first_fail < 0) {
                    first_fail = i;
                    memcpy(r, w, (size_t)n * sizeof(double));
                }
            }
            if (first_fail < 0) { status = 0; break; }
            t = first_fail + 1; /* resume (R9) */
            all_conv = 0;
        }
        rho = th[t - 1];
        if (P->precond == 2)
            orc_jacobi_diag(n, P->a_rowptr, P->a_col, P->a_val, P->b_rowptr, P->b_col, P->b_val, rho, 1e-8, M);
        for (int64_t i = 0; i < n; ++i) u[i] = r[i];
        prec_apply(&pc, u);
        c.prec++;
        if (b > 1) { /* residuals of the next targets: one A-matvec each (B1) */
            nub = b - 1 < ph - t ? b - 1 : ph - t;
            if (nub > m - 1) nub = m - 1 > 0 ? m - 1 : 0;
            for (int i = 1; i <= nub; ++i) {
                double* ui = ub + (size_t)n * (i - 1);
                residual(&c, U + (size_t)n * (t - 1 + i), th[t - 1 + i], w, s);
                for (int64_t j = 0; j < n; ++j) ui[j] = w[j];
                prec_apply(&pc, ui);
                c.prec++;
            }
        }
    }
    if (status != 0) {
        /* NOT_CONVERGED (R19) / BREAKDOWN: report the current best with verified residuals */
        for (int i = 0; i < p; ++i) {
            resid[i] = residual(&c, U + (size_t)n * i, th[i], w, s);
            verify_mv++;
        }
    }
    for (int i = 0; i < p; ++i) evals[i] = th[i];
    if (evecs) memcpy(evecs, U, (size_t)n * p * sizeof(double));
    if (rep && rep->n_sample > 0 && rep->sample_rows && rep->sample_vals)
        for (int cc = 0; cc < p; ++cc)
            for (int i = 0; i < rep->n_sample; ++i)
                rep->sample_vals[i + (size_t)rep->n_sample * cc] = U[rep->sample_rows[i] + (size_t)n * cc];
    if (rep) rep->cycles = cyc > P->max_cycles ? P->max_cycles : cyc;
    goto done;

done_init_fail:
    for (int i = 0; i < p; ++i) { evals[i] = NAN; resid[i] = NAN; }
done:
    if (rep) {
        rep->status = status;
        rep->a_matvecs = c.a_mv;
        rep->b_matvecs = c.b_mv;
        rep->precond_applies = c.prec;
        rep->verify_matvecs = verify_mv;
        rep->inner_steps = inner_steps;
        rep->random_draws = draws;
    }
    free(ub);
    free(pc.rp); free(pc.ci); free(pc.val);
    free(M); free(U); free(W); free(Xp); free(w); free(Bw); free(z);
    free(s); free(r); free(u); free(T); free(Tk); free(Y); free(th);
    return status;
}

/* =====================================================================================
 * PL+1, Algorithm 2 (alg:pl+1) -- NEXT-1 of SURVEY 8(f).
 * Readings:
 *  P1 step 4: G_k = B-orthonormal basis of span{M(A-rho_k B)x_k, ..., [M(A-rho_k B)]^m x_k}
 *     built as v_1 = M r_k, v_{j+1} = M(A - rho_k B) g_j, each v CGS2-orthogonalised (B-inner
 *     product, R3) against g_1..g_{j-1} only (x_k and p_{k-1} are not projected out: step 5
 *     solves the pencil (Q^T A Q, Q^T B Q)); a breakdown (R16 threshold) ends G_k early.
 *  P2 step 5: lowest eigenpair of the projected pencil by Cholesky reduction S = L L^T,
 *     C = L^-1 H L^-T and the Jacobi eig; w = L^-T y_1 (w^T S w = 1), sign fixed
 *     so that w(1) >= 0 (the coefficient of x_k).
 *  P3 a Cholesky pivot d_j <= 1e-24 S_jj (component of the column outside the span of the
 *     previous ones below 1e-12 relative) drops p_{k-1} from Q_k (SPEC "columns dropped");
 *     if the failing column is not p_{k-1}: BREAKDOWN.
 *  P4 step 7: rho_{k-1} = rho(x_{k-1}), the Rayleigh quotient of the previous iterate (the
 *     shift of iteration k-1; Lemma 8's proof uses p_{k-1}^T(A - rho(x_{k-1})B)p_k = 0);
 *     |p_{k-1}^T(A - rho_{k-1}B)p_{k-1}| <= 1e-14 ||A||_F -> coefficient 0 (SPEC fallback).
 *  P5 step 6: rho_{k+1} and r_{k+1} from explicit products A x_{k+1}, B x_{k+1}; A p_{k-1} by an
 *     explicit product when Q_k is formed.  A-matvecs: 1 (x_0) + per iteration m (A g_j) +
 *     1 (A x_{k+1}) + [k > 0] (A p_{k-1}).
 *  P6 x_0(i) = u01(seed, 3, i) (R13 generator, stream 3), then B-normalised (step 2).
 *  P7 quasi-optimality diagnostic (Def. defnglbopt): rho(y*_k) = min of the
 *     Rayleigh quotient over U_k = span{x_0} + span{g_0..g_{k-1}}, from a
 *     B-orthonormal basis of U_k (CGS2_B, g_j dropped at the R16 threshold) and the smallest
 *     eigenvalue of Z^T A Z.  lambda_1 of the ratio is the caller's (e.g. the converged rho).
 * ===================================================================================== */

/* S = L L^T in place (lower triangle of L, column-major nq x nq); returns the index of the
 * first pivot that fails the P3 test, or -1. */
static int pl1_chol(int nq, const double* S, double* L) {
    for (int i = 0; i < nq * nq; ++i) L[i] = 0.0;
    for (int j = 0; j < nq; ++j) {
        double d = S[j + nq * j];
        for (int k = 0; k < j; ++k) d -= L[j + nq * k] * L[j + nq * k];
        if (!(d > 1e-24 * S[j + nq * j])) return j;
        const double ljj = sqrt(d);
        L[j + nq * j] = ljj;
        for (int i = j + 1; i < nq; ++i) {
            double s = S[i + nq * j];
            for (int k = 0; k < j; ++k) s -= L[i + nq * k] * L[j + nq * k];
            L[i + nq * j] = s / ljj;
        }
    }
    return -1;
}

int orc_pl1_solve(const orc_pl1_problem* P, double* x_out, orc_pl1_report* rep) {
    const int64_t n = P->n;
    const int m = P->m;
    if (rep) { rep->status = 1; rep->cycles = 0; rep->log_len = 0; rep->a_matvecs = rep->b_matvecs = 0; }
    if (n < 2 || m < 1 || m > 32 || !(P->tol > 0.0) || P->max_cycles < 1) return 1;
    orc_problem Q;
    memset(&Q, 0, sizeof(Q));
    Q.n = n;
    Q.a_rowptr = P->a_rowptr; Q.a_col = P->a_col; Q.a_val = P->a_val;
    Q.b_rowptr = P->b_rowptr; Q.b_col = P->b_col; Q.b_val = P->b_val;
    Q.seed = P->seed;
    ctx_t c = {&Q, n, 0, 0, 0};
    const size_t nb = (size_t)n * sizeof(double);
    double* M = (double*)malloc(nb);
    if (P->use_precond)
        orc_jacobi_diag(n, P->a_rowptr, P->a_col, P->a_val, P->b_rowptr, P->b_col, P->b_val, P->sigma, 1e-8, M);
    else
        for (int64_t i = 0; i < n; ++i) M[i] = 1.0;
    const double normF = orc_frobenius(P->a_rowptr[n] - P->a_rowptr[0], P->a_val + 0);
    double *x = malloc(nb), *Ax = malloc(nb), *Bx = malloc(nb), *r = malloc(nb);
    double *p = malloc(nb), *Ap = malloc(nb), *Bp = malloc(nb);
    double *v = malloc(nb), *tmp = malloc(nb), *g = malloc(nb), *xt = malloc(nb), *d = malloc(nb);
    double *G = malloc(nb * m), *AG = malloc(nb * m), *BG = malloc(nb * m);
    const int qmax = m + 2;
    double H[34 * 34], S[34 * 34], L[34 * 34], C[34 * 34], Y[34 * 34], th[34], w[34];
    const double* Qc[34];
    const double* AQc[34];
    const double* BQc[34];
    int status = 2, has_p = 0, k = 0;
    double beta;

    /* step 2: x_0 with ||x_0||_B = 1, rho_0, r_0 */
    for (int64_t i = 0; i < n; ++i) x[i] = P->x0 ? P->x0[i] : orc_u01(P->seed, 3, (uint64_t)i);
    applyB(&c, x, Bx);
    double nx = sqrt(orc_dot(n, x, Bx));
    for (int64_t i = 0; i < n; ++i) x[i] /= nx;
    applyA(&c, x, Ax);
    applyB(&c, x, Bx);
    double rho = orc_dot(n, x, Ax) / orc_dot(n, x, Bx);
    for (int64_t i = 0; i < n; ++i) r[i] = Ax[i] - rho * Bx[i];
    double res = sqrt(orc_dot(n, r, r));
    double rho_prev = rho;  /* rho(x_{k-1}) for step 7 (P4) */
    double conj_next = 0.0;
    /* quasi-optimality diagnostic (P7): B-orthonormal basis Z of U_k, Hz = Z^T A Z */
    const int qcap = (rep && rep->log_qopt && rep->log_qdim) ? rep->qopt_cap : 0;
    ctx_t cq = {&Q, n, 0, 0, 0};  /* its own counters: not the algorithm's matvecs */
    double *Z = NULL, *Hz = NULL, *Tq = NULL, *Yq = NULL, *thq = NULL, *vq = NULL, *Bvq = NULL, *Azq = NULL;
    int dq = 0;
    if (qcap > 0) {
        Z = malloc(nb * qcap); Hz = calloc((size_t)qcap * qcap, sizeof(double));
        Tq = malloc(sizeof(double) * qcap * qcap); Yq = malloc(sizeof(double) * qcap * qcap);
        thq = malloc(sizeof(double) * qcap);
        vq = malloc(nb); Bvq = malloc(nb); Azq = malloc(nb);
        memcpy(Z, x, nb);  /* U_0 = span{x_0}, x_0 B-normalised */
        applyA(&cq, Z, Azq);
        Hz[0] = orc_dot(n, Z, Azq);
        dq = 1;
        rep->log_qopt[0] = Hz[0];
        rep->log_qdim[0] = 1;
    }

    for (k = 0;; ++k) {
        if (rep && k < rep->log_cap) {
            rep->log_rho[k] = rho;
            rep->log_res[k] = res;
            rep->log_conj[k] = conj_next;
            rep->log_ritz[k] = 0.0;
            rep->log_mg[k] = 0;
            rep->log_nq[k] = 0;
            rep->log_len = k + 1;
        }
        if (res <= P->tol) { status = 0; break; }  /* step 3 */
        if (k >= P->max_cycles) { status = 2; break; }
        /* step 4 (P1): G_k */
        int mg = 0;
        for (int j = 0; j < m; ++j) {
            if (j == 0)
                for (int64_t i = 0; i < n; ++i) v[i] = M[i] * r[i];  /* M (A - rho_k B) x_k */
            else
                for (int64_t i = 0; i < n; ++i)
                    v[i] = M[i] * (AG[i + (size_t)n * (j - 1)] - rho * BG[i + (size_t)n * (j - 1)]);
            if (cgs2_ctx(&c, mg, G, v, tmp, NULL, &beta, NULL)) break;  /* breakdown: G_k ends */
            double* gj = G + (size_t)n * mg;
            for (int64_t i = 0; i < n; ++i) gj[i] = v[i] / beta;
            applyA(&c, gj, AG + (size_t)n * mg);
            applyB(&c, gj, BG + (size_t)n * mg);
            ++mg;
        }
        if (rep && k < rep->log_cap) rep->log_mg[k] = mg;
        /* step 5: Q_k = [x_k, G_k, p_{k-1}], RR on the projected pencil (P2, P3) */
        int nq = 1 + mg;
        Qc[0] = x; AQc[0] = Ax; BQc[0] = Bx;
        for (int j = 0; j < mg; ++j) {
            Qc[1 + j] = G + (size_t)n * j;
            AQc[1 + j] = AG + (size_t)n * j;
            BQc[1 + j] = BG + (size_t)n * j;
        }
        if (has_p) {
            applyA(&c, p, Ap);
            applyB(&c, p, Bp);
            Qc[nq] = p; AQc[nq] = Ap; BQc[nq] = Bp;
            ++nq;
        }
        int use_p = has_p, fail;
        for (;;) {
            for (int i = 0; i < nq; ++i)
                for (int jj = 0; jj < nq; ++jj) {
                    H[i + nq * jj] = orc_dot(n, Qc[i], AQc[jj]);
                    S[i + nq * jj] = orc_dot(n, Qc[i], BQc[jj]);
                }
            for (int i = 0; i < nq; ++i)
                for (int jj = 0; jj < i; ++jj) {
                    const double h = 0.5 * (H[i + nq * jj] + H[jj + nq * i]);
                    const double s = 0.5 * (S[i + nq * jj] + S[jj + nq * i]);
                    H[i + nq * jj] = H[jj + nq * i] = h;
                    S[i + nq * jj] = S[jj + nq * i] = s;
                }
            fail = pl1_chol(nq, S, L);
            if (fail < 0) break;
            if (use_p && fail == nq - 1) { use_p = 0; --nq; continue; }  /* P3: drop p_{k-1} */
            break;
        }
        if (fail >= 0) { status = 3; break; }
        /* C = L^-1 H L^-T: forward substitution on the columns, then on the rows */
        for (int jj = 0; jj < nq; ++jj)
            for (int i = 0; i < nq; ++i) {
                double s = H[i + nq * jj];
                for (int t = 0; t < i; ++t) s -= L[i + nq * t] * C[t + nq * jj];
                C[i + nq * jj] = s / L[i + nq * i];
            }  /* C = L^-1 H */
        for (int i = 0; i < nq; ++i)
            for (int jj = 0; jj < nq; ++jj) {
                double s = C[i + nq * jj];
                for (int t = 0; t < jj; ++t) s -= L[jj + nq * t] * Y[i + nq * t];
                Y[i + nq * jj] = s / L[jj + nq * jj];
            }  /* Y = (L^-1 H) L^-T */
        memcpy(C, Y, sizeof(double) * nq * nq);
        if (orc_sym_eig(nq, C, th, Y) < 0) { status = 3; break; }
        for (int i = nq - 1; i >= 0; --i) {  /* w = L^-T y_1 */
            double s = Y[i];
            for (int t = i + 1; t < nq; ++t) s -= L[t + nq * i] * w[t];
            w[i] = s / L[i + nq * i];
        }
        if (w[0] < 0.0)
            for (int i = 0; i < nq; ++i) w[i] = -w[i];
        if (rep && k < rep->log_cap) {
            rep->log_ritz[k] = th[0];
            rep->log_nq[k] = nq;
        }
        /* step 6: g_k, x~_{k+1}, x_{k+1}, rho_{k+1}, r_{k+1} (P5) */
        for (int64_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < mg; ++j) s += w[1 + j] * G[i + (size_t)n * j];
            g[i] = s;
            xt[i] = w[0] * x[i] + s + (use_p ? w[nq - 1] * p[i] : 0.0);
        }
        if (qcap > 0 && k + 1 < qcap) {  /* U_{k+1} = U_k + span{g_k} (P7) */
            if (rep->log_g) memcpy(rep->log_g + (size_t)n * k, g, nb);
            memcpy(vq, g, nb);
            double bq;
            if (!cgs2_ctx(&cq, dq, Z, vq, Bvq, NULL, &bq, NULL)) {
                double* zd = Z + (size_t)n * dq;
                for (int64_t i = 0; i < n; ++i) zd[i] = vq[i] / bq;
                applyA(&cq, zd, Azq);
                for (int i = 0; i <= dq; ++i) Hz[i + qcap * dq] = Hz[dq + qcap * i] = orc_dot(n, Z + (size_t)n * i, Azq);
                ++dq;
            }
            for (int jj = 0; jj < dq; ++jj)
                for (int i = 0; i < dq; ++i) Tq[i + dq * jj] = Hz[i + qcap * jj];
            if (orc_sym_eig(dq, Tq, thq, Yq) < 0) { status = 3; break; }
            rep->log_qopt[k + 1] = thq[0];
            rep->log_qdim[k + 1] = dq;
        }
        applyB(&c, xt, tmp);
        const double nxt = sqrt(orc_dot(n, xt, tmp));
        const double rho_k = rho;
        for (int64_t i = 0; i < n; ++i) x[i] = xt[i] / nxt;
        applyA(&c, x, Ax);
        applyB(&c, x, Bx);
        rho = orc_dot(n, x, Ax) / orc_dot(n, x, Bx);
        for (int64_t i = 0; i < n; ++i) r[i] = Ax[i] - rho * Bx[i];
        res = sqrt(orc_dot(n, r, r));
        /* step 7 (P4): p~_k and p_k */
        conj_next = 0.0;
        if (!has_p) {
            memcpy(v, g, nb);
        } else if (P->variant == 1) {
            const double wp = use_p ? w[nq - 1] : 0.0;
            for (int64_t i = 0; i < n; ++i) v[i] = g[i] + wp * p[i];
        } else {
            for (int64_t i = 0; i < n; ++i) d[i] = Ap[i] - rho_prev * Bp[i];  /* (A - rho_{k-1} B) p_{k-1} */
            const double num = orc_dot(n, d, g), den = orc_dot(n, d, p);
            const double coef = fabs(den) <= 1e-14 * normF ? 0.0 : num / den;
            for (int64_t i = 0; i < n; ++i) v[i] = g[i] - coef * p[i];
        }
        applyB(&c, v, tmp);
        const double np_ = sqrt(orc_dot(n, v, tmp));
        if (np_ > 0.0) {
            if (has_p && P->variant == 0) conj_next = orc_dot(n, d, v) / np_ / normF;
            for (int64_t i = 0; i < n; ++i) p[i] = v[i] / np_;
            has_p = 1;
        } else {
            has_p = 0;
        }
        rho_prev = rho_k;
    }
    if (x_out) memcpy(x_out, x, nb);
    if (rep) {
        rep->status = status;
        rep->cycles = k;
        rep->a_matvecs = c.a_mv;
        rep->b_matvecs = c.b_mv;
        rep->rho = rho;
        rep->resid = res;
    }
    (void)qmax;
    free(M); free(x); free(Ax); free(Bx); free(r); free(p); free(Ap); free(Bp); free(v); free(tmp);
    free(g); free(xt); free(d); free(G); free(AG); free(BG);
    free(Z); free(Hz); free(Tq); free(Yq); free(thq); free(vq); free(Bvq); free(Azq);
    return status;
}
