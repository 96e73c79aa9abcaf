// Small kernels of PL+1 (Algorithm 2; NEXT-1 of SURVEY 8(f)), readings P1-P6
// of DESIGN.md section 2.  The n-length work reuses the TRPL+K kernels (SpMV, CGS2 in the
// B-inner product, Gram columns by the fused dot kernel, the DMMA rotation, the Jacobi eig);
// these add the projected-pencil reduction of step 5 and the vector updates of steps 4, 6, 7.
// Included by kernels.cu (mat_diag, warp_sum).
#pragma once

namespace trplk {

// v = M (z - rho s), M = Jacobi of A - sigma B (R1, floor R12); s = x when B = I.
__global__ void k_pl1_prec(const Sell A, const Sell B, int64_t n, double sigma, double mfloor, const double* z,
                           const double* s, const double* rhop, double* v, int prec) {
    const double rho = rhop ? *rhop : 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (!prec) {  // M = I
            v[i] = z[i] - rho * s[i];
            continue;
        }
        const double ad = mat_diag(A, i >> 5, (int)(i & 31));
        const double bd = B.nrows ? mat_diag(B, i >> 5, (int)(i & 31)) : 1.0;
        double d = fabs(ad - sigma * bd);
        d = d > mfloor ? d : mfloor;
        v[i] = (1.0 / d) * (z[i] - rho * s[i]);
    }
}

// Deterministic dot products of up to 4 vector pairs (Pl1Pairs): CTA partials, then one CTA
// sums them in CTA order (k_pl1_dots_fin).  out[slot[t]] = a_t . b_t.
constexpr int PL1_DOT_CTAS = 296;

__global__ void __launch_bounds__(256) k_pl1_dots(Pl1Pairs P, int64_t n, double* part) {
    __shared__ double sw[8][4];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (t < P.np) acc[t] = fma(P.a[t][i], P.b[t][i], acc[t]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        double v = acc[t];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sw[warp][t] = v;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sw[w][threadIdx.x];
        part[(int64_t)blockIdx.x * 4 + threadIdx.x] = s;
    }
}

__global__ void k_pl1_dots_fin(Pl1Pairs P, const double* part, int nblk, double* out) {
    const int t = threadIdx.x;
    if (t >= P.np) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[b * 4 + t];
    out[P.slot[t]] = s;
}

// several ranks: out[slot] = sum over ranks (in rank order) of the gathered local sums
__global__ void k_pl1_dots_ranks(Pl1Pairs P, const double* all, int nranks, int stride, double* out) {
    const int t = threadIdx.x;
    if (t >= P.np) return;
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += all[(int64_t)r * stride + P.slot[t]];
    out[P.slot[t]] = s;
}

// Step 5 Gram matrices in one pass: H = Q^T (A Q), S = Q^T (B Q) for the NC columns of Q (upper
// triangles, thread-per-row register accumulators, fixed-order CTA then grid sums).  BQ = NULL:
// B = I.  Columns of Q past a breakdown hold finite stale data (their entries are ignored).
template <int NC>
__global__ void __launch_bounds__(256) k_pl1_gram(const double* __restrict__ Q, const double* __restrict__ AQ,
                                                  const double* __restrict__ BQ, int64_t ld, int64_t n,
                                                  double* part) {
    constexpr int NT = NC * (NC + 1) / 2;
    __shared__ double sw[8][2 * NT];
    double h[NT], s[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) h[t] = s[t] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double q[NC], a[NC], b[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            q[c] = Q[i + c * ld];
            a[c] = AQ[i + c * ld];
            b[c] = BQ ? BQ[i + c * ld] : q[c];
        }
        int t = 0;
#pragma unroll
        for (int r = 0; r < NC; ++r)
#pragma unroll
            for (int c = r; c < NC; ++c, ++t) {
                h[t] = fma(q[r], a[c], h[t]);
                s[t] = fma(q[r], b[c], s[t]);
            }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        double x = h[t], y = s[t];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, o);
            y += __shfl_xor_sync(0xffffffffu, y, o);
        }
        if (lane == 0) {
            sw[warp][t] = x;
            sw[warp][NT + t] = y;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * NT; t += blockDim.x) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += sw[w][t];
        part[(int64_t)blockIdx.x * 2 * NT + t] = x;
    }
}

// grid sums in CTA order -> H, S (nc x nc, ld nc, mirrored)
template <int NC>
__global__ void k_pl1_gram_fin(const double* part, int nblk, double* H, double* S) {
    constexpr int NT = NC * (NC + 1) / 2;
    const int t = threadIdx.x;
    if (t >= 2 * NT) return;
    double x = 0.0;
    for (int b = 0; b < nblk; ++b) x += part[(int64_t)b * 2 * NT + t];
    const int tt = t < NT ? t : t - NT;
    int r = 0, c = 0, u = 0;
    for (r = 0; r < NC; ++r) {
        if (tt < u + NC - r) {
            c = r + (tt - u);
            break;
        }
        u += NC - r;
    }
    double* M = t < NT ? H : S;
    M[r + NC * c] = x;
    M[c + NC * r] = x;
}

// Step 5 (P2, P3): compact the Gram columns of Q = [x, G(:, 0:mg), p] out of the (m+2)-wide
// H = Q^T A Q and S = Q^T B Q (column-major, ld = ldq), symmetrise, Cholesky S = L L^T with the
// P3 pivot test (a failing p column is dropped), C = L^-1 H L^-T into T (ld ldT).  One CTA.
// mg = ctl->k (columns CGS2 appended in step 4); on exit ctl->k = nq for the eig kernel.
__global__ void k_pl1_reduce(const double* Hq, const double* Sq, int ldq, int m, Ctl* ctl, int has_p, double* T,
                             int ldT, Pl1Dev* d) {
    const int mg = ctl->k;
    __shared__ double H[PL1_QP * PL1_QP], S[PL1_QP * PL1_QP], L[PL1_QP * PL1_QP], C[PL1_QP * PL1_QP];
    __shared__ int cols[PL1_QP];
    __shared__ int snq, sfail;
    const int tid = threadIdx.x;
    if (tid == 0) {
        int nq = 0;
        cols[nq++] = 0;
        for (int j = 0; j < mg; ++j) cols[nq++] = 1 + j;
        if (has_p) cols[nq++] = m + 1;
        snq = nq;
        sfail = -1;
    }
    __syncthreads();
    int nq = snq;
    for (int idx = tid; idx < nq * nq; idx += blockDim.x) {
        const int i = idx % nq, j = idx / nq;
        const int ci = cols[i], cj = cols[j];
        H[i + PL1_QP * j] = 0.5 * (Hq[ci + (int64_t)ldq * cj] + Hq[cj + (int64_t)ldq * ci]);
        S[i + PL1_QP * j] = 0.5 * (Sq[ci + (int64_t)ldq * cj] + Sq[cj + (int64_t)ldq * ci]);
        L[i + PL1_QP * j] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < nq; ++j) {
        if (tid == 0) {
            double dd = S[j + PL1_QP * j];
            for (int k = 0; k < j; ++k) dd -= L[j + PL1_QP * k] * L[j + PL1_QP * k];
            if (!(dd > 1e-24 * S[j + PL1_QP * j])) {
                if (has_p && j == nq - 1) snq = nq - 1;  // P3: drop p_{k-1}
                else sfail = j;
            } else {
                L[j + PL1_QP * j] = sqrt(dd);
            }
        }
        __syncthreads();
        if (sfail >= 0 || snq < nq) break;
        const double ljj = L[j + PL1_QP * j];
        for (int i = j + 1 + tid; i < nq; i += blockDim.x) {
            double s = S[i + PL1_QP * j];
            for (int k = 0; k < j; ++k) s -= L[i + PL1_QP * k] * L[j + PL1_QP * k];
            L[i + PL1_QP * j] = s / ljj;
        }
        __syncthreads();
    }
    nq = snq;
    if (sfail >= 0) {
        if (tid == 0) {
            d->nq = nq;
            d->fail = sfail;
            d->mg = mg;
            ctl->k = 1;  // keep the (discarded) eig of this iteration well defined
        }
        return;
    }
    // C = L^-1 H (forward substitution, one column per thread), then (L^-1 H) L^-T (one row per thread)
    for (int j = tid; j < nq; j += blockDim.x)
        for (int i = 0; i < nq; ++i) {
            double s = H[i + PL1_QP * j];
            for (int t = 0; t < i; ++t) s -= L[i + PL1_QP * t] * C[t + PL1_QP * j];
            C[i + PL1_QP * j] = s / L[i + PL1_QP * i];
        }
    __syncthreads();
    for (int i = tid; i < nq; i += blockDim.x)
        for (int j = 0; j < nq; ++j) {
            double s = C[i + PL1_QP * j];
            for (int t = 0; t < j; ++t) s -= L[j + PL1_QP * t] * H[i + PL1_QP * t];  // H reused as Y
            H[i + PL1_QP * j] = s / L[j + PL1_QP * j];
        }
    __syncthreads();
    for (int idx = tid; idx < nq * nq; idx += blockDim.x) {
        const int i = idx % nq, j = idx / nq;
        T[i + (int64_t)ldT * j] = H[i + PL1_QP * j];
        d->L[i + PL1_QP * j] = L[i + PL1_QP * j];
    }
    if (tid < PL1_QP) d->cols[tid] = tid < nq ? cols[tid] : -1;
    if (tid == 0) {
        d->nq = nq;
        d->fail = -1;
        d->mg = mg;
        ctl->k = nq;
    }
}

// w = L^-T y_1 (y_1 = column 0 of Y, ld ldY), sign w(1) >= 0 (P2), scattered to the m+2 slots of
// Q (zeros for unused slots) in d->w.  One thread.
__global__ void k_pl1_back(const double* Y, int ldY, int m, Pl1Dev* d) {
    if (threadIdx.x != 0) return;
    const int nq = d->nq;
    double w[PL1_QP];
    for (int i = nq - 1; i >= 0; --i) {
        double s = Y[i];
        for (int t = i + 1; t < nq; ++t) s -= d->L[t + PL1_QP * i] * w[t];
        w[i] = s / d->L[i + PL1_QP * i];
    }
    const double sg = w[0] < 0.0 ? -1.0 : 1.0;
    for (int i = 0; i < m + 2; ++i) d->w[i] = 0.0;
    for (int i = 0; i < nq; ++i) d->w[d->cols[i]] = sg * w[i];
}

// xt = w(1) x + g + w(m+2) p (step 6)
__global__ void k_pl1_xt(int64_t n, const double* x, const double* g, const double* p, const Pl1Dev* d, int m,
                         double* xt) {
    const double a = d->w[0], b = d->w[m + 1];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        xt[i] = a * x[i] + g[i] + b * p[i];
}

// y = x / sqrt(*nrm2)
__global__ void k_pl1_scale(int64_t n, const double* x, const double* nrm2, double* y) {
    const double s = sqrt(*nrm2);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i] / s;
}

// p_k = p~_k / ||p~_k||_B, or (zero norm: g_k = 0) no search direction for the next iteration
__global__ void k_pl1_scale_p(int64_t n, const double* x, const double* nrm2, double* y, Pl1Dev* d) {
    const double q = *nrm2;
    if (blockIdx.x == 0 && threadIdx.x == 0) d->has_p = q > 0.0 ? 1 : 0;
    if (!(q > 0.0)) return;
    const double s = sqrt(q);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i] / s;
}

// r = Ax - rho Bx with rho = xAx / xBx from the device scalars (step 6)
__global__ void k_pl1_res(int64_t n, const double* Ax, const double* Bx, const double* xAx, const double* xBx,
                          double* r) {
    const double rho = *xAx / *xBx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = Ax[i] - rho * Bx[i];
}

// y = a x + b z (host scalars)
__global__ void k_pl1_axpby(int64_t n, double a, const double* x, double b, const double* z, double* y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = a * x[i] + b * z[i];
}

// step 7 (P4): pt = g - (num/den) p, coefficient 0 when |den| <= 1e-14 ||A||_F; variant 1: g + w(m+2) p
__global__ void k_pl1_pt(int64_t n, const double* g, const double* p, const double* num, const double* den,
                         double den_floor, int variant, const Pl1Dev* d, int m, double* pt) {
    double c;
    if (variant == 1) c = d->w[m + 1];
    else c = fabs(*den) <= den_floor ? 0.0 : -(*num / *den);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        pt[i] = g[i] + c * p[i];
}

static int pl1_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g < 1 ? 1 : g);
}

void pl1_prec(const Sell& A, const Sell& B, int64_t n, double sigma, double mfloor, const double* z,
              const double* s, const double* rho, double* v, int prec, cudaStream_t st) {
    k_pl1_prec<<<pl1_grid(n), 256, 0, st>>>(A, B, n, sigma, mfloor, z, s, rho, v, prec);
}

__global__ void k_pl1_begin(Ctl* ctl) {
    ctl->k = 0;
    ctl->flags = ~0u;
    ctl->pass3 = 0;
}

__global__ void k_pl1_shift_rho(Pl1Dev* d, const double* sc) {
    d->rho_prev = d->rho_cur;
    d->rho_cur = sc[1] / sc[2];
}

// v = (A - rho_{k-1} B) p_{k-1} from the stored products (P4)
__global__ void k_pl1_dvec(int64_t n, const double* Ap, const double* Bp, const Pl1Dev* d, double* v) {
    const double r = d->rho_prev;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = Ap[i] - r * Bp[i];
}

// quasi-optimality diagnostic (P7): H(j, i) = H(i, j) for i < j < d (the Gram columns fill i <= j)
__global__ void k_pl1_qmirror(double* H, int ldH, int d) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < d * d; idx += gridDim.x * blockDim.x) {
        const int i = idx % d, j = idx / d;
        if (i < j) H[j + (int64_t)i * ldH] = H[i + (int64_t)j * ldH];
    }
}

void pl1_qmirror(double* H, int ldH, int d, cudaStream_t st) { k_pl1_qmirror<<<4, 256, 0, st>>>(H, ldH, d); }
void pl1_begin(Ctl* ctl, cudaStream_t st) { k_pl1_begin<<<1, 1, 0, st>>>(ctl); }
void pl1_shift_rho(Pl1Dev* d, const double* sc, cudaStream_t st) { k_pl1_shift_rho<<<1, 1, 0, st>>>(d, sc); }
void pl1_dvec(int64_t n, const double* Ap, const double* Bp, const Pl1Dev* d, double* v, cudaStream_t st) {
    k_pl1_dvec<<<pl1_grid(n), 256, 0, st>>>(n, Ap, Bp, d, v);
}

void pl1_dots(const Pl1Pairs& P, int64_t n, double* part, double* out, cudaStream_t st) {
    int g = (int)std::min<int64_t>(PL1_DOT_CTAS, (n + 255) / 256);
    if (g < 1) g = 1;
    k_pl1_dots<<<g, 256, 0, st>>>(P, n, part);
    k_pl1_dots_fin<<<1, 32, 0, st>>>(P, part, g, out);
}

void pl1_dots_ranks(const Pl1Pairs& P, const double* all, int nranks, int stride, double* out, cudaStream_t st) {
    k_pl1_dots_ranks<<<1, 32, 0, st>>>(P, all, nranks, stride, out);
}

void pl1_reduce(const double* Hq, const double* Sq, int ldq, int m, Ctl* ctl, int has_p, double* T, int ldT,
                Pl1Dev* d, cudaStream_t st) {
    k_pl1_reduce<<<1, 64, 0, st>>>(Hq, Sq, ldq, m, ctl, has_p, T, ldT, d);
}

void pl1_scale_p(int64_t n, const double* x, const double* nrm2, double* y, Pl1Dev* d, cudaStream_t st) {
    k_pl1_scale_p<<<pl1_grid(n), 256, 0, st>>>(n, x, nrm2, y, d);
}

template <int NC>
static void pl1_gram_k(const double* Q, const double* AQ, const double* BQ, int64_t ld, int64_t n, double* part,
                       double* H, double* S, cudaStream_t st) {
    constexpr int NT = NC * (NC + 1) / 2;
    int g = (int)std::min<int64_t>(PL1_PART / (2 * NT), (n + 255) / 256);
    if (g > 296) g = 296;
    if (g < 1) g = 1;
    k_pl1_gram<NC><<<g, 256, 0, st>>>(Q, AQ, BQ, ld, n, part);
    k_pl1_gram_fin<NC><<<1, 2 * NT <= 32 ? 32 : ((2 * NT + 31) / 32) * 32, 0, st>>>(part, g, H, S);
}

bool pl1_gram(int nc, const double* Q, const double* AQ, const double* BQ, int64_t ld, int64_t n, double* part,
              double* H, double* S, cudaStream_t st) {
    switch (nc) {
        case 3: pl1_gram_k<3>(Q, AQ, BQ, ld, n, part, H, S, st); return true;
        case 4: pl1_gram_k<4>(Q, AQ, BQ, ld, n, part, H, S, st); return true;
        case 5: pl1_gram_k<5>(Q, AQ, BQ, ld, n, part, H, S, st); return true;
        case 6: pl1_gram_k<6>(Q, AQ, BQ, ld, n, part, H, S, st); return true;
        case 7: pl1_gram_k<7>(Q, AQ, BQ, ld, n, part, H, S, st); return true;
        case 8: pl1_gram_k<8>(Q, AQ, BQ, ld, n, part, H, S, st); return true;
        default: return false;
    }
}

void pl1_back(const double* Y, int ldY, int m, Pl1Dev* d, cudaStream_t st) { k_pl1_back<<<1, 32, 0, st>>>(Y, ldY, m, d); }

void pl1_xt(int64_t n, const double* x, const double* g, const double* p, const Pl1Dev* d, int m, double* xt,
            cudaStream_t st) {
    k_pl1_xt<<<pl1_grid(n), 256, 0, st>>>(n, x, g, p, d, m, xt);
}

void pl1_scale(int64_t n, const double* x, const double* nrm2, double* y, cudaStream_t st) {
    k_pl1_scale<<<pl1_grid(n), 256, 0, st>>>(n, x, nrm2, y);
}

void pl1_res(int64_t n, const double* Ax, const double* Bx, const double* xAx, const double* xBx, double* r,
             cudaStream_t st) {
    k_pl1_res<<<pl1_grid(n), 256, 0, st>>>(n, Ax, Bx, xAx, xBx, r);
}

void pl1_axpby(int64_t n, double a, const double* x, double b, const double* z, double* y, cudaStream_t st) {
    k_pl1_axpby<<<pl1_grid(n), 256, 0, st>>>(n, a, x, b, z, y);
}

void pl1_pt(int64_t n, const double* g, const double* p, const double* num, const double* den, double den_floor,
            int variant, const Pl1Dev* d, int m, double* pt, cudaStream_t st) {
    k_pl1_pt<<<pl1_grid(n), 256, 0, st>>>(n, g, p, num, den, den_floor, variant, d, m, pt);
}

}  // namespace trplk
