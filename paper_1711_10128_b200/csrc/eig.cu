// K6: the Rayleigh-Ritz eigensolve T = Y Theta Y^T (Alg.1 step 11) in one
// CTA by parallel-ordered cyclic Jacobi (north_star item 4).
//
// Round-robin ordering: in each of the kk-1 rounds of a sweep, kk/2 disjoint pairs (p,q) are
// rotated at once.  Because the pairs are disjoint, the two-sided update A <- J^T A J splits
// into independent 2x2 blocks J_i^T A[P_i,P_j] J_j, so a round needs only two barriers:
// [rotation parameters] -> barrier -> [2x2 block updates of A (upper triangle, mirrored) and
// column updates of V] -> barrier.  Rotation formula and skip rule as the oracle
// (|a_pq| <= eps sqrt|a_pp a_qq| or <= 1e-30 ||T||_F is not rotated; a sweep without rotations
// ends the iteration); the rotated entry is set to exactly 0.  Output: ascending Theta (stable
// on ties), Y with the largest-magnitude entry of each column positive (R11); T is then reset
// to diag(Theta(1:p^)) for the restart (R10).
#include "trplk_internal.cuh"

namespace trplk {

constexpr int EIG_THREADS = 512;
constexpr int ELD = QMAX + 1;
constexpr int MAXPAIRS = QMAX / 2;
constexpr int MAXBLK = MAXPAIRS * (MAXPAIRS + 1) / 2;

__device__ __forceinline__ int rr_player(int pos, int r, int kk) {
    return pos == 0 ? 0 : 1 + (pos - 1 + r) % (kk - 1);
}

__global__ void __launch_bounds__(EIG_THREADS) k_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph,
                                                     int k_fixed, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k;
    extern __shared__ double sm[];
    double* A = sm;
    double* V = sm + QMAX * ELD;
    __shared__ double cs[MAXPAIRS], sn[MAXPAIRS], red[EIG_THREADS];
    __shared__ int pp[MAXPAIRS], qq[MAXPAIRS], act[MAXPAIRS], ord[QMAX];
    __shared__ unsigned char tabp[QMAX - 1][MAXPAIRS], tabq[QMAX - 1][MAXPAIRS];
    __shared__ unsigned char bi[MAXBLK], bj[MAXBLK];
    __shared__ int rotated;
    __shared__ double fro;
    const int tid = threadIdx.x;
    double f = 0.0;
    for (int idx = tid; idx < k * k; idx += EIG_THREADS) {
        const int i = idx % k, j = idx / k;
        const double a = 0.5 * (T[i + (int64_t)j * ldT] + T[j + (int64_t)i * ldT]);  // sym(T)
        A[i + j * ELD] = a;
        V[i + j * ELD] = (i == j) ? 1.0 : 0.0;
        f += a * a;
    }
    const int kk = k + (k & 1);
    const int npairs = kk / 2;
    const int nblk = npairs * (npairs + 1) / 2;
    for (int idx = tid; idx < (kk - 1) * npairs; idx += EIG_THREADS) {
        const int r = idx / npairs, i = idx % npairs;
        int p = rr_player(i, r, kk), q = rr_player(kk - 1 - i, r, kk);
        if (p > q) { const int t = p; p = q; q = t; }
        tabp[r][i] = (unsigned char)p;
        tabq[r][i] = (unsigned char)q;
    }
    if (tid == 0) {
        int b = 0;
        for (int i = 0; i < npairs; ++i)
            for (int j = i; j < npairs; ++j) {
                bi[b] = (unsigned char)i;
                bj[b] = (unsigned char)j;
                ++b;
            }
    }
    red[tid] = f;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < EIG_THREADS; ++i) s += red[i];
        fro = sqrt(s);
    }
    __syncthreads();
    const double eps = 2.220446049250313e-16;
    for (int sweep = 0; sweep < 100 && k > 1; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int r = 0; r < kk - 1; ++r) {
            if (tid < npairs) {
                const int p = tabp[r][tid], q = tabq[r][tid];
                int a_ = 0;
                double c = 1.0, s = 0.0;
                if (q < k) {
                    const double apq = A[p + q * ELD], app = A[p + p * ELD], aqq = A[q + q * ELD];
                    if (!(fabs(apq) <= eps * sqrt(fabs(app * aqq)) || fabs(apq) <= 1e-30 * fro)) {
                        // t = sgn(tau)/(|tau| + sqrt(1+tau^2)), tau = (aqq-app)/(2apq), division-light
                        const double d = aqq - app, b = 2.0 * apq;
                        const double t = ((d == 0.0 || ((d > 0.0) == (b > 0.0))) ? 1.0 : -1.0) * fabs(b) /
                                         (fabs(d) + sqrt(d * d + b * b));
                        c = rsqrt(1.0 + t * t);
                        s = t * c;
                        a_ = 1;
                        rotated = 1;
                    }
                }
                pp[tid] = p;
                qq[tid] = q;
                cs[tid] = c;
                sn[tid] = s;
                act[tid] = a_;
            }
            __syncthreads();
            // A <- J^T A J on the 2x2 blocks (i <= j, mirrored); rotated pairs get exact zeros
            for (int b = tid; b < nblk; b += EIG_THREADS) {
                const int i = bi[b], j = bj[b];
                if (!act[i] && !act[j]) continue;
                const int p1 = pp[i], q1 = qq[i], p2 = pp[j], q2 = qq[j];
                const bool q1ok = q1 < k, q2ok = q2 < k;
                const double c1 = cs[i], s1 = sn[i], c2 = cs[j], s2 = sn[j];
                const double a = A[p1 + p2 * ELD];
                const double bb = q2ok ? A[p1 + q2 * ELD] : 0.0;
                const double cc = q1ok ? A[q1 + p2 * ELD] : 0.0;
                const double dd = (q1ok && q2ok) ? A[q1 + q2 * ELD] : 0.0;
                const double n00 = a * c2 - bb * s2, n01 = a * s2 + bb * c2;   // M J_j
                const double n10 = cc * c2 - dd * s2, n11 = cc * s2 + dd * c2;
                const double m00 = c1 * n00 - s1 * n10, m01 = c1 * n01 - s1 * n11;  // J_i^T (M J_j)
                double m10 = s1 * n00 + c1 * n10, m11 = s1 * n01 + c1 * n11;
                double m01w = m01;
                if (i == j) {
                    if (act[i]) { m01w = 0.0; m10 = 0.0; }
                    A[p1 + p1 * ELD] = m00;
                    if (q1ok) {
                        A[q1 + q1 * ELD] = m11;
                        A[p1 + q1 * ELD] = m01w;
                        A[q1 + p1 * ELD] = m10;
                    }
                } else {
                    A[p1 + p2 * ELD] = m00;
                    A[p2 + p1 * ELD] = m00;
                    if (q2ok) {
                        A[p1 + q2 * ELD] = m01;
                        A[q2 + p1 * ELD] = m01;
                    }
                    if (q1ok) {
                        A[q1 + p2 * ELD] = m10;
                        A[p2 + q1 * ELD] = m10;
                    }
                    if (q1ok && q2ok) {
                        A[q1 + q2 * ELD] = m11;
                        A[q2 + q1 * ELD] = m11;
                    }
                }
            }
            // V <- V J (rows x pairs)
            for (int e = tid; e < k * MAXPAIRS; e += EIG_THREADS) {
                const int pi = e & (MAXPAIRS - 1), i = e / MAXPAIRS;
                if (pi >= npairs || !act[pi]) continue;
                const int p = pp[pi], q = qq[pi];
                const double c = cs[pi], s = sn[pi];
                const double vip = V[i + p * ELD], viq = V[i + q * ELD];
                V[i + p * ELD] = c * vip - s * viq;
                V[i + q * ELD] = s * vip + c * viq;
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    // ascending order, stable on ties (R11)
    if (tid < k) {
        const double ti = A[tid + tid * ELD];
        int rank = 0;
        for (int j = 0; j < k; ++j) {
            const double tj = A[j + j * ELD];
            rank += (tj < ti) || (tj == ti && j < tid);
        }
        ord[rank] = tid;
    }
    __syncthreads();
    if (tid < k) {
        const int src = ord[tid];
        int imax = 0;
        double vmax = -1.0;
        for (int i = 0; i < k; ++i) {
            const double a = fabs(V[i + src * ELD]);
            if (a > vmax) { vmax = a; imax = i; }
        }
        const double sg = V[imax + src * ELD] < 0.0 ? -1.0 : 1.0;  // sign rule (R11)
        for (int i = 0; i < k; ++i) Y[i + (int64_t)tid * ldY] = sg * V[i + src * ELD];
        ctl->theta[tid] = A[src + src * ELD];
    }
    __syncthreads();
    if (ph > 0) {  // restart: T <- diag(Theta(1:p^)) (R10)
        for (int idx = tid; idx < QMAX * QMAX; idx += EIG_THREADS) {
            const int i = idx % QMAX, j = idx / QMAX;
            T[i + (int64_t)j * ldT] = (i == j && i < ph) ? ctl->theta[i] : 0.0;
        }
    }
    if (tid == 0) ctl->k_rr = k;
}

void launch_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph, int k_fixed, unsigned gate,
                cudaStream_t s) {
    static bool init = false;
    const int smem = 2 * QMAX * ELD * (int)sizeof(double);
    if (!init) {
        cudaFuncSetAttribute(k_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        init = true;
    }
    k_eig<<<1, EIG_THREADS, smem, s>>>(ctl, T, ldT, Y, ldY, ph, k_fixed, gate);
}

}  // namespace trplk
