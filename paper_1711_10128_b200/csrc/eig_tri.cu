// K6 alternative (TRPLK_EIG=tri): the Rayleigh-Ritz eigensolve T = Y Theta Y^T (Alg.1 step 11,
// PAPER.md:191-193) for the nev lowest pairs only -- the restart keeps p^ Ritz pairs (P:193,
// R5), so the other k - p^ are never used.  One CTA:
//   1. Householder tridiagonalisation Q^T T Q = tridiag(d, e) (reflectors kept below the
//      subdiagonal, as LAPACK dsytd2 does);
//   2. eigenvalues lambda_0..lambda_{nev-1} by multisection on Sturm counts (one warp per
//      eigenvalue, 32 trial points per round: the interval shrinks 33x per round);
//   3. tridiagonal eigenvectors by inverse iteration on the pivoted LU of T - lambda I, three
//      iterations, members of a cluster (gap <= 1e-3 ||T||) orthogonalised against the
//      earlier members in every iteration (the dstein recipe);
//   4. back-transformation by the reflectors, sign rule R11, ascending Theta; restart T reset
//      (R10) as k_eig.
// Same outputs as k_eig for the first nev columns (eig.cu).  Backward stable like Jacobi: Ritz
// values to O(eps ||T||), Y orthonormal to O(eps) (tests/test_gpu_kernels.py).
#include <cfloat>
#include <cstdlib>
#include <cstring>

#include "trplk_internal.cuh"

namespace trplk {

constexpr int TRI_THREADS = 512;
__device__ long long tri_clk[8];  // phase-boundary clocks of the last launch (tools/eig_time.py)
constexpr int TRI_WARPS = TRI_THREADS / 32;
constexpr int TRLD = QMAX + 1;

__device__ __forceinline__ double tri_rcp(double x) {  // ~correctly rounded 1/x (normal range)
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// number of eigenvalues of tridiag(d, e) below lam (Sturm sequence, LAPACK dlaebz guard)
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int k, double lam, double pivmin) {
    int c = 0;
    double q = d[0] - lam;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
    for (int i = 1; i < k; ++i) {
        q = (d[i] - lam) - e2[i - 1] * tri_rcp(q);
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

__global__ void __launch_bounds__(TRI_THREADS) k_eig_tri(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph,
                                                         int k_fixed, int nev_in, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k;
    const int nev = nev_in > 0 && nev_in < k ? nev_in : k;
    extern __shared__ double tsm[];
    double* A = tsm;                 // k x k, column-major, ld TRLD; reflectors below the subdiagonal
    double* Z = tsm + QMAX * TRLD;   // k x nev eigenvectors, ld TRLD
    __shared__ double d[QMAX], e[QMAX], e2[QMAX], tau[QMAX], lam[QMAX], pv[QMAX], wv[QMAX];
    __shared__ double sred[TRI_WARPS];
    __shared__ double sK, sbnorm, spivmin;
    __shared__ int cl_first[QMAX + 1], ncl;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) tri_clk[0] = clock64();
    for (int idx = tid; idx < k * k; idx += TRI_THREADS) {
        const int i = idx % k, j = idx / k;
        A[i + j * TRLD] = 0.5 * (T[i + (int64_t)j * ldT] + T[j + (int64_t)i * ldT]);  // sym(T)
    }
    __syncthreads();
    if (tid == 0) tri_clk[1] = clock64();
    // ---- 1. tridiagonalisation (lower), j = 0 .. k-3
    for (int j = 0; j + 2 < k; ++j) {
        const int L = k - j - 1;  // length of x = A[j+1 .. k-1, j]
        if (warp == 0) {
            double s = 0.0;
            for (int i = lane; i < L; i += 32) {
                const double x = A[j + 1 + i + j * TRLD];
                s = fma(x, x, s);
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) {
                const double x0 = A[j + 1 + j * TRLD];
                const double nrm = sqrt(s);
                if (nrm == 0.0) {
                    tau[j] = 0.0;
                    e[j] = 0.0;
                } else {
                    const double alpha = x0 >= 0.0 ? -nrm : nrm;
                    const double v0 = x0 - alpha;
                    const double vtv = s - x0 * x0 + v0 * v0;
                    tau[j] = 2.0 / vtv;
                    e[j] = alpha;
                    A[j + 1 + j * TRLD] = v0;
                }
                d[j] = A[j + j * TRLD];
            }
        }
        __syncthreads();
        const double tj = tau[j];
        if (tj == 0.0) continue;  // uniform: no reflection needed
        const double* v = A + (j + 1) + j * TRLD;  // v_i = v[i], i < L
        // p = tau A22 v: 8 lanes per row, strided columns, shuffle-combined in lane order
        {
            const int row = tid >> 3, part = tid & 7;
            double s = 0.0;
            if (row < L)
                for (int l = part; l < L; l += 8) s = fma(A[j + 1 + row + (j + 1 + l) * TRLD], v[l], s);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            if (row < L && part == 0) pv[row] = tj * s;
        }
        __syncthreads();
        if (warp == 0) {
            double s = 0.0;
            for (int i = lane; i < L; i += 32) s = fma(v[i], pv[i], s);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) sK = 0.5 * tj * s;
        }
        __syncthreads();
        if (tid < L) wv[tid] = pv[tid] - sK * v[tid];
        __syncthreads();
        for (int l = warp; l < L; l += TRI_WARPS) {  // A22 -= v w^T + w v^T (warp per column)
            const double vl = v[l], wl = wv[l];
            for (int i = lane; i < L; i += 32)
                A[j + 1 + i + (j + 1 + l) * TRLD] -= fma(v[i], wl, wv[i] * vl);
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (k >= 2) {
            d[k - 2] = A[k - 2 + (k - 2) * TRLD];
            e[k - 2] = A[k - 1 + (k - 2) * TRLD];
            if (k == 2) tau[0] = 0.0;
        }
        d[k - 1] = A[k - 1 + (k - 1) * TRLD];
        double gl = DBL_MAX, gu = -DBL_MAX, emax = 0.0;
        for (int i = 0; i < k; ++i) {
            const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < k ? fabs(e[i]) : 0.0);
            gl = fmin(gl, d[i] - r);
            gu = fmax(gu, d[i] + r);
            if (i + 1 < k) {
                e2[i] = e[i] * e[i];
                emax = fmax(emax, e2[i]);
            }
        }
        sbnorm = fmax(fabs(gl), fabs(gu));
        spivmin = DBL_MIN * fmax(1.0, emax);
        lam[QMAX - 1] = gl;  // scratch: Gershgorin bounds
        wv[QMAX - 1] = gu;
    }
    __syncthreads();
    const double bnorm = sbnorm, pivmin = spivmin;
    if (tid == 0) tri_clk[2] = clock64();
    // ---- 2. eigenvalues by multisection (one warp per eigenvalue)
    {
        const double gl0 = lam[QMAX - 1] - 2.0 * DBL_EPSILON * bnorm - 2.0 * pivmin;
        const double gu0 = wv[QMAX - 1] + 2.0 * DBL_EPSILON * bnorm + 2.0 * pivmin;
        __syncthreads();
        for (int i = warp; i < nev; i += TRI_WARPS) {
            double lo = gl0, hi = gu0;
            for (int round = 0; round < 60; ++round) {
                if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin) break;
                const double x = lo + (hi - lo) * (double)(lane + 1) * (1.0 / 33.0);
                const int c = sturm_count(d, e2, k, x, pivmin);
                const unsigned m = __ballot_sync(0xffffffffu, c >= i + 1);
                const int l = m ? __ffs(m) - 1 : 32;
                const double xl = __shfl_sync(0xffffffffu, x, l > 0 ? l - 1 : 0);
                const double xh = __shfl_sync(0xffffffffu, x, l < 32 ? l : 31);
                const double nlo = l == 0 ? lo : xl;
                const double nhi = l == 32 ? hi : xh;
                if (nlo == lo && nhi == hi) break;  // no representable progress
                lo = nlo;
                hi = nhi;
            }
            if (lane == 0) lam[i] = 0.5 * (lo + hi);
        }
    }
    __syncthreads();
    if (tid == 0) tri_clk[3] = clock64();
    // clusters of close eigenvalues (processed sequentially by one thread each)
    if (tid == 0) {
        int n = 0;
        for (int i = 0; i < nev; ++i)
            if (i == 0 || lam[i] - lam[i - 1] > 1e-3 * bnorm) cl_first[n++] = i;
        cl_first[n] = nev;
        ncl = n;
    }
    __syncthreads();
    // ---- 3. inverse iteration (one thread per cluster)
    if (tid < ncl) {
        const int i0 = cl_first[tid], i1 = cl_first[tid + 1];
        double u0[QMAX], u1[QMAX], u2[QMAX], ml[QMAX], z[QMAX];
        bool sw[QMAX];
        double lprev = 0.0;
        for (int i = i0; i < i1; ++i) {
            double lm = lam[i];
            if (i > i0 && lm - lprev < 10.0 * DBL_EPSILON * fabs(lm)) lm = lprev + 10.0 * DBL_EPSILON * fabs(lm);
            lprev = lm;
            // pivoted LU of T - lm I: rows (u0 diag, u1 super, u2 super-super), multipliers ml
            const double tiny = DBL_EPSILON * bnorm + pivmin;
            double a = d[0] - lm, b = k > 1 ? e[0] : 0.0, c2 = 0.0;
            for (int r = 0; r + 1 < k; ++r) {
                const double sub = e[r], dn = d[r + 1] - lm, sn = r + 2 < k ? e[r + 1] : 0.0;
                if (fabs(a) >= fabs(sub)) {  // no interchange
                    if (fabs(a) < tiny) a = a < 0.0 ? -tiny : tiny;
                    const double m = sub / a;
                    sw[r] = false;
                    ml[r] = m;
                    u0[r] = a;
                    u1[r] = b;
                    u2[r] = c2;
                    a = dn - m * b;
                    b = sn;
                    c2 = 0.0;
                } else {  // interchange rows r and r+1
                    const double m = a / sub;
                    sw[r] = true;
                    ml[r] = m;
                    u0[r] = sub;
                    u1[r] = dn;
                    u2[r] = sn;
                    a = b - m * dn;
                    b = -m * sn;
                    c2 = 0.0;
                }
            }
            if (fabs(a) < tiny) a = a < 0.0 ? -tiny : tiny;
            u0[k - 1] = a;
            for (int r = 0; r < k; ++r) u0[r] = 1.0 / u0[r];  // reciprocal pivots for the solves
            // start vector: a fixed pseudo-random vector (deterministic)
            for (int r = 0; r < k; ++r) {
                const unsigned h = (unsigned)(r + 1) * 2654435761u ^ (unsigned)(i + 7) * 40503u;
                z[r] = 0.5 + (double)(h & 0xffff) * (1.0 / 65536.0);
            }
            for (int it = 0; it < 3; ++it) {
                // forward: apply the row interchanges and multipliers
                for (int r = 0; r + 1 < k; ++r) {
                    if (sw[r]) {
                        const double t = z[r];
                        z[r] = z[r + 1];
                        z[r + 1] = t - ml[r] * z[r];
                    } else {
                        z[r + 1] -= ml[r] * z[r];
                    }
                }
                // back substitution with U (diag u0, super u1, super-super u2)
                for (int r = k - 1; r >= 0; --r) {
                    double s = z[r];
                    if (r + 1 < k) s -= u1[r] * z[r + 1];
                    if (r + 2 < k) s -= u2[r] * z[r + 2];
                    z[r] = s * u0[r];
                }
                // orthogonalise against the earlier members of the cluster, then scale
                for (int j = i0; j < i; ++j) {
                    double dt = 0.0;
                    for (int r = 0; r < k; ++r) dt = fma(Z[r + j * TRLD], z[r], dt);
                    for (int r = 0; r < k; ++r) z[r] = fma(-dt, Z[r + j * TRLD], z[r]);
                }
                double nn = 0.0;
                for (int r = 0; r < k; ++r) nn = fma(z[r], z[r], nn);
                const double inv = 1.0 / sqrt(nn);
                for (int r = 0; r < k; ++r) z[r] *= inv;
            }
            for (int r = 0; r < k; ++r) Z[r + i * TRLD] = z[r];
        }
    }
    __syncthreads();
    if (tid == 0) tri_clk[4] = clock64();
    // ---- 4. back-transformation z <- H_0 ... H_{k-3} z (warp per vector), sign rule, output
    for (int c = warp; c < nev; c += TRI_WARPS) {
        double* zc = Z + c * TRLD;
        for (int j = k - 3; j >= 0; --j) {
            const double tj = tau[j];
            if (tj == 0.0) continue;
            const int L = k - j - 1;
            const double* v = A + (j + 1) + j * TRLD;
            double s = 0.0;
            for (int i = lane; i < L; i += 32) s = fma(v[i], zc[j + 1 + i], s);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            s *= tj;
            for (int i = lane; i < L; i += 32) zc[j + 1 + i] = fma(-s, v[i], zc[j + 1 + i]);
            __syncwarp();
        }
        // sign rule (R11): the largest-magnitude entry positive (first on ties)
        double vmax = -1.0;
        int imax = 0;
        for (int i = lane; i < k; i += 32) {
            const double a = fabs(zc[i]);
            if (a > vmax) {
                vmax = a;
                imax = i;
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, vmax, o);
            const int oi = __shfl_xor_sync(0xffffffffu, imax, o);
            if (ov > vmax || (ov == vmax && oi < imax)) {
                vmax = ov;
                imax = oi;
            }
        }
        const double sg = zc[imax] < 0.0 ? -1.0 : 1.0;
        for (int i = lane; i < k; i += 32) Y[i + (int64_t)c * ldY] = sg * zc[i];
        if (lane == 0) ctl->theta[c] = lam[c];
    }
    __syncthreads();
    if (ph > 0) {  // restart: T <- diag(Theta(1:p^)) (R10)
        for (int idx = tid; idx < QMAX * QMAX; idx += TRI_THREADS) {
            const int i = idx % QMAX, j = idx / QMAX;
            T[i + (int64_t)j * ldT] = (i == j && i < ph) ? ctl->theta[i] : 0.0;
        }
    }
    if (tid == 0) {
        ctl->k_rr = k;
        ctl->eig_sweeps = 0;
        tri_clk[5] = clock64();
    }
}

void launch_eig_tri(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph, int k_fixed, int nev, unsigned gate,
                    cudaStream_t s) {
    static int init = 0;
    const int smem = 2 * QMAX * TRLD * (int)sizeof(double);
    if (!init) {
        cudaFuncSetAttribute(k_eig_tri, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        init = 1;
    }
    static const int nev_env = getenv("TRPLK_EIG_NEV") ? atoi(getenv("TRPLK_EIG_NEV")) : 0;  // timing knob
    k_eig_tri<<<1, TRI_THREADS, smem, s>>>(ctl, T, ldT, Y, ldY, ph, k_fixed, nev_env > 0 ? nev_env : nev, gate);
}

}  // namespace trplk

// debug (tools/eig_time.py): phase clocks of the last k_eig_tri launch
extern "C" void trplk_debug_tri_clk(long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, trplk::tri_clk, sizeof(long long) * 8);
}
