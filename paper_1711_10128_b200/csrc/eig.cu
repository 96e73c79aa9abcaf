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
#include <cstdlib>
#include <cstring>

#include "trplk_internal.cuh"

namespace trplk {

constexpr int ELD = QMAX + 1;
constexpr int MAXPAIRS = QMAX / 2;
constexpr int MAXBLK = MAXPAIRS * (MAXPAIRS + 1) / 2;

__device__ __forceinline__ int rr_player(int pos, int r, int kk) {
    return pos == 0 ? 0 : 1 + (pos - 1 + r) % (kk - 1);
}

// ------------------------------------------------------------------------------------------
// One barrier per round.  A is double-buffered: round r reads A_r and writes
// A_{r+1}, so within one phase
//   warp 0      computes the rotation parameters of round r+1: for its pivot (x, y) it forms
//               the new entry A_{r+1}[x,y] from A_r and the round-r rotations of the two pairs
//               holding x and y (the same 2x2 formula the block update uses) and takes the new
//               diagonal entries from the round-r parameter step;
//   warps 1..7  apply the round-r rotations: 2x2 blocks J_i^T A_r[P_i,P_j] J_j -> A_{r+1}
//               (every entry of A is in exactly one block) and V <- V J;
// and a round costs one barrier (a two-barrier version of the same rotations measured
// 244 vs 154 us at k = 30 and was removed).  Same skip rule and sweep-end test as the oracle.
#ifdef EIG_TRACE
__device__ unsigned long long eig_trace[32];  // per-warp cycles to the round barrier; [30] rounds, [31] round cycles
#endif
// Warp roles (warp w runs on scheduler w % 4): warp 0 computes the next round's rotation
// parameters -- the critical path -- and has scheduler 0 to itself (warps 4, 8, 12 idle);
// warps 1-3, 5-7 update the 2x2 blocks of A, warps 9-11, 13-15 the columns of V.
constexpr int EIG1_THREADS = 512;
constexpr int BLK_WARPS = 6;
__device__ __forceinline__ int eig_role(int w, int& rank) {  // 0 params, 1 blocks, 2 V, 3 idle
    if (w == 0) { rank = 0; return 0; }
    if ((w & 3) == 0) { rank = 0; return 3; }
    const int sub = (w & 3) - 1;  // 0..2
    if (w < 8) { rank = (w >> 2) * 3 + sub; return 1; }
    rank = ((w - 8) >> 2) * 3 + sub;
    return 2;
}

__device__ __forceinline__ int rr_pos(int x, int r, int kk) {  // position of player x in round r
    if (x == 0) return 0;
    const int m = kk - 1;
    int v = (x - 1 - r) % m;
    if (v < 0) v += m;
    return v + 1;
}

__device__ __forceinline__ int pair_of_pos(int pos, int kk) { return pos < kk / 2 ? pos : kk - 1 - pos; }

// 2x2 block update J_i^T [a b; c d] J_j (rotation (c1,s1) of pair i, (c2,s2) of pair j)
__device__ __forceinline__ void block22(double a, double b, double c, double d, double c1, double s1, double c2,
                                        double s2, double& m00, double& m01, double& m10, double& m11) {
    const double n00 = a * c2 - b * s2, n01 = a * s2 + b * c2;
    const double n10 = c * c2 - d * s2, n11 = c * s2 + d * c2;
    m00 = c1 * n00 - s1 * n10;
    m01 = c1 * n01 - s1 * n11;
    m10 = s1 * n00 + c1 * n10;
    m11 = s1 * n01 + c1 * n11;
}

// Rotation of the pivot (p,q), p < q < k, from a_pp, a_qq, a_pq (skip rule of the oracle:
// |a_pq| <= eps sqrt|a_pp a_qq| or <= 1e-30 ||T||_F is not rotated); also the new diagonal.
// fp64 reciprocal and reciprocal square root: hardware approximation + two Newton steps (~1 ulp).
// Measured on B200 (tools/micro_fp64lat.cu): the IEEE sqrt / div / rsqrt chains cost 99 / 79 / 74
// cycles of dependent latency, the original parameter formula 551 cycles per rotation.
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double h = x * y;
    double e = fma(-h, y, 1.0);
    y = fma(0.5 * y, e, y);
    h = x * y;
    e = fma(-h, y, 1.0);
    return fma(0.5 * y, e, y);
}

// 2^-e for the binary exponent e of x > 0 (x = 0: 1): scaling by it is exact.
__device__ __forceinline__ double pow2_inv(double x) {
    long long e = (__double_as_longlong(x) >> 52) & 0x7ff;  // biased exponent (x >= 0)
    if (e == 0) return 1.0;                                   // zero / subnormal: leave as is
    e = 2046 - e;                                             // 2^(1023 - (e - 1023))
    if (e < 1) e = 1;
    return __longlong_as_double(e << 52);
}

// Rotation of the pivot (p,q), p < q < k, from a_pp, a_qq, a_pq (skip rule of the oracle:
// |a_pq| <= eps sqrt|a_pp a_qq| or <= 1e-30 ||T||_F is not rotated, tested on squares); also
// the new diagonal.  t = sgn(tau) / (|tau| + sqrt(1 + tau^2)) in the division-free form
// t = sgn |b| / (|d| + sqrt(d^2 + b^2)), c = 1/sqrt(1 + t^2), s = t c.
__device__ __forceinline__ void jacobi_param(double app, double aqq, double apq, double fro, double& c, double& s,
                                             double& dp, double& dq, int& act) {
    const double eps = 2.220446049250313e-16;
    c = 1.0;
    s = 0.0;
    dp = app;
    dq = aqq;
    act = 0;
    // The squared quantities are formed from values scaled by a power of two (exact, so the
    // decision and t are those of the unscaled formula) -- no overflow / flush to zero for any
    // finite T, whatever its magnitude.
    const double s3 = pow2_inv(fmax(fmax(fabs(app), fabs(aqq)), fabs(apq)));
    const double app3 = app * s3, aqq3 = aqq * s3, apq3 = apq * s3;
    if (!(apq3 * apq3 <= eps * eps * fabs(app3 * aqq3) || fabs(apq) <= 1e-30 * fro)) {
        double d = aqq - app, b = 2.0 * apq;
        const double s2 = pow2_inv(fmax(fabs(d), fabs(b)));  // t is invariant under d, b -> s2 d, s2 b
        d *= s2;
        b *= s2;
        const double h = fma(d, d, b * b);
        const double den = fma(h, rsqrt_nr(h), fabs(d));  // |d| + sqrt(d^2 + b^2)
        const double t = ((d == 0.0 || ((d > 0.0) == (b > 0.0))) ? 1.0 : -1.0) * fabs(b) * rcp_nr(den);
        c = rsqrt(fma(t, t, 1.0));  // CUDA rsqrt: c^2 + s^2 = 1 to ~1 ulp (orthogonality of V)
        s = t * c;
        double m00, m01, m10, m11;
        block22(app, apq, apq, aqq, c, s, c, s, m00, m01, m10, m11);
        dp = m00;
        dq = m11;
        act = 1;
    }
}

__global__ void __launch_bounds__(EIG1_THREADS) k_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph,
                                                      int k_fixed, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k;
    extern __shared__ double sm[];
    double* V = sm + 2 * QMAX * ELD;  // A_r, A_{r+1} at sm + (r & 1) * QMAX * ELD
    __shared__ double pc[2][MAXPAIRS], ps[2][MAXPAIRS], pdp[2][MAXPAIRS], pdq[2][MAXPAIRS];
    __shared__ int pp[2][MAXPAIRS], pq[2][MAXPAIRS], pact[2][MAXPAIRS];
    __shared__ double red[EIG1_THREADS];
    __shared__ int ord[QMAX];
    __shared__ unsigned char bi[MAXBLK], bj[MAXBLK];
    __shared__ int rot[101];
    __shared__ double fro;
    const int tid = threadIdx.x;
    double f = 0.0;
    // Static schedule table for the parameter warp: for round r and pair m of round r+1,
    // .x = players x < y of that pair and the round-r pairs i, j holding them, .y = the players
    // (p1 < q1) of pair i and (p2 < q2) of pair j -- so the pivot's operands are one table load
    // away instead of a chain of dependent index loads.
    __shared__ uint2 nxtab[QMAX - 1][MAXPAIRS];
    {
        const int kk0 = k + (k & 1), nr0 = kk0 - 1, np0 = kk0 / 2;
        for (int idx = tid; idx < nr0 * np0; idx += EIG1_THREADS) {
            const int r = idx / np0, m = idx % np0, rn = r + 1 == nr0 ? 0 : r + 1;
            int x = rr_player(m, rn, kk0), y = rr_player(kk0 - 1 - m, rn, kk0);
            if (x > y) { const int t = x; x = y; y = t; }
            const int i = pair_of_pos(rr_pos(x, r, kk0), kk0), j = pair_of_pos(rr_pos(y, r, kk0), kk0);
            int p1 = rr_player(i, r, kk0), q1 = rr_player(kk0 - 1 - i, r, kk0);
            int p2 = rr_player(j, r, kk0), q2 = rr_player(kk0 - 1 - j, r, kk0);
            if (p1 > q1) { const int t = p1; p1 = q1; q1 = t; }
            if (p2 > q2) { const int t = p2; p2 = q2; q2 = t; }
            nxtab[r][m] = make_uint2((unsigned)x | (unsigned)y << 8 | (unsigned)i << 16 | (unsigned)j << 24,
                                     (unsigned)p1 | (unsigned)q1 << 8 | (unsigned)p2 << 16 | (unsigned)q2 << 24);
        }
    }
    for (int idx = tid; idx < k * k; idx += EIG1_THREADS) {
        const int i = idx % k, j = idx / k;
        const double a = 0.5 * (T[i + (int64_t)j * ldT] + T[j + (int64_t)i * ldT]);  // sym(T)
        sm[i + j * ELD] = a;
        V[i + j * ELD] = (i == j) ? 1.0 : 0.0;
        f += a * a;
    }
    const int kk = k + (k & 1);
    const int npairs = kk / 2;
    const int nblk = npairs * (npairs + 1) / 2;
    const int nr = kk - 1;  // rounds per sweep
    if (tid == 0) {
        int b = 0;
        for (int i = 0; i < npairs; ++i)
            for (int j = i; j < npairs; ++j) {
                bi[b] = (unsigned char)i;
                bj[b] = (unsigned char)j;
                ++b;
            }
    }
    for (int i = tid; i < 101; i += EIG1_THREADS) rot[i] = 0;
    red[tid] = f;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < EIG1_THREADS; ++i) s += red[i];
        fro = sqrt(s);
    }
    __syncthreads();
    const int maxsweep = 100;
    if (k > 1 && tid < npairs) {  // parameters of round 0 of sweep 0
        int p = rr_player(tid, 0, kk), q = rr_player(kk - 1 - tid, 0, kk);
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0, dp = sm[p + p * ELD], dq = 0.0;
        int act = 0;
        if (q < k) jacobi_param(sm[p + p * ELD], sm[q + q * ELD], sm[p + q * ELD], fro, c, s, dp, dq, act);
        pc[0][tid] = c; ps[0][tid] = s; pdp[0][tid] = dp; pdq[0][tid] = dq;
        pp[0][tid] = p; pq[0][tid] = q; pact[0][tid] = act;
        if (act) rot[0] = 1;
    }
    __syncthreads();
    int sweep = 0, r = 0, cur = 0;
    const int warp = tid >> 5;
#ifdef EIG_TRACE
    long long tr0 = clock64();
#endif
    while (k > 1) {
#ifdef EIG_TRACE
        tr0 = clock64();
#endif
        const int nxt = cur ^ 1;
        const int rn = r + 1 == nr ? 0 : r + 1;
        const int sn = r + 1 == nr ? sweep + 1 : sweep;
        const double* __restrict__ Ac = sm + cur * (QMAX * ELD);
        double* __restrict__ An = sm + nxt * (QMAX * ELD);
        if (warp == 0) {
            // rotation parameters of round r+1 (pair m = lane)
            const int m = tid;
            if (m < npairs && sn < maxsweep) {
                const uint2 tb = nxtab[r][m];
                const int x = tb.x & 255, y = (tb.x >> 8) & 255, i = (tb.x >> 16) & 255, j = tb.x >> 24;
                const int p1 = tb.y & 255, q1 = (tb.y >> 8) & 255, p2 = (tb.y >> 16) & 255, q2 = tb.y >> 24;
                double c = 1.0, s = 0.0, dx, dy = 0.0;
                int act = 0;
                const bool xp = p1 == x;
                dx = xp ? pdp[cur][i] : pdq[cur][i];
                if (y < k) {
                    const bool yp = p2 == y;
                    dy = yp ? pdp[cur][j] : pdq[cur][j];
                    double axy;
                    if (i == j) {
                        axy = pact[cur][i] ? 0.0 : Ac[x + y * ELD];
                    } else {
                        const bool q1ok = q1 < k, q2ok = q2 < k;
                        const double a = Ac[p1 + p2 * ELD];
                        const double bb = q2ok ? Ac[p1 + q2 * ELD] : 0.0;
                        const double cc = q1ok ? Ac[q1 + p2 * ELD] : 0.0;
                        const double dd = (q1ok && q2ok) ? Ac[q1 + q2 * ELD] : 0.0;
                        double m00, m01, m10, m11;
                        block22(a, bb, cc, dd, pc[cur][i], ps[cur][i], pc[cur][j], ps[cur][j], m00, m01, m10, m11);
                        axy = xp ? (yp ? m00 : m01) : (yp ? m10 : m11);
                    }
#ifdef EIG_TRACE
                    long long tb = clock64();
                    if (m == 0) atomicAdd(&eig_trace[16], (unsigned long long)(tb - tr0));
#endif
                    jacobi_param(dx, dy, axy, fro, c, s, dx, dy, act);
#ifdef EIG_TRACE
                    if (m == 0) atomicAdd(&eig_trace[17], (unsigned long long)(clock64() - tb));
#endif
                }
                pc[nxt][m] = c; ps[nxt][m] = s; pdp[nxt][m] = dx; pdq[nxt][m] = dy;
                pp[nxt][m] = x; pq[nxt][m] = y; pact[nxt][m] = act;
                if (act) rot[sn] = 1;
            }
        } else {
            int rank = 0;
            const int role = eig_role(warp, rank);
            if (role == 1) {
                // 2x2 block updates of round r: A_r -> A_{r+1} (A_r and A_{r+1} are distinct
                // buffers, so the loads of later blocks are not ordered after earlier stores)
                const int t2 = rank * 32 + (tid & 31);
                for (int b = t2; b < nblk; b += 32 * BLK_WARPS) {
                    const int i = bi[b], j = bj[b];
                    const int p1 = pp[cur][i], q1 = pq[cur][i], p2 = pp[cur][j], q2 = pq[cur][j];
                    const bool q1ok = q1 < k, q2ok = q2 < k;
                    const double a = Ac[p1 + p2 * ELD];
                    const double bb = q2ok ? Ac[p1 + q2 * ELD] : 0.0;
                    const double cc = q1ok ? Ac[q1 + p2 * ELD] : 0.0;
                    const double dd = (q1ok && q2ok) ? Ac[q1 + q2 * ELD] : 0.0;
                    const int ai = pact[cur][i], aj = pact[cur][j];
                    double m00 = a, m01 = bb, m10 = cc, m11 = dd;
                    if (i == j) {
                        if (ai) {
                            m00 = pdp[cur][i];
                            m11 = pdq[cur][i];
                            m01 = m10 = 0.0;
                        }
                    } else if (ai || aj) {
                        block22(a, bb, cc, dd, pc[cur][i], ps[cur][i], pc[cur][j], ps[cur][j], m00, m01, m10, m11);
                    }
                    An[p1 + p2 * ELD] = m00;
                    An[p2 + p1 * ELD] = m00;
                    if (q2ok) {
                        An[p1 + q2 * ELD] = m01;
                        An[q2 + p1 * ELD] = m01;
                    }
                    if (q1ok) {
                        An[q1 + p2 * ELD] = m10;
                        An[p2 + q1 * ELD] = m10;
                    }
                    if (q1ok && q2ok) {
                        An[q1 + q2 * ELD] = m11;
                        An[q2 + q1 * ELD] = m11;
                    }
                }
            } else if (role == 2) {
                // V <- V J for the pairs of round r: tasks (pair, row) packed densely over the
                // V warps (consecutive lanes = consecutive rows of one pair: conflict-free)
                const int tv = rank * 32 + (tid & 31);
                constexpr int NVT = 32 * 6;
                const int ntask = npairs * k;
                const float inv_k = 1.0f / (float)k;
                for (int e = tv; e < ntask; e += NVT) {
                    const int pi = __float2int_rz(((float)e + 0.5f) * inv_k);
                    if (!pact[cur][pi]) continue;
                    const int row = e - pi * k;
                    const int ip = row + pp[cur][pi] * ELD, iq = row + pq[cur][pi] * ELD;
                    const double c = pc[cur][pi], sn_ = ps[cur][pi];
                    const double vp = V[ip], vq = V[iq];
                    V[ip] = c * vp - sn_ * vq;
                    V[iq] = sn_ * vp + c * vq;
                }
            }
        }
#ifdef EIG_TRACE
        if ((tid & 31) == 0) atomicAdd(&eig_trace[warp], (unsigned long long)(clock64() - tr0));
#endif
        __syncthreads();
#ifdef EIG_TRACE
        if (tid == 0) atomicAdd(&eig_trace[31], (unsigned long long)(clock64() - tr0));
        if (tid == 0) atomicAdd(&eig_trace[30], 1ull);
#endif
        cur = nxt;
        if (r + 1 == nr) {  // end of a sweep: stop after a sweep without rotations
            if (!rot[sweep] || sn >= maxsweep) break;
            // ... or when no pivot passes the skip rule any more: the next sweep would rotate
            // nothing (no entry changes without a rotation), so stopping here gives the same A, V
            const double* __restrict__ Ar = sm + cur * (QMAX * ELD);
            const double eps2 = 2.220446049250313e-16 * 2.220446049250313e-16;
            int live = 0;
            for (int idx = tid; idx < k * k; idx += EIG1_THREADS) {
                const int pr = idx % k, qr = idx / k;
                if (pr < qr) {
                    // the skip rule of jacobi_param, on values scaled by a power of two (exact: no
                    // overflow / flush of the squares for any finite T)
                    const double apq = Ar[pr + qr * ELD], app = Ar[pr + pr * ELD], aqq = Ar[qr + qr * ELD];
                    const double s3 = pow2_inv(fmax(fmax(fabs(app), fabs(aqq)), fabs(apq)));
                    const double apq3 = apq * s3;
                    if (!(apq3 * apq3 <= eps2 * fabs((app * s3) * (aqq * s3)) || fabs(apq) <= 1e-30 * fro))
                        live = 1;
                }
            }
            if (!__syncthreads_or(live)) {
                ++sweep;  // report the sweep the test replaced
                break;
            }
        }
        r = rn;
        sweep = sn;
    }
    const double* __restrict__ A = sm + cur * (QMAX * ELD);
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
        for (int idx = tid; idx < QMAX * QMAX; idx += EIG1_THREADS) {
            const int i = idx % QMAX, j = idx / QMAX;
            T[i + (int64_t)j * ldT] = (i == j && i < ph) ? ctl->theta[i] : 0.0;
        }
    }
    if (tid == 0) {
        ctl->k_rr = k;
        ctl->eig_sweeps = sweep + 1;
    }
}

// TRPLK_EIG=tri selects the tridiagonal eigensolver (eig_tri.cu) for the p^ wanted pairs.
void launch_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph, int k_fixed, unsigned gate,
                cudaStream_t s) {
    static int init = 0;
    const int smem1 = 3 * QMAX * ELD * (int)sizeof(double);
    if (!init) {
        cudaFuncSetAttribute(k_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
        init = 1;
    }
    static const int tri = [] {
        const char* e = getenv("TRPLK_EIG");
        return e && !strcmp(e, "tri") ? 1 : 0;
    }();
    if (tri) launch_eig_tri(ctl, T, ldT, Y, ldY, ph, k_fixed, ph, gate, s);  // ph > 0: only p^ pairs needed
    else k_eig<<<1, EIG1_THREADS, smem1, s>>>(ctl, T, ldT, Y, ldY, ph, k_fixed, gate);
}

}  // namespace trplk
