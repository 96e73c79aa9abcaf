// Device kernels of the TRPL+K hot path, hand-written for sm_100a (B200).
//
//   k_sdots   K1/K7/K4: SELL-32 SpMV with A (and B) fused with the Jacobi preconditioner
//             (or the residual) and with the dot products of a basis block against the
//             result -- eq 3.1, R1, Alg.1 steps 12-15.
//   k_upd     K2/K3: classical Gram-Schmidt update y = x - U h fused with the next pass's
//             dots, or with the final normalisation (reading R3).
//   k_eig     K6: one-CTA parallel-ordered cyclic Jacobi of T (Alg.1 step 11).
//   k_rotate  K5: X = U Y on fp64 DMMA tensor cores (mma.sync m8n8k4 f64).
//
// Every reduction is deterministic: fixed per-warp butterfly shuffles, a fixed-order CTA
// sum, per-CTA partials and a fixed-order final sum by the last CTA to finish.
#include <cstdio>

#include "trplk_internal.cuh"

namespace trplk {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double shx(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += shx(v, o);
    return v;
}

// Reduce NV = 2^LOG values across the warp with one shuffle per value per halving step.
// Afterwards lane l holds in v[0] the warp sum of value index (l >> (5-LOG)) & (NV-1).
template <int LOG>
__device__ __forceinline__ void warp_butterfly(double (&v)[1 << LOG], int lane) {
#pragma unroll
    for (int s = 0; s < LOG; ++s) {
        const int off = 16 >> s;
        const int half = (1 << LOG) >> (s + 1);
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const double send = upper ? v[j] : v[j + half];
            const double keep = upper ? v[j + half] : v[j];
            v[j] = keep + shx(send, off);
        }
    }
#pragma unroll
    for (int off = (16 >> LOG); off >= 1; off >>= 1) v[0] += shx(v[0], off);
}

// SELL-32 row of lane `lane` in slice s: returns sum_j val*x[col], diag = slot-0 value.
__device__ __forceinline__ double sell_row(const Sell& M, int64_t s, int lane, const double* __restrict__ x,
                                           double& diag) {
    const int64_t b = __ldg(M.sptr + s), e = __ldg(M.sptr + s + 1);
    const int w = (int)((e - b) >> 5);
    const double* vp = M.val + b + lane;
    const int* cp = M.col + b + lane;
    double acc = 0.0;
    diag = __ldg(vp);
    int j = 0;
    for (; j + 4 <= w; j += 4) {
        const double v0 = __ldg(vp + 32 * j), v1 = __ldg(vp + 32 * (j + 1));
        const double v2 = __ldg(vp + 32 * (j + 2)), v3 = __ldg(vp + 32 * (j + 3));
        const int c0 = __ldg(cp + 32 * j), c1 = __ldg(cp + 32 * (j + 1));
        const int c2 = __ldg(cp + 32 * (j + 2)), c3 = __ldg(cp + 32 * (j + 3));
        const double x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2), x3 = __ldg(x + c3);
        acc = fma(v0, x0, acc);
        acc = fma(v1, x1, acc);
        acc = fma(v2, x2, acc);
        acc = fma(v3, x3, acc);
    }
    for (; j < w; ++j) acc = fma(__ldg(vp + 32 * j), __ldg(x + __ldg(cp + 32 * j)), acc);
    return acc;
}

// Last-CTA-done pattern.  Returns true in exactly one CTA, after all CTAs wrote their partials.
__device__ __forceinline__ bool last_cta(unsigned* counter) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(counter, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

// Fixed-order sum of the per-CTA partials part[v*maxcta + c], c < ncta, into out[v] (smem).
__device__ void reduce_partials(const double* part, int maxcta, int ncta, int nv, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int v = warp; v < nv; v += WARPS) {
        double s = 0.0;
        for (int c = lane; c < ncta; c += 32) s += __ldcg(part + (int64_t)v * maxcta + c);
        s = warp_sum(s);
        if (lane == 0) out[v] = s;
    }
    __syncthreads();
}

// ------------------------------------------------------------ K1: fused SpMV + dots
__device__ void sdots_finalize(const SdotsArgs& a, const double* r, int k1, int k2) {
    Ctl* ctl = a.ctl;
    if (a.dest1 == D_TCOL) {
        const int col = a.tcol_fixed >= 0 ? a.tcol_fixed : ctl->k - 1;
        for (int i = threadIdx.x; i < k1; i += blockDim.x) {
            a.T[i + (int64_t)col * a.ldT] = r[i];
            if (a.tcol_fixed < 0) a.T[col + (int64_t)i * a.ldT] = r[i];
        }
    } else if (a.dest1 >= D_H0) {
        for (int i = threadIdx.x; i < k1; i += blockDim.x) ctl->h[a.dest1 - D_H0][i] = r[i];
    }
    if (a.dest2 >= D_H0)
        for (int i = threadIdx.x; i < k2; i += blockDim.x) ctl->h[a.dest2 - D_H0][i] = r[k1 + i];
    if (threadIdx.x == 0) {
        int o = k1 + k2;
        if (a.norm1) ctl->nrm[a.nslot1] = r[o++];
        if (a.norm2) ctl->nrm[a.nslot2] = r[o];
    }
}

__device__ __forceinline__ const double* resolve_x(const double* x, int dyn, int64_t ld, int off, const Ctl* ctl) {
    if (dyn == 1) return x + ld * (int64_t)(ctl->t - 1 + off);
    if (dyn == 2) return x + ld * (int64_t)(ctl->xprev_col + off);
    return x;
}

__device__ __forceinline__ void sdots_counts(const SdotsArgs& a, const Ctl* ctl, bool two, int& k1, int& k2) {
    const int kc = ctl->k;
    k1 = a.set1 ? (a.k_from_ctl ? kc : a.k1) : 0;
    k2 = (two && a.set2) ? (a.k_from_ctl ? kc : a.k2) : 0;
}

template <int RPT, bool TWO>
__global__ void __launch_bounds__(CTA) k_sdots(const SdotsArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    int k1, k2;
    sdots_counts(a, ctl, TWO, k1, k2);
    double theta = 0.0;
    if (a.out_mode >= 3)
        theta = a.theta_idx >= 0 ? ctl->theta[a.theta_idx]
                                 : (a.theta_idx == -1 ? ctl->theta[ctl->t - 1] : a.theta_val);
    const double rho = ctl->rho;
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const int kmx = k1 > k2 ? k1 : k2;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);

    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    for (int i = threadIdx.x; i < WARPS * NV_MAX; i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nslices = (a.nrows + 31) >> 5;
    const int64_t ntiles = (nslices + RPT - 1) / RPT;
    for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles; tile += (int64_t)gridDim.x * WARPS) {
        double xv[RPT], zv[RPT], ov[RPT];
        int64_t row[RPT];
        bool ok[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int64_t s = tile * RPT + i;
            row[i] = s * 32 + lane;
            ok[i] = (s < nslices) && (row[i] < a.nrows);
            xv[i] = zv[i] = ov[i] = 0.0;
            if (s < nslices) {
                double ad = 1.0, bd = 1.0, z = 0.0, sv = 0.0;
                const double xr = ok[i] ? X[row[i]] : 0.0;
                if (a.out_mode == 4) {
                    ad = __ldg(a.A.val + __ldg(a.A.sptr + s) + lane);
                } else if (a.A.nrows) {
                    z = sell_row(a.A, s, lane, X, ad);
                } else {
                    z = xr;
                }
                if (a.out_mode >= 2) {
                    if (a.B.nrows) sv = sell_row(a.B, s, lane, X, bd);
                    else sv = xr;
                }
                double o = 0.0, minv = 1.0;
                if (a.out_mode >= 2) {
                    double d = fabs(ad - a.sigma * bd);
                    d = d > a.mfloor ? d : a.mfloor;
                    minv = 1.0 / d;  // M_ii
                }
                switch (a.out_mode) {
                    case 1: o = z; break;
                    case 2: o = minv * (z - rho * sv); break;  // w = M (z - rho B g), R1
                    case 3: o = z - theta * sv; break;         // r = A x - theta B x
                    case 4: o = (ok[i] ? a.wext[row[i]] : 0.0) - theta * sv; break;
                    default: break;
                }
                if (ok[i]) {
                    if (a.out) a.out[row[i]] = o;
                    if (a.uout) a.uout[row[i]] = minv * o;
                    xv[i] = xr;
                    zv[i] = z;
                    ov[i] = o;
                }
            }
        }
        if (kmx > 0) {
            double v1[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) v1[i] = a.set1 == 1 ? zv[i] : (a.set1 == 2 ? ov[i] : xv[i]);
            for (int c0 = 0; c0 < kmx; c0 += 8) {
                double v[TWO ? 16 : 8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const int c = c0 + cc;
                    double s1 = 0.0, s2 = 0.0;
                    if (c < kmx) {
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            if (ok[i]) {
                                const double u = a.U[(int64_t)c * a.ldu + row[i]];
                                s1 = fma(u, v1[i], s1);
                                if (TWO) s2 = fma(u, ov[i], s2);
                            }
                        }
                    }
                    v[cc] = s1;
                    if constexpr (TWO) v[8 + cc] = s2;
                }
                if constexpr (TWO) {
                    warp_butterfly<4>(v, lane);
                    const int idx = (lane >> 1) & 15;
                    if ((lane & 1) == 0) {
                        const int col = c0 + (idx & 7);
                        if (idx < 8) {
                            if (col < k1) acc[warp][col] += v[0];
                        } else {
                            if (col < k2) acc[warp][k1 + col] += v[0];
                        }
                    }
                } else {
                    warp_butterfly<3>(v, lane);
                    const int idx = (lane >> 2) & 7;
                    if ((lane & 3) == 0 && c0 + idx < k1) acc[warp][c0 + idx] += v[0];
                }
            }
        }
        if (nn) {
            double n1 = 0.0, n2 = 0.0;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const double o = ov[i], x = xv[i], z = zv[i];
                const double p1 = a.norm1 == 1 ? o * o : a.norm1 == 2 ? x * z : a.norm1 == 3 ? x * x : z * z;
                const double p2 = a.norm2 == 1 ? o * o : a.norm2 == 2 ? x * z : a.norm2 == 3 ? x * x : z * z;
                n1 += p1;
                n2 += p2;
            }
            n1 = warp_sum(n1);
            n2 = warp_sum(n2);
            if (lane == 0) {
                int o = k1 + k2;
                if (a.norm1) acc[warp][o++] += n1;
                if (a.norm2) acc[warp][o] += n2;
            }
        }
    }
    if (nv == 0) return;
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += CTA) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s += acc[w][v];
        a.part[(int64_t)v * a.maxcta + blockIdx.x] = s;
    }
    if (!last_cta(a.counter)) return;
    reduce_partials(a.part, a.maxcta, gridDim.x, nv, res);
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
    } else {
        sdots_finalize(a, res, k1, k2);
    }
    if (threadIdx.x == 0) *a.counter = 0u;
}

// --------------------------------------------------- K2/K3: CGS update (+dots / +norm)
__device__ void upd_finalize(const UpdArgs& a, const double* r, int kv) {
    Ctl* ctl = a.ctl;
    for (int i = threadIdx.x; i < kv; i += blockDim.x) ctl->h[a.hout][i] = r[i];
    if (threadIdx.x == 0) ctl->nrm[a.mode == 1 ? N_1SQ : N_2SQ_EXP] = r[kv];
}

template <int KMAX>
__global__ void __launch_bounds__(CTA) k_upd(const UpdArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.mode == 3 && ctl->pass3 == 0) return;
    const int kv = a.kv >= 0 ? a.kv : ctl->k;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    __shared__ double hs[KMAX > 0 ? KMAX : 1];
    __shared__ double acc[WARPS][QMAX + 1];
    __shared__ double res[QMAX + 1];
    for (int i = threadIdx.x; i < KMAX; i += CTA) hs[i] = i < kv ? ctl->h[a.hslot][i] : 0.0;
    __syncthreads();

    // Decisions of FINAL / FIX, computed identically in every CTA from global values (R3).
    bool pass3 = false, brk = false;
    double binv = 0.0;
    if (a.mode >= 2) {
        double hn = 0.0;
        for (int i = 0; i < kv; ++i) hn += hs[i] * hs[i];
        const double nin = sqrt(ctl->nrm[N_IN2]);
        double b;
        if (a.mode == 2) {
            const double n1sq = ctl->nrm[N_1SQ];
            const double n2sq = n1sq - hn;    // ||w''||^2 = ||w'||^2 - ||h2||^2 (U B-orthonormal)
            pass3 = !(n2sq >= 0.5 * n1sq);    // second pass dropped the norm by > 1/sqrt2
            b = sqrt(n2sq > 0.0 ? n2sq : 0.0);
        } else {
            const double n3sq = ctl->nrm[N_2SQ_EXP] - hn;
            b = sqrt(n3sq > 0.0 ? n3sq : 0.0);
        }
        if (!pass3) {
            brk = !(b >= 1e-14 * nin) || nin == 0.0;
            binv = 1.0 / b;
        }
    }
    const bool write_y = a.mode <= 1 || (a.mode == 2 && pass3);
    const bool do_dots = a.dots && (a.mode == 1 || (a.mode == 2 && pass3));
    const bool write_dest = (a.mode >= 2) && !pass3 && !brk;
    double* dest = a.dest;
    if (write_dest && a.dest_dyn) dest = a.dest + a.dest_ld * (int64_t)ctl->k;

    if (do_dots)
        for (int i = threadIdx.x; i < WARPS * (QMAX + 1); i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (a.nrows + 31) >> 5;
    if (write_y || write_dest) {
        for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles;
             tile += (int64_t)gridDim.x * WARPS) {
            const int64_t row = tile * 32 + lane;
            const bool ok = row < a.nrows;
            double ur[KMAX];
#pragma unroll
            for (int c = 0; c < KMAX; ++c) ur[c] = (ok && c < kv) ? a.U[(int64_t)c * a.ldu + row] : 0.0;
            double y = ok ? X[row] : 0.0;
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < kv) y = fma(-hs[c], ur[c], y);  // y = x - U h, columns in order
            if (ok) {
                if (write_y && a.out) a.out[row] = y;
                if (write_dest) {
                    const double g = y * binv;
                    dest[row] = g;
                    if (a.dest2) a.dest2[row] = g;
                }
            }
            if (do_dots) {
#pragma unroll
                for (int c0 = 0; c0 < KMAX; c0 += 16) {
                    if (c0 < kv) {
                        double v[16];
#pragma unroll
                        for (int cc = 0; cc < 16; ++cc) v[cc] = (c0 + cc < KMAX) ? ur[(c0 + cc) % KMAX] * y : 0.0;
                        warp_butterfly<4>(v, lane);
                        const int idx = (lane >> 1) & 15;
                        if ((lane & 1) == 0 && c0 + idx < kv) acc[warp][c0 + idx] += v[0];
                    }
                }
                const double yy = warp_sum(y * y);
                if (lane == 0) acc[warp][kv] += yy;
            }
        }
    }
    if (a.mode == 0) return;
    const int nv = do_dots ? kv + 1 : 0;
    if (nv) {
        __syncthreads();
        for (int v = threadIdx.x; v < nv; v += CTA) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) s += acc[w][v];
            a.part[(int64_t)v * a.maxcta + blockIdx.x] = s;
        }
    }
    if (!last_cta(a.counter)) return;
    if (nv) {
        reduce_partials(a.part, a.maxcta, gridDim.x, nv, res);
        if (a.red_local) {
            for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
        } else {
            upd_finalize(a, res, kv);
        }
    }
    if (threadIdx.x == 0) {
        if (a.mode == 2) {
            if (pass3) {
                ctl->pass3 = 1;
                ctl->pass3_count += 1;
            } else if (brk) {
                ctl->flags &= ~a.clear_on_brk;
                ctl->brk += 1;
            } else if (a.inc_k) {
                ctl->k += 1;
            }
        } else if (a.mode == 3) {
            ctl->pass3 = 0;
            if (brk) {
                ctl->flags &= ~a.clear_on_brk;
                ctl->brk += 1;
            } else if (a.inc_k) {
                ctl->k += 1;
            }
        }
        *a.counter = 0u;
    }
}

// ------------------------------------------------ multi-rank: sum gathered partials
__global__ void k_finalize_multi(const SdotsArgs sd, const UpdArgs up, int which, const double* red_all,
                                 int nranks, int stride) {
    __shared__ double res[NV_MAX];
    Ctl* ctl = which == 0 ? sd.ctl : up.ctl;
    int k1 = 0, k2 = 0, nv = 0;
    if (which == 0) {
        if ((ctl->flags & sd.gate) != sd.gate) return;
        if (sd.gate_pass3 && ctl->pass3 == 0) return;
        sdots_counts(sd, ctl, true, k1, k2);
        nv = k1 + k2 + (sd.norm1 ? 1 : 0) + (sd.norm2 ? 1 : 0);
    } else {
        if ((ctl->flags & up.gate) != up.gate) return;
        if (up.mode == 2 && ctl->pass3 == 0) return;  // FINAL without pass 3: no dots
        k1 = up.kv >= 0 ? up.kv : ctl->k;
        nv = k1 + 1;
    }
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s += red_all[(int64_t)r * stride + v];
        res[v] = s;
    }
    __syncthreads();
    if (which == 0) sdots_finalize(sd, res, k1, k2);
    else upd_finalize(up, res, k1);
}

// ------------------------------------------------------- K6: one-CTA cyclic Jacobi
constexpr int LDA = QMAX + 1;

__device__ __forceinline__ int rr_player(int pos, int r, int kk) {
    return pos == 0 ? 0 : 1 + (pos - 1 + r) % (kk - 1);
}

__global__ void __launch_bounds__(256) k_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph,
                                             int k_fixed, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k;
    extern __shared__ double sm[];
    double* A = sm;
    double* V = sm + QMAX * LDA;
    __shared__ double cs[QMAX / 2], sn[QMAX / 2], red[256];
    __shared__ int pp[QMAX / 2], qq[QMAX / 2], ord[QMAX];
    __shared__ int rotated;
    __shared__ double fro;
    const int tid = threadIdx.x;
    double f = 0.0;
    for (int idx = tid; idx < k * k; idx += blockDim.x) {
        const int i = idx % k, j = idx / k;
        const double a = 0.5 * (T[i + (int64_t)j * ldT] + T[j + (int64_t)i * ldT]);  // sym(T)
        A[i + j * LDA] = a;
        V[i + j * LDA] = (i == j) ? 1.0 : 0.0;
        f += a * a;
    }
    red[tid] = f;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) s += red[i];
        fro = sqrt(s);
    }
    __syncthreads();
    const double eps = 2.220446049250313e-16;
    const int kk = k + (k & 1);
    const int npairs = kk / 2;
    for (int sweep = 0; sweep < 100 && k > 1; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int r = 0; r < kk - 1; ++r) {
            if (tid < npairs) {
                int p = rr_player(tid, r, kk), q = rr_player(kk - 1 - tid, r, kk);
                if (p > q) { const int tmp = p; p = q; q = tmp; }
                pp[tid] = -1;
                if (q < k) {
                    const double apq = A[p + q * LDA], app = A[p + p * LDA], aqq = A[q + q * LDA];
                    if (!(fabs(apq) <= eps * sqrt(fabs(app * aqq)) || fabs(apq) <= 1e-30 * fro)) {
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        const double c = 1.0 / sqrt(1.0 + t * t);
                        cs[tid] = c;
                        sn[tid] = t * c;
                        pp[tid] = p;
                        qq[tid] = q;
                        rotated = 1;
                    }
                }
            }
            __syncthreads();
            // A <- A J and V <- V J (columns p, q of every rotated pair)
            for (int idx = tid; idx < npairs * k; idx += blockDim.x) {
                const int pi = idx / k, i = idx % k;
                const int p = pp[pi];
                if (p < 0) continue;
                const int q = qq[pi];
                const double c = cs[pi], s = sn[pi];
                const double aip = A[i + p * LDA], aiq = A[i + q * LDA];
                A[i + p * LDA] = c * aip - s * aiq;
                A[i + q * LDA] = s * aip + c * aiq;
                const double vip = V[i + p * LDA], viq = V[i + q * LDA];
                V[i + p * LDA] = c * vip - s * viq;
                V[i + q * LDA] = s * vip + c * viq;
            }
            __syncthreads();
            // A <- J^T A (rows p, q); the rotated entries (p,q), (q,p) are set to exactly 0
            for (int idx = tid; idx < npairs * k; idx += blockDim.x) {
                const int pi = idx / k, j = idx % k;
                const int p = pp[pi];
                if (p < 0) continue;
                const int q = qq[pi];
                const double c = cs[pi], s = sn[pi];
                const double apj = A[p + j * LDA], aqj = A[q + j * LDA];
                A[p + j * LDA] = (j == q) ? 0.0 : c * apj - s * aqj;
                A[q + j * LDA] = (j == p) ? 0.0 : s * apj + c * aqj;
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    // ascending order, stable on ties (R11)
    if (tid < k) {
        const double ti = A[tid + tid * LDA];
        int rank = 0;
        for (int j = 0; j < k; ++j) {
            const double tj = A[j + j * LDA];
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
            const double a = fabs(V[i + src * LDA]);
            if (a > vmax) { vmax = a; imax = i; }
        }
        const double sg = V[imax + src * LDA] < 0.0 ? -1.0 : 1.0;  // sign rule (R11)
        for (int i = 0; i < k; ++i) Y[i + (int64_t)tid * ldY] = sg * V[i + src * LDA];
        ctl->theta[tid] = A[src + src * LDA];
    }
    __syncthreads();
    // restart: T <- diag(Theta(1:p^)) (R10)
    if (ph > 0) {
        for (int idx = tid; idx < QMAX * QMAX; idx += blockDim.x) {
            const int i = idx % QMAX, j = idx / QMAX;
            T[i + (int64_t)j * ldT] = (i == j && i < ph) ? ctl->theta[i] : 0.0;
        }
    }
    if (tid == 0) ctl->k_rr = k;
}

// ------------------------------------------------------- K5: DMMA rotation X = U Y
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(256) k_rotate(const double* __restrict__ U, int64_t ldu, int64_t nrows,
                                                const Ctl* ctl, int k_fixed, const double* __restrict__ Y,
                                                int ldY, int ncol, double* __restrict__ X, int64_t ldx,
                                                unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k_rr;
    const int ksteps = (k + 3) >> 2;
    __shared__ double Ys[QMAX][8 * NT + 1];
    for (int idx = threadIdx.x; idx < QMAX * 8 * NT; idx += blockDim.x) {
        const int kk = idx / (8 * NT), j = idx % (8 * NT);
        Ys[kk][j] = (kk < k && j < ncol) ? Y[kk + (int64_t)j * ldY] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t ntile = (nrows + 7) >> 3;
    const int ar = lane >> 2, ac = lane & 3;
    for (int64_t tile = gw; tile < ntile; tile += nw) {
        const int64_t r = tile * 8 + ar;
        const bool ok = r < nrows;
        double acc[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        int ks = 0;
        for (; ks + 4 <= ksteps; ks += 4) {
            double av[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int kk = 4 * (ks + u) + ac;
                av[u] = (ok && kk < k) ? U[(int64_t)kk * ldu + r] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt], av[u], Ys[4 * (ks + u) + ac][8 * nt + ar]);
        }
        for (; ks < ksteps; ++ks) {
            const int kk = 4 * ks + ac;
            const double av = (ok && kk < k) ? U[(int64_t)kk * ldu + r] : 0.0;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt], av, Ys[4 * ks + ac][8 * nt + ar]);
        }
        if (ok) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * nt + 2 * ac + e;
                    if (col < ncol) X[(int64_t)col * ldx + r] = acc[nt][e];
                }
        }
    }
}

// ---------------------------------------------------------------- small kernels
__device__ __forceinline__ double u01(uint64_t seed, uint64_t stream, uint64_t index) {
    // counter-based U[0,1): splitmix64 finaliser over (seed, stream, index), reading R13
    uint64_t key = (seed * 0xD1B54A32D192ED03ULL) ^ (stream * 0xABC98388FB8FAC03ULL);
    uint64_t z = key + (index + 1ULL) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_random(double* x, int64_t nrows, int64_t row0, int64_t n_global, uint64_t seed,
                         uint64_t stream, uint64_t col) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = u01(seed, stream, col * (uint64_t)n_global + (uint64_t)(row0 + i));
}

__global__ void k_copy_cols(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t nrows, int ncols) {
    const int c = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
        dst[(int64_t)c * ldd + i] = src[(int64_t)c * lds + i];
}

__global__ void k_gather(const double* x, const int* idx, int64_t n, double* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = x[idx[i]];
}

// ---------------------------------------------------------------- launchers
static int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

constexpr int SD_RPT = 2;

int sdots_grid(int64_t nrows) {
    const int64_t nslices = (nrows + 31) / 32;
    const int64_t warps_needed = (nslices + SD_RPT - 1) / SD_RPT;
    int64_t g = (warps_needed + WARPS - 1) / WARPS;
    const int64_t cap = (int64_t)num_sms() * 4;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

int kmax_bucket(int k) {
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 24) return 24;
    if (k <= 32) return 32;
    if (k <= 40) return 40;
    if (k <= 48) return 48;
    return 64;
}

int upd_grid(int64_t nrows, int kmax) {
    const int64_t tiles = (nrows + 31) / 32;
    int64_t g = (tiles + WARPS - 1) / WARPS;
    const int per_sm = kmax <= 16 ? 6 : kmax <= 32 ? 4 : kmax <= 48 ? 3 : 2;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

void launch_sdots(const SdotsArgs& a, int grid, cudaStream_t s) {
    if (a.set2) k_sdots<SD_RPT, true><<<grid, CTA, 0, s>>>(a);
    else k_sdots<SD_RPT, false><<<grid, CTA, 0, s>>>(a);
}

void launch_upd(const UpdArgs& a, int kmax, int grid, cudaStream_t s) {
    switch (kmax) {
        case 8: k_upd<8><<<grid, CTA, 0, s>>>(a); break;
        case 16: k_upd<16><<<grid, CTA, 0, s>>>(a); break;
        case 24: k_upd<24><<<grid, CTA, 0, s>>>(a); break;
        case 32: k_upd<32><<<grid, CTA, 0, s>>>(a); break;
        case 40: k_upd<40><<<grid, CTA, 0, s>>>(a); break;
        case 48: k_upd<48><<<grid, CTA, 0, s>>>(a); break;
        default: k_upd<64><<<grid, CTA, 0, s>>>(a); break;
    }
}

void launch_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph, int k_fixed, unsigned gate,
                cudaStream_t s) {
    static bool init = false;
    const int smem = 2 * QMAX * LDA * (int)sizeof(double);
    if (!init) {
        cudaFuncSetAttribute(k_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        init = true;
    }
    k_eig<<<1, 256, smem, s>>>(ctl, T, ldT, Y, ldY, ph, k_fixed, gate);
}

void launch_rotate(const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed, const double* Y,
                   int ldY, int ncol, double* X, int64_t ldx, unsigned gate, cudaStream_t s) {
    const int64_t tiles = (nrows + 7) / 8;
    int64_t g = (tiles + 7) / 8;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    if (ncol <= 8) k_rotate<1><<<(int)g, 256, 0, s>>>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate);
    else if (ncol <= 16) k_rotate<2><<<(int)g, 256, 0, s>>>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate);
    else k_rotate<3><<<(int)g, 256, 0, s>>>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate);
}

void launch_random(double* x, int64_t nrows, int64_t row0, int64_t n_global, uint64_t seed, uint64_t stream,
                   uint64_t col, cudaStream_t s) {
    int64_t g = (nrows + 255) / 256;
    if (g > 4096) g = 4096;
    if (g < 1) g = 1;
    k_random<<<(int)g, 256, 0, s>>>(x, nrows, row0, n_global, seed, stream, col);
}

void launch_copy_cols(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t nrows, int ncols,
                      cudaStream_t s) {
    int64_t g = (nrows + 255) / 256;
    if (g > 1024) g = 1024;
    if (g < 1) g = 1;
    k_copy_cols<<<dim3((unsigned)g, (unsigned)ncols), 256, 0, s>>>(src, lds, dst, ldd, nrows, ncols);
}

void launch_gather(const double* x, const int* idx, int64_t n, double* out, cudaStream_t s) {
    int64_t g = (n + 255) / 256;
    if (g > 1024) g = 1024;
    if (g < 1) g = 1;
    k_gather<<<(int)g, 256, 0, s>>>(x, idx, n, out);
}

void launch_finalize_sdots_multi(const SdotsArgs& sd, const double* red_all, int nranks, int stride,
                                 cudaStream_t s) {
    UpdArgs up{};
    k_finalize_multi<<<1, 256, 0, s>>>(sd, up, 0, red_all, nranks, stride);
}

void launch_finalize_upd_multi(const UpdArgs& up, const double* red_all, int nranks, int stride,
                               cudaStream_t s) {
    SdotsArgs sd{};
    k_finalize_multi<<<1, 256, 0, s>>>(sd, up, 1, red_all, nranks, stride);
}

}  // namespace trplk
