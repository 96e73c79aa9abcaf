// Device kernels of the TRPL+K hot path, hand-written for sm_100a (B200).
//
//   k_sdots_mma / k_spmv_nd  K1/K7/K4 fallbacks: SpMV with A (and B) fused with the Jacobi
//             preconditioner (or the residual) and the dot products of a basis block against
//             the result -- eq 3.1, R1, Alg.1 steps 12-15 (the default K1
//             kernels are in stream_rs.cuh / k1_pipe.cuh, the other dot launches stream_tp.cuh).
//   k_upd     K2/K3: classical Gram-Schmidt update y = x - U h fused with the next pass's
//             dots, or with the final normalisation (reading R3).
//   k_rotate_t K5 for 48 < k <= 64: X = U Y on fp64 DMMA tensor cores (mma.sync m8n8k4 f64;
//             P:193); k <= 48 uses k_rotate_s (rotate.cuh).  K6 (the RR eig) is eig.cu.
//
// Streaming kernels use one lane per row (32-row SELL slice = one warp tile) and issue the
// whole row of the basis block U (k loads per lane) before the SpMV's dependent gathers, so
// the basis stream overlaps the gather latency.  Every reduction is deterministic: per-warp
// shuffle butterflies in a fixed pattern, a fixed-order CTA sum, then a two-level grid
// reduction (groups of 32 CTAs, then groups) whose order does not depend on scheduling.
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include <cooperative_groups.h>

#include "trplk_internal.cuh"

namespace trplk {

thread_local const void* g_last_kern = nullptr;

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

// Row `32 s + lane` of a local matrix times x: returns sum_j a_ij x_j and the diagonal a_ii.
// DIA: every load address is computed, so all values and gathers of a chunk of 8 diagonals
// are in flight at once (one memory round trip); the sum runs in ascending column order.
// SELL: column ids are loaded first (two round trips per chunk of 8 entries).
// XNC = false: x is gathered with ld.global.cg (L2) instead of the read-only path -- for
// kernels that read x after other CTAs wrote it inside the same launch (inner_grid.cuh).
template <bool XNC = true>
__device__ __forceinline__ double mat_row(const Sell& M, int64_t s, int lane, const double* __restrict__ x,
                                          double& diag) {
    double acc = 0.0;
    if (M.fmt == 1) {
        const int64_t row = s * 32 + lane;
        const int nl = (int)M.nrows, top = (int)(M.nrows + M.nghost - 1), glo = (int)M.glo;
        const bool halo = M.nghost != 0;
        const double* dv = M.dval + row;
        diag = __ldg(dv + (int64_t)M.diag_slot * M.ldv);
        for (int d0 = 0; d0 < M.ndiag; d0 += 8) {
            double v[8], xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int d = d0 + u;
                v[u] = 0.0;
                xv[u] = 0.0;
                if (d < M.ndiag) {
                    int idx = (int)row + M.offs[d];  // local rows + ghosts < 2^31 (checked at create)
                    if (halo) idx = idx < 0 ? idx + nl + glo : (idx >= nl ? idx + glo : idx);
                    idx = idx < 0 ? 0 : (idx > top ? top : idx);  // out-of-matrix slots hold 0
                    v[u] = __ldg(dv + (int64_t)d * M.ldv);
                    xv[u] = XNC ? __ldg(x + idx) : __ldcg(x + idx);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = fma(v[u], xv[u], acc);
        }
        return acc;
    }
    const int64_t b = __ldg(M.sptr + s), e = __ldg(M.sptr + s + 1);
    const int w = (int)((e - b) >> 5);
    const double* vp = M.val + b + lane;
    const int* cp = M.col + b + lane;
    diag = __ldg(vp);
    for (int j0 = 0; j0 < w; j0 += 8) {
        double v[8];
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool in = j0 + u < w;
            v[u] = in ? __ldg(vp + 32 * (j0 + u)) : 0.0;
            c[u] = in ? __ldg(cp + 32 * (j0 + u)) : 0;
        }
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = (j0 + u < w) ? (XNC ? __ldg(x + c[u]) : __ldcg(x + c[u])) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(v[u], xv[u], acc);
    }
    return acc;
}

// Diagonal entry of row 32 s + lane (DIA: the offset-0 array; SELL: slot 0).
__device__ __forceinline__ double mat_diag(const Sell& M, int64_t s, int lane) {
    if (M.fmt == 1) return __ldg(M.dval + (int64_t)M.diag_slot * M.ldv + s * 32 + lane);
    return __ldg(M.val + __ldg(M.sptr + s) + lane);
}

// Deterministic grid reduction of the CTA's nv values `mine` (smem).  Returns true in exactly
// one CTA, whose smem `out` then holds the grid sums.  The summation order is fixed.
// Grids of <= 1024 CTAs: one level -- the last CTA to arrive sums, per value, CTA partials
// lane, lane+32, ... in order and then the 32 lanes by an xor butterfly (one global round trip
// less than two levels).  Larger grids: CTAs in groups of RG (lane = CTA in group, butterfly),
// then the groups likewise.
constexpr int RG = 32;
constexpr int ONE_LEVEL_MAX = 1024;
__device__ bool grid_reduce(const double* mine, int nv, double* part, double* gpart, unsigned* cnt, int maxcta,
                            double* out, int bid_off = 0, int ncta_tot = 0) {
    __shared__ bool flag;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // a reduction may span several launches in stream order (halo overlap: interior rows, then
    // the boundary rows): CTA slots bid_off.. of ncta_tot; the last CTA to arrive is in the last one
    const int bid = blockIdx.x + bid_off, ncta = ncta_tot > 0 ? ncta_tot : (int)gridDim.x;
    // only the threads that wrote partials fence (a fence waits for ALL of the thread's
    // outstanding stores, e.g. its rows of the output vector, which need no ordering here)
    if (tid < nv) {
        for (int v = tid; v < nv; v += blockDim.x) part[(int64_t)v * maxcta + bid] = mine[v];
        __threadfence();
    }
    __syncthreads();
    if (ncta <= ONE_LEVEL_MAX) {
        if (tid == 0) flag = atomicAdd(&cnt[0], 1u) == (unsigned)(ncta - 1);
        __syncthreads();
        if (!flag) return false;
        __threadfence();
        // warp w sums values w*VB .. w*VB+VB-1 (then + nwarps*VB ...): VB*U partial loads in
        // flight per lane, so a 296-CTA x 60-value reduction is ~3 dependent L2 round trips
        const int nwarps = blockDim.x >> 5;
        constexpr int VB = 4, U = 4;
        for (int v0 = warp * VB; v0 < nv; v0 += nwarps * VB) {
            double sv[VB];
#pragma unroll
            for (int b = 0; b < VB; ++b) sv[b] = 0.0;
            for (int c0 = lane; c0 < ncta; c0 += 32 * U) {
                double t[VB][U];
#pragma unroll
                for (int b = 0; b < VB; ++b)
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        t[b][u] = (v0 + b < nv && c0 + 32 * u < ncta)
                                      ? __ldcg(part + (int64_t)(v0 + b) * maxcta + c0 + 32 * u)
                                      : 0.0;
#pragma unroll
                for (int b = 0; b < VB; ++b)
#pragma unroll
                    for (int u = 0; u < U; ++u) sv[b] += t[b][u];
            }
#pragma unroll
            for (int b = 0; b < VB; ++b) {
                const double s = warp_sum(sv[b]);
                if (lane == 0 && v0 + b < nv) out[v0 + b] = s;
            }
        }
        __syncthreads();
        if (tid == 0) cnt[0] = 0u;
        return true;
    }
    const int g = bid / RG, g0 = g * RG, gs = min(RG, ncta - g0), ng = (ncta + RG - 1) / RG;
    if (tid == 0) flag = atomicAdd(&cnt[1 + g], 1u) == (unsigned)(gs - 1);
    __syncthreads();
    if (!flag) return false;
    __threadfence();
    constexpr int VPC = 4;  // values per warp in flight (register budget of the host kernel)
    double val[VPC];
    for (int base = warp; base < nv; base += VPC * WARPS) {
#pragma unroll
        for (int i = 0; i < VPC; ++i) {
            const int v = base + i * WARPS;
            val[i] = (v < nv && lane < gs) ? __ldcg(part + (int64_t)v * maxcta + g0 + lane) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < VPC; ++i) {
            const int v = base + i * WARPS;
            if (v < nv) {
                const double s = warp_sum(val[i]);
                if (lane == 0) gpart[(int64_t)v * MAXG + g] = s;
            }
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        cnt[1 + g] = 0u;
        flag = atomicAdd(&cnt[0], 1u) == (unsigned)(ng - 1);
    }
    __syncthreads();
    if (!flag) return false;
    __threadfence();
    for (int base = warp; base < nv; base += VPC * WARPS) {
#pragma unroll
        for (int i = 0; i < VPC; ++i) {
            const int v = base + i * WARPS;
            double s = 0.0;
            if (v < nv) {
                if (lane < ng) s = __ldcg(gpart + (int64_t)v * MAXG + lane);
                if (lane + 32 < ng) s += __ldcg(gpart + (int64_t)v * MAXG + lane + 32);
            }
            val[i] = s;
        }
#pragma unroll
        for (int i = 0; i < VPC; ++i) {
            const int v = base + i * WARPS;
            if (v < nv) {
                const double s = warp_sum(val[i]);
                if (lane == 0) out[v] = s;
            }
        }
    }
    __syncthreads();
    if (tid == 0) cnt[0] = 0u;
    return true;
}

__device__ __forceinline__ const double* resolve_x(const double* x, int dyn, int64_t ld, int off, const Ctl* ctl) {
    if (dyn == 1) return x + ld * (int64_t)(ctl->t - 1 + off);
    if (dyn == 2) return x + ld * (int64_t)(ctl->xprev_col + off);
    return x;
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
        if (a.clear_done) ctl->flags &= ~a.clear_done;
    }
}

__device__ __forceinline__ void sdots_counts(const SdotsArgs& a, const Ctl* ctl, bool two, int& k1, int& k2) {
    const int kc = ctl->k;
    k1 = a.set1 ? (a.k_from_ctl ? kc : a.k1) : 0;
    k2 = (two && a.set2) ? (a.k_from_ctl ? kc : a.k2) : 0;
}

// KMAX = basis columns held in registers per chunk (the first chunk is issued before the SpMV);
// wider blocks are processed in chunks of KMAX columns.
// -------------------------------------- SpMV-only launches (no basis dots): residual K7 etc.
// r = A x - theta B x (u = M r), z = A x, w = M (z - rho B x) with up to two norms; R row tiles
// per warp iteration so R tiles' value loads and gathers are in flight together, norms in
// per-lane registers (one warp reduction at the end), <= 80 registers for 3 CTAs per SM.
template <int R>
__global__ void __launch_bounds__(CTA, 3) k_spmv_nd(const SdotsArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    double theta = 0.0;
    if (a.out_mode >= 3)
        theta = a.theta_idx >= 0 ? ctl->theta[a.theta_idx]
                                 : (a.theta_idx == -1 ? ctl->theta[ctl->t - 1 + (a.x_dyn == 1 ? a.x_off : 0)] : a.theta_val);
    const double rho = ctl->rho;
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    __shared__ double acc[WARPS][2];
    __shared__ double res[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nslices = (a.nrows + 31) >> 5;
    const int64_t stride = (int64_t)gridDim.x * WARPS;
    double n1 = 0.0, n2 = 0.0;
    for (int64_t s0 = (int64_t)blockIdx.x * WARPS + warp; s0 < nslices; s0 += stride * R) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t s = s0 + r * stride;
            if (s >= nslices) break;
            const int64_t row = s * 32 + lane;
            const bool ok = row < a.nrows;
            double ad = 1.0, bd = 1.0, z = 0.0, sv = 0.0, xr = 0.0;
            if (ok) {
                xr = X[row];
                if (a.out_mode == 4) ad = mat_diag(a.A, s, lane);
                else if (a.A.nrows) z = mat_row(a.A, s, lane, X, ad);
                else z = xr;
                if (a.out_mode >= 2) sv = a.B.nrows ? mat_row(a.B, s, lane, X, bd) : xr;
            }
            double o = 0.0, minv = 1.0;
            if (a.out_mode >= 2) {
                minv = jacobi_minv(ad, bd, a.pmode == 2 ? (a.out_mode == 2 ? rho : theta) : a.sigma, a.mfloor);  // M_ii
            }
            switch (a.out_mode) {
                case 1: o = z; break;
                case 2: o = minv * (z - rho * sv); break;  // w = M (z - rho B g), R1
                case 3: o = z - theta * sv; break;         // r = A x - theta B x
                case 4: o = (ok ? a.wext[row] : 0.0) - theta * sv; break;
                default: break;
            }
            if (ok) {
                if (a.out) a.out[row] = o;
                if (a.uout) a.uout[row] = minv * o;
                if (nn) {
                    n1 += a.norm1 == 1 ? o * o : a.norm1 == 2 ? xr * z : a.norm1 == 3 ? xr * xr : z * z;
                    if (a.norm2) n2 += a.norm2 == 1 ? o * o : a.norm2 == 2 ? xr * z : a.norm2 == 3 ? xr * xr : z * z;
                }
            }
        }
    }
    if (nn == 0) return;
    n1 = warp_sum(n1);
    n2 = warp_sum(n2);
    if (lane == 0) {
        acc[warp][0] = n1;
        acc[warp][1] = n2;
    }
    __syncthreads();
    if (threadIdx.x < nn) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) t += acc[w][threadIdx.x];
        res[threadIdx.x] = t;
    }
    __syncthreads();
    if (!grid_reduce(res, nn, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nn; v += CTA) a.red_local[v] = res[v];
    } else {
        sdots_finalize(a, res, 0, 0);
    }
}

// ---------------------------------------------- K1 (DMMA dots): fused SpMV + U^T [z w]
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// The dot products of K1 are the tall-skinny contraction U(:,1:k)^T [z w] (n x k by n x 2).
// Each warp accumulates it over all of its 32-row tiles in DMMA m8n8k4 fragments
// (A = 8 columns x 4 rows of U, B = rows of [z w 0..0], C = 8 x 8, columns 0/1 useful) and
// reduces across warps/CTAs once at the end: no per-tile shuffle reductions.  The CUDA-core
// version of this kernel was issue-bound (ncu: 'wait' + math-pipe throttle, 31% DRAM).
// NG = column groups of 8 held in accumulators (k <= 8 NG).
template <int NG, bool TWO>
__global__ void __launch_bounds__(CTA, 2) k_sdots_mma(const SdotsArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    int k1, k2;
    sdots_counts(a, ctl, TWO, k1, k2);
    const double rho = ctl->rho;
    double theta = 0.0;
    if (a.out_mode >= 3)
        theta = a.theta_idx >= 0 ? ctl->theta[a.theta_idx]
                                 : (a.theta_idx == -1 ? ctl->theta[ctl->t - 1 + (a.x_dyn == 1 ? a.x_off : 0)] : a.theta_val);
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const int kmx = k1 > k2 ? k1 : k2;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    const double* __restrict__ Ub = a.U;

    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;  // fragment row/col ids
    double cacc[NG][2];
#pragma unroll
    for (int g = 0; g < NG; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0, n2 = 0.0;
    const int64_t nslices = (a.nrows + 31) >> 5;
    for (int64_t s = (int64_t)blockIdx.x * WARPS + warp; s < nslices; s += (int64_t)gridDim.x * WARPS) {
        const int64_t r0 = s * 32;
        const int64_t row = r0 + lane;
        const bool ok = row < a.nrows;
        double ad = 1.0, bd = 1.0, z = 0.0, sv = 0.0;
        const double xr = ok ? X[row] : 0.0;
        if (a.A.nrows) z = mat_row(a.A, s, lane, X, ad);
        else z = xr;
        if (a.out_mode >= 2) {
            if (a.B.nrows) sv = mat_row(a.B, s, lane, X, bd);
            else sv = xr;
        }
        double o = 0.0, minv = 1.0;
        if (a.out_mode >= 2) {
            minv = jacobi_minv(ad, bd, a.pmode == 2 ? (a.out_mode == 2 ? rho : theta) : a.sigma, a.mfloor);  // M_ii
        }
        if (a.out_mode == 1) o = z;
        else if (a.out_mode == 2) o = minv * (z - rho * sv);  // w = M (z - rho B g), R1
        else if (a.out_mode == 3) o = z - theta * sv;
        if (ok) {
            if (a.out) a.out[row] = o;
            if (a.uout) a.uout[row] = minv * o;
        } else {
            z = 0.0;
            o = 0.0;
        }
        const double v1 = a.set1 == 1 ? z : (a.set1 == 2 ? o : xr);
        if (nn) {
            const double p1 = a.norm1 == 1 ? o * o : a.norm1 == 2 ? xr * z : a.norm1 == 3 ? xr * xr : z * z;
            const double p2 = a.norm2 == 1 ? o * o : a.norm2 == 2 ? xr * z : a.norm2 == 3 ? xr * xr : z * z;
            n1 += ok ? p1 : 0.0;
            n2 += ok ? p2 : 0.0;
        }
        // B fragments of the 8 row quads: B[fj][fi] = (fi == 0 ? v1 : fi == 1 ? o : 0) at row 4q + fj
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, v1, 4 * q + fj);
            const double t2 = TWO ? __shfl_sync(0xffffffffu, o, 4 * q + fj) : 0.0;
            bq[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
        }
        const int64_t nrows = a.nrows;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            if (8 * g < kmx) {
                const int c = 8 * g + fi;
                const bool cok = c < kmx;
                const double* up = Ub + (int64_t)c * a.ldu + r0 + fj;
                double av[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) av[q] = (cok && r0 + 4 * q + fj < nrows) ? __ldg(up + 4 * q) : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884(cacc[g], av[q], bq[q]);
            }
        }
    }
    // per-warp results: lane with fj == 0 holds C[fi][0] (set 1) and C[fi][1] (set 2) of group g
    for (int i = threadIdx.x; i < WARPS * NV_MAX; i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (fj == 0) {
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int c = 8 * g + fi;
            if (c < k1) acc[warp][c] = cacc[g][0];
            if (TWO && c < k2) acc[warp][k1 + c] = cacc[g][1];
        }
    }
    if (nn) {
        n1 = warp_sum(n1);
        n2 = warp_sum(n2);
        if (lane == 0) {
            int oo = k1 + k2;
            if (a.norm1) acc[warp][oo++] = n1;
            if (a.norm2) acc[warp][oo] = n2;
        }
    }
    if (nv == 0) return;
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += CTA) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s += acc[w][v];
        res[v] = s;
    }
    __syncthreads();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
    } else {
        sdots_finalize(a, res, k1, k2);
    }
}

// --------------------------------------------------- K2/K3: CGS update (+dots / +norm)
__device__ void upd_finalize(const UpdArgs& a, const double* r, int kv) {
    Ctl* ctl = a.ctl;
    for (int i = threadIdx.x; i < kv; i += blockDim.x) ctl->h[a.hout][i] = r[i];
    if (threadIdx.x == 0) ctl->nrm[a.mode == 1 ? N_1SQ : N_2SQ_EXP] = r[kv];
}

// Third CGS pass inside a cooperatively launched FINAL kernel (reading R3; one rank, B = I):
// w2 = w1 - U h2 is in a.out (written by all CTAs; the grid barrier below makes every row
// visible before any CTA reads it -- a CTA's rows are not the rows it wrote with the two-tile
// mapping); h3 = U^T w2 and ||w2||^2 are reduced
// over the grid (per-CTA partials, grid barrier, the same fixed-order sum in every CTA), then
// g = (w2 - U h3) / beta3 with beta3^2 = ||w2||^2 - ||h3||^2.  Rare path (a second pass that
// loses more than half the norm): written for few registers, not speed.  Returns breakdown.
__device__ __noinline__ bool final_pass3_coop(const double* __restrict__ U, int64_t ldu, int64_t nrows, const double* w2,
                                              double* part, int maxcta, double* dest2, int kv, double nin, double* dest,
                                              double* sred) {
    namespace cg = cooperative_groups;
    __shared__ double acc3[WARPS][QMAX + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < WARPS * (QMAX + 1); i += CTA) (&acc3[0][0])[i] = 0.0;
    // w2 was written by the two-tile loop, whose row mapping is not this pass's: every CTA's
    // rows must be visible before they are read back (only on the rare third pass)
    __threadfence();
    cg::this_grid().sync();
    const int64_t ntiles = (nrows + 31) >> 5;
    double yy = 0.0;
    for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles; tile += (int64_t)gridDim.x * WARPS) {
        const int64_t row = tile * 32 + lane;
        const bool ok = row < nrows;
        const double y = ok ? w2[row] : 0.0;
        yy += y * y;
        for (int c = 0; c < kv; ++c) {
            const double v = warp_sum(ok ? __ldg(U + (int64_t)c * ldu + row) * y : 0.0);
            if (lane == 0) acc3[warp][c] += v;
        }
    }
    yy = warp_sum(yy);
    if (lane == 0) acc3[warp][kv] = yy;
    __syncthreads();
    for (int v = threadIdx.x; v <= kv; v += CTA) {
        double t = 0.0;
        for (int w = 0; w < WARPS; ++w) t += acc3[w][v];
        part[(int64_t)v * maxcta + blockIdx.x] = t;
    }
    __threadfence();
    cg::this_grid().sync();
    for (int v = threadIdx.x; v <= kv; v += CTA) {  // every CTA: the same fixed-order sum
        double t = 0.0;
        for (int c = 0; c < (int)gridDim.x; ++c) t += __ldcg(part + (int64_t)v * maxcta + c);
        sred[v] = t;
    }
    __syncthreads();
    double hn = 0.0;
    for (int i = 0; i < kv; ++i) hn += sred[i] * sred[i];
    const double n3sq = sred[kv] - hn;
    const double b = sqrt(n3sq > 0.0 ? n3sq : 0.0);
    const bool brk = !(b >= 1e-14 * nin) || nin == 0.0;
    if (!brk) {
        const double binv = 1.0 / b;
        for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles; tile += (int64_t)gridDim.x * WARPS) {
            const int64_t row = tile * 32 + lane;
            if (row >= nrows) continue;
            double y = w2[row];
            for (int c = 0; c < kv; ++c) y = fma(-sred[c], __ldg(U + (int64_t)c * ldu + row), y);
            const double g = y * binv;
            dest[row] = g;
            if (dest2) dest2[row] = g;
        }
    }
    cg::this_grid().sync();  // the partials buffer is free again before any CTA leaves
    return brk;
}

// DOTS = true: mode 1 (update + U^T y dots); DOTS = false: modes 0 / 2 / 3 (no dots; the rare
// third-pass dots are a separate gated k_sdots launch).
template <int KMAX, bool DOTS>
__global__ void __launch_bounds__(CTA, DOTS ? 2 : (KMAX <= 32 ? 2 : 1)) k_upd(const UpdArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.mode == 3 && ctl->pass3 == 0) return;
    const int kv = a.kv >= 0 ? a.kv : ctl->k;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    __shared__ double hs[KMAX];
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
            pass3 = !(n2sq >= 0.5 * n1sq) || a.force3;  // second pass dropped the norm by > 1/sqrt2
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
    const bool do_dots = DOTS && a.mode == 1;
    const bool write_dest = (a.mode >= 2) && !pass3 && !brk;
    double* dest = a.dest;
    if (write_dest && a.dest_dyn) dest = a.dest + a.dest_ld * (int64_t)ctl->k;

    if (do_dots)
        for (int i = threadIdx.x; i < WARPS * (QMAX + 1); i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (a.nrows + 31) >> 5;
    double dacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) dacc[g][0] = dacc[g][1] = 0.0;
    double yy_acc = 0.0;
    static_assert(KMAX > 0, "");
    if constexpr (!DOTS && KMAX <= 24) {
        // two 32-row tiles per warp iteration (as k_step1_rs2 / k_upd2_wp2): both rows of U in
        // flight together, half the dependent load round trips per warp
        const int64_t npair = (ntiles + 1) >> 1;
        if (write_y || write_dest) {
            for (int64_t tp = (int64_t)blockIdx.x * WARPS + warp; tp < npair; tp += (int64_t)gridDim.x * WARPS) {
                const int64_t r0 = (2 * tp) * 32 + lane, r1 = r0 + 32;
                const bool ok0 = r0 < a.nrows, ok1 = r1 < a.nrows;
                double y0 = ok0 ? X[r0] : 0.0, y1 = ok1 ? X[r1] : 0.0;
                double u0[KMAX], u1[KMAX];
#pragma unroll
                for (int c = 0; c < KMAX; ++c) {
                    u0[c] = (ok0 && c < kv) ? __ldg(a.U + (int64_t)c * a.ldu + r0) : 0.0;
                    u1[c] = (ok1 && c < kv) ? __ldg(a.U + (int64_t)c * a.ldu + r1) : 0.0;
                }
#pragma unroll
                for (int c = 0; c < KMAX; ++c) {
                    y0 = fma(-hs[c], u0[c], y0);
                    y1 = fma(-hs[c], u1[c], y1);
                }
                if (ok0) {
                    if (write_y && a.out) a.out[r0] = y0;
                    if (write_dest) {
                        dest[r0] = y0 * binv;
                        if (a.dest2) a.dest2[r0] = y0 * binv;
                    }
                }
                if (ok1) {
                    if (write_y && a.out) a.out[r1] = y1;
                    if (write_dest) {
                        dest[r1] = y1 * binv;
                        if (a.dest2) a.dest2[r1] = y1 * binv;
                    }
                }
            }
        }
    } else if (write_y || write_dest) {
        for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles;
             tile += (int64_t)gridDim.x * WARPS) {
            const int64_t row = tile * 32 + lane;
            const bool ok = row < a.nrows;
            // y = x - U h, columns in order; the whole row of U is loaded before the first FMA
            // (KMAX loads in flight per lane)
            double y = ok ? X[row] : 0.0;
            const double* up = a.U + row;
            double uk[KMAX];
#pragma unroll
            for (int c = 0; c < KMAX; ++c) uk[c] = (ok && c < kv) ? __ldg(up + (int64_t)c * a.ldu) : 0.0;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) y = fma(-hs[c], uk[c], y);
            if (ok) {
                if (write_y && a.out) a.out[row] = y;
                if (write_dest) {
                    const double g = y * binv;
                    dest[row] = g;
                    if (a.dest2) a.dest2[row] = g;
                }
            }
            if (DOTS && do_dots) {
                // U^T y accumulated in DMMA fragments over the warp's tiles: A = y^T (row 0, 4 rows
                // per quad), B = U(4 rows, 8 columns) re-read in fragment order (cache hits).
                yy_acc += ok ? y * y : 0.0;
                const int fi = lane >> 2, fj = lane & 3;
                double ya[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double t = __shfl_sync(0xffffffffu, y, 4 * q + fj);
                    ya[q] = fi == 0 ? t : 0.0;
                }
                const int64_t r0 = tile * 32;
#pragma unroll
                for (int g = 0; g < KMAX / 8; ++g) {
                    if (8 * g < kv) {
                        const int c = 8 * g + fi;
                        const bool cok = c < kv;
                        const double* up = a.U + (int64_t)c * a.ldu + r0 + fj;
                        double bu[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) bu[q] = (cok && r0 + 4 * q + fj < a.nrows) ? __ldg(up + 4 * q) : 0.0;
#pragma unroll
                        for (int q = 0; q < 8; ++q) dmma884(dacc[g], ya[q], bu[q]);
                    }
                }
            }
        }
    }
    if (a.mode == 0) return;
    bool brk3 = false, done3 = false;
    if (a.mode == 2 && pass3 && a.coop) {
        __syncthreads();
        double* d3 = a.dest_dyn ? a.dest + a.dest_ld * (int64_t)ctl->k : a.dest;
        brk3 = final_pass3_coop(a.U, a.ldu, a.nrows, a.out, a.part, a.maxcta, a.dest2, kv, sqrt(ctl->nrm[N_IN2]), d3,
                                res);
        done3 = true;
    }
    const int nv = do_dots ? kv + 1 : 0;
    __shared__ bool is_last;
    if (nv) {
        // per-warp results: lane fi == 0 holds D[0][2 fj + e] = dot of column 8g + 2fj + e
        const int fi = lane >> 2, fj = lane & 3;
        if (fi == 0) {
#pragma unroll
            for (int g = 0; g < KMAX / 8; ++g)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 8 * g + 2 * fj + e;
                    if (c < kv) acc[warp][c] = dacc[g][e];
                }
        }
        const double yy = warp_sum(yy_acc);
        if (lane == 0) acc[warp][kv] = yy;
        __syncthreads();
        for (int v = threadIdx.x; v < nv; v += CTA) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) s += acc[w][v];
            res[v] = s;
        }
        __syncthreads();
        if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
        if (a.red_local) {
            for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
        } else {
            upd_finalize(a, res, kv);
        }
    } else {
        // no dots: one ticket so exactly one CTA -- the last to finish, after every CTA has
        // read the control block -- applies the control-block side effects (no data is handed
        // between CTAs, so no fence)
        __syncthreads();
        if (threadIdx.x == 0) is_last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!is_last) return;
        if (threadIdx.x == 0) *a.counter = 0u;
    }
    if (threadIdx.x == 0) {
        if (a.mode == 2 && done3) {  // third pass done in this kernel
            for (int i = 0; i < kv; ++i) ctl->h[2][i] = res[i];  // h3 and ||w2||^2 (reported by the API)
            ctl->nrm[N_2SQ_EXP] = res[kv];
            ctl->pass3_count += 1;
            if (brk3) {
                ctl->flags &= ~a.clear_on_brk;
                ctl->brk += 1;
            } else if (a.inc_k) {
                ctl->k += 1;
            }
        } else if (a.mode == 2) {
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

// ------------------------------------------------------- K5: DMMA rotation X = U Y

// Transposed-operand DMMA rotation (default): X^T = Y^T U^T, so the A operand (Y^T, p^ x k) is
// loaded into registers once per warp and reused for every row tile, and the B operand is
// U^T: lane (kk = l&3, n = l>>2) loads U[row0 + n, 4 ks + kk] -- 4 columns x 8 consecutive rows
// per instruction, each column's 32 bytes x 4 row blocks of a 32-row tile forming full lines.
// The accumulator D = X^T (8 output columns x 8 rows) holds 2 consecutive rows per lane,
// written as one 16-byte store.  NJ = 8-column groups of X (p^ <= 8 NJ), KS4 = k-steps of 4
// (k <= 4 KS4), RB = 8-row blocks per warp iteration (all RB*KS4 loads issued first).
constexpr int ROT_CTA = 128;
template <int NJ, int KS4, int RB>
__global__ void __launch_bounds__(ROT_CTA, 2) k_rotate_t(const double* __restrict__ U, int64_t ldu, int64_t nrows,
                                                       const Ctl* ctl, int k_fixed, const double* __restrict__ Y,
                                                       int ldY, int ncol, double* __restrict__ X, int64_t ldx,
                                                       unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k_rr;
    const int lane = threadIdx.x & 31;
    const int lq = lane & 3, lr = lane >> 2;
    double yf[NJ][KS4];
#pragma unroll
    for (int jb = 0; jb < NJ; ++jb)
#pragma unroll
        for (int ks = 0; ks < KS4; ++ks) {
            const int kk = 4 * ks + lq, j = 8 * jb + lr;
            yf[jb][ks] = (kk < k && j < ncol) ? __ldg(Y + kk + (int64_t)j * ldY) : 0.0;
        }
    const int64_t gw = ((int64_t)blockIdx.x * ROT_CTA + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * ROT_CTA) >> 5;
    const int64_t ntile = (nrows + 8 * RB - 1) / (8 * RB);
    const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && ((ldx & 1) == 0);
    for (int64_t tile = gw; tile < ntile; tile += nw) {
        const int64_t r0 = tile * (8 * RB);
        double b[RB][KS4];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const int64_t row = r0 + 8 * rb + lr;
#pragma unroll
            for (int ks = 0; ks < KS4; ++ks) {
                const int kk = 4 * ks + lq;
                b[rb][ks] = (row < nrows && kk < k) ? __ldg(U + (int64_t)kk * ldu + row) : 0.0;
            }
        }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            double acc[NJ][2];
#pragma unroll
            for (int jb = 0; jb < NJ; ++jb) {
                acc[jb][0] = acc[jb][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS4; ++ks) dmma884(acc[jb], yf[jb][ks], b[rb][ks]);
            }
            const int64_t row = r0 + 8 * rb + 2 * lq;
#pragma unroll
            for (int jb = 0; jb < NJ; ++jb) {
                const int j = 8 * jb + lr;
                if (j < ncol) {
                    double* xp = X + (int64_t)j * ldx + row;
                    if (vec && row + 1 < nrows) {
                        *reinterpret_cast<double2*>(xp) = make_double2(acc[jb][0], acc[jb][1]);
                    } else {
                        if (row < nrows) xp[0] = acc[jb][0];
                        if (row + 1 < nrows) xp[1] = acc[jb][1];
                    }
                }
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

}  // namespace trplk

#include "stream_rs.cuh"  // register-stream + DMMA K1 (shares the device helpers above)
#include "stream_tp.cuh"   // thread-per-row K1 / K2
#include "rotate.cuh"      // shared-memory-staged DMMA rotation (default)
#include "block.cuh"       // multi-vector Gram / update / SpMM (block +K)
#include "ic0.cuh"         // IC(0) factor and sync-free triangular solves (NEXT-2)
#include "k1_pipe.cuh"     // software-pipelined K1 (DIA, B = I, k <= 24)
#include "small.cuh"       // single-CTA inner loop for small n (latency path)
#include "inner_grid.cuh"  // cooperative grid-wide inner loop for mid-size n (latency path)
#include "pl1.cuh"         // PL+1 (Algorithm 2) small kernels
#include "fused.cuh"       // K3 of step j + K1 of step j+1 in one kernel (lagged rounds)
#include "lean_k1.cuh"     // thread-per-row K1 (register accumulators) for k <= 24

namespace trplk {

// ---------------------------------------------------------------- launchers
// K1 variant: default = the pipelined kernel (k1_pipe.cuh) for k <= 16 on slabs of >= 2^24 rows
// (the C5 steps), else the two-tile register-stream kernel (stream_rs.cuh).  TRPLK_K1=pipe /
// TRPLK_K1=rs force one of them wherever it applies (parity tests of both on every shape);
// TRPLK_K1=tpdots keeps the first-pass CGS dots on the thread-per-row kernel.
static int k1var() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TRPLK_K1");
        v = (e && !strcmp(e, "pipe")) ? 2 : (e && !strcmp(e, "rs")) ? 1 : (e && !strcmp(e, "tpdots")) ? 3
            : (e && !strcmp(e, "lean")) ? 4 : 0;
    }
    return v;
}

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

// Grid of a persistent streaming kernel: resident CTAs (occupancy API) x SMs, balanced so
// that every CTA processes the same number of 32-row tiles.
static int occupancy(const void* kernel) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(kernel);
    if (it != cache.end()) return it->second;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, CTA, 0);
    if (occ < 1) occ = 1;
    cache[kernel] = occ;
    return occ;
}

template <typename K>
static int stream_grid(K kernel, int64_t nrows) {
    const int occ = occupancy(reinterpret_cast<const void*>(kernel));
    const int64_t tiles = (nrows + 31) / 32;
    const int64_t need = (tiles + WARPS - 1) / WARPS;
    int64_t cap = (int64_t)num_sms() * occ;
    if (cap > MAXCTA) cap = MAXCTA;
    if (need <= cap) return (int)(need < 1 ? 1 : need);
    const int64_t waves = (need + cap - 1) / cap;
    return (int)((need + waves - 1) / waves);
}

int kmax_bucket(int k) {
    if (k <= 0) return 0;
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 24) return 24;
    if (k <= 32) return 32;
    if (k <= 40) return 40;
    if (k <= 48) return 48;
    return 64;
}

#define SDM_CASE(NG)                                                                     \
    case NG:                                                                             \
        if (a.set2) {                                                                    \
            auto kern = k_sdots_mma<NG, true>;                                           \
            NOTE_KERN(kern);                                                             \
            kern<<<stream_grid(kern, a.nrows), CTA, 0, s>>>(a);                          \
        } else {                                                                         \
            auto kern = k_sdots_mma<NG, false>;                                          \
            NOTE_KERN(kern);                                                             \
            kern<<<stream_grid(kern, a.nrows), CTA, 0, s>>>(a);                          \
        }                                                                                \
        break;

void launch_sdots(const SdotsArgs& a, int kmax, cudaStream_t s) {
    // inner-step K1 shape: z = A g, w = M (z - rho B g), U^T z (+ U^T w, ||w||^2)
    const bool k1_shape = a.A.nrows && a.out_mode <= 2 && a.set1 == 1 && (a.set2 == 0 || a.set2 == 2 || a.set2 == 4) &&
                          (a.norm1 >= 0 && a.norm1 <= 2) && (a.norm2 == 0 || (a.norm2 == 5 && a.set2 == 4)) &&
                          a.x_dyn == 0 && a.uout == nullptr;
    if (kmax > 0 && k1_shape) {
        const bool split = a.row0 != 0 || a.cta_tot != 0;  // row-range launches: rs2 / pipe only
        // thread-per-row K1 with the DIA-C decode: default for k <= 16 on slabs of >= 2^24 rows with
        // constant diagonals (C5: 4.46 vs 4.72 ms for the pipelined kernel at k = 15), or forced
        const bool lean_default = k1var() == 0 && kmax <= 16 && a.nrows >= ((int64_t)1 << 24) && a.A.cmask;
        if (!split && a.set2 != 4 && (k1var() == 4 || lean_default) && kmax <= 24 && launch_step1_lean(a, kmax, s))
            return;
        // pipelined K1: measured faster on long tile loops with a register-resident row (C5,
        // k <= 16: 10.98 vs 11.53 ms per inner step); equal or slower elsewhere
        if ((k1var() == 2 || (k1var() == 0 && kmax <= 16 && a.nrows >= (int64_t)1 << 24)) &&
            launch_step1_pipe(a, kmax, s))
            return;
        if (launch_step1_rs(a, kmax, s)) return;
    }
    // first-pass CGS dots U^T x, x^T x (seed, +K; B = I): the register-stream DMMA kernel with A
    // absent (measured at C5, k = 24: the thread-per-row kernel streamed at 0.66 of DRAM peak with
    // 192 registers and one CTA per SM)
    const bool xdots = a.A.nrows == 0 && a.B.nrows == 0 && a.set1 == 3 && a.set2 == 0 && a.out_mode == 0 &&
                       (a.norm1 == 0 || a.norm1 == 3) && a.norm2 == 0 && a.uout == nullptr && a.out == nullptr;
    if (kmax > 0 && xdots && k1var() != 3) {
        SdotsArgs b = a;
        b.set1 = 1;                          // z = x when A is absent
        b.norm1 = a.norm1 == 3 ? 2 : 0;      // x.z = x.x
        if (launch_step1_rs(b, kmax, s)) return;
    }
    // every other dot launch (+K T columns with B != I, start-block Gram, ...): thread-per-row
    if (kmax > 0 && a.out_mode != 4 && launch_step1_tp(a, kmax, s)) return;
    if (kmax > 0 && a.out_mode != 4) {  // dots beyond the bucketed widths: DMMA accumulator kernel
        switch ((kmax + 7) / 8) {
            SDM_CASE(1)
            SDM_CASE(2)
            SDM_CASE(3)
            SDM_CASE(4)
            SDM_CASE(5)
            SDM_CASE(6)
            SDM_CASE(7)
            default:
            SDM_CASE(8)
        }
        return;
    }
    // SpMV-only launch (residual, plain SpMV, start-block residual from W)
    auto kern = k_spmv_nd<2>;
    NOTE_KERN(kern);
    kern<<<stream_grid(kern, (a.nrows + 1) / 2), CTA, 0, s>>>(a);
}

#define UP_CASE(KM)                                                \
    case KM: {                                                     \
        if (a.mode == 1 && a.dots) {                               \
            auto kern = k_upd<KM, true>;                           \
            NOTE_KERN(kern);                                       \
            kern<<<stream_grid(kern, a.nrows), CTA, 0, s>>>(a);    \
        } else {                                                   \
            auto kern = k_upd<KM, false>;                          \
            NOTE_KERN(kern);                                       \
            if (a.mode == 2 && a.coop) {                           \
                cudaLaunchConfig_t cfg{};                          \
                cfg.gridDim = stream_grid(kern, KM <= 24 ? (a.nrows + 1) / 2 : a.nrows); \
                cfg.blockDim = CTA;                                \
                cfg.stream = s;                                    \
                cudaLaunchAttribute at[1];                         \
                at[0].id = cudaLaunchAttributeCooperative;         \
                at[0].val.cooperative = 1;                         \
                cfg.attrs = at;                                    \
                cfg.numAttrs = 1;                                  \
                cudaLaunchKernelEx(&cfg, kern, a);                 \
            } else {  /* k <= 24: two 32-row tiles per warp iteration */ \
                kern<<<stream_grid(kern, KM <= 24 ? (a.nrows + 1) / 2 : a.nrows), CTA, 0, s>>>(a); \
            }                                                      \
        }                                                          \
    } break;

void launch_upd(const UpdArgs& a, int kmax, cudaStream_t s) {
    // CGS pass 2 with dots: warp-group two-tile kernel (stream_tp.cuh)
    if (a.mode == 1 && a.dots && launch_upd2_wp(a, kmax, s)) return;
    switch (kmax) {
        UP_CASE(8)
        UP_CASE(16)
        UP_CASE(24)
        UP_CASE(32)
        UP_CASE(40)
        UP_CASE(48)
        default:
        UP_CASE(64)
    }
}


template <int NJ, int KS4>
static void rot_t(const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed, const double* Y,
                  int ldY, int ncol, double* X, int64_t ldx, unsigned gate, cudaStream_t s) {
    constexpr int RB = 2;
    auto kern = k_rotate_t<NJ, KS4, RB>;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, ROT_CTA, 0);
    if (occ < 1) occ = 1;
    const int64_t tiles = (nrows + 8 * RB - 1) / (8 * RB);
    int64_t g = (tiles + ROT_CTA / 32 - 1) / (ROT_CTA / 32);
    const int64_t cap = (int64_t)num_sms() * occ;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    kern<<<(int)g, ROT_CTA, 0, s>>>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate);
}

template <int NJ>
static void rot_t_k(int kmax, const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed,
                    const double* Y, int ldY, int ncol, double* X, int64_t ldx, unsigned gate, cudaStream_t s) {
    (void)kmax;  // only 48 < k <= 64 comes here
    rot_t<NJ, 16>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
}

// kmax: upper bound of the device-side width (k_fixed, or the solve's max basis q).
// k <= 48: k_rotate_s (rotate.cuh, U tile staged in shared memory); 48 < k <= 64: the
// register-fragment k_rotate_t (the shared-memory slab of 64 columns would leave one CTA per SM).
void launch_rotate(const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed, const double* Y,
                   int ldY, int ncol, double* X, int64_t ldx, unsigned gate, cudaStream_t s, int kmax) {
    if (k_fixed > 0) kmax = k_fixed;
    const bool done = ncol <= 8    ? rot_s_k<1>(kmax, U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s)
                      : ncol <= 16 ? rot_s_k<2>(kmax, U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s)
                                   : rot_s_k<3>(kmax, U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    if (done) return;
    if (ncol <= 8) rot_t_k<1>(kmax, U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else if (ncol <= 16) rot_t_k<2>(kmax, U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else rot_t_k<3>(kmax, U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
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

struct DiaOffs {
    int o[DIA_MAX];
};

// create-time CSR -> DIA scatter (rows of a local block; ci holds global column ids)
__global__ void k_csr_to_dia(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                             const double* __restrict__ va, int64_t nrows, int64_t row0, DiaOffs offs, int nd,
                             int64_t ldv, double* __restrict__ dval) {
    const int64_t base = rp[0];
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p1 = rp[r + 1] - base;
        for (int64_t p = rp[r] - base; p < p1; ++p) {
            const int64_t off = ci[p] - (row0 + r);
            int d = 0;
            while (d < nd - 1 && offs.o[d] != off) ++d;
            dval[(int64_t)d * ldv + r] = va[p];
        }
    }
}

void launch_csr_to_dia(const int64_t* rp, const int64_t* ci, const double* va, int64_t nrows, int64_t row0,
                       const int* offs, int nd, int64_t ldv, double* dval, cudaStream_t s) {
    DiaOffs o{};
    for (int d = 0; d < nd && d < DIA_MAX; ++d) o.o[d] = offs[d];
    int64_t g = (nrows + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_csr_to_dia<<<(int)g, 256, 0, s>>>(rp, ci, va, nrows, row0, o, nd, ldv, dval);
}

// DIA-C detection: per diagonal, the min and max bit pattern of its stored (non-+0.0) entries.
__global__ void k_dia_const_scan(const double* __restrict__ dval, int64_t nrows, int64_t ldv, int nd,
                                 unsigned long long* __restrict__ mnmx) {
    const int d = blockIdx.y;
    unsigned long long mn = ~0ull, mx = 0ull;
    const unsigned long long* v = reinterpret_cast<const unsigned long long*>(dval + (int64_t)d * ldv);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = __ldg(v + r);
        if (b != 0ull) {
            mn = b < mn ? b : mn;
            mx = b > mx ? b : mx;
        }
    }
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mnmx + 2 * d, mn);
        atomicMax(mnmx + 2 * d + 1, mx);
    }
}

// DIA-C presence words: bit d of row r = stored entry of constant diagonal d (rows >= nrows: 0).
template <typename T>
__global__ void k_dia_pmask(const double* __restrict__ dval, int64_t nrows, int64_t ldv, int nd, unsigned cmask,
                            T* __restrict__ pm) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < ldv; r += (int64_t)gridDim.x * blockDim.x) {
        unsigned m = 0;
        if (r < nrows)
            for (int d = 0; d < nd; ++d)
                if (((cmask >> d) & 1u) &&
                    __double_as_longlong(__ldg(dval + (int64_t)d * ldv + r)) != 0ll)
                    m |= 1u << d;
        pm[r] = (T)m;
    }
}

void launch_dia_const_scan(const double* dval, int64_t nrows, int64_t ldv, int nd, unsigned long long* mnmx,
                           cudaStream_t s) {
    int64_t g = (nrows + 255) / 256;
    if (g > 148 * 4) g = 148 * 4;
    if (g < 1) g = 1;
    k_dia_const_scan<<<dim3((unsigned)g, (unsigned)nd), 256, 0, s>>>(dval, nrows, ldv, nd, mnmx);
}

void launch_dia_pmask(const double* dval, int64_t nrows, int64_t ldv, int nd, unsigned cmask, unsigned char* pm,
                      cudaStream_t s) {
    int64_t g = (ldv + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_dia_pmask<unsigned char><<<(int)g, 256, 0, s>>>(dval, nrows, ldv, nd, cmask, pm);
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
