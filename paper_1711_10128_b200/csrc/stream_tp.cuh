// Streaming dot kernels of the solver besides the inner-step K1 (stream_rs.cuh / k1_pipe.cuh):
//
//   k_step1_tp  thread-per-row: every dot launch that is not the inner-step K1 -- the CGS first
//               pass U^T B x of the seed and +K vectors (reading R3), the +K T columns
//               (Alg. 1 step 8), the start-block Gram -- all modes of
//               SdotsArgs (z = A x, w = M (z - rho B x), residual r = A x - theta B x, u = M r).
//   k_upd2_wp2  K2, warp-group: w' = w - U h1, h2 = U^T w', ||w'||^2  (CGS pass 2, reading R3)
//
// Layout: a warp tile is TR = 32/S consecutive rows; the k basis columns are split over the S
// lane groups (group g owns columns [g*KS, g*KS+KS)), so each lane keeps its KS values of U
// and its KS (or 2*KS) dot accumulators in registers for the whole kernel.  Every column read
// of a warp is TR consecutive doubles (S <= 2: a full 128-byte line), all KS loads of a lane
// are issued before any arithmetic (K1: before the SpMV's gathers), and the cross-lane
// reduction happens once per kernel instead of once per tile.  Measured on B200 with
// tools/micro_cgs.cu: 6.2 TB/s for the K2 shape at k = 24 (95% of the measured copy peak),
// where the shared-memory-transpose + DMMA variant streams at 2.6-3 TB/s.
//
// Sums: each lane accumulates its rows in row order; lanes of a group are combined by a fixed
// xor butterfly, warps in index order, CTAs by grid_reduce (fixed two-level order), so the
// result is bitwise reproducible for a given grid.  Included by kernels.cu (same translation
// unit: mat_row, grid_reduce, sdots_finalize, upd_finalize).
#pragma once

namespace trplk {

// A row of a local matrix times x at an arbitrary row index (mat_row works on 32-row slices).
__device__ __forceinline__ double mat_row_at(const Sell& M, int64_t row, const double* __restrict__ x,
                                             double& diag) {
    return mat_row(M, row >> 5, (int)(row & 31), x, diag);
}

template <int KS, int S, bool TWO, bool PF>
__global__ void __launch_bounds__(CTA, 1) k_step1_tp(const SdotsArgs a) {
    constexpr int TR = 32 / S;
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    int k1, k2;
    sdots_counts(a, ctl, TWO, k1, k2);
    const int kmx = k1 > k2 ? k1 : k2;
    const double rho = ctl->rho;
    double theta = 0.0;
    if (a.out_mode >= 3)
        theta = a.theta_idx >= 0 ? ctl->theta[a.theta_idx]
                                 : (a.theta_idx == -1 ? ctl->theta[ctl->t - 1 + (a.x_dyn == 1 ? a.x_off : 0)] : a.theta_val);
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / TR, rr = lane % TR;
    const int c0 = grp * KS;
    double a1[KS], a2[TWO ? KS : 1];
#pragma unroll
    for (int c = 0; c < KS; ++c) {
        a1[c] = 0.0;
        if (TWO) a2[c] = 0.0;
    }
    double n1 = 0.0, n2 = 0.0;
    const int64_t ntile = (a.nrows + TR - 1) / TR;
    const double* ub = a.U + (int64_t)c0 * a.ldu;
    const int64_t tstride = (int64_t)gridDim.x * WARPS;
    double un[PF ? KS : 1];
    if (PF) {  // prefetch: the next tile's U row is in flight while this tile is processed
        const int64_t row = ((int64_t)blockIdx.x * WARPS + warp) * TR + rr;
#pragma unroll
        for (int c = 0; c < KS; ++c)
            un[c] = (row < a.nrows && c0 + c < kmx) ? __ldg(ub + (int64_t)c * a.ldu + row) : 0.0;
    }
    for (int64_t t = (int64_t)blockIdx.x * WARPS + warp; t < ntile; t += tstride) {
        const int64_t row = t * TR + rr;
        const bool ok = row < a.nrows;
        double u[KS];
        if (PF) {
            const int64_t rn = row + tstride * TR;
#pragma unroll
            for (int c = 0; c < KS; ++c) {
                u[c] = un[c];
                un[c] = (rn < a.nrows && c0 + c < kmx) ? __ldg(ub + (int64_t)c * a.ldu + rn) : 0.0;
            }
        } else {
#pragma unroll
            for (int c = 0; c < KS; ++c) u[c] = (ok && c0 + c < kmx) ? __ldg(ub + (int64_t)c * a.ldu + row) : 0.0;
        }
        double z = 0.0, o = 0.0, xr = 0.0;
        if (ok) {
            double ad = 1.0, bd = 1.0, sv = 0.0;
            xr = X[row];
            z = a.A.nrows ? mat_row_at(a.A, row, X, ad) : xr;
            if (a.out_mode >= 2) sv = a.B.nrows ? mat_row_at(a.B, row, X, bd) : xr;
            double minv = 1.0;
            if (a.out_mode >= 2) {
                minv = jacobi_minv(ad, bd, a.pmode == 2 ? (a.out_mode == 2 ? rho : theta) : a.sigma, a.mfloor);  // M_ii
            }
            if (a.out_mode == 1) o = z;
            else if (a.out_mode == 2) o = minv * (z - rho * sv);  // w = M (z - rho B g), R1
            else if (a.out_mode == 3) o = z - theta * sv;          // r = A x - theta B x
            if (grp == 0) {
                if (a.out) a.out[row] = o;
                if (a.uout) a.uout[row] = minv * o;
            }
        }
        if (nn && grp == 0) {
            const double p1 = a.norm1 == 1 ? o * o : a.norm1 == 2 ? xr * z : a.norm1 == 3 ? xr * xr : z * z;
            const double p2 = a.norm2 == 1 ? o * o : a.norm2 == 2 ? xr * z : a.norm2 == 3 ? xr * xr : z * z;
            n1 += p1;
            n2 += p2;
        }
        const double v1 = a.set1 == 1 ? z : (a.set1 == 2 ? o : xr);
#pragma unroll
        for (int c = 0; c < KS; ++c) {
            a1[c] = fma(u[c], v1, a1[c]);
            if (TWO) a2[c] = fma(u[c], o, a2[c]);
        }
    }
    // lanes of a group -> lane rr == 0 (fixed butterfly), then per-warp slots
#pragma unroll
    for (int c = 0; c < KS; ++c) {
#pragma unroll
        for (int off = 1; off < TR; off <<= 1) {
            a1[c] += __shfl_xor_sync(0xffffffffu, a1[c], off);
            if (TWO) a2[c] += __shfl_xor_sync(0xffffffffu, a2[c], off);
        }
    }
    if (rr == 0) {
#pragma unroll
        for (int c = 0; c < KS; ++c) {
            if (c0 + c < k1) acc[warp][c0 + c] = a1[c];
            if (TWO && c0 + c < k2) acc[warp][k1 + c0 + c] = a2[c];
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

// ------------------------------------------------------------------ launchers
template <typename K>
static int tp_grid(K kern, int64_t nrows, int tr) {
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (nsm <= 0) nsm = 148;
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, 0);
    if (occ < 1) occ = 1;
    const int64_t need = ((nrows + tr - 1) / tr + WARPS - 1) / WARPS;
    int64_t cap = (int64_t)nsm * occ;
    if (cap > MAXCTA) cap = MAXCTA;
    if (need <= cap) return (int)(need < 1 ? 1 : need);
    const int64_t waves = (need + cap - 1) / cap;
    return (int)((need + waves - 1) / waves);
}

template <int KS, int S, bool TWO>
static void launch_step1_tp_k(const SdotsArgs& a, cudaStream_t s) {
    auto kern = k_step1_tp<KS, S, TWO, false>;
    NOTE_KERN(kern);
    kern<<<tp_grid(kern, a.nrows, 32 / S), CTA, 0, s>>>(a);
}

// Column split by width: k <= 24 one group of KS columns (S = 1); k <= 64 two groups (S = 2).
bool launch_step1_tp(const SdotsArgs& a, int kmax, cudaStream_t s) {
    const bool two = a.set2 != 0;
#define TP1(KS, S) two ? launch_step1_tp_k<KS, S, true>(a, s) : launch_step1_tp_k<KS, S, false>(a, s)
    switch (kmax) {
        case 8: TP1(8, 1); break;
        case 16: TP1(16, 1); break;
        case 24: TP1(24, 1); break;
        case 32: TP1(16, 2); break;
        case 40: TP1(20, 2); break;
        case 48: TP1(24, 2); break;
        case 64: TP1(32, 2); break;
        default: return false;
    }
#undef TP1
    return true;
}

// K2 (CGS pass 2 with dots) with the columns split over a group of G = 2 (k <= 32) or 4 warps ("wp"): warp w of a group
// owns columns [w*KS, w*KS+KS) of the same 32-row tile (lane = row, every column read a full 256-byte
// segment), keeps its KS values of U and KS dot accumulators in registers, and the two halves
// parts of y = x - U h are combined through shared memory behind a group barrier (bar.sync,
// 32 G threads).  All k column loads of a tile are in flight at once with <= 128 registers, so
// k <= 48 runs 2 CTAs (16 warps) per SM -- the register budget the single-warp `tp` misses.
// Two 32-row tiles per warp-group iteration: both tiles' column loads in flight together, one
// group barrier for both, half the dependent load round trips per warp (as k_step1_rs2 for K1;
// the one-tile kernel measured slower and was removed).
template <int KS, int G>
__global__ void __launch_bounds__(CTA, 2) k_upd2_wp2(const UpdArgs a) {
    pdl_wait();
    constexpr int NGR = WARPS / G;
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int kv = a.kv >= 0 ? a.kv : ctl->k;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    __shared__ double hs[G * KS];
    __shared__ double sb[2][NGR][G][64];
    __shared__ double acc[WARPS][QMAX + 1];
    __shared__ double res[QMAX + 1];
    for (int i = threadIdx.x; i < G * KS; i += CTA) hs[i] = i < kv ? ctl->h[a.hslot][i] : 0.0;
    for (int i = threadIdx.x; i < WARPS * (QMAX + 1); i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = warp / G, wg = warp % G;
    const int c0 = wg * KS;
    double d[KS];
#pragma unroll
    for (int c = 0; c < KS; ++c) d[c] = 0.0;
    double yy = 0.0;
    const int64_t ntile = (a.nrows + 31) >> 5;
    const int64_t npair = (ntile + 1) >> 1;
    const double* ub = a.U + (int64_t)c0 * a.ldu;
    int par = 0;
    for (int64_t tp = (int64_t)blockIdx.x * NGR + grp; tp < npair; tp += (int64_t)gridDim.x * NGR) {
        const int64_t r0 = (2 * tp) * 32 + lane, r1 = r0 + 32;
        const bool ok0 = r0 < a.nrows, ok1 = r1 < a.nrows;
        double u0[KS], u1[KS];
#pragma unroll
        for (int c = 0; c < KS; ++c) {
            const bool cv = c0 + c < kv;
            u0[c] = (ok0 && cv) ? __ldg(ub + (int64_t)c * a.ldu + r0) : 0.0;
            u1[c] = (ok1 && cv) ? __ldg(ub + (int64_t)c * a.ldu + r1) : 0.0;
        }
        const double x0 = ok0 ? X[r0] : 0.0, x1 = ok1 ? X[r1] : 0.0;
        double sp0 = 0.0, sp1 = 0.0;
#pragma unroll
        for (int c = 0; c < KS; ++c) {
            sp0 = fma(hs[c0 + c], u0[c], sp0);
            sp1 = fma(hs[c0 + c], u1[c], sp1);
        }
        sb[par][grp][wg][lane] = sp0;
        sb[par][grp][wg][32 + lane] = sp1;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * G) : "memory");
        double s0 = sb[par][grp][0][lane], s1 = sb[par][grp][0][32 + lane];
#pragma unroll
        for (int w = 1; w < G; ++w) {
            s0 += sb[par][grp][w][lane];
            s1 += sb[par][grp][w][32 + lane];
        }
        par ^= 1;
        const double y0 = ok0 ? x0 - s0 : 0.0, y1 = ok1 ? x1 - s1 : 0.0;
        if (wg == 0) {
            if (a.out) {
                if (ok0) a.out[r0] = y0;
                if (ok1) a.out[r1] = y1;
            }
            yy = fma(y0, y0, yy);
            yy = fma(y1, y1, yy);
        }
#pragma unroll
        for (int c = 0; c < KS; ++c) d[c] = fma(u1[c], y1, fma(u0[c], y0, d[c]));
    }
#pragma unroll
    for (int c = 0; c < KS; ++c) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) d[c] += __shfl_xor_sync(0xffffffffu, d[c], off);
    }
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < KS; ++c)
            if (c0 + c < kv) acc[warp][c0 + c] = d[c];
    }
    const double ys = warp_sum(yy);
    __syncthreads();
    if (lane == 0 && wg == 0) acc[warp][kv] = ys;
    __syncthreads();
    const int nv = kv + 1;
    for (int v = threadIdx.x; v < nv; v += CTA) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) sum += acc[w][v];
        res[v] = sum;
    }
    __syncthreads();
    pdl_trigger();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
    } else {
        upd_finalize(a, res, kv);
    }
}

template <int KS, int G>
static void launch_upd2_wp_k(const UpdArgs& a, cudaStream_t s) {
    auto kern2 = k_upd2_wp2<KS, G>;
    NOTE_KERN(kern2);
    launch_pdl(kern2, tp_grid(kern2, (a.nrows + 1) / 2, 8 * G), CTA, 0, s, a);
}

bool launch_upd2_wp(const UpdArgs& a, int kmax, cudaStream_t s) {
    switch (kmax) {
        case 8: launch_upd2_wp_k<4, 2>(a, s); break;
        case 16: launch_upd2_wp_k<8, 2>(a, s); break;
        case 24: launch_upd2_wp_k<12, 2>(a, s); break;
        case 32: launch_upd2_wp_k<16, 2>(a, s); break;
        case 40: launch_upd2_wp_k<10, 4>(a, s); break;
        case 48: launch_upd2_wp_k<12, 4>(a, s); break;
        case 64: launch_upd2_wp_k<16, 4>(a, s); break;
        default: return false;
    }
    return true;
}

}  // namespace trplk
