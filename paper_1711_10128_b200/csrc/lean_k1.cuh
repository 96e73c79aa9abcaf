// Thread-per-row inner-step K1 for DIA matrices (<= 8 diagonals, DIA-C aware), B = I, k <= 24
// (k_step1_lean):  z = A g, w = M (z - rho g), T(1:k,k) = U^T z, h1 = U^T w, ||w||^2
// (eq 3.1; R1 at P:143; R3 pass-1 coefficients).
//
// Lane = row of a 32-row tile; every lane keeps the k values of its basis row and the 2k dot
// accumulators in registers for the whole kernel and adds its rows in row order (FMA, no
// tensor core: the two dot vectors would fill 2 of the 8 DMMA columns), so the cross-lane
// reduction (xor butterfly) runs once per kernel instead of a shared-memory transpose and DMMA
// chain per tile.  All loads of a tile -- k basis values, the DIA values / presence word and
// the gathers -- are issued before any arithmetic; PF additionally keeps the next tile's basis
// row in flight during this tile's SpMV.  <= 128 registers: 2 CTAs (16 warps) per SM.
// Included by kernels.cu after stream_rs.cuh (grid_reduce, sdots_finalize, warp_sum_s).
#pragma once

namespace trplk {

template <int KMAX, bool TWO, bool PF>
__global__ void __launch_bounds__(CTA, 2) k_step1_lean(const SdotsArgs a) {
    pdl_wait();
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int kc = ctl->k;
    const int k1 = a.k_from_ctl ? kc : a.k1;
    const int k2 = TWO ? (a.k_from_ctl ? kc : a.k2) : 0;
    const int kmx = k1 > k2 ? k1 : k2;
    const double rho = ctl->rho;
    const int nn = a.norm1 ? 1 : 0;
    const int nv = k1 + k2 + nn;
    const double* __restrict__ X = a.x;
    const Sell& M = a.A;
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    __shared__ double cv_s[8];
    if (threadIdx.x < 8)
        cv_s[threadIdx.x] = (threadIdx.x < M.ndiag && ((M.cmask >> threadIdx.x) & 1u)) ? M.cv[threadIdx.x] : 0.0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nd = M.ndiag;
    const int top = (int)(M.nrows + M.nghost - 1), nl = (int)M.nrows, glo = (int)M.glo;
    const bool halo = M.nghost != 0;
    const double shift = a.pmode == 2 ? rho : a.sigma;
    double a1[KMAX], a2[TWO ? KMAX : 1];
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
        a1[c] = 0.0;
        if (TWO) a2[c] = 0.0;
    }
    double n1 = 0.0;
    const int64_t nsl = (a.nrows + 31) >> 5;
    const int64_t stride = (int64_t)gridDim.x * WARPS;
    double un[PF ? KMAX : 1];
    int64_t sl = (int64_t)blockIdx.x * WARPS + warp;
    if (PF && sl < nsl) {
        const int64_t row = sl * 32 + lane;
#pragma unroll
        for (int c = 0; c < KMAX; ++c) un[c] = (row < a.nrows && c < kmx) ? __ldg(a.U + (int64_t)c * a.ldu + row) : 0.0;
    }
    for (; sl < nsl; sl += stride) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        double u[KMAX];
        if (PF) {
            const int64_t rn = row + stride * 32;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) {
                u[c] = un[c];
                un[c] = (rn < a.nrows && c < kmx) ? __ldg(a.U + (int64_t)c * a.ldu + rn) : 0.0;
            }
        } else {
#pragma unroll
            for (int c = 0; c < KMAX; ++c) u[c] = (ok && c < kmx) ? __ldg(a.U + (int64_t)c * a.ldu + row) : 0.0;
        }
        double z = 0.0, o = 0.0;
        if (ok) {
            const double* dv = M.dval + row;
            const unsigned pm = M.cmask ? dia_pmask(M, row) : 0u;
            double v[8], xv[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                v[d] = 0.0;
                xv[d] = 0.0;
                if (d < nd) {
                    int idx = (int)row + M.offs[d];
                    if (halo) idx = idx < 0 ? idx + nl + glo : (idx >= nl ? idx + glo : idx);
                    idx = idx < 0 ? 0 : (idx > top ? top : idx);  // out-of-matrix slots hold 0
                    if (!((M.cmask >> d) & 1u)) v[d] = __ldg(dv + (int64_t)d * M.ldv);
                    xv[d] = __ldg(X + idx);
                }
            }
            double dg = ((M.cmask >> M.diag_slot) & 1u) ? (((pm >> M.diag_slot) & 1u) ? cv_s[M.diag_slot] : 0.0)
                                                       : __ldg(dv + (int64_t)M.diag_slot * M.ldv);
            const double xr = __ldg(X + row);
#pragma unroll
            for (int d = 0; d < 8; ++d)
                if (d < nd && ((M.cmask >> d) & 1u)) v[d] = ((pm >> d) & 1u) ? cv_s[d] : 0.0;
#pragma unroll
            for (int d = 0; d < 8; ++d) z = fma(v[d], xv[d], z);  // ascending diagonal order (mat_row)
            if (a.out_mode == 2) {
                o = jacobi_minv(dg, 1.0, shift, a.mfloor) * (z - rho * xr);  // w = M (z - rho g), R1
                if (a.out) a.out[row] = o;
            }
        }
        if (a.norm1 == 1) n1 += o * o;
#pragma unroll
        for (int c = 0; c < KMAX; ++c) {
            a1[c] = fma(u[c], z, a1[c]);
            if (TWO) a2[c] = fma(u[c], o, a2[c]);
        }
    }
    // lanes -> lane 0 (fixed xor butterfly), warps in index order, CTAs by grid_reduce
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
        a1[c] = warp_sum_s(a1[c]);
        if (TWO) a2[c] = warp_sum_s(a2[c]);
    }
    n1 = warp_sum_s(n1);
    for (int i = threadIdx.x; i < WARPS * NV_MAX; i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < KMAX; ++c) {
            if (c < k1) acc[warp][c] = a1[c];
            if (TWO && c < k2) acc[warp][k1 + c] = a2[c];
        }
        if (nn) acc[warp][k1 + k2] = n1;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += CTA) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s += acc[w][v];
        res[v] = s;
    }
    __syncthreads();
    pdl_trigger();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
    } else {
        sdots_finalize(a, res, k1, k2);
    }
}

template <int KMAX, bool TWO, bool PF>
static void launch_step1_lean_k(const SdotsArgs& a, cudaStream_t s) {
    auto kern = k_step1_lean<KMAX, TWO, PF>;
    NOTE_KERN(kern);
    launch_pdl(kern, rs_grid(kern, 0, a.nrows), CTA, 0, s, a);
}

bool kern_reads_diac(const void* k) {
    const void* ks[] = {
        (const void*)k_step1_lean<8, true, true>,    (const void*)k_step1_lean<8, false, true>,
        (const void*)k_step1_lean<16, true, false>,  (const void*)k_step1_lean<16, false, false>,
        (const void*)k_step1_lean<24, true, false>,  (const void*)k_step1_lean<24, false, false>,
        (const void*)k_fin_step1<8>,  (const void*)k_fin_step1<16>, (const void*)k_fin_step1<24>,
        (const void*)k_fin_step1<32>, (const void*)k_fin_step1<40>, (const void*)k_fin_step1<48>};
    for (const void* x : ks)
        if (x == k) return true;
    return false;
}

// DIA (<= 8 diagonals), B = I, out_mode 0 / 2, ||w||^2 only; k <= 24.  PF for k <= 16.
bool launch_step1_lean(const SdotsArgs& a, int kmax, cudaStream_t s) {
    if (a.A.fmt != 1 || a.A.ndiag > 8 || a.B.nrows || a.out_mode == 1 || a.out_mode > 2 || a.norm1 > 1 ||
        a.set1 != 1 || (a.set2 != 0 && a.set2 != 2) || a.x_dyn != 0)
        return false;
    const bool two = a.set2 != 0;
    switch (kmax) {
        case 8: two ? launch_step1_lean_k<8, true, true>(a, s) : launch_step1_lean_k<8, false, true>(a, s); break;
        case 16: two ? launch_step1_lean_k<16, true, false>(a, s) : launch_step1_lean_k<16, false, false>(a, s); break;
        case 24: two ? launch_step1_lean_k<24, true, false>(a, s) : launch_step1_lean_k<24, false, false>(a, s); break;
        default: return false;
    }
    return true;
}

}  // namespace trplk
