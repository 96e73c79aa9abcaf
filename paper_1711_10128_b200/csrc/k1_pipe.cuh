// Software-pipelined K1 for DIA matrices with <= 8 diagonals and B = I (C2, C3, C5 shapes):
//   z = A g, w = M (z - rho g) (eq 3.1 + R1), T(1:k,k) = U^T z, h1 = U^T w, ||w||^2.
// Same per-tile arithmetic and summation order as k_step1_rs2 (stream_rs.cuh), but a warp issues the
// basis-row loads AND the DIA value / gather loads of its NEXT tile before it contracts the
// current one (DMMA from the shared-memory slab), so the SpMV's dependent gathers -- the top
// stall of k_step1_rs at C5 in ncu -- overlap a whole tile of work.
// k <= 24 (one slab chunk); wider blocks use k_step1_rs.  Included by kernels.cu after
// stream_rs.cuh (WLD, dmma884_s, warp_sum_s).
#pragma once

namespace trplk {

template <int KMAX, bool TWO>
__global__ void __launch_bounds__(CTA, 2) k_step1_pipe(const SdotsArgs a) {
    pdl_wait();
    static_assert(KMAX <= 24, "one slab chunk");
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    const int kc = ctl->k;
    const int k1 = a.set1 ? (a.k_from_ctl ? kc : a.k1) : 0;
    const int k2 = (TWO && a.set2) ? (a.k_from_ctl ? kc : a.k2) : 0;
    const int kmx = k1 > k2 ? k1 : k2;
    const double rho = ctl->rho;
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 == 5 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const double* __restrict__ X = a.x;
    const double* __restrict__ X2 = a.set2 == 4 ? resolve_x(a.x2, a.x2_dyn, a.x2_ld, a.x2_off, ctl) : nullptr;
    double n2 = 0.0;
    const Sell& M = a.A;
    extern __shared__ __align__(128) double wsm[];  // WARPS x KMAX x WLD
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* W = wsm + (size_t)warp * KMAX * WLD;
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0;
    const int nd = M.ndiag;
    const int nl = (int)M.nrows, top = (int)(M.nrows + M.nghost - 1), glo = (int)M.glo;
    const bool halo = M.nghost != 0;
    const int64_t nslices = (a.nrows + 31) >> 5;
    const int64_t sbeg = a.row0 >> 5;  // first tile of the row range
    const int64_t stride = (int64_t)gridDim.x * WARPS;
    // registers of the tile in flight: basis row, DIA values, gathered x, diagonal, own x
    double ur[KMAX], v[8], xv[8], dg = 0.0, xr = 0.0;
    auto issue = [&](int64_t sl) {
        const int64_t row = sl * 32 + lane;
        const bool ok = sl < nslices && row < a.nrows;
#pragma unroll
        for (int c = 0; c < KMAX; ++c) ur[c] = (ok && c < kmx) ? __ldg(a.U + (int64_t)c * a.ldu + row) : 0.0;
        const double* dv = M.dval + row;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            v[d] = 0.0;
            xv[d] = 0.0;
            if (ok && d < nd) {
                int idx = (int)row + M.offs[d];
                if (halo) idx = idx < 0 ? idx + nl + glo : (idx >= nl ? idx + glo : idx);
                idx = idx < 0 ? 0 : (idx > top ? top : idx);
                v[d] = __ldg(dv + (int64_t)d * M.ldv);
                xv[d] = __ldg(X + idx);
            }
        }
        dg = ok ? __ldg(dv + (int64_t)M.diag_slot * M.ldv) : 1.0;
        xr = ok ? X[row] : 0.0;
    };
    int64_t sl = sbeg + (int64_t)blockIdx.x * WARPS + warp;
    if (sl < nslices) issue(sl);
    for (; sl < nslices; sl += stride) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        // SpMV of this tile (ascending column order, as mat_row)
        double z = 0.0;
#pragma unroll
        for (int d = 0; d < 8; ++d) z = fma(v[d], xv[d], z);
        double o = 0.0;
        if (a.out_mode == 2) {
            o = jacobi_minv(dg, 1.0, a.pmode == 2 ? rho : a.sigma, a.mfloor) * (z - rho * xr);  // w = M (z - rho g), R1
        } else if (a.out_mode == 1) {
            o = z;
        }
        if (ok) {
            if (a.out) a.out[row] = o;
        } else {
            z = 0.0;
            o = 0.0;
        }
        if (a.norm1 == 1) n1 += o * o;
        if (TWO && a.set2 == 4) {  // second dot set on the external vector x2
            const double x2 = ok ? X2[row] : 0.0;
            n2 += x2 * x2;
            o = x2;
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < KMAX; ++c) W[c * WLD + lane] = ur[c];
        __syncwarp();
        if (sl + stride < nslices) issue(sl + stride);  // next tile's loads fly during the DMMAs
        const double v1 = a.set1 == 1 ? z : o;
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, v1, 4 * q + fj);
            const double t2 = TWO ? __shfl_sync(0xffffffffu, o, 4 * q + fj) : 0.0;
            bq[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
        }
        // (interleaving the chunks' DMMA chains measured 1 % slower here: 4.84 vs 4.79 ms at C5)
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            if (8 * g < kmx) {
                const double* sp = W + (8 * g + fi) * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(cacc[g], sp[4 * q], bq[q]);
            }
        }
        __syncwarp();
    }
    for (int i = threadIdx.x; i < WARPS * NV_MAX; i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (fj == 0) {
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            const int c = 8 * g + fi;
            if (c < k1) acc[warp][c] = cacc[g][0];
            if (TWO && c < k2) acc[warp][k1 + c] = cacc[g][1];
        }
    }
    if (nn) {
        const double s1 = warp_sum_s(n1);
        if (lane == 0 && a.norm1) acc[warp][k1 + k2] = s1;
        if (a.norm2 == 5) {
            const double s2 = warp_sum_s(n2);
            if (lane == 0) acc[warp][k1 + k2 + (a.norm1 ? 1 : 0)] = s2;
        }
    }
    if (nv == 0) return;
    __syncthreads();
    for (int vv = threadIdx.x; vv < nv; vv += CTA) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s += acc[w][vv];
        res[vv] = s;
    }
    __syncthreads();
    pdl_trigger();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res, a.cta_off, a.cta_tot)) return;
    if (a.red_local) {
        for (int vv = threadIdx.x; vv < nv; vv += CTA) a.red_local[vv] = res[vv];
    } else {
        sdots_finalize(a, res, k1, k2);
    }
}

template <int KMAX, bool TWO>
static void launch_step1_pipe_k(const SdotsArgs& a, cudaStream_t s) {
    const int smem = WARPS * KMAX * WLD * (int)sizeof(double);
    auto kern = k_step1_pipe<KMAX, TWO>;
    NOTE_KERN(kern);
    launch_pdl(kern, a.grid_force > 0 ? a.grid_force : rs_grid(kern, smem, a.nrows - a.row0), CTA, smem, s, a);
}

bool launch_step1_pipe(const SdotsArgs& a, int kmax, cudaStream_t s) {
    if (a.A.fmt != 1 || a.A.ndiag > 8 || a.B.nrows || a.out_mode > 2 || a.norm1 > 1 || (a.norm2 != 0 && a.norm2 != 5))
        return false;
    const bool two = a.set2 != 0;
    switch (kmax) {
        case 8: two ? launch_step1_pipe_k<8, true>(a, s) : launch_step1_pipe_k<8, false>(a, s); break;
        case 16: two ? launch_step1_pipe_k<16, true>(a, s) : launch_step1_pipe_k<16, false>(a, s); break;
        case 24: two ? launch_step1_pipe_k<24, true>(a, s) : launch_step1_pipe_k<24, false>(a, s); break;
        default: return false;
    }
    return true;
}

}  // namespace trplk
