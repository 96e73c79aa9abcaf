// Small-n latency path: the m inner steps of one cycle (eq 3.1, PAPER.md:
// 133-143, with the Jacobi preconditioner of P:143 as reading R1 and CGS2 as R3) in ONE CTA.
//
// For a problem whose rows fit one CTA's threads a few times over (C1: n = 1,000), the
// inner step is latency-bound: three grid-wide reductions per step cost more than the data.
// Here one 256-thread CTA owns every row (row = tid + 256 i), the basis stays in L1/L2, and
// every reduction is a block reduction (warp butterflies + shared memory) -- the three kernel
// launches and three grid reductions of a step become three __syncthreads-separated phases:
//   1  z = A g, w = M (z - rho g), T(1:k,k) = U^T z, h1 = U^T w, ||w||^2
//   2  w' = w - U h1, h2 = U^T w', ||w'||^2
//   3  beta^2 = ||w'||^2 - ||h2||^2 (Pythagoras), g_{j+1} = (w' - U h2) / beta, or a third pass
//      (h3 = U^T w'', ...) when the second pass lost more than half the norm, or a breakdown
//      (flag cleared, the inner loop stops with the columns built so far, R16).
// Same readings and decisions as the multi-kernel path; one rank, B = I.  Included by
// kernels.cu (mat_row, warp_butterfly, warp_sum).
#pragma once

namespace trplk {

constexpr int SMALL_CTA = 256;
constexpr int SMALL_WARPS = SMALL_CTA / 32;

// Block sum of NV8 * 8 per-thread values (v[i] = 0 beyond the live count): warp butterflies in
// chunks of 8, per-warp partials in shared memory, warps summed in index order.
template <int NV8>
__device__ __forceinline__ void small_block_sum(double (&v)[NV8 * 8], double (*sacc)[NV8 * 8], double* out, int nv) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < NV8; ++c) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = v[8 * c + u];
        warp_butterfly<3>(t, lane);
        if ((lane & 3) == 0) sacc[warp][8 * c + ((lane >> 2) & 7)] = t[0];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nv; i += SMALL_CTA) {
        double s = 0.0;
        for (int w = 0; w < SMALL_WARPS; ++w) s += sacc[w][i];
        out[i] = s;
    }
    __syncthreads();
}

template <int KMAX>
__global__ void __launch_bounds__(SMALL_CTA, 1) k_inner_small(const SmallArgs a) {
    constexpr int NV8 = (2 * KMAX + 1 + 7) / 8;  // 2k+1 values of phase 1, in chunks of 8
    constexpr int NW8 = (KMAX + 1 + 7) / 8;      // k+1 values of phases 2 and 3
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    __shared__ double sacc[SMALL_WARPS][NV8 * 8];
    __shared__ double red[NV8 * 8];
    __shared__ int sk, sbrk;
    const int tid = threadIdx.x;
    if (tid == 0) {
        sk = ctl->k;
        sbrk = 0;
    }
    __syncthreads();
    const double rho = ctl->rho;
    const int64_t n = a.nrows;
    for (int j = 1; j <= a.m; ++j) {
        const int k = sk;
        const double* g = a.U + (int64_t)(k - 1) * a.ldu;
        const bool cgs = j < a.m;
        // ---- phase 1: SpMV + preconditioner + T column / h1 / ||w||^2
        {
        double v[NV8 * 8];
#pragma unroll
        for (int i = 0; i < NV8 * 8; ++i) v[i] = 0.0;
        for (int64_t row = tid; row < n; row += SMALL_CTA) {
            double ad = 1.0;
            const double z = mat_row(a.A, row >> 5, (int)(row & 31), g, ad);
            const double w = jacobi_minv(ad, 1.0, a.pmode == 2 ? rho : a.sigma, a.mfloor) * (z - rho * g[row]);  // w = M (z - rho g), R1
            if (cgs) a.w[row] = w;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) {
                if (c < k) {
                    const double u = a.U[(int64_t)c * a.ldu + row];
                    v[c] = fma(u, z, v[c]);
                    if (cgs) v[KMAX + c] = fma(u, w, v[KMAX + c]);
                }
            }
            if (cgs) v[2 * KMAX] = fma(w, w, v[2 * KMAX]);
        }
        small_block_sum<NV8>(v, sacc, red, 2 * KMAX + 1);
        }
        for (int i = tid; i < k; i += SMALL_CTA) {  // T(1:k,k), mirrored (eq 3.1)
            a.T[i + (int64_t)(k - 1) * a.ldT] = red[i];
            a.T[(k - 1) + (int64_t)i * a.ldT] = red[i];
        }
        if (!cgs) break;
        // ---- phase 2: w' = w - U h1, h2 = U^T w', ||w'||^2
        double hr[KMAX];
#pragma unroll
        for (int c = 0; c < KMAX; ++c) hr[c] = c < k ? red[KMAX + c] : 0.0;
        const double nin2 = red[2 * KMAX];
        __syncthreads();  // red is rewritten below
        double v[NW8 * 8];
#pragma unroll
        for (int i = 0; i < NW8 * 8; ++i) v[i] = 0.0;
        for (int64_t row = tid; row < n; row += SMALL_CTA) {
            double y = a.w[row];
            double u[KMAX];
#pragma unroll
            for (int c = 0; c < KMAX; ++c) u[c] = c < k ? a.U[(int64_t)c * a.ldu + row] : 0.0;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) y = fma(-hr[c], u[c], y);
            a.w1[row] = y;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) v[c] = fma(u[c], y, v[c]);
            v[KMAX] = fma(y, y, v[KMAX]);
        }
        small_block_sum<NW8>(v, reinterpret_cast<double(*)[NW8 * 8]>(&sacc[0][0]), red, KMAX + 1);
        double hn = 0.0;
#pragma unroll
        for (int c = 0; c < KMAX; ++c) {
            hr[c] = c < k ? red[c] : 0.0;
            hn += hr[c] * hr[c];
        }
        const double n1sq = red[KMAX];
        __syncthreads();
        // ---- phase 3: FINAL (R3 decisions as k_upd FINAL / FIX)
        const double nin = sqrt(nin2);
        const double n2sq = n1sq - hn;
        const bool pass3 = !(n2sq >= 0.5 * n1sq) || a.force3;
        const double* src = a.w1;
        double b = sqrt(n2sq > 0.0 ? n2sq : 0.0);
        if (pass3) {
#pragma unroll
            for (int i = 0; i < NW8 * 8; ++i) v[i] = 0.0;
            for (int64_t row = tid; row < n; row += SMALL_CTA) {
                double y = a.w1[row];
                double u[KMAX];
#pragma unroll
                for (int c = 0; c < KMAX; ++c) u[c] = c < k ? a.U[(int64_t)c * a.ldu + row] : 0.0;
#pragma unroll
                for (int c = 0; c < KMAX; ++c) y = fma(-hr[c], u[c], y);
                a.w2[row] = y;
#pragma unroll
                for (int c = 0; c < KMAX; ++c) v[c] = fma(u[c], y, v[c]);
                v[KMAX] = fma(y, y, v[KMAX]);
            }
            small_block_sum<NW8>(v, reinterpret_cast<double(*)[NW8 * 8]>(&sacc[0][0]), red, KMAX + 1);
            hn = 0.0;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) {
                hr[c] = c < k ? red[c] : 0.0;
                hn += hr[c] * hr[c];
            }
            const double n3sq = red[KMAX] - hn;
            b = sqrt(n3sq > 0.0 ? n3sq : 0.0);
            src = a.w2;
            if (tid == 0) {
                for (int i = 0; i < k; ++i) ctl->h[2][i] = red[i];
                ctl->nrm[N_2SQ_EXP] = red[KMAX];
                ctl->pass3_count += 1;
            }
            __syncthreads();
        }
        const bool brk = !(b >= 1e-14 * nin) || nin == 0.0;
        if (brk) {  // inner breakdown (R16): stop with the columns built so far
            if (tid == 0) {
                ctl->flags &= ~a.clear;
                ctl->brk += 1;
            }
            break;
        }
        const double binv = 1.0 / b;
        double* dst = a.U + (int64_t)k * a.ldu;
        for (int64_t row = tid; row < n; row += SMALL_CTA) {
            double y = src[row];
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < k) y = fma(-hr[c], a.U[(int64_t)c * a.ldu + row], y);
            dst[row] = y * binv;
        }
        if (tid == 0) sk = k + 1;
        __syncthreads();  // g_{j+1} complete before the next SpMV gathers it
    }
    if (tid == 0) ctl->k = sk;
}

template <int KMAX>
static void launch_small_k(const SmallArgs& a, cudaStream_t s) {
    NOTE_KERN(k_inner_small<KMAX>);
    k_inner_small<KMAX><<<1, SMALL_CTA, 0, s>>>(a);
}

bool launch_inner_small(const SmallArgs& a, int kmax, cudaStream_t s) {
    if (a.nrows > SMALL_NMAX) return false;
    if (kmax <= 16) launch_small_k<16>(a, s);
    else if (kmax <= 24) launch_small_k<24>(a, s);
    else return false;  // wider blocks: the per-thread partial sums no longer fit the registers
    return true;
}

}  // namespace trplk
