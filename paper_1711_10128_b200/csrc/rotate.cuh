// K5 rotation X = U Y(:, 1:p^) (Alg.1 steps 11/15) on fp64 DMMA with the
// basis tile staged through shared memory ("s" variant, default).
//
// A warp owns a 32-row tile: lane = row, it issues the loads of all k basis columns at once
// (each load instruction one column's contiguous 256 bytes), parks the tile in a private
// shared-memory slab (column stride WLD = 36 doubles), then forms X^T = Y^T U^T per 8-row
// block with mma.sync.m8n8k4.f64: the A operand (Y^T, <= 3 x 16 fragments) stays in registers
// for the whole kernel, the B operand (U^T: lane (kk, n) = U[8 rb + n, 4 ks + kk]) comes from
// the slab, and the accumulator holds 2 consecutive rows of one output column per lane,
// written as one 16-byte store.  For KMAX >= 32 the slab is double-buffered and filled by
// cp.async, so the next tile streams in during the current tile's DMMA (round 2; measured alone:
// C3 k = 32 3.98 -> 4.54 TB/s, k = 48 3.83 -> 3.88, C2 k = 30 1.51 -> 1.58; narrower bases keep
// the register-staged single slab, two CTAs per SM: C5 k = 24 5.43 TB/s against 4.91 pipelined).
// The ncu capture of the register-fragment version at C5 showed
// lg_throttle + long_scoreboard stalls: its loads touched 4 columns x 64 bytes per instruction.
// Included by kernels.cu after stream_rs.cuh (WLD, dmma884_s).
#pragma once

namespace trplk {

template <int NJ, int KMAX>
__global__ void __launch_bounds__(CTA, (NJ * KMAX > 64 || KMAX >= 32) ? 1 : 2) k_rotate_s(const double* __restrict__ U, int64_t ldu, int64_t nrows,
                                                     const Ctl* ctl, int k_fixed, const double* __restrict__ Y,
                                                     int ldY, int ncol, double* __restrict__ X, int64_t ldx,
                                                     unsigned gate) {
    constexpr int KS4 = KMAX / 4;
    if ((ctl->flags & gate) != gate) return;
    const int k = k_fixed > 0 ? k_fixed : ctl->k_rr;
    extern __shared__ __align__(128) double wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lq = lane & 3, lr = lane >> 2;
    double* W = wsm + (size_t)warp * KMAX * WLD;
    double yf[NJ][KS4];
#pragma unroll
    for (int jb = 0; jb < NJ; ++jb)
#pragma unroll
        for (int ks = 0; ks < KS4; ++ks) {
            const int kk = 4 * ks + lq, j = 8 * jb + lr;
            yf[jb][ks] = (kk < k && j < ncol) ? __ldg(Y + kk + (int64_t)j * ldY) : 0.0;
        }
    const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && ((ldx & 1) == 0);
    const int64_t ntile = (nrows + 31) >> 5;
    const int64_t tstride = (int64_t)gridDim.x * WARPS;
    // KMAX >= 32: two slabs per warp, filled by cp.async (LDGSTS, no register staging): the next
    // tile's KMAX x 256 B are in flight while the current one goes through the DMMA.  Columns >= k
    // and rows >= nrows are zero-filled (src-size 0).  KMAX < 32: one slab filled through
    // registers, two CTAs per SM (measured: C5 k = 24 rotation 5.4 TB/s against 4.9 pipelined,
    // C3 k = 32 4.5 against 4.0 the other way; profiles/r02_variants.md).
    constexpr bool PIPE = KMAX >= 32;
    auto fill = [&](int64_t t, double* Wb) {
        const int64_t row = t * 32 + lane;
        const bool ok = row < nrows;
#pragma unroll
        for (int c = 0; c < KMAX; ++c) {
            const bool v = ok && c < k;
            const double* src = v ? U + (int64_t)c * ldu + row : U;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(Wb + c * WLD + lane);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int64_t t = (int64_t)blockIdx.x * WARPS + warp;
    if (PIPE && t < ntile) fill(t, W);
    for (int it = 0; t < ntile; t += tstride, ++it) {
        const int64_t r0 = t * 32;
        double* Wc = PIPE ? W + (it & 1) * (WARPS * KMAX * WLD) : W;
        if (PIPE) {
            if (t + tstride < ntile) {
                fill(t + tstride, W + ((it + 1) & 1) * (WARPS * KMAX * WLD));
                asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            }
        } else {
            const int64_t row = r0 + lane;
            const bool ok = row < nrows;
            double ur[PIPE ? 1 : KMAX];
#pragma unroll
            for (int c = 0; c < (PIPE ? 1 : KMAX); ++c) ur[c] = (ok && c < k) ? __ldg(U + (int64_t)c * ldu + row) : 0.0;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < (PIPE ? 1 : KMAX); ++c) W[c * WLD + lane] = ur[c];
        }
        __syncwarp();
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
            double acc[NJ][2];
#pragma unroll
            for (int jb = 0; jb < NJ; ++jb) acc[jb][0] = acc[jb][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS4; ++ks) {
                const double b = Wc[(4 * ks + lq) * WLD + 8 * rb + lr];
#pragma unroll
                for (int jb = 0; jb < NJ; ++jb) dmma884_s(acc[jb], yf[jb][ks], b);
            }
            const int64_t rr = r0 + 8 * rb + 2 * lq;
#pragma unroll
            for (int jb = 0; jb < NJ; ++jb) {
                const int j = 8 * jb + lr;
                if (j < ncol) {
                    double* xp = X + (int64_t)j * ldx + rr;
                    if (vec && rr + 1 < nrows) {
                        *reinterpret_cast<double2*>(xp) = make_double2(acc[jb][0], acc[jb][1]);
                    } else {
                        if (rr < nrows) xp[0] = acc[jb][0];
                        if (rr + 1 < nrows) xp[1] = acc[jb][1];
                    }
                }
            }
        }
        __syncwarp();  // every lane is done with Wc before the next iteration refills it
    }
}

template <int NJ, int KMAX>
static void rot_s(const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed, const double* Y,
                  int ldY, int ncol, double* X, int64_t ldx, unsigned gate, cudaStream_t s) {
    auto kern = k_rotate_s<NJ, KMAX>;
    const int smem = (KMAX >= 32 ? 2 : 1) * WARPS * KMAX * WLD * (int)sizeof(double);  // KMAX >= 32: two slabs per warp
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 1, nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, smem);
    if (occ < 1) occ = 1;
    const int64_t need = ((nrows + 31) / 32 + WARPS - 1) / WARPS;
    int64_t g = (int64_t)nsm * occ;
    if (need < g) g = need;
    if (g < 1) g = 1;
    NOTE_KERN(kern);
    kern<<<(int)g, CTA, smem, s>>>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate);
}

template <int NJ>
static bool rot_s_k(int kmax, const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed,
                    const double* Y, int ldY, int ncol, double* X, int64_t ldx, unsigned gate, cudaStream_t s) {
    if (kmax <= 8) rot_s<NJ, 8>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else if (kmax <= 16) rot_s<NJ, 16>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else if (kmax <= 24) rot_s<NJ, 24>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else if (kmax <= 32) rot_s<NJ, 32>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else if (kmax <= 48) rot_s<NJ, 48>(U, ldu, nrows, ctl, k_fixed, Y, ldY, ncol, X, ldx, gate, s);
    else return false;
    return true;
}

}  // namespace trplk
