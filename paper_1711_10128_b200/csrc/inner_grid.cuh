// Mid-size latency path: the m inner steps of one cycle (eq 3.1; Jacobi
// preconditioner R1, CGS2 with Pythagorean beta and gated third pass R3, breakdown R16) in ONE
// cooperative launch of one 512-thread CTA per SM.
//
// Below a few million rows the multi-kernel inner step (K1, K2, K3: three launches and three
// last-CTA grid reductions) spends as long on launch, ramp, tail and reduction as on moving
// bytes (C2, 262k rows: ~55 us per step for ~150 MB).  Here every kernel boundary becomes a
// grid barrier and every grid reduction an all-reduce that each CTA finishes by itself:
//   phase 1   z = A g, w = M (z - rho g), CTA partials of U^T z, U^T w, ||w||^2  -> all-reduce
//             (CTA 0 writes T(1:k,k), mirrored)
//   phase 2   w' = w - U h1, partials of U^T w', ||w'||^2                      -> all-reduce
//   [pass 3   w'' = w' - U h2, partials of U^T w'', ||w''||^2                  -> all-reduce]
//   final     g_{j+1} = (w' - U h) / beta                                      -> grid barrier
// Every CTA sums the CTA partials in the same fixed order, so all CTAs hold bit-identical
// totals and take the same third-pass / breakdown decisions without a broadcast.  The dot
// products use the DMMA fragment scheme of k_step1_rs2 (stream_rs.cuh): each warp parks its
// 32-row tile of U in a shared-memory slab (row layout in registers -> fragment order).
// Vectors written inside the launch (w, w', the new basis columns, the partials) are read
// with ld.global.cg, never through the read-only path.  One rank, B = I, k <= 32.
// Included by kernels.cu after stream_rs.cuh (mat_row, dmma884_s, WLD, rs_chunk, warp_sum_s).
#pragma once

namespace trplk {

constexpr int GW = 16;               // warps per CTA
constexpr int GCTA = GW * 32;        // one CTA per SM
constexpr int GNVP = GRID_NVP;       // partial stride (nv <= 2 * 32 + 1)
constexpr int GSPLIT = 8;            // CTA ranges summed in parallel by the all-reduce

// All-reduce of the CTA sums res[0..nv) over the grid; res holds the totals on return in
// every CTA.  Fixed order: GSPLIT contiguous CTA ranges, each summed in CTA order, then the
// ranges in order.  `part` alternates between two buffers (the caller flips it) so a CTA that
// runs ahead cannot overwrite partials another CTA is still reading.
__device__ __forceinline__ void grid_allreduce(double* res, int nv, double* part, double (*tmp)[GNVP],
                                               double* stage) {
    for (int v = threadIdx.x; v < nv; v += GCTA) part[(size_t)blockIdx.x * GNVP + v] = res[v];
    cooperative_groups::this_grid().sync();
    const int G = gridDim.x, chunk = (G + GSPLIT - 1) / GSPLIT;
    // all G x nv partials into shared memory first: independent loads, all in flight at once
    const int tot = G * nv;
#pragma unroll 4
    for (int t = threadIdx.x; t < tot; t += GCTA) {
        const int b = t / nv;
        stage[t] = __ldcg(part + (size_t)b * GNVP + (t - b * nv));
    }
    __syncthreads();
    for (int t = threadIdx.x; t < GSPLIT * nv; t += GCTA) {
        const int c = t / nv, v = t - c * nv;
        const int b1 = min(G, (c + 1) * chunk);
        double s = 0.0;
        for (int b = c * chunk; b < b1; ++b) s += stage[b * nv + v];
        tmp[c][v] = s;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += GCTA) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < GSPLIT; ++c) s += tmp[c][v];
        res[v] = s;
    }
    __syncthreads();
}

// Warp DMMA accumulators -> CTA sums: res[0..k) = set 1, res[k..2k) = set 2 (if two), then the
// per-warp scalar `nrm` at res[nv - 1].  Warps summed in index order.
template <int KMAX>
__device__ __forceinline__ void grid_cta_sums(const double (&cacc)[KMAX / 8][2], double nrm, int k, bool two,
                                              bool with_nrm, double (*acc)[GNVP], double* res) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, fi = lane >> 2, fj = lane & 3;
    const int nv = (two ? 2 * k : k) + (with_nrm ? 1 : 0);
    if (fj == 0) {
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            const int c = 8 * g + fi;
            if (c < k) {
                acc[warp][c] = cacc[g][0];
                if (two) acc[warp][k + c] = cacc[g][1];
            }
        }
    }
    if (with_nrm) {
        const double s = warp_sum_s(nrm);
        if (lane == 0) acc[warp][nv - 1] = s;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += GCTA) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < GW; ++w) s += acc[w][v];
        res[v] = s;
    }
    __syncthreads();
}

// Phase 1 of inner step j: SpMV + preconditioner + dots (k_step1_rs arithmetic, B = I).
template <int KMAX>
__device__ __forceinline__ void grid_phase1(const SmallArgs& a, int k, bool cgs, double rho, const double* g,
                                            double* W, double (*acc)[GNVP], double* res) {
    constexpr int CH = rs_chunk(KMAX);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, fi = lane >> 2, fj = lane & 3;
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int q = 0; q < KMAX / 8; ++q) cacc[q][0] = cacc[q][1] = 0.0;
    double n1 = 0.0;
    const int64_t nsl = (a.nrows + 31) >> 5;
    for (int64_t sl = (int64_t)blockIdx.x * GW + warp; sl < nsl; sl += (int64_t)gridDim.x * GW) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        const double* up = a.U + row;
        double ur[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) ur[c] = (ok && c < k) ? __ldcg(up + (int64_t)c * a.ldu) : 0.0;
        double ad = 1.0;
        double z = mat_row<false>(a.A, sl, lane, g, ad);
        const double xr = ok ? __ldcg(g + row) : 0.0;
        double o = jacobi_minv(ad, 1.0, a.pmode == 2 ? rho : a.sigma, a.mfloor) * (z - rho * xr);  // w = M (z - rho g), R1
        if (!ok) {
            z = 0.0;
            o = 0.0;
        }
        if (cgs) {
            if (ok) a.w[row] = o;
            n1 = fma(o, o, n1);
        }
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, z, 4 * q + fj);
            const double t2 = __shfl_sync(0xffffffffu, o, 4 * q + fj);
            bq[q] = fi == 0 ? t1 : ((fi == 1 && cgs) ? t2 : 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {
            const bool more = cb + CH < KMAX && cb + CH < k;
            if (more) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int cc = cb + CH + c;
                    ur[c] = (ok && cc < k && cc < KMAX) ? __ldcg(up + (int64_t)cc * a.ldu) : 0.0;
                }
            }
            if (cb < k) {
#pragma unroll
                for (int q8 = cb / 8; q8 < (cb + CH) / 8 && q8 < KMAX / 8; ++q8) {
                    if (8 * q8 < k) {
                        const double* sp = W + (8 * q8 - cb + fi) * WLD + fj;
#pragma unroll
                        for (int q = 0; q < 8; ++q) dmma884_s(cacc[q8], sp[4 * q], bq[q]);
                    }
                }
            }
            if (more) {
                __syncwarp();
#pragma unroll
                for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
                __syncwarp();
            }
        }
    }
    grid_cta_sums<KMAX>(cacc, n1, k, cgs, cgs, acc, res);
}

// A CGS pass: y = x - U h (columns in order), y written to `yout`; CTA sums of U^T y, ||y||^2.
template <int KMAX>
__device__ __forceinline__ void grid_pass(const SmallArgs& a, int k, const double* x, const double* hs, double* yout,
                                          double* W, double (*acc)[GNVP], double* res) {
    constexpr int CH = KMAX < 24 ? KMAX : 24;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, fi = lane >> 2, fj = lane & 3;
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int q = 0; q < KMAX / 8; ++q) cacc[q][0] = cacc[q][1] = 0.0;
    double yy = 0.0;
    const int64_t nsl = (a.nrows + 31) >> 5;
    for (int64_t sl = (int64_t)blockIdx.x * GW + warp; sl < nsl; sl += (int64_t)gridDim.x * GW) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        const double* up = a.U + row;
        double y = ok ? __ldcg(x + row) : 0.0;
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {
            if (cb < k) {
                double ur[CH];
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    ur[c] = (ok && cb + c < k && cb + c < KMAX) ? __ldcg(up + (int64_t)(cb + c) * a.ldu) : 0.0;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (cb + c < KMAX) {
                        y = fma(-hs[cb + c], ur[c], y);
                        W[(cb + c) * WLD + lane] = ur[c];
                    }
            }
        }
        if (!ok) y = 0.0;
        if (ok) yout[row] = y;
        yy = fma(y, y, yy);
        __syncwarp();
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t = __shfl_sync(0xffffffffu, y, 4 * q + fj);
            bq[q] = fi == 0 ? t : 0.0;
        }
#pragma unroll
        for (int q8 = 0; q8 < KMAX / 8; ++q8) {
            if (8 * q8 < k) {
                const double* sp = W + (8 * q8 + fi) * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(cacc[q8], sp[4 * q], bq[q]);
            }
        }
    }
    grid_cta_sums<KMAX>(cacc, yy, k, false, true, acc, res);
}

// g_{j+1} = (x - U h) * binv into column k of U (thread per row, columns in order).
template <int KMAX>
__device__ __forceinline__ void grid_final(const SmallArgs& a, int k, const double* x, const double* hs,
                                           double binv) {
    double* dst = a.U + (int64_t)k * a.ldu;
    for (int64_t row = (int64_t)blockIdx.x * GCTA + threadIdx.x; row < a.nrows; row += (int64_t)gridDim.x * GCTA) {
        double u[KMAX];
#pragma unroll
        for (int c = 0; c < KMAX; ++c) u[c] = c < k ? __ldcg(a.U + (int64_t)c * a.ldu + row) : 0.0;
        double y = __ldcg(x + row);
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
            if (c < k) y = fma(-hs[c], u[c], y);
        dst[row] = y * binv;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int KMAX>
__global__ void __launch_bounds__(GCTA, 1) k_inner_grid(const GridArgs ga) {
    const SmallArgs& a = ga.s;
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;  // same value in every CTA: the whole grid returns
    extern __shared__ __align__(128) double gsm[];  // GW x KMAX x WLD: one slab per warp
    __shared__ double acc[GW][GNVP];
    __shared__ double red[GNVP];
    __shared__ double tmp[GSPLIT][GNVP];
    __shared__ double hs[KMAX];
    const int warp = threadIdx.x >> 5;
    double* W = gsm + (size_t)warp * KMAX * WLD;
    const double rho = ctl->rho;
    int k = ctl->k;
    int pb = 0;
    const size_t pstride = (size_t)GRID_MAXCTA * GNVP;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    unsigned long long* tr = ga.trace;
#define GTR(i) \
    if (tr && lead) tr[(j - 1) * 8 + (i)] = gtimer();
    for (int j = 1; j <= a.m; ++j) {
        GTR(0)
        const double* g = a.U + (int64_t)(k - 1) * a.ldu;
        const bool cgs = j < a.m;
        // ---- phase 1
        grid_phase1<KMAX>(a, k, cgs, rho, g, W, acc, red);
        GTR(1)
        grid_allreduce(red, cgs ? 2 * k + 1 : k, ga.part + pb * pstride, tmp, gsm);
        GTR(2)
        pb ^= 1;
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < k; i += GCTA) {  // T(1:k,k), mirrored (eq 3.1)
                a.T[i + (int64_t)(k - 1) * a.ldT] = red[i];
                a.T[(k - 1) + (int64_t)i * a.ldT] = red[i];
            }
        if (!cgs) break;
        const double nin2 = red[2 * k];
        for (int i = threadIdx.x; i < k; i += GCTA) hs[i] = red[k + i];
        __syncthreads();
        // ---- phase 2: second CGS pass
        grid_pass<KMAX>(a, k, a.w, hs, a.w1, W, acc, red);
        GTR(3)
        grid_allreduce(red, k + 1, ga.part + pb * pstride, tmp, gsm);
        GTR(4)
        pb ^= 1;
        double hn = 0.0;
        for (int c = 0; c < k; ++c) hn += red[c] * red[c];
        const double n1sq = red[k];
        for (int i = threadIdx.x; i < k; i += GCTA) hs[i] = red[i];
        __syncthreads();
        const double nin = sqrt(nin2);
        const double n2sq = n1sq - hn;
        double b = sqrt(n2sq > 0.0 ? n2sq : 0.0);
        const double* src = a.w1;
        if (!(n2sq >= 0.5 * n1sq) || a.force3) {  // R3: the second pass lost more than half the norm
            grid_pass<KMAX>(a, k, a.w1, hs, a.w2, W, acc, red);
            grid_allreduce(red, k + 1, ga.part + pb * pstride, tmp, gsm);
            pb ^= 1;
            hn = 0.0;
            for (int c = 0; c < k; ++c) hn += red[c] * red[c];
            const double n3sq = red[k] - hn;
            b = sqrt(n3sq > 0.0 ? n3sq : 0.0);
            src = a.w2;
            if (lead) {
                for (int i = 0; i < k; ++i) ctl->h[2][i] = red[i];
                ctl->nrm[N_2SQ_EXP] = red[k];
                ctl->pass3_count += 1;
            }
            for (int i = threadIdx.x; i < k; i += GCTA) hs[i] = red[i];
            __syncthreads();
        }
        if (!(b >= 1e-14 * nin) || nin == 0.0) {  // inner breakdown (R16): stop with the columns built so far
            if (lead) {
                ctl->flags &= ~a.clear;
                ctl->brk += 1;
            }
            break;
        }
        // ---- final: g_{j+1}
        grid_final<KMAX>(a, k, src, hs, 1.0 / b);
        GTR(5)
        k += 1;
        cooperative_groups::this_grid().sync();  // g_{j+1} complete before the next SpMV gathers it
        GTR(6)
    }
#undef GTR
    if (lead) ctl->k = k;
}

template <int KMAX>
static bool launch_grid_k(const GridArgs& a, cudaStream_t s) {
    static int grid = -1;
    const int smem = GW * KMAX * WLD * (int)sizeof(double);
    auto kern = k_inner_grid<KMAX>;
    if (grid < 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int occ = 0, dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, GCTA, smem);
        grid = occ >= 1 ? std::min(nsm * occ, GRID_MAXCTA) : 0;
    }
    if (grid <= 0) return false;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = GCTA;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    NOTE_KERN(kern);
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess;
}

bool launch_inner_grid(const GridArgs& a, int kmax, cudaStream_t s) {
    if (kmax <= 16) return launch_grid_k<16>(a, s);
    if (kmax <= 24) return launch_grid_k<24>(a, s);
    if (kmax <= 32) return launch_grid_k<32>(a, s);
    return false;
}

}  // namespace trplk
