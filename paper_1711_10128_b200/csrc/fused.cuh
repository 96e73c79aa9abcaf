// K3 + K1 of consecutive inner steps in one kernel (k_fin_step1): the FINAL CGS2 update of
// step j, g_{j+1} = (w' - U h2) / beta (reading R3), and the fused SpMV + Jacobi + dots
// of step j+1 on that g (eq 3.1; R1 at P:143):
//
//   z = A g, w = M (z - rho g), T(1:k+1, k+1) = U^T z, h1 = U^T w, ||w||^2.
//
// The unfused step streams the basis U three times (K1 dots, K2 update + dots, K3 update).  K3
// and the next K1 read the same rows of U, but K1 of a row needs g at the row's stencil
// neighbours, which other warps produce.  Here every warp walks its 32-row tiles in rounds
// (tile = round * NW + global warp id, NW warps in the grid): in round r it runs the FINAL of
// its round-r tile, publishes the round (per-round completion counter), and runs the K1 of its
// tile of round r - lag once every CTA has completed the rounds that tile's stencil reaches
// (lag = ceil(max |offset| / round rows) + slack).  The K1 re-read of U hits L2 while the
// distance is below its capacity (C3: 0.5 rounds of 49 columns; C5: ~3.5 rounds of <= 25), so
// HBM sees U about twice per inner step instead of three times.  All CTAs must be co-resident
// (cooperative launch); the rare third CGS pass (R3) and breakdown (R16) are handled in-kernel
// (third pass: grid-wide, then the K1 over all tiles without lag).  Per-tile arithmetic and
// order are those of k_upd FINAL and of the K1 kernels; only the grid's partial-sum grouping
// of the dots differs.  DIA (<= 8 diagonals, DIA-C aware), B = I, one rank.
// Included by kernels.cu after stream_rs.cuh (WLD, dmma884_nv, warp_sum_s, grid_reduce,
// sdots_finalize, final_pass3_coop).
#pragma once

namespace trplk {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int KMAX>
__global__ void __launch_bounds__(CTA, 2) k_fin_step1(const FusedArgs f) {
    const UpdArgs& u = f.u;
    const SdotsArgs& a = f.a;
    Ctl* ctl = u.ctl;
    if ((ctl->flags & u.gate) != u.gate) return;
    const int kv = ctl->k;  // basis width before g_{j+1}
    constexpr int CH = 8;
    __shared__ double hs[KMAX];
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    extern __shared__ __align__(128) double wsm[];  // WARPS x CH x WLD
    for (int i = threadIdx.x; i < KMAX; i += CTA) hs[i] = i < kv ? ctl->h[u.hslot][i] : 0.0;
    __syncthreads();
    // FINAL decisions (k_upd mode 2), identical in every CTA
    bool pass3, brk = false;
    double binv = 0.0;
    {
        double hn = 0.0;
        for (int i = 0; i < kv; ++i) hn += hs[i] * hs[i];
        const double nin = sqrt(ctl->nrm[N_IN2]);
        const double n1sq = ctl->nrm[N_1SQ];
        const double n2sq = n1sq - hn;  // ||w''||^2 = ||w'||^2 - ||h2||^2
        pass3 = !(n2sq >= 0.5 * n1sq) || u.force3;
        const double b = sqrt(n2sq > 0.0 ? n2sq : 0.0);
        if (!pass3) {
            brk = !(b >= 1e-14 * nin) || nin == 0.0;
            binv = 1.0 / b;
        }
    }
    double* g = u.dest + u.dest_ld * (int64_t)kv;  // U(:, kv) = g_{j+1}
    const int k1 = kv + 1;
    const int k2 = a.set2 ? kv + 1 : 0;
    const int nn = a.norm1 ? 1 : 0;
    const double rho = ctl->rho;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* W = wsm + (size_t)warp * CH * WLD;
    const int64_t nrows = u.nrows;
    const int64_t nsl = (nrows + 31) >> 5;
    const int64_t NW = (int64_t)gridDim.x * WARPS;
    const int64_t R = (nsl + NW - 1) / NW;
    const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
    const double* __restrict__ Ub = u.U;
    const int64_t ldu = u.ldu;
    const Sell& M = a.A;
    const int nd = M.ndiag;
    const int top = (int)(M.nrows - 1);

    // y = w' - U h2 of one tile: columns in order (as k_upd), 16 row loads in flight per lane
    auto fin_tile = [&](int64_t sl, bool to_g) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < nrows;
        double y = ok ? __ldcs(u.x + row) : 0.0;
        const double* up = Ub + row;
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += 16) {
            if (cb < kv) {
                double uk[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) uk[c] = (ok && cb + c < kv) ? __ldg(up + (int64_t)(cb + c) * ldu) : 0.0;
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    if (cb + c < KMAX) y = fma(-hs[cb + c < KMAX ? cb + c : 0], uk[c], y);
            }
        }
        if (ok) {
            if (to_g) g[row] = y * binv;
            else u.out[row] = y;  // third pass follows: w2
        }
    };

    double cacc[KMAX / 8][2];
#pragma unroll
    for (int q = 0; q < KMAX / 8; ++q) cacc[q][0] = cacc[q][1] = 0.0;
    double n1 = 0.0;
    __shared__ double cv_s[8];  // DIA-C constants of the first 8 diagonals
    if (threadIdx.x < 8) cv_s[threadIdx.x] = (threadIdx.x < nd && ((M.cmask >> threadIdx.x) & 1u)) ? M.cv[threadIdx.x] : 0.0;
    __syncthreads();
    const double minv_shift = a.pmode == 2 ? rho : a.sigma;

    // One warp iteration of the round loop: the FINAL of tile sa (>= 0) and the K1 of tile sb
    // (>= 0, its stencil rows complete), with the loads of both tiles in flight together: the
    // FINAL's w' and first 16 basis columns, the K1's first 8 basis columns (L2), DIA values
    // and gathers.
    auto pair_tile = [&](int64_t sa, int64_t sb) {
        const int64_t ra = sa * 32 + lane, rb = sb * 32 + lane;
        const bool oka = sa >= 0 && ra < nrows, okb = sb >= 0 && rb < nrows;
        // ---- issue
        double y = oka ? __ldcs(u.x + ra) : 0.0;
        double ua[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) ua[c] = (oka && c < kv) ? __ldg(Ub + ra + (int64_t)c * ldu) : 0.0;
        const double* upb = Ub + rb;
        double ur[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) ur[c] = (okb && c < k1) ? __ldcg(upb + (int64_t)c * ldu) : 0.0;
        double v[8], xv[8], dg = 1.0, xr = 0.0;
        unsigned pm = 0;
        if (okb) {
            pm = M.cmask ? dia_pmask(M, rb) : 0u;
            const double* dv = M.dval + rb;
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                v[d] = 0.0;
                xv[d] = 0.0;
                if (d < nd) {
                    int idx = (int)rb + M.offs[d];
                    idx = idx < 0 ? 0 : (idx > top ? top : idx);  // out-of-matrix slots hold 0
                    if (!((M.cmask >> d) & 1u)) v[d] = __ldg(dv + (int64_t)d * M.ldv);
                    xv[d] = __ldcg(g + idx);
                }
            }
            if (!((M.cmask >> M.diag_slot) & 1u)) dg = __ldg(dv + (int64_t)M.diag_slot * M.ldv);
            xr = __ldcg(g + rb);
        } else {
#pragma unroll
            for (int d = 0; d < 8; ++d) v[d] = xv[d] = 0.0;
        }
        // ---- FINAL: y = w' - U h2, columns in order (as k_upd), g = y / beta
        if (sa >= 0) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < KMAX) y = fma(-hs[c < KMAX ? c : 0], ua[c], y);
#pragma unroll
            for (int cb = 16; cb < KMAX; cb += 16) {
                if (cb < kv) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) ua[c] = (oka && cb + c < kv) ? __ldg(Ub + ra + (int64_t)(cb + c) * ldu) : 0.0;
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        if (cb + c < KMAX) y = fma(-hs[cb + c < KMAX ? cb + c : 0], ua[c], y);
                }
            }
            if (oka) g[ra] = y * binv;
        }
        if (sb < 0) return;
        // ---- K1: SpMV (ascending diagonal order, as mat_row), w, ||w||^2, dots on DMMA
        double z = 0.0;
        if (M.cmask) {
#pragma unroll
            for (int d = 0; d < 8; ++d)
                if (d < nd && ((M.cmask >> d) & 1u)) v[d] = ((pm >> d) & 1u) ? cv_s[d] : 0.0;
            if (okb && ((M.cmask >> M.diag_slot) & 1u)) dg = ((pm >> M.diag_slot) & 1u) ? cv_s[M.diag_slot] : 0.0;
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) z = fma(v[d], xv[d], z);
        double o = 0.0;
        if (a.out_mode == 2) o = jacobi_minv(dg, 1.0, minv_shift, a.mfloor) * (z - rho * xr);
        if (okb) {
            if (a.out_mode == 2 && a.out) __stcs(a.out + rb, o);
        } else {
            z = 0.0;
            o = 0.0;
        }
        if (a.norm1 == 1) n1 += o * o;
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, z, 4 * q + fj);
            const double t2 = __shfl_sync(0xffffffffu, o, 4 * q + fj);
            bq[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {
            const bool more = cb + CH < KMAX && cb + CH < k1;
            if (more) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int cc = cb + CH + c;
                    ur[c] = (okb && cc < k1) ? __ldcg(upb + (int64_t)cc * ldu) : 0.0;
                }
            }
            if (cb < k1) {
                const double* sp = W + fi * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_nv(cacc[cb / 8], sp[4 * q], bq[q]);
            }
            if (more) {
                __syncwarp();
#pragma unroll
                for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
                __syncwarp();
            }
        }
        __syncwarp();
    };
    // K1 of one tile on g (complete at its stencil rows): SpMV in ascending diagonal order (as
    // mat_row), w, ||w||^2, then U(rows, 0:kv+1)^T [z w] on DMMA through the warp's slab
    auto k1_tile = [&](int64_t sl) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < nrows;
        const double* up = Ub + row;
        double ur[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) ur[c] = (ok && c < k1) ? __ldcg(up + (int64_t)c * ldu) : 0.0;
        double z = 0.0, dg = 1.0, xr = 0.0;
        if (ok) {
            const unsigned pm = M.cmask ? dia_pmask(M, row) : 0u;
            const double* dv = M.dval + row;
            double v[8], xv[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                v[d] = 0.0;
                xv[d] = 0.0;
                if (d < nd) {
                    int idx = (int)row + M.offs[d];
                    idx = idx < 0 ? 0 : (idx > top ? top : idx);  // out-of-matrix slots hold 0
                    v[d] = dia_val(M, d, pm, dv);
                    xv[d] = __ldca(g + idx);
                }
            }
#pragma unroll
            for (int d = 0; d < 8; ++d) z = fma(v[d], xv[d], z);
            dg = dia_val(M, M.diag_slot, pm, dv);
            xr = __ldca(g + row);
        }
        double o = 0.0;
        if (a.out_mode == 2) o = jacobi_minv(dg, 1.0, a.pmode == 2 ? rho : a.sigma, a.mfloor) * (z - rho * xr);
        if (ok) {
            if (a.out_mode == 2 && a.out) __stcs(a.out + row, o);
        } else {
            z = 0.0;
            o = 0.0;
        }
        if (a.norm1 == 1) n1 += o * o;
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, z, 4 * q + fj);
            const double t2 = __shfl_sync(0xffffffffu, o, 4 * q + fj);
            bq[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {
            const bool more = cb + CH < KMAX && cb + CH < k1;
            if (more) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int cc = cb + CH + c;
                    ur[c] = (ok && cc < k1) ? __ldcg(up + (int64_t)cc * ldu) : 0.0;
                }
            }
            if (cb < k1) {
                const double* sp = W + fi * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_nv(cacc[cb / 8], sp[4 * q], bq[q]);
            }
            if (more) {
                __syncwarp();
#pragma unroll
                for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
                __syncwarp();
            }
        }
        __syncwarp();
    };

    bool run_k1 = false, done3 = false, brk3 = false;
    if (!pass3 && !brk) {
        run_k1 = true;
        // round r: the FINAL of round r and the K1 of round r - lag, whose stencil reaches round
        // r - lag + dn <= r - 1 (lag >= dn + 1): wait until every CTA has published that round
        // (bar.sync + one release per CTA / one acquire per CTA + bar.sync, as a grid semaphore)
        const int lag = f.lag;
        for (int64_t r = 0; r < R + lag; ++r) {
            const int64_t r1 = r - lag;
            if (r1 >= 0) {
                int64_t need = r1 + f.dn;
                if (need > R - 1) need = R - 1;
                if (threadIdx.x == 0) {
                    long long spins = 0;
                    while (ld_acquire_u32(f.rcnt + need) < gridDim.x) {
                        __nanosleep(32);
                        if (++spins > (1ll << 27)) __trap();  // watchdog: a dirty counter would hang the GPU
                    }
                }
                __syncthreads();
            }
            const int64_t sa = (r < R && r * NW + gw < nsl) ? r * NW + gw : -1;
            const int64_t sb = (r1 >= 0 && r1 * NW + gw < nsl) ? r1 * NW + gw : -1;
            if (sa >= 0 || sb >= 0) pair_tile(sa, sb);
            if (r < R) {
                __syncthreads();
                if (threadIdx.x == 0) red_release_add(f.rcnt + r, 1u);
            }
        }
    } else if (pass3) {
        // rare: w2 = w' - U h2 everywhere, the grid-wide third pass writes g (or breaks down),
        // then the K1 over all tiles (final_pass3_coop ends with a grid barrier)
        for (int64_t sl = gw; sl < nsl; sl += NW) fin_tile(sl, false);
        __syncthreads();
        brk3 = final_pass3_coop(Ub, ldu, nrows, u.out, u.part, u.maxcta, nullptr, kv, sqrt(ctl->nrm[N_IN2]), g, res);
        done3 = true;
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // h3, ||w2||^2 (the same in every CTA; reported by the API)
            for (int i = 0; i < kv; ++i) ctl->h[2][i] = res[i];
            ctl->nrm[N_2SQ_EXP] = res[kv];
        }
        __syncthreads();
        if (!brk3) {
            run_k1 = true;
            __threadfence();
            for (int64_t sl = gw; sl < nsl; sl += NW) k1_tile(sl);
        }
    }
    // K1 dots: per-warp fragments -> CTA sums -> deterministic grid sum (as k_step1_rs2)
    const int nv = run_k1 ? k1 + k2 + nn : 0;
    for (int i = threadIdx.x; i < WARPS * NV_MAX; i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (run_k1) {
        if (fj == 0) {
#pragma unroll
            for (int q = 0; q < KMAX / 8; ++q) {
                const int c = 8 * q + fi;
                if (c < k1) acc[warp][c] = cacc[q][0];
                if (c < k2) acc[warp][k1 + c] = cacc[q][1];
            }
        }
        if (nn) {
            const double s1 = warp_sum_s(n1);
            if (lane == 0) acc[warp][k1 + k2] = s1;
        }
        __syncthreads();
        for (int v = threadIdx.x; v < nv; v += CTA) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) s += acc[w][v];
            res[v] = s;
        }
        __syncthreads();
    }
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    // the last CTA: every CTA has left the round loop -- reset the counters, apply the FINAL's
    // control-block effects (k += 1 before the T column lands in column k - 1), then the K1's
    if (!pass3 && !brk)
        for (int64_t r = threadIdx.x; r < R; r += CTA) f.rcnt[r] = 0u;
    if (threadIdx.x == 0) {
        if (done3) {
            ctl->pass3_count += 1;
            if (brk3) {
                ctl->flags &= ~u.clear_on_brk;
                ctl->brk += 1;
            } else {
                ctl->k += 1;
            }
        } else if (brk) {
            ctl->flags &= ~u.clear_on_brk;
            ctl->brk += 1;
        } else {
            ctl->k += 1;
        }
    }
    if (run_k1) {  // sdots_finalize of the K1 with the T column index known here (kv)
        for (int i = threadIdx.x; i < k1; i += CTA) {
            a.T[i + (int64_t)kv * a.ldT] = res[i];
            a.T[kv + (int64_t)i * a.ldT] = res[i];
        }
        if (a.dest2 >= D_H0)
            for (int i = threadIdx.x; i < k2; i += CTA) ctl->h[a.dest2 - D_H0][i] = res[k1 + i];
        if (threadIdx.x == 0 && a.norm1) ctl->nrm[a.nslot1] = res[k1 + k2];
    }
}

template <int KMAX>
static bool launch_fin_step1_k(const FusedArgs& f0, cudaStream_t s, int maxoff, int slack) {
    auto kern = k_fin_step1<KMAX>;
    const int smem = WARPS * 8 * WLD * (int)sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, smem);
    if (occ < 1) return false;
    int64_t grid = (int64_t)nsm_s() * occ;
    if (grid > MAXCTA) grid = MAXCTA;
    const int64_t nsl = (f0.u.nrows + 31) / 32;
    const int64_t need = (nsl + WARPS - 1) / WARPS;
    if (grid > need) grid = need < 1 ? 1 : need;
    FusedArgs f = f0;
    const int64_t NW = grid * WARPS, R = (nsl + NW - 1) / NW;
    if (R > f.rcnt_cap) return false;
    f.dn = (int)((maxoff + 32 * NW - 1) / (32 * NW));
    f.lag = f.dn + slack;
    NOTE_KERN(kern);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(CTA);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, f) == cudaSuccess;
}

bool launch_fin_step1(const FusedArgs& f, int kmax, int maxoff, int slack, cudaStream_t s) {
    switch (kmax) {
        case 8: return launch_fin_step1_k<8>(f, s, maxoff, slack);
        case 16: return launch_fin_step1_k<16>(f, s, maxoff, slack);
        case 24: return launch_fin_step1_k<24>(f, s, maxoff, slack);
        case 32: return launch_fin_step1_k<32>(f, s, maxoff, slack);
        case 40: return launch_fin_step1_k<40>(f, s, maxoff, slack);
        case 48: return launch_fin_step1_k<48>(f, s, maxoff, slack);
        default: return false;
    }
}

}  // namespace trplk
