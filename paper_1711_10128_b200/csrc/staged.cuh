// TMA-staged variants of the two dot-product kernels of the inner step (K1, K2).
//
// The basis block U is streamed HBM -> shared memory by the bulk-copy engine
// (cp.async.bulk ... mbarrier::complete_tx, one elected thread per CTA, NSTAGE-deep ring), so
// the bytes in flight no longer depend on registers or warps: while the 8 warps of a CTA
// consume tile i (SpMV from global, dot products by DMMA from shared memory), the copies of
// tile i+1 are already outstanding.  A CTA tile is TR = 256 rows (one 32-row slice per warp);
// each of the k columns of the tile is one contiguous 2 KB bulk copy.  The column stride in
// shared memory, TLD = TR + 4 doubles (= 8 mod 32 banks), makes the DMMA fragment reads
// (8 columns x 4 consecutive rows per warp request) and the row-wise reads conflict-free.
//
//   k_step1_tma  K1: z = A g, w = M (z - rho B g), T(1:k,k) = U^T z, h1 = U^T w, ||w||^2
//   k_upd2_tma   K2: w' = w - U h1, h2 = U^T w', ||w'||^2
// Arithmetic, order and outputs are those of k_sdots_mma / k_upd<.., true> (kernels.cu).
// Included by kernels.cu (same translation unit: mat_row, grid_reduce, sdots_finalize and
// upd_finalize are shared and inlined).
#pragma once

namespace trplk {

constexpr int TR = 256;
constexpr int TLD = TR + 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TRPLK_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TRPLK_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void dmma884_s(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum_s(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Issue the bulk copies of CTA tile `t` (columns 0..ncols-1 of U) into stage buffer `st`.
__device__ __forceinline__ void issue_tile(double* st, const double* U, int64_t ldu, int64_t nrows, int64_t t,
                                           int ncols, uint64_t* bar) {
    const int64_t r0 = t * TR;
    int64_t rows = nrows - r0;
    if (rows > TR) rows = TR;
    const unsigned bytes = (unsigned)(((rows + 1) & ~(int64_t)1) * 8);  // 16-byte multiple (ld even)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the stage
    mbar_expect_tx(bar, bytes * (unsigned)ncols);
    for (int c = 0; c < ncols; ++c) bulk_g2s(st + c * TLD, U + (int64_t)c * ldu + r0, bytes, bar);
}

template <int KMAX, bool TWO, int NS>
__global__ void __launch_bounds__(CTA, 1) k_step1_tma(const SdotsArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    const int kc = ctl->k;
    const int k1 = a.set1 ? (a.k_from_ctl ? kc : a.k1) : 0;
    const int k2 = (TWO && a.set2) ? (a.k_from_ctl ? kc : a.k2) : 0;
    const int kmx = k1 > k2 ? k1 : k2;
    const double rho = ctl->rho;
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const double* __restrict__ X = a.x;  // K1 input is a fixed column (no x_dyn)

    extern __shared__ __align__(128) double stg[];  // NS stages of KMAX x TLD
    __shared__ __align__(8) uint64_t bar[NS];
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    const int64_t ntile = (a.nrows + TR - 1) / TR;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < NS; ++s) {
            const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
            if (t < ntile) issue_tile(stg + (size_t)s * KMAX * TLD, a.U, a.ldu, a.nrows, t, kmx, &bar[s]);
        }
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x, ++it) {
        const int s = it % NS;
        const unsigned phase = (unsigned)((it / NS) & 1);
        const double* S = stg + (size_t)s * KMAX * TLD;
        const int64_t sl = t * (TR / 32) + warp;  // slice of this warp
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        double z = 0.0, o = 0.0, ad = 1.0, bd = 1.0, sv = 0.0;
        const double xr = ok ? X[row] : 0.0;
        if (sl * 32 < a.nrows) {
            z = mat_row(a.A, sl, lane, X, ad);
            if (a.out_mode == 2) {
                if (a.B.nrows) sv = mat_row(a.B, sl, lane, X, bd);
                else sv = xr;
                double d = fabs(ad - a.sigma * bd);
                d = d > a.mfloor ? d : a.mfloor;
                o = (1.0 / d) * (z - rho * sv);  // w = M (z - rho B g), R1
            } else if (a.out_mode == 1) {
                o = z;
            }
        }
        if (ok) {
            if (a.out) a.out[row] = o;
        } else {
            z = 0.0;
            o = 0.0;
        }
        if (a.norm1 == 1) n1 += o * o;
        const double v1 = a.set1 == 1 ? z : o;
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, v1, 4 * q + fj);
            const double t2 = TWO ? __shfl_sync(0xffffffffu, o, 4 * q + fj) : 0.0;
            bq[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
        }
        mbar_wait(&bar[s], phase);
        const int lr = warp * 32 + fj;
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            if (8 * g < kmx) {
                const int c = 8 * g + fi;
                const double* sp = S + c * TLD + lr;
                double av[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) av[q] = c < kmx ? sp[4 * q] : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(cacc[g], av[q], bq[q]);
            }
        }
        __syncthreads();  // every warp is done with stage s
        if (threadIdx.x == 0) {
            const int64_t tn = t + (int64_t)NS * gridDim.x;
            if (tn < ntile) issue_tile(stg + (size_t)s * KMAX * TLD, a.U, a.ldu, a.nrows, tn, kmx, &bar[s]);
        }
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
        if (lane == 0) acc[warp][k1 + k2] = s1;
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

template <int KMAX, int NS>
__global__ void __launch_bounds__(CTA, 1) k_upd2_tma(const UpdArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int kv = a.kv >= 0 ? a.kv : ctl->k;
    const double* __restrict__ X = a.x_dyn == 2 ? a.x + a.x_ld * (int64_t)(ctl->xprev_col + a.x_off)
                                 : (a.x_dyn == 1 ? a.x + a.x_ld * (int64_t)(ctl->t - 1 + a.x_off) : a.x);
    extern __shared__ __align__(128) double stg[];
    __shared__ __align__(8) uint64_t bar[NS];
    __shared__ double hs[KMAX];
    __shared__ double acc[WARPS][QMAX + 1];
    __shared__ double res[QMAX + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    const int64_t ntile = (a.nrows + TR - 1) / TR;
    for (int i = threadIdx.x; i < KMAX; i += CTA) hs[i] = i < kv ? ctl->h[a.hslot][i] : 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < NS; ++s) {
            const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
            if (t < ntile) issue_tile(stg + (size_t)s * KMAX * TLD, a.U, a.ldu, a.nrows, t, kv, &bar[s]);
        }
    double dacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) dacc[g][0] = dacc[g][1] = 0.0;
    double yy = 0.0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x, ++it) {
        const int s = it % NS;
        const unsigned phase = (unsigned)((it / NS) & 1);
        const double* S = stg + (size_t)s * KMAX * TLD;
        const int64_t row = t * TR + warp * 32 + lane;
        const bool ok = row < a.nrows;
        double y = ok ? X[row] : 0.0;
        mbar_wait(&bar[s], phase);
        const int lrow = warp * 32 + lane;
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
            if (c < kv) y = fma(-hs[c], S[c * TLD + lrow], y);  // y = x - U h, columns in order
        if (!ok) y = 0.0;
        if (ok && a.out) a.out[row] = y;
        yy += y * y;
        double ya[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double tq = __shfl_sync(0xffffffffu, y, 4 * q + fj);
            ya[q] = fi == 0 ? tq : 0.0;
        }
        const int lr = warp * 32 + fj;
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            if (8 * g < kv) {
                const int c = 8 * g + fi;
                const double* sp = S + c * TLD + lr;
                double bu[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) bu[q] = c < kv ? sp[4 * q] : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(dacc[g], ya[q], bu[q]);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t tn = t + (int64_t)NS * gridDim.x;
            if (tn < ntile) issue_tile(stg + (size_t)s * KMAX * TLD, a.U, a.ldu, a.nrows, tn, kv, &bar[s]);
        }
    }
    for (int i = threadIdx.x; i < WARPS * (QMAX + 1); i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (fi == 0) {
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = 8 * g + 2 * fj + e;
                if (c < kv) acc[warp][c] = dacc[g][e];
            }
    }
    const double ys = warp_sum_s(yy);
    if (lane == 0) acc[warp][kv] = ys;
    __syncthreads();
    const int nv = kv + 1;
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
}

// ------------------------------------------- register-stream + shared-memory transpose variant
// Each warp loads its 32-row tile of U in row layout (lane = row, all k column loads issued
// at once, before the SpMV's dependent gathers), parks it in a private shared-memory slab
// (column stride 36 doubles = 8 mod 32 banks), and reads it back in DMMA fragment order.
// U is read from HBM/L2 exactly once; no block-level barriers in the main loop.
constexpr int WLD = 36;

// Slab width of k_step1_rs: 24 columns up to k = 32; 16 beyond, where 24 registers of the basis
// row plus 2 k/8 DMMA accumulators no longer fit 128 registers without spilling.
__host__ __device__ constexpr int rs_chunk(int kmax) { return kmax < 24 ? kmax : (kmax > 32 ? 16 : 24); }

template <int KMAX, bool TWO>
__global__ void __launch_bounds__(CTA, 2) k_step1_rs(const SdotsArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    const int kc = ctl->k;
    const int k1 = a.set1 ? (a.k_from_ctl ? kc : a.k1) : 0;
    const int k2 = (TWO && a.set2) ? (a.k_from_ctl ? kc : a.k2) : 0;
    const int kmx = k1 > k2 ? k1 : k2;
    const double rho = ctl->rho;
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const double* __restrict__ X = a.x;
    constexpr int CH = rs_chunk(KMAX);               // columns per chunk (= slab width)
    extern __shared__ __align__(128) double wsm[];  // WARPS x CH x WLD: one chunk per warp
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* W = wsm + (size_t)warp * CH * WLD;
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0;
    const int64_t nslices = (a.nrows + 31) >> 5;
    for (int64_t sl = (int64_t)blockIdx.x * WARPS + warp; sl < nslices; sl += (int64_t)gridDim.x * WARPS) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        double ur[CH];
        const double* up = a.U + row;
#pragma unroll
        for (int c = 0; c < CH; ++c) ur[c] = (ok && c < kmx) ? __ldg(up + (int64_t)c * a.ldu) : 0.0;
        double z = 0.0, o = 0.0, ad = 1.0, bd = 1.0, sv = 0.0;
        const double xr = ok ? X[row] : 0.0;
        z = mat_row(a.A, sl, lane, X, ad);
        if (a.out_mode == 2) {
            if (a.B.nrows) sv = mat_row(a.B, sl, lane, X, bd);
            else sv = xr;
            double d = fabs(ad - a.sigma * bd);
            d = d > a.mfloor ? d : a.mfloor;
            o = (1.0 / d) * (z - rho * sv);  // w = M (z - rho B g), R1
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
        else if (a.norm1 == 2) n1 += xr * z;  // x^T B x of a CGS first pass (z = B x)
        const double v1 = a.set1 == 1 ? z : o;
        double bq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, v1, 4 * q + fj);
            const double t2 = TWO ? __shfl_sync(0xffffffffu, o, 4 * q + fj) : 0.0;
            bq[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
        }
        // chunks of CH columns through the warp's slab: the next chunk's loads are issued
        // (into the registers just parked) before this chunk's DMMAs
        __syncwarp();
#pragma unroll
        for (int c = 0; c < CH; ++c) W[c * WLD + lane] = ur[c];
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {
            const bool more = cb + CH < KMAX && cb + CH < kmx;
            if (more) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int cc = cb + CH + c;
                    ur[c] = (ok && cc < kmx && cc < KMAX) ? __ldg(up + (int64_t)cc * a.ldu) : 0.0;
                }
            }
            if (cb < kmx) {
#pragma unroll
                for (int g = cb / 8; g < (cb + CH) / 8 && g < KMAX / 8; ++g) {
                    if (8 * g < kmx) {
                        const double* sp = W + (8 * g - cb + fi) * WLD + fj;
#pragma unroll
                        for (int q = 0; q < 8; ++q) dmma884_s(cacc[g], sp[4 * q], bq[q]);
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
        if (lane == 0) acc[warp][k1 + k2] = s1;
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

// K1 with two 32-row tiles per warp per iteration (default; TRPLK_RS1=1 selects the one-tile
// k_step1_rs): the loads of both tiles (basis rows, DIA values, gathers) are in flight
// together, so a warp walks half as many dependent load round trips; 8-column slab chunks,
// one slab per tile.  C2: K1 24.5 -> 22.6 us, solve -2.7 %; C3: K1 145 -> 135 us, -2.9 %.
template <int KMAX, bool TWO>
__global__ void __launch_bounds__(CTA, 2) k_step1_rs2(const SdotsArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    if (a.gate_pass3 && ctl->pass3 == 0) return;
    const int kc = ctl->k;
    const int k1 = a.set1 ? (a.k_from_ctl ? kc : a.k1) : 0;
    const int k2 = (TWO && a.set2) ? (a.k_from_ctl ? kc : a.k2) : 0;
    const int kmx = k1 > k2 ? k1 : k2;
    const double rho = ctl->rho;
    const int nn = (a.norm1 ? 1 : 0) + (a.norm2 ? 1 : 0);
    const int nv = k1 + k2 + nn;
    const double* __restrict__ X = a.x;
    constexpr int CH = 8;
    extern __shared__ __align__(128) double wsm[];  // WARPS x 2 x CH x WLD
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* W0 = wsm + (size_t)warp * 2 * CH * WLD;
    double* W1 = W0 + CH * WLD;
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0;
    const int64_t nslices = (a.nrows + 31) >> 5;
    const int64_t npairs = (nslices + 1) >> 1;
    auto tile = [&](int64_t sl, bool live, double& v1, double& o) {
        const int64_t row = sl * 32 + lane;
        const bool ok = live && row < a.nrows;
        double z = 0.0, ad = 1.0, bd = 1.0, sv = 0.0;
        o = 0.0;
        const double xr = ok ? X[row] : 0.0;
        if (live) {
            z = mat_row(a.A, sl, lane, X, ad);
            if (a.out_mode == 2) {
                if (a.B.nrows) sv = mat_row(a.B, sl, lane, X, bd);
                else sv = xr;
                double d = fabs(ad - a.sigma * bd);
                d = d > a.mfloor ? d : a.mfloor;
                o = (1.0 / d) * (z - rho * sv);  // w = M (z - rho B g), R1
            } else if (a.out_mode == 1) {
                o = z;
            }
        }
        if (ok) {
            if (a.out) a.out[row] = o;
        } else {
            z = 0.0;
            o = 0.0;
        }
        if (a.norm1 == 1) n1 += o * o;
        else if (a.norm1 == 2) n1 += xr * z;
        v1 = a.set1 == 1 ? z : o;
    };
    for (int64_t pr = (int64_t)blockIdx.x * WARPS + warp; pr < npairs; pr += (int64_t)gridDim.x * WARPS) {
        const int64_t s0 = 2 * pr, s1 = 2 * pr + 1;
        const bool has1 = s1 < nslices;
        const int64_t r0 = s0 * 32 + lane, r1 = s1 * 32 + lane;
        const bool ok0 = r0 < a.nrows, ok1 = has1 && r1 < a.nrows;
        const double* up0 = a.U + r0;
        const double* up1 = a.U + r1;
        double u0[CH], u1[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            u0[c] = (ok0 && c < kmx) ? __ldg(up0 + (int64_t)c * a.ldu) : 0.0;
            u1[c] = (ok1 && c < kmx) ? __ldg(up1 + (int64_t)c * a.ldu) : 0.0;
        }
        double va, oa, vb, ob;
        tile(s0, true, va, oa);
        tile(s1, has1, vb, ob);
        double bq0[8], bq1[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double t1 = __shfl_sync(0xffffffffu, va, 4 * q + fj);
            const double t2 = TWO ? __shfl_sync(0xffffffffu, oa, 4 * q + fj) : 0.0;
            bq0[q] = fi == 0 ? t1 : (fi == 1 ? t2 : 0.0);
            const double t3 = __shfl_sync(0xffffffffu, vb, 4 * q + fj);
            const double t4 = TWO ? __shfl_sync(0xffffffffu, ob, 4 * q + fj) : 0.0;
            bq1[q] = fi == 0 ? t3 : (fi == 1 ? t4 : 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            W0[c * WLD + lane] = u0[c];
            W1[c * WLD + lane] = u1[c];
        }
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {
            const bool more = cb + CH < KMAX && cb + CH < kmx;
            if (more) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const int cc = cb + CH + c;
                    u0[c] = (ok0 && cc < kmx) ? __ldg(up0 + (int64_t)cc * a.ldu) : 0.0;
                    u1[c] = (ok1 && cc < kmx) ? __ldg(up1 + (int64_t)cc * a.ldu) : 0.0;
                }
            }
            if (cb < kmx) {
                const double* sp0 = W0 + fi * WLD + fj;
                const double* sp1 = W1 + fi * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(cacc[cb / 8], sp0[4 * q], bq0[q]);
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(cacc[cb / 8], sp1[4 * q], bq1[q]);
            }
            if (more) {
                __syncwarp();
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    W0[c * WLD + lane] = u0[c];
                    W1[c * WLD + lane] = u1[c];
                }
                __syncwarp();
            }
        }
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
        if (lane == 0) acc[warp][k1 + k2] = s1;
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

template <int KMAX>
__global__ void __launch_bounds__(CTA, 2) k_upd2_rs(const UpdArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int kv = a.kv >= 0 ? a.kv : ctl->k;
    const double* __restrict__ X = a.x_dyn == 2 ? a.x + a.x_ld * (int64_t)(ctl->xprev_col + a.x_off)
                                 : (a.x_dyn == 1 ? a.x + a.x_ld * (int64_t)(ctl->t - 1 + a.x_off) : a.x);
    extern __shared__ __align__(128) double wsm[];
    __shared__ double hs[KMAX];
    __shared__ double acc[WARPS][QMAX + 1];
    __shared__ double res[QMAX + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* W = wsm + (size_t)warp * KMAX * WLD;
    for (int i = threadIdx.x; i < KMAX; i += CTA) hs[i] = i < kv ? ctl->h[a.hslot][i] : 0.0;
    __syncthreads();
    double dacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) dacc[g][0] = dacc[g][1] = 0.0;
    double yy = 0.0;
    const int64_t nslices = (a.nrows + 31) >> 5;
    for (int64_t sl = (int64_t)blockIdx.x * WARPS + warp; sl < nslices; sl += (int64_t)gridDim.x * WARPS) {
        const int64_t row = sl * 32 + lane;
        const bool ok = row < a.nrows;
        constexpr int CH = KMAX < 24 ? KMAX : 24;
        double ur[CH];
        const double* up = a.U + row;
        double y = ok ? X[row] : 0.0;
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < KMAX; cb += CH) {  // y = x - U h, columns in order; park U rows
            if (cb < kv) {
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    ur[c] = (ok && cb + c < kv && cb + c < KMAX) ? __ldg(up + (int64_t)(cb + c) * a.ldu) : 0.0;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (cb + c < KMAX) {
                        y = fma(-hs[cb + c], ur[c], y);
                        W[(cb + c) * WLD + lane] = ur[c];
                    }
            }
        }
        if (!ok) y = 0.0;
        if (ok && a.out) a.out[row] = y;
        yy += y * y;
        __syncwarp();
        double ya[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double tq = __shfl_sync(0xffffffffu, y, 4 * q + fj);
            ya[q] = fi == 0 ? tq : 0.0;
        }
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            if (8 * g < kv) {
                const double* sp = W + (8 * g + fi) * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(dacc[g], ya[q], sp[4 * q]);
            }
        }
    }
    for (int i = threadIdx.x; i < WARPS * (QMAX + 1); i += CTA) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    if (fi == 0) {
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = 8 * g + 2 * fj + e;
                if (c < kv) acc[warp][c] = dacc[g][e];
            }
    }
    const double ys = warp_sum_s(yy);
    if (lane == 0) acc[warp][kv] = ys;
    __syncthreads();
    const int nv = kv + 1;
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
}

// ------------------------------------------------------------------ launchers
static int nsm_s() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <typename K>
static int tma_grid(K kern, int smem, int64_t nrows) {
    static bool dummy = false;
    (void)dummy;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, smem);
    if (occ < 1) occ = 1;
    const int64_t ntile = (nrows + TR - 1) / TR;
    int64_t cap = (int64_t)nsm_s() * occ;
    if (cap > MAXCTA) cap = MAXCTA;
    int64_t g = ntile < cap ? ntile : cap;
    return (int)(g < 1 ? 1 : g);
}

template <int KMAX, bool TWO>
static void launch_step1_k(const SdotsArgs& a, cudaStream_t s) {
    constexpr int NS = KMAX <= 48 ? 2 : 1;
    const int smem = NS * KMAX * TLD * (int)sizeof(double);
    auto kern = k_step1_tma<KMAX, TWO, NS>;
    kern<<<tma_grid(kern, smem, a.nrows), CTA, smem, s>>>(a);
}

template <int KMAX>
static void launch_upd2_k(const UpdArgs& a, cudaStream_t s) {
    constexpr int NS = KMAX <= 48 ? 2 : 1;
    const int smem = NS * KMAX * TLD * (int)sizeof(double);
    auto kern = k_upd2_tma<KMAX, NS>;
    kern<<<tma_grid(kern, smem, a.nrows), CTA, smem, s>>>(a);
}

template <typename K>
static int rs_grid(K kern, int smem, int64_t nrows) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, smem);
    if (occ < 1) occ = 1;
    const int64_t need = ((nrows + 31) / 32 + WARPS - 1) / WARPS;
    static const int spw = getenv("TRPLK_RS_SPW") ? atoi(getenv("TRPLK_RS_SPW")) : 0;  // experiment knob
    if (spw > 0) {
        int64_t g = (need + spw - 1) / spw;
        if (g > MAXCTA) g = MAXCTA;
        return (int)(g < 1 ? 1 : g);
    }
    int64_t cap = (int64_t)nsm_s() * occ;
    if (cap > MAXCTA) cap = MAXCTA;
    if (need <= cap) return (int)(need < 1 ? 1 : need);
    const int64_t waves = (need + cap - 1) / cap;
    return (int)((need + waves - 1) / waves);
}

template <int KMAX, bool TWO>
static void launch_step1_rs_k(const SdotsArgs& a, cudaStream_t s) {
    static const bool two_tiles = !(getenv("TRPLK_RS1") && getenv("TRPLK_RS1")[0] == '1');
    if (two_tiles) {
        const int smem2 = WARPS * 2 * 8 * WLD * (int)sizeof(double);
        auto kern2 = k_step1_rs2<KMAX, TWO>;
        kern2<<<rs_grid(kern2, smem2, (a.nrows + 1) / 2), CTA, smem2, s>>>(a);
        return;
    }
    const int smem = WARPS * rs_chunk(KMAX) * WLD * (int)sizeof(double);
    auto kern = k_step1_rs<KMAX, TWO>;
    kern<<<rs_grid(kern, smem, a.nrows), CTA, smem, s>>>(a);
}

template <int KMAX>
static void launch_upd2_rs_k(const UpdArgs& a, cudaStream_t s) {
    const int smem = WARPS * KMAX * WLD * (int)sizeof(double);
    auto kern = k_upd2_rs<KMAX>;
    kern<<<rs_grid(kern, smem, a.nrows), CTA, smem, s>>>(a);
}

bool launch_step1_rs(const SdotsArgs& a, int kmax, cudaStream_t s) {
    const bool two = a.set2 != 0;
    switch (kmax) {
        case 8: two ? launch_step1_rs_k<8, true>(a, s) : launch_step1_rs_k<8, false>(a, s); break;
        case 16: two ? launch_step1_rs_k<16, true>(a, s) : launch_step1_rs_k<16, false>(a, s); break;
        case 24: two ? launch_step1_rs_k<24, true>(a, s) : launch_step1_rs_k<24, false>(a, s); break;
        case 32: two ? launch_step1_rs_k<32, true>(a, s) : launch_step1_rs_k<32, false>(a, s); break;
        case 40: two ? launch_step1_rs_k<40, true>(a, s) : launch_step1_rs_k<40, false>(a, s); break;
        case 48: two ? launch_step1_rs_k<48, true>(a, s) : launch_step1_rs_k<48, false>(a, s); break;
        default: return false;
    }
    return true;
}

bool launch_upd2_rs(const UpdArgs& a, int kmax, cudaStream_t s) {
    switch (kmax) {
        case 8: launch_upd2_rs_k<8>(a, s); break;
        case 16: launch_upd2_rs_k<16>(a, s); break;
        case 24: launch_upd2_rs_k<24>(a, s); break;
        case 32: launch_upd2_rs_k<32>(a, s); break;
        case 40: launch_upd2_rs_k<40>(a, s); break;
        case 48: launch_upd2_rs_k<48>(a, s); break;
        default: return false;
    }
    return true;
}

bool launch_step1_tma(const SdotsArgs& a, int kmax, cudaStream_t s) {
    const bool two = a.set2 != 0;
    switch (kmax) {
        case 8: two ? launch_step1_k<8, true>(a, s) : launch_step1_k<8, false>(a, s); break;
        case 16: two ? launch_step1_k<16, true>(a, s) : launch_step1_k<16, false>(a, s); break;
        case 24: two ? launch_step1_k<24, true>(a, s) : launch_step1_k<24, false>(a, s); break;
        case 32: two ? launch_step1_k<32, true>(a, s) : launch_step1_k<32, false>(a, s); break;
        case 40: two ? launch_step1_k<40, true>(a, s) : launch_step1_k<40, false>(a, s); break;
        case 48: two ? launch_step1_k<48, true>(a, s) : launch_step1_k<48, false>(a, s); break;
        case 64: two ? launch_step1_k<64, true>(a, s) : launch_step1_k<64, false>(a, s); break;
        default: return false;
    }
    return true;
}

bool launch_upd2_tma(const UpdArgs& a, int kmax, cudaStream_t s) {
    switch (kmax) {
        case 8: launch_upd2_k<8>(a, s); break;
        case 16: launch_upd2_k<16>(a, s); break;
        case 24: launch_upd2_k<24>(a, s); break;
        case 32: launch_upd2_k<32>(a, s); break;
        case 40: launch_upd2_k<40>(a, s); break;
        case 48: launch_upd2_k<48>(a, s); break;
        case 64: launch_upd2_k<64>(a, s); break;
        default: return false;
    }
    return true;
}

}  // namespace trplk
