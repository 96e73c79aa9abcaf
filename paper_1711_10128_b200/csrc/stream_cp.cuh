// Asynchronous-copy pipelined variants of the inner-step dot kernels (HBM regime).
//
//   k_upd2_cp   K2: w' = w - U h1, h2 = U^T w', ||w'||^2   (CGS pass 2, reading R3)
//   k_step1_cp  K1: z = A g, w = M (z - rho B g), T(1:k,k) = U^T z, h1 = U^T w, ||w||^2
//               (eq 3.1; preconditioner of P:143 as reading R1)
//
// Each warp streams its 32-row tiles of the basis block U (and of the vector being updated)
// HBM -> shared memory with cp.async (16-byte copies: lane pairs cover one column's 256-byte
// segment, L1 bypassed) into an NST-deep ring of per-warp stages, so the bytes in flight do
// not cost registers: while a warp consumes tile t from shared memory (row-wise update, DMMA
// m8n8k4 dots from fragment reads, column stride WLD = 36 doubles), the copies of tiles t+1 ..
// t+NST-1 are outstanding.  The ncu capture of the register-staged `rs` variant at C3 showed
// its warps stalled on the loads feeding the shared-memory stores (two dependent HBM round
// trips per 48-column tile, 3.0-4.4 TB/s); here every warp keeps NST-1 tiles in flight.
// Arithmetic and summation order are those of the `rs` kernels (staged.cuh): identical
// results.  Included by kernels.cu (mat_row, grid_reduce, sdots_finalize, upd_finalize).
#pragma once

namespace trplk {

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int n = valid ? 16 : 0;  // src-size 0: zero fill (ragged tail)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Issue the copies of tile `t` (rows t*32 .. t*32+31) of columns [0, ncol) of U (ld ldu) into
// stage `W` (column c at W + c*WLD), plus optionally the vector x into W + ncolmax*WLD.
// Lane l copies rows 2*(l&15), +1 of columns c = (l>>4), (l>>4)+2, ... (16-byte copies); a
// row pair beyond nrows is zero-filled.  Requires U, x, ldu 16-byte aligned (ld % 2 == 0).
__device__ __forceinline__ void cp_tile(double* W, const double* U, int64_t ldu, int ncol, int ncolmax,
                                        const double* x, int64_t nrows, int64_t t, int lane, bool vec16) {
    const int64_t r0 = t * 32;
    const int rp = 2 * (lane & 15);
    const int64_t row = r0 + rp;
    if (vec16) {
        const bool ok = row + 1 < nrows;  // full pair (nrows even or interior)
        for (int c = lane >> 4; c < ncol; c += 2) {
            const double* src = U + (int64_t)c * ldu + row;
            if (ok || row >= nrows) {
                cp_async16(W + c * WLD + rp, ok ? src : U, ok);
            } else {  // the single last row of an odd nrows
                cp_async8(W + c * WLD + rp, src, true);
                cp_async8(W + c * WLD + rp + 1, U, false);
            }
        }
        if (x && (lane >> 4) == 0) {
            if (ok || row >= nrows) {
                cp_async16(W + ncolmax * WLD + rp, ok ? x + row : x, ok);
            } else {
                cp_async8(W + ncolmax * WLD + rp, x + row, true);
                cp_async8(W + ncolmax * WLD + rp + 1, x, false);
            }
        }
    } else {  // 8-byte copies, lane = row
        const int64_t rr = r0 + lane;
        const bool ok = rr < nrows;
        for (int c = 0; c < ncol; ++c) cp_async8(W + c * WLD + lane, ok ? U + (int64_t)c * ldu + rr : U, ok);
        if (x) cp_async8(W + ncolmax * WLD + lane, ok ? x + rr : x, ok);
    }
}

template <int KMAX, int NST, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_upd2_cp(const UpdArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int kv = a.kv >= 0 ? a.kv : ctl->k;
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    constexpr int SW = (KMAX + 1) * WLD;  // doubles per stage (KMAX columns + x)
    extern __shared__ __align__(128) double wsm[];
    __shared__ double hs[KMAX];
    __shared__ double acc[NW][QMAX + 1];
    __shared__ double res[QMAX + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* Wb = wsm + (size_t)warp * NST * SW;
    for (int i = threadIdx.x; i < KMAX; i += 32 * NW) hs[i] = i < kv ? ctl->h[a.hslot][i] : 0.0;
    const bool vec16 = ((a.ldu & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.U) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const int64_t ntile = (a.nrows + 31) >> 5;
    const int64_t t0 = (int64_t)blockIdx.x * NW + warp, ts = (int64_t)gridDim.x * NW;
    // prologue: tiles t0, t0+ts, ... into stages 0..NST-2
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        const int64_t t = t0 + s * ts;
        if (t < ntile) cp_tile(Wb + s * SW, a.U, a.ldu, kv, KMAX, X, a.nrows, t, lane, vec16);
        cp_commit();
    }
    __syncthreads();  // hs
    double dacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) dacc[g][0] = dacc[g][1] = 0.0;
    double yy = 0.0;
    int st = 0;
    for (int64_t t = t0; t < ntile; t += ts) {
        {  // refill: tile t + (NST-1) ts into the stage consumed last iteration
            const int64_t tn = t + (int64_t)(NST - 1) * ts;
            const int sn = (st + NST - 1) % NST;
            if (tn < ntile) cp_tile(Wb + sn * SW, a.U, a.ldu, kv, KMAX, X, a.nrows, tn, lane, vec16);
            cp_commit();
        }
        cp_wait<NST - 1>();
        __syncwarp();
        const double* W = Wb + st * SW;
        const int64_t row = t * 32 + lane;
        const bool ok = row < a.nrows;
        // y = x - U h, columns in order
        double y = W[KMAX * WLD + lane];
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
            if (c < kv) y = fma(-hs[c], W[c * WLD + lane], y);
        if (!ok) y = 0.0;
        if (ok && a.out) a.out[row] = y;
        yy += y * y;
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
                for (int q = 0; q < 8; ++q) dmma884_s(dacc[g], ya[q], (8 * g + fi < kv) ? sp[4 * q] : 0.0);
            }
        }
        __syncwarp();
        st = (st + 1) % NST;
    }
    cp_wait<0>();
    for (int i = threadIdx.x; i < NW * (QMAX + 1); i += 32 * NW) (&acc[0][0])[i] = 0.0;
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
    for (int v = threadIdx.x; v < nv; v += 32 * NW) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += acc[w][v];
        res[v] = s;
    }
    __syncthreads();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += 32 * NW) a.red_local[v] = res[v];
    } else {
        upd_finalize(a, res, kv);
    }
}


template <int KMAX, bool TWO, int NST, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_step1_cp(const SdotsArgs a) {
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
    constexpr int SW = KMAX * WLD;
    extern __shared__ __align__(128) double wsm[];
    __shared__ double acc[NW][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* Wb = wsm + (size_t)warp * NST * SW;
    const bool vec16 = ((a.ldu & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.U) & 15) == 0);
    const int64_t ntile = (a.nrows + 31) >> 5;
    const int64_t t0 = (int64_t)blockIdx.x * NW + warp, ts = (int64_t)gridDim.x * NW;
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        const int64_t t = t0 + s * ts;
        if (t < ntile) cp_tile(Wb + s * SW, a.U, a.ldu, kmx, KMAX, nullptr, a.nrows, t, lane, vec16);
        cp_commit();
    }
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0;
    int st = 0;
    for (int64_t t = t0; t < ntile; t += ts) {
        {
            const int64_t tn = t + (int64_t)(NST - 1) * ts;
            const int sn = (st + NST - 1) % NST;
            if (tn < ntile) cp_tile(Wb + sn * SW, a.U, a.ldu, kmx, KMAX, nullptr, a.nrows, tn, lane, vec16);
            cp_commit();
        }
        // SpMV + preconditioner of this tile's rows (gathers overlap the stage copies)
        const int64_t row = t * 32 + lane;
        const bool ok = row < a.nrows;
        double z = 0.0, o = 0.0, ad = 1.0, bd = 1.0, sv = 0.0;
        if (ok) {
            const double xr = X[row];
            z = mat_row(a.A, t, lane, X, ad);
            if (a.out_mode == 2) {
                if (a.B.nrows) sv = mat_row(a.B, t, lane, X, bd);
                else sv = xr;
                double d = fabs(ad - a.sigma * bd);
                d = d > a.mfloor ? d : a.mfloor;
                o = (1.0 / d) * (z - rho * sv);  // w = M (z - rho B g), R1
            } else if (a.out_mode == 1) {
                o = z;
            }
            if (a.out) a.out[row] = o;
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
        cp_wait<NST - 1>();
        __syncwarp();
        const double* W = Wb + st * SW;
#pragma unroll
        for (int g = 0; g < KMAX / 8; ++g) {
            if (8 * g < kmx) {
                const bool cok = 8 * g + fi < kmx;
                const double* sp = W + (8 * g + fi) * WLD + fj;
#pragma unroll
                for (int q = 0; q < 8; ++q) dmma884_s(cacc[g], cok ? sp[4 * q] : 0.0, bq[q]);
            }
        }
        __syncwarp();
        st = (st + 1) % NST;
    }
    cp_wait<0>();
    for (int i = threadIdx.x; i < NW * NV_MAX; i += 32 * NW) (&acc[0][0])[i] = 0.0;
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
    for (int v = threadIdx.x; v < nv; v += 32 * NW) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) sum += acc[w][v];
        res[v] = sum;
    }
    __syncthreads();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += 32 * NW) a.red_local[v] = res[v];
    } else {
        sdots_finalize(a, res, k1, k2);
    }
}

// ------------------------------------------------------------------ launchers
template <typename K>
static int cp_grid(K kern, int smem, int nthreads, int64_t nrows, int nw) {
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (nsm <= 0) nsm = 148;
    }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthreads, smem);
    if (occ < 1) occ = 1;
    const int64_t need = ((nrows + 31) / 32 + nw - 1) / nw;
    int64_t cap = (int64_t)nsm * occ;
    if (cap > MAXCTA) cap = MAXCTA;
    if (need <= cap) return (int)(need < 1 ? 1 : need);
    const int64_t waves = (need + cap - 1) / cap;
    return (int)((need + waves - 1) / waves);
}

// warps per CTA so that the NST stages of all warps stay within ~110 KB (two CTAs per SM)
template <int KMAX>
static void launch_upd2_cp_k(const UpdArgs& a, cudaStream_t s) {
    constexpr int NST = 3;
    constexpr int SWB = (KMAX + 1) * WLD * 8 * NST;
    constexpr int NW = (110 * 1024) / SWB >= 8 ? 8 : ((110 * 1024) / SWB >= 4 ? 4 : ((110 * 1024) / SWB >= 2 ? 2 : 1));
    auto kern = k_upd2_cp<KMAX, NST, NW>;
    const int smem = NW * SWB;
    kern<<<cp_grid(kern, smem, 32 * NW, a.nrows, NW), 32 * NW, smem, s>>>(a);
}

template <int KMAX, bool TWO>
static void launch_step1_cp_k(const SdotsArgs& a, cudaStream_t s) {
    constexpr int NST = 3;
    constexpr int SWB = KMAX * WLD * 8 * NST;
    constexpr int NW = (110 * 1024) / SWB >= 8 ? 8 : ((110 * 1024) / SWB >= 4 ? 4 : ((110 * 1024) / SWB >= 2 ? 2 : 1));
    auto kern = k_step1_cp<KMAX, TWO, NST, NW>;
    const int smem = NW * SWB;
    kern<<<cp_grid(kern, smem, 32 * NW, a.nrows, NW), 32 * NW, smem, s>>>(a);
}

bool launch_step1_cp(const SdotsArgs& a, int kmax, cudaStream_t s) {
    const bool two = a.set2 != 0;
    switch (kmax) {
        case 8: two ? launch_step1_cp_k<8, true>(a, s) : launch_step1_cp_k<8, false>(a, s); break;
        case 16: two ? launch_step1_cp_k<16, true>(a, s) : launch_step1_cp_k<16, false>(a, s); break;
        case 24: two ? launch_step1_cp_k<24, true>(a, s) : launch_step1_cp_k<24, false>(a, s); break;
        case 32: two ? launch_step1_cp_k<32, true>(a, s) : launch_step1_cp_k<32, false>(a, s); break;
        case 40: two ? launch_step1_cp_k<40, true>(a, s) : launch_step1_cp_k<40, false>(a, s); break;
        case 48: two ? launch_step1_cp_k<48, true>(a, s) : launch_step1_cp_k<48, false>(a, s); break;
        default: return false;
    }
    return true;
}

bool launch_upd2_cp(const UpdArgs& a, int kmax, cudaStream_t s) {
    switch (kmax) {
        case 8: launch_upd2_cp_k<8>(a, s); break;
        case 16: launch_upd2_cp_k<16>(a, s); break;
        case 24: launch_upd2_cp_k<24>(a, s); break;
        case 32: launch_upd2_cp_k<32>(a, s); break;
        case 40: launch_upd2_cp_k<40>(a, s); break;
        case 48: launch_upd2_cp_k<48>(a, s); break;
        default: return false;
    }
    return true;
}

}  // namespace trplk
