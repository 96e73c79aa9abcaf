// Register-stream K1 of the inner step (default for every shape but the long C5 slabs, where
// k1_pipe.cuh runs):
//
//   k_step1_rs2  z = A g, w = M (z - rho B g), T(1:k,k) = U^T z, h1 = U^T w, ||w||^2
//                (eq 3.1; the preconditioned next vector of P:143 as reading R1;
//                the first CGS2 pass coefficients of reading R3); with A absent the first-pass
//                dots U^T x, x^T x of every other CGS2 (seed, +K: reading R3)
//
// A warp owns two 32-row tiles per iteration (lane = row): it issues the loads of both tiles'
// basis rows, DIA values and gathers together, parks the rows in a private shared-memory slab
// (column stride WLD = 36 doubles: conflict-free row-wise and in DMMA fragment order) and
// contracts U^T [z w] on fp64 DMMA (mma.sync m8n8k4), accumulators in registers for the whole
// kernel.  Measured choices: profiles/r01_variants.md.  Included by kernels.cu (mat_row,
// grid_reduce and sdots_finalize are shared and inlined); k1_pipe.cuh, rotate.cuh and
// inner_grid.cuh use the helpers below.
#pragma once

namespace trplk {

__device__ __forceinline__ void dmma884_s(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// fp64 DMMA without `volatile`: the compiler may interleave independent accumulator chains
__device__ __forceinline__ void dmma884_nv(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum_s(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------- register-stream + shared-memory transpose variant
// Each warp loads its 32-row tile of U in row layout (lane = row, all k column loads issued
// at once, before the SpMV's dependent gathers), parks it in a private shared-memory slab
// (column stride 36 doubles = 8 mod 32 banks), and reads it back in DMMA fragment order.
// U is read from HBM/L2 exactly once; no block-level barriers in the main loop.
constexpr int WLD = 36;

// Slab width of the one-tile-per-warp streaming kernels (inner_grid.cuh): 24 columns up to k = 32;
// 16 beyond, where 24 registers of the basis row plus 2 k/8 DMMA accumulators no longer fit 128
// registers without spilling.
__host__ __device__ constexpr int rs_chunk(int kmax) { return kmax < 24 ? kmax : (kmax > 32 ? 16 : 24); }

// K1 with two 32-row tiles per warp per iteration (the one-tile kernel it replaced measured
// slower and was removed): the loads of both tiles (basis rows, DIA values, gathers) are in flight
// together, so a warp walks half as many dependent load round trips; 8-column slab chunks,
// one slab per tile.  C2: K1 24.5 -> 22.6 us, solve -2.7 %; C3: K1 145 -> 135 us, -2.9 %.
template <int KMAX, bool TWO>
__global__ void __launch_bounds__(CTA, 2) k_step1_rs2(const SdotsArgs a) {
    pdl_wait();
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
    const double* __restrict__ X = resolve_x(a.x, a.x_dyn, a.x_ld, a.x_off, ctl);
    const double* __restrict__ X2 = a.set2 == 4 ? resolve_x(a.x2, a.x2_dyn, a.x2_ld, a.x2_off, ctl) : nullptr;
    double n2 = 0.0;
    constexpr int CH = 8;
    extern __shared__ __align__(128) double wsm[];  // WARPS x 2 x CH x WLD
    __shared__ double acc[WARPS][NV_MAX];
    __shared__ double res[NV_MAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* W0 = wsm + (size_t)warp * 2 * CH * WLD;
    double* W1 = W0 + CH * WLD;
    // one accumulator chain per 8-column chunk, the two tiles' DMMAs in order (volatile): the
    // round-2 variant with the tiles in separate, interleaved chains measured slower (C2 solve
    // 63.7 vs 62.6 ms, C5 K1 at k = 23 6.91 vs 6.67 ms; profiles/r02_variants.md)
    double cacc[KMAX / 8][2];
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
    double n1 = 0.0;
    const int64_t nslices = (a.nrows + 31) >> 5;
    const int64_t sbeg = a.row0 >> 5;  // first tile of the row range
    const int64_t npairs = (nslices - sbeg + 1) >> 1;
    auto tile = [&](int64_t sl, bool live, double& v1, double& o) {
        const int64_t row = sl * 32 + lane;
        const bool ok = live && row < a.nrows;
        double z = 0.0, ad = 1.0, bd = 1.0, sv = 0.0;
        o = 0.0;
        const double xr = ok ? X[row] : 0.0;
        if (live) {
            z = a.A.nrows ? mat_row(a.A, sl, lane, X, ad) : xr;  // A absent: dots of x itself
            if (a.out_mode == 2) {
                if (a.B.nrows) sv = mat_row(a.B, sl, lane, X, bd);
                else sv = xr;
                o = jacobi_minv(ad, bd, a.pmode == 2 ? rho : a.sigma, a.mfloor) * (z - rho * sv);  // w = M (z - rho B g), R1
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
        if (TWO && a.set2 == 4) {  // second dot set on the external vector x2
            const double x2 = ok ? X2[row] : 0.0;
            n2 += x2 * x2;
            o = x2;
        }
    };
    for (int64_t pr = (int64_t)blockIdx.x * WARPS + warp; pr < npairs; pr += (int64_t)gridDim.x * WARPS) {
        const int64_t s0 = sbeg + 2 * pr, s1 = s0 + 1;
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
        if (lane == 0 && a.norm1) acc[warp][k1 + k2] = s1;
        if (a.norm2 == 5) {
            const double s2 = warp_sum_s(n2);
            if (lane == 0) acc[warp][k1 + k2 + (a.norm1 ? 1 : 0)] = s2;
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
    pdl_trigger();
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res, a.cta_off, a.cta_tot)) return;
    if (a.red_local) {
        for (int v = threadIdx.x; v < nv; v += CTA) a.red_local[v] = res[v];
    } else {
        sdots_finalize(a, res, k1, k2);
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
    const int smem2 = WARPS * 2 * 8 * WLD * (int)sizeof(double);
    auto kern2 = k_step1_rs2<KMAX, TWO>;
    NOTE_KERN(kern2);
    launch_pdl(kern2, a.grid_force > 0 ? a.grid_force : rs_grid(kern2, smem2, (a.nrows - a.row0 + 1) / 2), CTA, smem2, s, a);
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

}  // namespace trplk
