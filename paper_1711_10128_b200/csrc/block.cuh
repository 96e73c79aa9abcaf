// Multi-vector ("block") kernels: c <= 8 vectors against a basis block of k <= 64 columns in ONE
// pass over the basis -- the +K augmentation of Alg. 1 steps 6-8 (the l
// previous Ritz vectors are orthogonalised and multiplied by A together, "l matrix-vector
// products") as block classical Gram-Schmidt with Cholesky-QR inside the block (BCGS2),
// instead of l sequential column-by-column CGS2 + SpMV passes.  SURVEY 8(a) S5 ("Block CGS2
// (K4 Gram (n x k)^T (n x c)) + SpMM over c vectors").
//
//   k_blk<KMAX, BM_GRAM>  sums = [U^T Y (k x c) | Y^T Y (c x c)]
//   k_blk<KMAX, BM_UPD>   Q = Y Rinv (optional c x c upper triangle), Y' = Q - U H -> Yout,
//                         sums = [U^T Y' | Y'^T Y']
//   k_blk<KMAX, BM_SPMM>  Z = A Y (c SpMVs sharing the matrix tile), sums = [U^T Z]
//
// A warp owns a 32-row tile (lane = row): all k basis loads of the tile in flight, the tile parked
// in a private shared-memory slab (column stride WLD = 36: conflict-free for both fragment
// orders), the vectors in a second slab.  U H is formed on fp64 DMMA as (H^T U^T)^T per 8-row
// block (A operand H^T in registers, as the rotation kernel), the dots U^T V and V^T V on DMMA with
// V from the slab as the B operand (m8n8k4: n = 8 vectors).  Per-CTA sums are added warp by warp
// in a fixed order, then grid_reduce (fixed order): bitwise reproducible for a given grid.
// Included by kernels.cu after stream_rs.cuh (WLD, dmma884_s, mat_row, grid_reduce).
#pragma once

namespace trplk {

__device__ __forceinline__ int blk_count(const BlkArgs& a, const Ctl* ctl) {
    int c = a.c_dyn ? *a.c_dyn : a.c;
    if (a.c_cap && *a.c_cap < c) c = *a.c_cap;
    return c;
}

__device__ __forceinline__ int blk_nv(int mode, int k, int c) {
    return mode == BM_SPMM ? k * c : (mode == BM_SPMW ? 2 * k * c + c * c : k * c + c * c);
}

// last CTA (or the multi-rank finalize): scatter the sums r = [U^T V (k x c) | V^T V (c x c)]
// (SPMW: [U^T Z | U^T W | W^T W])
__device__ void blk_finalize(const BlkArgs& a, const double* r, int k, int c) {
    const int64_t nkc = (int64_t)k * c;
    if (a.mode == BM_SPMW) {
        const int k0 = *a.k0p;
        for (int64_t v = threadIdx.x; v < nkc; v += blockDim.x) {
            const int i = (int)(v % k), j = (int)(v / k);
            if (i <= k0 + j) {
                a.T[i + (int64_t)(k0 + j) * a.ldT] = r[v];
                if (i < k0 + j) a.T[(k0 + j) + (int64_t)i * a.ldT] = r[v];
            }
            a.HV[i + (int64_t)QMAX * j] = r[nkc + v];
        }
        for (int v = threadIdx.x; v < c * c; v += blockDim.x) a.G[(v % c) + BC * (v / c)] = r[2 * nkc + v];
        return;
    }
    if (a.T) {  // SPMM: T columns k0 .. k0+c-1 of eq 3.1 (T(1:k, col) = U^T A x~), mirrored
        // entry (i, k0 + j) with i <= k0 + j, mirrored below the diagonal: as the column-by-column
        // order (each entry from the later column's product), so no address is written twice
        const int k0 = *a.k0p;
        for (int64_t v = threadIdx.x; v < nkc; v += blockDim.x) {
            const int i = (int)(v % k), j = (int)(v / k);
            if (i > k0 + j) continue;
            a.T[i + (int64_t)(k0 + j) * a.ldT] = r[v];
            if (i < k0 + j) a.T[(k0 + j) + (int64_t)i * a.ldT] = r[v];
        }
        return;
    }
    for (int64_t v = threadIdx.x; v < nkc; v += blockDim.x) {
        const int i = (int)(v % k), j = (int)(v / k);
        a.HV[i + (int64_t)QMAX * j] = r[v];
    }
    if (a.mode != BM_SPMM)
        for (int v = threadIdx.x; v < c * c; v += blockDim.x) a.G[(v % c) + BC * (v / c)] = r[nkc + v];
}

template <int KMAX, int MODE, int LB>
__global__ void __launch_bounds__(CTA, LB) k_blk(const BlkArgs a) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int k = a.k_from_ctl ? ctl->k + a.k_off : a.k;
    const int c = blk_count(a, ctl);
    if (c <= 0) return;
    constexpr bool SPW = MODE == BM_SPMW;
    const int nv = blk_nv(MODE, k, c);
    extern __shared__ __align__(128) double bsm[];
    __shared__ double res[BLK_NV];
    __shared__ double Rs[BC * BC];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fi = lane >> 2, fj = lane & 3;
    double* Wt = bsm + (size_t)warp * (KMAX + (SPW ? 2 : 1) * BC) * WLD;  // basis tile: column j at Wt[j * WLD]
    double* Vs = Wt + KMAX * WLD;                          // vector slab: vector j at Vs[j * WLD]
    double* Ws = Vs + BC * WLD;                            // SPMW: preconditioned vectors
    const double rho = ctl->rho;
    const bool useR = MODE == BM_UPD && a.Rinv != nullptr;
    // Y may alias Yout (in-place update): each warp reads its whole tile before writing it
    const double* Yp = a.y_dyn == 2 ? a.Y + a.ldy * (int64_t)ctl->xprev_col : a.Y;
    for (int i = threadIdx.x; i < BC * BC; i += CTA) Rs[i] = useR ? a.Rinv[i] : 0.0;
    for (int i = threadIdx.x; i < BLK_NV; i += CTA) res[i] = 0.0;
    __syncthreads();
    // A operand H^T of the product U H (lane (fi, fj): vector fi, basis index 4 ks + fj)
    double hf[KMAX / 4];
#pragma unroll
    for (int ks = 0; ks < KMAX / 4; ++ks)
        hf[ks] = (MODE == BM_UPD && 4 * ks + fj < k && fi < c) ? __ldg(a.H + (4 * ks + fj) + (int64_t)QMAX * fi) : 0.0;
    double cacc[KMAX / 8][2], wacc[SPW ? KMAX / 8 : 1][2], gacc[2] = {0.0, 0.0};
#pragma unroll
    for (int g = 0; g < KMAX / 8; ++g) cacc[g][0] = cacc[g][1] = 0.0;
#pragma unroll
    for (int g = 0; g < (SPW ? KMAX / 8 : 1); ++g) wacc[g][0] = wacc[g][1] = 0.0;
    const int64_t ntile = (a.nrows + 31) >> 5;
    const int64_t tstride = (int64_t)gridDim.x * WARPS;
    // KMAX <= 32: the next tile's basis rows are loaded while this tile is contracted (one tile of
    // loads always in flight per warp; measured necessary: without it a warp's loads and its DMMA /
    // shared-memory phase alternate and the kernel streamed at ~1/3 of the DRAM peak at C5)
    constexpr bool PF = KMAX <= 32 && LB == 1;
    double un[PF ? KMAX : 1];
    if (PF) {
        const int64_t t0 = (int64_t)blockIdx.x * WARPS + warp, row0 = t0 * 32 + lane;
#pragma unroll
        for (int j = 0; j < (PF ? KMAX : 1); ++j)
            un[j] = (row0 < a.nrows && j < k) ? __ldg(a.U + (int64_t)j * a.ldu + row0) : 0.0;
    }
    for (int64_t t = (int64_t)blockIdx.x * WARPS + warp; t < ntile; t += tstride) {
        const int64_t r0 = t * 32, row = r0 + lane;
        const bool ok = row < a.nrows;
        double ur[KMAX];
        if (PF) {
            const int64_t rown = row + tstride * 32;
#pragma unroll
            for (int j = 0; j < KMAX; ++j) {
                ur[j] = un[PF ? j : 0];
                un[PF ? j : 0] = (rown < a.nrows && j < k) ? __ldg(a.U + (int64_t)j * a.ldu + rown) : 0.0;
            }
        } else {
#pragma unroll
            for (int j = 0; j < KMAX; ++j) ur[j] = (ok && j < k) ? __ldg(a.U + (int64_t)j * a.ldu + row) : 0.0;
        }
        double v[BC], wv[SPW ? BC : 1];
        if (MODE == BM_SPMM || SPW) {
#pragma unroll
            for (int j = 0; j < BC; ++j) {
                double d = 1.0;
                v[j] = (j < c) ? mat_row(a.A, t, lane, Yp + (int64_t)j * a.ldy, d) : 0.0;
                if (!ok) v[j] = 0.0;
                if (SPW) {  // w = M (z - rho g), reading R1, one shift for the block (reading B1)
                    const double yr = (ok && j < c) ? Yp[(int64_t)j * a.ldy + row] : 0.0;
                    wv[j] = (ok && j < c) ? jacobi_minv(d, 1.0, a.sigma, a.mfloor) * (v[j] - rho * yr) : 0.0;
                    if (ok && j < c) a.Yout[(int64_t)j * a.ldyo + row] = wv[j];
                }
            }
        } else {
            double y[BC];
#pragma unroll
            for (int j = 0; j < BC; ++j) y[j] = (ok && j < c) ? Yp[(int64_t)j * a.ldy + row] : 0.0;
            if (useR) {
#pragma unroll
                for (int j = 0; j < BC; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int i = 0; i <= j; ++i) s = fma(y[i], Rs[i + BC * j], s);
                    v[j] = s;
                }
            } else {
#pragma unroll
                for (int j = 0; j < BC; ++j) v[j] = y[j];
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < KMAX; ++j) Wt[j * WLD + lane] = ur[j];
#pragma unroll
        for (int j = 0; j < BC; ++j) Vs[j * WLD + lane] = v[j];
        if (SPW) {
#pragma unroll
            for (int j = 0; j < BC; ++j) Ws[j * WLD + lane] = wv[SPW ? j : 0];
        }
        __syncwarp();
        if (MODE == BM_UPD) {  // Y' = Q - U H: (H^T U^T) per 8-row block, lane: vector fi, rows 2 fj, 2 fj + 1
            // the four 8-row blocks' accumulators interleaved: four independent DMMA chains
            double d4[4][2];
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) d4[rb][0] = d4[rb][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KMAX / 4; ++ks)
#pragma unroll
                for (int rb = 0; rb < 4; ++rb) dmma884_nv(d4[rb], hf[ks], Wt[(4 * ks + fj) * WLD + 8 * rb + fi]);
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) {
                const double* d2 = d4[rb];
                const int rr = 8 * rb + 2 * fj;
                const double y0 = Vs[fi * WLD + rr] - d2[0], y1 = Vs[fi * WLD + rr + 1] - d2[1];
                Vs[fi * WLD + rr] = y0;
                Vs[fi * WLD + rr + 1] = y1;
                if (fi < c && a.Yout) {
                    double* yo = a.Yout + (int64_t)fi * a.ldyo + r0 + rr;
                    if (r0 + rr < a.nrows) yo[0] = y0;
                    if (r0 + rr + 1 < a.nrows) yo[1] = y1;
                }
            }
            __syncwarp();
        }
        // dots: U^T V (basis chunk g, vectors) and V^T V on DMMA over the 32 rows (8 k-steps of 4);
        // the chunks' accumulators (independent chains) interleaved per k-step
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double bv = Vs[fi * WLD + 4 * q + fj];  // B operand (vector fi, row 4q + fj) = A of V^T V
            const double bw = SPW ? Ws[fi * WLD + 4 * q + fj] : 0.0;
#pragma unroll
            for (int g = 0; g < KMAX / 8; ++g) {
                if (8 * g < k) {
                    const double au = Wt[(8 * g + fi) * WLD + 4 * q + fj];
                    dmma884_nv(cacc[g], au, bv);
                    if (SPW) dmma884_nv(wacc[SPW ? g : 0], au, bw);
                }
            }
            if (MODE != BM_SPMM) {
                const double b2 = SPW ? bw : bv;
                dmma884_nv(gacc, b2, b2);
            }
        }
        __syncwarp();
    }
    // per-CTA sums, warp by warp in index order (lane: basis 8 g + fi, vectors 2 fj, 2 fj + 1)
    for (int w = 0; w < WARPS; ++w) {
        if (warp == w) {
#pragma unroll
            for (int g = 0; g < KMAX / 8; ++g) {
                const int i = 8 * g + fi;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 2 * fj + e;
                    if (i < k && j < c) {
                        res[i + k * j] += cacc[g][e];
                        if (SPW) res[k * c + i + k * j] += wacc[SPW ? g : 0][e];
                    }
                }
            }
            if (MODE != BM_SPMM) {
                const int go = SPW ? 2 * k * c : k * c;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 2 * fj + e;
                    if (fi < c && j < c) res[go + fi + c * j] += gacc[e];
                }
            }
        }
        __syncthreads();
    }
    if (!grid_reduce(res, nv, a.part, a.gpart, a.counter, a.maxcta, res)) return;
    if (a.red_local) {
        for (int i = threadIdx.x; i < nv; i += CTA) a.red_local[i] = res[i];
        return;
    }
    blk_finalize(a, res, k, c);
}

// k <= 24: two CTAs per SM (<= 128 registers, no register prefetch) -- measured at C5 (k = 24,
// c = 2, through trplk_k_block): GRAM 5.5 -> 6.2 TB/s, UPD 3.1 -> 4.2, SPMM 3.2 -> 4.4 against
// one CTA with the next tile's rows prefetched into registers.  TRPLK_BLK_LB=1 selects the latter.
static int blk_lb() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TRPLK_BLK_LB");
        v = (e && e[0] == '1') ? 1 : 2;
    }
    return v;
}

template <int KMAX, int MODE, int LB>
static void launch_blk_kl(const BlkArgs& a, cudaStream_t s) {
    const int smem = WARPS * (KMAX + (MODE == BM_SPMW ? 2 : 1) * BC) * WLD * (int)sizeof(double);
    auto kern = k_blk<KMAX, MODE, LB>;
    static bool init = false;
    static int grid_cap = 0;
    if (!init) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, smem);
        grid_cap = nsm_s() * (occ < 1 ? 1 : occ);
        if (grid_cap > MAXCTA) grid_cap = MAXCTA;
        init = true;
    }
    const int64_t need = ((a.nrows + 31) / 32 + WARPS - 1) / WARPS;
    int64_t g = need < grid_cap ? need : grid_cap;
    if (g < 1) g = 1;
    NOTE_KERN(kern);
    kern<<<(int)g, CTA, smem, s>>>(a);
}

template <int KMAX, int MODE>
static void launch_blk_k(const BlkArgs& a, cudaStream_t s) {
    if (KMAX <= 24 && blk_lb() == 2) launch_blk_kl<KMAX, MODE, 2>(a, s);
    else launch_blk_kl<KMAX, MODE, 1>(a, s);
}

template <int MODE>
static bool launch_blk_m(const BlkArgs& a, int kmax, cudaStream_t s) {
    if (kmax <= 8) launch_blk_k<8, MODE>(a, s);
    else if (kmax <= 16) launch_blk_k<16, MODE>(a, s);
    else if (kmax <= 24) launch_blk_k<24, MODE>(a, s);
    else if (kmax <= 32) launch_blk_k<32, MODE>(a, s);
    else if (kmax <= 48) launch_blk_k<48, MODE>(a, s);
    else if (kmax <= 64) launch_blk_k<64, MODE>(a, s);
    else return false;
    return true;
}

bool launch_block(const BlkArgs& a, int kmax, cudaStream_t s) {
    if (a.mode == BM_GRAM) return launch_blk_m<BM_GRAM>(a, kmax, s);
    if (a.mode == BM_UPD) return launch_blk_m<BM_UPD>(a, kmax, s);
    if (a.mode == BM_SPMM) return launch_blk_m<BM_SPMM>(a, kmax, s);
    if (a.mode == BM_SPMW) return launch_blk_m<BM_SPMW>(a, kmax, s);
    return false;
}

// ------------------------------------------------------------ BCGS2 control (one CTA, c <= 8)
// Cholesky-QR of the block Gram G (c x c, ld BC) restricted to the vectors not yet dropped; a
// pivot that leaves less than 1e-14 of the input norm of vector j (lprod_j * sqrt(d_j) <
// 1e-14 ||x_j||, the CGS2 breakdown rule of R3 / R16) drops j.  Writes Rinv = R^-1 (upper).
__device__ void blk_cholqr(BlkCtl* b, const double* G, int c) {
    double L[BC][BC];
    for (int i = 0; i < BC; ++i)
        for (int j = 0; j < BC; ++j) L[i][j] = 0.0;
    for (int j = 0; j < c; ++j) {
        if (b->drop[j]) continue;
        double d = G[j + BC * j];
        for (int p = 0; p < j; ++p) d -= L[j][p] * L[j][p];
        const double keep = b->lprod[j] * b->lprod[j] * (d > 0.0 ? d : 0.0);
        if (!(d > 0.0) || keep < 1e-28 * b->g0[j]) {
            b->drop[j] = 1;
            continue;
        }
        L[j][j] = sqrt(d);
        b->lprod[j] *= L[j][j];
        for (int i = j + 1; i < c; ++i) {
            if (b->drop[i]) continue;
            double s = G[i + BC * j];
            for (int p = 0; p < j; ++p) s -= L[i][p] * L[j][p];
            L[i][j] = s / L[j][j];
        }
    }
    // Rinv = (L^T)^-1: upper triangular, column j solves L^T r = e_j by back substitution
    for (int i = 0; i < BC * BC; ++i) b->Rinv[i] = 0.0;
    for (int j = 0; j < c; ++j) {
        if (b->drop[j]) continue;
        for (int i = j; i >= 0; --i) {
            if (b->drop[i]) continue;
            double s = (i == j) ? 1.0 : 0.0;
            for (int p = i + 1; p <= j; ++p)
                if (!b->drop[p]) s -= L[p][i] * b->Rinv[p + BC * j];
            b->Rinv[i + BC * j] = s / L[i][i];
        }
    }
}

__global__ void k_blk_ctl(BlkCtl* b, Ctl* ctl, int stage, int cst, const int* c_dyn, int seed, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    if (threadIdx.x == 0) {
        const int k = ctl->k;
        const int c = c_dyn ? *c_dyn : cst;
        if (stage == 1) {  // after GRAM + first UPD: inputs' norms, first Cholesky-QR
            b->c = c;
            for (int j = 0; j < BC; ++j) {
                b->drop[j] = 0;
                b->lprod[j] = 1.0;
                b->g0[j] = j < c ? b->G[0][j + BC * j] : 0.0;
                if (j < c && !(b->g0[j] > 0.0)) b->drop[j] = 1;
            }
        }
        const double* G = b->G[stage];
        blk_cholqr(b, G, c);
        bool pass3 = false;
        if (stage == 2)  // R3: the second pass kept less than 1/sqrt2 of the (unit) first-pass norm
            for (int j = 0; j < c; ++j)
                if (!b->drop[j] && G[j + BC * j] < 0.5) pass3 = true;
        // next coefficients: Hs = (U^T W) Rinv
        const double* HV = b->HV[stage];
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < c; ++j) {
                double s = 0.0;
                for (int p = 0; p <= j; ++p) s += HV[i + QMAX * p] * b->Rinv[p + BC * j];
                b->Hs[i + QMAX * j] = s;
            }
        if (stage == 2 && pass3) {
            ctl->flags |= F_BPASS3;
            b->pass3 = 1;
            ctl->pass3_count += 1;
        } else if (stage >= 2) {  // placement: accepted vectors appended after the current basis
            ctl->flags &= ~F_BPASS3;
            b->pass3 = 0;
            int acc = 0;
            for (int j = 0; j < c; ++j) {
                if (b->drop[j]) {
                    if (!seed) ctl->flags &= ~(F_KCOL0 << j);
                    ctl->brk += 1;
                    b->pos[j] = -1;
                } else {
                    b->pos[j] = acc++;
                }
            }
            for (int j = c; j < BC; ++j) b->pos[j] = -1;
            b->acc = acc;
            b->k0 = k;
            ctl->k = k + acc;
            // seed block: the target's own seed dependent -> the cycle has no seed (R16: the host
            // injects a random vector and repeats the cycle)
            if (seed && b->drop[0]) ctl->flags &= ~F_CYCLE;
            // inner groups: the images that still fit the basis (room = kcap - k); 0 ends the loop
            b->cin = acc;
        }
    }
}

void launch_blk_ctl(BlkCtl* b, Ctl* ctl, int stage, int c, const int* c_dyn, int seed, unsigned gate,
                    cudaStream_t s) {
    k_blk_ctl<<<1, 32, 0, s>>>(b, ctl, stage, c, c_dyn, seed, gate);
}

// block inner loop: the next group's size, the accepted vectors that still fit the basis
__global__ void k_blk_room(BlkCtl* b, const Ctl* ctl, int kcap, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    if (threadIdx.x == 0) {
        const int room = kcap - ctl->k;
        b->cin = b->acc < room ? b->acc : (room > 0 ? room : 0);
    }
}

void launch_blk_room(BlkCtl* b, const Ctl* ctl, int kcap, unsigned gate, cudaStream_t s) {
    k_blk_room<<<1, 32, 0, s>>>(b, ctl, kcap, gate);
}

// Q = W Rinv for the accepted vectors, into the basis (U(:, k0 + pos_j)) and the +K scratch block
__global__ void k_blk_place(const double* __restrict__ W, int64_t ldw, const BlkCtl* b, const Ctl* ctl,
                            double* U, int64_t ldu, double* xk, int64_t ldx, int64_t nrows, int cst, unsigned gate) {
    if ((ctl->flags & gate) != gate) return;
    const int c = cst > 0 ? cst : b->c;
    if (ctl->flags & F_BPASS3) return;  // (never: the placement follows the last pass)
    __shared__ double R[BC * BC];
    __shared__ int pos[BC];
    for (int i = threadIdx.x; i < BC * BC; i += blockDim.x) R[i] = b->Rinv[i];
    if (threadIdx.x < BC) pos[threadIdx.x] = threadIdx.x < c ? b->pos[threadIdx.x] : -1;
    __syncthreads();
    const int k0 = b->k0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        double w[BC];
#pragma unroll
        for (int i = 0; i < BC; ++i) w[i] = i < c ? W[(int64_t)i * ldw + r] : 0.0;
#pragma unroll
        for (int j = 0; j < BC; ++j) {
            if (j >= c || pos[j] < 0) continue;
            double s = 0.0;
#pragma unroll
            for (int i = 0; i <= j; ++i) s = fma(w[i], R[i + BC * j], s);
            U[(int64_t)(k0 + pos[j]) * ldu + r] = s;
            if (xk) xk[(int64_t)pos[j] * ldx + r] = s;
        }
    }
}

void launch_blk_place(const double* W, int64_t ldw, const BlkCtl* b, const Ctl* ctl, double* U, int64_t ldu,
                      double* xk, int64_t ldx, int64_t nrows, int c, unsigned gate, cudaStream_t s) {
    int64_t g = (nrows + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_blk_place<<<(int)g, 256, 0, s>>>(W, ldw, b, ctl, U, ldu, xk, ldx, nrows, c, gate);
}

// multi-rank: the gathered per-rank sums added in rank order on every rank, then scattered
__global__ void k_blk_finalize_multi(const BlkArgs a, const double* red_all, int nranks, int stride) {
    Ctl* ctl = a.ctl;
    if ((ctl->flags & a.gate) != a.gate) return;
    const int k = a.k_from_ctl ? ctl->k + a.k_off : a.k;
    const int c = blk_count(a, ctl);
    if (c <= 0) return;
    const int nv = blk_nv(a.mode, k, c);
    __shared__ double r[BLK_NV];
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < nranks; ++q) s += red_all[(int64_t)q * stride + v];
        r[v] = s;
    }
    __syncthreads();
    blk_finalize(a, r, k, c);
}

void launch_blk_finalize_multi(const BlkArgs& a, const double* red_all, int nranks, int stride, cudaStream_t s) {
    k_blk_finalize_multi<<<1, 256, 0, s>>>(a, red_all, nranks, stride);
}

}  // namespace trplk
