// IC(0) preconditioner on the device (NEXT-2 of SURVEY 8(f); "incomplete ILU or LDL
// factorization"; reading P2a of DESIGN.md) for DIA matrices, one rank, B = I:
//   factor  L with the lower pattern of K = A - sigma I (no fill): for the lower offsets o_a in
//           ascending order, L(i, i+o_a) = (K(i, i+o_a) - sum_{o_b < o_a} L(i, i+o_b) L(i+o_a, i+o_b))
//           / L(i+o_a, i+o_a);  L(i, i) = sqrt(K_ii - sum_a L(i, i+o_a)^2) (pivot floor: R12's)
//   apply   M v = (L L^T)^-1 v: forward solve L y = v, backward solve L^T w = y.
// A slot of A whose value is 0 is outside the pattern (the DIA scatter stores 0 for absent
// entries; an explicitly stored zero of the CSR input would be in the oracle's pattern only).
//
// Scheduling is sync-free (no level analysis): 32-row chunks (a warp, lane = row) are claimed in
// row order through an atomic ticket (reverse order for L^T); a warp spins on the done-flags of the
// earlier chunks its rows depend on (claimed by running warps, so it always makes progress), then
// resolves the dependencies inside its own chunk: offset -1 (+1 for L^T) by an affine scan across
// the lanes (y_l = p_l - b_l y_{l-1}: five shuffle rounds), any other offset shorter than 32 by a
// lane-by-lane loop.  The critical path is the grid's wavefront (x + y + z for a 7-point stencil);
// the rest streams.  Included by kernels.cu (DIA helpers).
#pragma once

namespace trplk {


// spin on a done-flag; a dependency that never completes (a scheduling bug) traps after ~10 s
// instead of hanging the device
__device__ __forceinline__ int ic0_chunk_wait(const int* flags, int64_t c) {
    if (c < 0) return 1;
    const volatile int* f = flags + c;
    unsigned long long spins = 0;
    while (*f == 0) {
        __nanosleep(64);
        if (++spins > (1ull << 27)) __trap();
    }
    return 1;
}

// the warp waits for every chunk (other than its own) that one of its lanes depends on:
// lane-specific chunk ids, deduplicated by a ballot loop; reverse = the chunks after c (L^T)
__device__ __forceinline__ void ic0_wait_deps(const int* flags, int64_t c, int64_t dc, bool reverse, int64_t nchunk) {
    const bool need = dc >= 0 && (reverse ? (dc > c && dc < nchunk) : dc < c);
    unsigned m = __ballot_sync(0xffffffffu, need);
    while (m) {
        const int src = __ffs(m) - 1;
        const int64_t w = __shfl_sync(0xffffffffu, dc, src);
        if ((threadIdx.x & 31) == 0) ic0_chunk_wait(flags, w);
        m &= ~__ballot_sync(0xffffffffu, need && dc == w);
    }
}

// ----------------------------------------------------------------------------- factorization
__global__ void __launch_bounds__(256) k_ic0_factor(const Ic0Args a) {
    if (a.ctl && (a.ctl->flags & a.gate) != a.gate) return;
    const int lane = threadIdx.x & 31;
    const int64_t nchunk = (a.n + 31) >> 5;
    unsigned* ticket = reinterpret_cast<unsigned*>(a.flags + nchunk);
    for (;;) {
        int64_t c = 0;
        if (lane == 0) c = atomicAdd(ticket, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= nchunk) return;
        const int64_t r0 = c * 32, i = r0 + lane;
        const bool ok = i < a.n;
        // dependencies on earlier chunks, only where the entry exists (K_ij != 0): a Dirichlet
        // boundary row has no left neighbour, so a grid line does not wait for the previous one
        for (int d = 0; d < a.nlow; ++d) {
            const int64_t j = i + a.loff[d];
            const bool dep = ok && j >= 0 && __ldg(a.A.dval + (int64_t)a.lslot[d] * a.A.ldv + i) != 0.0;
            ic0_wait_deps(a.flags, c, dep ? (j >> 5) : -1, false, (int64_t)0);
        }
        __syncwarp();
        __threadfence();
        // rows one at a time inside the chunk (their in-chunk dependencies come before them)
        for (int l = 0; l < 32; ++l) {
            if (lane == l && ok) {
                double Li[DIA_MAX];
                double dsum = 0.0;
                for (int d = 0; d < a.nlow; ++d) {
                    const int64_t j = i + a.loff[d];
                    const double kij = j >= 0 ? __ldg(a.A.dval + (int64_t)a.lslot[d] * a.A.ldv + i) : 0.0;
                    double lij = 0.0;
                    if (kij != 0.0) {
                        double s = kij;
                        for (int b = 0; b < d; ++b) {
                            const int e = a.pair[d][b];
                            if (e >= 0 && Li[b] != 0.0) s -= Li[b] * __ldcg(a.L + (int64_t)e * a.ldl + j);
                        }
                        lij = s / __ldcg(a.L + (int64_t)a.nlow * a.ldl + j);
                    }
                    Li[d] = lij;
                    dsum = fma(lij, lij, dsum);
                    a.L[(int64_t)d * a.ldl + i] = lij;
                }
                double dg = __ldg(a.A.dval + (int64_t)a.A.diag_slot * a.A.ldv + i) - a.sigma;
                // K_ii - sum L_ij^2 in the oracle's order: subtract term by term
                double dd = dg;
                for (int d = 0; d < a.nlow; ++d) dd -= Li[d] * Li[d];
                (void)dsum;
                if (!(dd > a.floor)) dd = a.floor;
                a.L[(int64_t)a.nlow * a.ldl + i] = sqrt(dd);
            }
            __syncwarp();
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(a.flags + c, 1);
    }
}

// ----------------------------------------------------------------------------- solves
// Forward: y_i = (v_i - sum_a L(i, i+o_a) y_{i+o_a}) / L_ii, terms in ascending column order.
// Backward (L^T): y_i = (v_i - sum_a L(i-o_a, i) y_{i-o_a}) / L_ii, over the rows below i.
__global__ void __launch_bounds__(256) k_ic0_solve(const Ic0Args a) {
    if (a.ctl && (a.ctl->flags & a.gate) != a.gate) return;
    const int lane = threadIdx.x & 31;
    const int64_t nchunk = (a.n + 31) >> 5;
    unsigned* ticket = reinterpret_cast<unsigned*>(a.flags + nchunk);
    // does any offset other than -1 (+1) reach inside a chunk?  then lane-by-lane
    bool seq = false;
    for (int d = 0; d < a.nlow; ++d)
        if (a.loff[d] > -32 && a.loff[d] != -1) seq = true;
    int dm1 = -1;  // lower diagonal of offset -1
    for (int d = 0; d < a.nlow; ++d)
        if (a.loff[d] == -1) dm1 = d;
    const double* Ld = a.L + (int64_t)a.nlow * a.ldl;
    for (;;) {
        int64_t t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nchunk) return;
        const int64_t c = a.trans ? nchunk - 1 - t : t;
        const int64_t r0 = c * 32, i = r0 + lane;
        const bool ok = i < a.n;
        for (int d = 0; d < a.nlow; ++d) {  // only the entries of L that exist (L != 0)
            if (!a.trans) {
                const int64_t j = i + a.loff[d];
                const bool dep = ok && j >= 0 && __ldg(a.L + (int64_t)d * a.ldl + i) != 0.0;
                ic0_wait_deps(a.flags, c, dep ? (j >> 5) : -1, false, nchunk);
            } else {
                const int64_t k = i - a.loff[d];
                const bool dep = ok && k < a.n && __ldg(a.L + (int64_t)d * a.ldl + k) != 0.0;
                ic0_wait_deps(a.flags, c, dep ? (k >> 5) : -1, true, nchunk);
            }
        }
        __syncwarp();
        __threadfence();
        const double lii = ok ? __ldg(Ld + i) : 1.0;
        // terms from other chunks (and, when seq, everything but the in-chunk ones)
        double s = ok ? a.v[i] : 0.0;
        double bcoef = 0.0;  // coefficient of the in-chunk neighbour (offset -1 / +1)
        if (!a.trans) {
            for (int d = 0; d < a.nlow; ++d) {
                const int64_t j = i + a.loff[d];
                if (!ok || j < 0) continue;
                const double lij = __ldg(a.L + (int64_t)d * a.ldl + i);
                if (lij == 0.0) continue;  // no entry: y_j was not waited for
                if (j >= r0) {  // inside this chunk
                    if (d == dm1 && !seq) bcoef = lij;
                    continue;
                }
                s -= lij * __ldcg(a.y + j);
            }
        } else {
            for (int d = 0; d < a.nlow; ++d) {
                const int64_t k = i - a.loff[d];
                if (!ok || k >= a.n) continue;
                const double lki = __ldg(a.L + (int64_t)d * a.ldl + k);
                if (lki == 0.0) continue;
                if (k < r0 + 32) {
                    if (d == dm1 && !seq) bcoef = lki;
                    continue;
                }
                s -= lki * __ldcg(a.y + k);
            }
        }
        if (!seq) {
            // y_l = p_l - b_l y_{l-1} (forward) / y_l = p_l - b_l y_{l+1} (backward): affine scan
            double p = s / lii, b = bcoef / lii;
            const int dir = a.trans ? -1 : 1;
#pragma unroll
            for (int sh = 1; sh < 32; sh <<= 1) {
                const int src = lane - dir * sh;
                const double pp = __shfl_sync(0xffffffffu, p, (src & 31));
                const double bp = __shfl_sync(0xffffffffu, b, (src & 31));
                if (src >= 0 && src < 32) {  // compose: y = p - b (pp - bp y') = (p - b pp) + (b bp) y'
                    p = p - b * pp;
                    b = -b * bp;
                }
            }
            if (ok) a.y[i] = p;
        } else {
            // lane by lane with every in-chunk term
            for (int l = 0; l < 32; ++l) {
                const int ll = a.trans ? 31 - l : l;
                if (lane == ll && ok) {
                    double ss = s;
                    for (int d = 0; d < a.nlow; ++d) {
                        if (!a.trans) {
                            const int64_t j = i + a.loff[d];
                            if (j >= r0 && j >= 0) {
                                const double lij = __ldg(a.L + (int64_t)d * a.ldl + i);
                                if (lij != 0.0) ss -= lij * __ldcg(a.y + j);
                            }
                        } else {
                            const int64_t k = i - a.loff[d];
                            if (k < r0 + 32 && k < a.n) {
                                const double lki = __ldg(a.L + (int64_t)d * a.ldl + k);
                                if (lki != 0.0) ss -= lki * __ldcg(a.y + k);
                            }
                        }
                    }
                    a.y[i] = ss / lii;
                }
                __syncwarp();
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(a.flags + c, 1);
    }
}

static int ic0_grid() {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ic0_solve, 256, 0);
    return nsm * (occ < 1 ? 1 : occ);
}

void launch_ic0_factor(const Ic0Args& a, cudaStream_t s) {
    const int64_t nchunk = (a.n + 31) >> 5;
    cudaMemsetAsync(a.flags, 0, sizeof(int) * (size_t)(nchunk + 1), s);
    NOTE_KERN(k_ic0_factor);
    k_ic0_factor<<<ic0_grid(), 256, 0, s>>>(a);
}

void launch_ic0_solve(const Ic0Args& a, cudaStream_t s) {
    const int64_t nchunk = (a.n + 31) >> 5;
    cudaMemsetAsync(a.flags, 0, sizeof(int) * (size_t)(nchunk + 1), s);
    NOTE_KERN(k_ic0_solve);
    k_ic0_solve<<<ic0_grid(), 256, 0, s>>>(a);
}

}  // namespace trplk
