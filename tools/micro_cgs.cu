// Micro-benchmark of CGS pass layouts (tools/, not product): y = x - U h, d = U^T y, yy = y.y
// for k columns of an n-row column-major basis, thread-per-row with the k columns split over
// S lane groups (tile = 32/S rows per warp), R tiles per warp iteration (all loads first).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/micro_cgs tools/micro_cgs.cu
//   ./micro_cgs n ld
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int CTA = 256;

template <int K, int S, int R, int MINB, bool DOTS>
__global__ void __launch_bounds__(CTA, MINB) kupd(const double* __restrict__ U, long ld, const double* __restrict__ h,
                                                  const double* __restrict__ x, double* __restrict__ y, long n,
                                                  double* __restrict__ part) {
    constexpr int KS = K / S, TR = 32 / S;
    __shared__ double hs[K];
    __shared__ double red[CTA / 32][K + 1];
    for (int i = threadIdx.x; i < K; i += CTA) hs[i] = h[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / TR, rr = lane % TR;
    const int c0 = grp * KS;
    double acc[DOTS ? KS : 1];
#pragma unroll
    for (int c = 0; c < (DOTS ? KS : 1); ++c) acc[c] = 0.0;
    double yy = 0.0;
    const long ntile = (n + TR - 1) / TR;
    const long gw = (long)blockIdx.x * (CTA / 32) + warp, nw = (long)gridDim.x * (CTA / 32);
    for (long t0 = gw * R; t0 < ntile; t0 += nw * R) {
        double u[R][KS], xv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const long row = (t0 + r) * TR + rr;
            const bool ok = row < n;
#pragma unroll
            for (int c = 0; c < KS; ++c) u[r][c] = ok ? __ldg(U + (long)(c0 + c) * ld + row) : 0.0;
            xv[r] = ok ? __ldg(x + row) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const long row = (t0 + r) * TR + rr;
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < KS; ++c) s = fma(hs[c0 + c], u[r][c], s);
#pragma unroll
            for (int o = TR; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double yv = xv[r] - s;
            if (grp == 0 && row < n) y[row] = yv;
            if (DOTS) {
#pragma unroll
                for (int c = 0; c < KS; ++c) acc[c] = fma(u[r][c], yv, acc[c]);
            }
            if (grp == 0) yy = fma(yv, yv, yy);
        }
    }
    // reduce over the TR lanes of each group
#pragma unroll
    for (int c = 0; c < (DOTS ? KS : 1); ++c) {
        double v = acc[c];
#pragma unroll
        for (int o = 1; o < TR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (DOTS && rr == 0) red[warp][c0 + c] = v;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) yy += __shfl_xor_sync(0xffffffffu, yy, o);
    if (lane == 0) red[warp][K] = yy;
    __syncthreads();
    for (int v = threadIdx.x; v <= K; v += CTA) {
        double s = 0.0;
        for (int w = 0; w < CTA / 32; ++w) s += red[w][v];
        part[(long)v * gridDim.x + blockIdx.x] = s;
    }
}

// pure read of k columns + x, write y = x - sum (no dots), lane per row: reference stream
template <int K>
__global__ void __launch_bounds__(CTA, 2) kread(const double* __restrict__ U, long ld, const double* __restrict__ x,
                                                double* __restrict__ y, long n) {
    const long stride = (long)gridDim.x * CTA;
    for (long row = (long)blockIdx.x * CTA + threadIdx.x; row < n; row += stride) {
        double s = __ldg(x + row);
#pragma unroll
        for (int c = 0; c < K; ++c) s -= __ldg(U + (long)c * ld + row);
        y[row] = s;
    }
}

int nsm;

template <typename F>
float timeit(F f, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

template <int K, int S, int R, int MINB, bool DOTS>
void run(const double* U, long ld, const double* h, const double* x, double* y, long n, double* part, int reps) {
    auto kern = kupd<K, S, R, MINB, DOTS>;
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTA, 0));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    for (int mult : {1, 2, 4}) {
        const int grid = nsm * occ * mult;
        if (mult > 1 && grid > 4096) continue;
        float ms = timeit([&] { kern<<<grid, CTA>>>(U, ld, h, x, y, n, part); }, reps);
        CK(cudaGetLastError());
        const double bytes = 8.0 * n * (K + 2);
        printf("kupd K=%2d S=%d R=%d MINB=%d dots=%d regs=%3d spill=%zu occ=%d grid=%5d: %8.2f us  %7.1f GB/s\n", K, S, R,
               MINB, (int)DOTS, fa.numRegs, fa.localSizeBytes, occ, grid, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    }
}

template <int K>
void sweep(const double* U, long ld, const double* h, const double* x, double* y, long n, double* part, int reps) {
    {
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kread<K>, CTA, 0));
        const int grid = nsm * occ;
        float ms = timeit([&] { kread<K><<<grid, CTA>>>(U, ld, x, y, n); }, reps);
        printf("kread K=%2d grid=%d: %8.2f us  %7.1f GB/s\n", K, grid, ms * 1e3, 8.0 * n * (K + 2) / (ms * 1e-3) / 1e9);
    }
    run<K, 1, 1, 1, true>(U, ld, h, x, y, n, part, reps);
    run<K, 2, 1, 2, true>(U, ld, h, x, y, n, part, reps);
    run<K, 2, 2, 1, true>(U, ld, h, x, y, n, part, reps);
    run<K, 4, 1, 2, true>(U, ld, h, x, y, n, part, reps);
    run<K, 4, 2, 2, true>(U, ld, h, x, y, n, part, reps);
    run<K, 8, 2, 2, true>(U, ld, h, x, y, n, part, reps);
    run<K, 8, 4, 2, true>(U, ld, h, x, y, n, part, reps);
    run<K, 2, 1, 2, false>(U, ld, h, x, y, n, part, reps);
    run<K, 4, 2, 2, false>(U, ld, h, x, y, n, part, reps);
}

int main(int argc, char** argv) {
    long n = argc > 1 ? atol(argv[1]) : 2097152;
    const long ld = n;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    double *U, *x, *y, *h, *part;
    CK(cudaMalloc(&U, sizeof(double) * ld * 48));
    CK(cudaMalloc(&x, sizeof(double) * n));
    CK(cudaMalloc(&y, sizeof(double) * n));
    CK(cudaMalloc(&h, sizeof(double) * 64));
    CK(cudaMalloc(&part, sizeof(double) * 65 * 8192));
    CK(cudaMemset(U, 0, sizeof(double) * ld * 48));
    CK(cudaMemset(x, 0, sizeof(double) * n));
    CK(cudaMemset(h, 0, sizeof(double) * 64));
    const int reps = n > 50000000 ? 5 : 30;
    // memcpy reference: same byte count as K=24 (read 26n, write... ) -> copy of 13n doubles
    {
        double* dst;
        CK(cudaMalloc(&dst, sizeof(double) * n * 13));
        float ms = timeit([&] { CK(cudaMemcpyAsync(dst, U, sizeof(double) * n * 13, cudaMemcpyDeviceToDevice)); }, reps);
        printf("memcpy %ld B: %.2f us  %.1f GB/s (read+write)\n", (long)(8 * n * 13), ms * 1e3, 2.0 * 8 * n * 13 / (ms * 1e-3) / 1e9);
        CK(cudaFree(dst));
    }
    printf("n=%ld nsm=%d\n", n, nsm);
    sweep<24>(U, ld, h, x, y, n, part, reps);
    sweep<48>(U, ld, h, x, y, n, part, reps);
    return 0;
}
