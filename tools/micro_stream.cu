// Micro-benchmark of the basis-stream access patterns of the CGS kernels (tools/, not product).
// y[i] = x[i] - sum_c U[c*ld + i] h[c] for k columns, n rows; variants of the thread->row map.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_stream tools/micro_stream.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

__constant__ double hc[64];

// A: lane per row, 32-row warp tiles, grid-stride over tiles, all k loads first
template <int K>
__global__ void vA(const double* __restrict__ U, long ld, const double* __restrict__ x, double* __restrict__ y, long n) {
    const int lane = threadIdx.x & 31;
    const long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
    for (long t = w; t < (n + 31) / 32; t += nw) {
        const long r = t * 32 + lane;
        if (r >= n) continue;
        double u[K];
#pragma unroll
        for (int c = 0; c < K; ++c) u[c] = U[c * ld + r];
        double a = x[r];
#pragma unroll
        for (int c = 0; c < K; ++c) a = fma(-hc[c], u[c], a);
        y[r] = a;
    }
}

// B: lane per 2 consecutive rows with 16-byte loads (64-row warp tiles)
template <int K>
__global__ void vB(const double* __restrict__ U, long ld, const double* __restrict__ x, double* __restrict__ y, long n) {
    const int lane = threadIdx.x & 31;
    const long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
    for (long t = w; t < (n + 63) / 64; t += nw) {
        const long r = t * 64 + 2 * lane;
        if (r >= n) continue;
        double2 u[K];
#pragma unroll
        for (int c = 0; c < K; ++c) u[c] = *reinterpret_cast<const double2*>(U + c * ld + r);
        double2 a = *reinterpret_cast<const double2*>(x + r);
#pragma unroll
        for (int c = 0; c < K; ++c) { a.x = fma(-hc[c], u[c].x, a.x); a.y = fma(-hc[c], u[c].y, a.y); }
        *reinterpret_cast<double2*>(y + r) = a;
    }
}

// C: block-contiguous partition (each CTA owns a contiguous row range), lane per row
template <int K>
__global__ void vC(const double* __restrict__ U, long ld, const double* __restrict__ x, double* __restrict__ y, long n) {
    const long per = (n + gridDim.x - 1) / gridDim.x;
    const long b = blockIdx.x * per, e = min(n, b + per);
    for (long r = b + threadIdx.x; r < e; r += blockDim.x) {
        double u[K];
#pragma unroll
        for (int c = 0; c < K; ++c) u[c] = U[c * ld + r];
        double a = x[r];
#pragma unroll
        for (int c = 0; c < K; ++c) a = fma(-hc[c], u[c], a);
        y[r] = a;
    }
}

__global__ void vcopy(const double2* __restrict__ a, double2* __restrict__ b, long n2) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += gridDim.x * (long)blockDim.x) b[i] = a[i];
}

template <typename F>
float timeit(F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<double> h(64, 0.01);
    CK(cudaMemcpyToSymbol(hc, h.data(), 64 * 8));
    for (long n : {262144L, 2097152L, 16777216L}) {
        const int K = 24;
        const long ld = n;
        double *U, *x, *y;
        CK(cudaMalloc(&U, sizeof(double) * ld * K));
        CK(cudaMalloc(&x, sizeof(double) * n));
        CK(cudaMalloc(&y, sizeof(double) * n));
        cudaMemset(U, 0, sizeof(double) * ld * K);
        cudaMemset(x, 0, sizeof(double) * n);
        const double bytes = 8.0 * n * (K + 2);
        for (int occ : {1, 2, 3, 4, 8}) {
            const int g = nsm * occ;
            float ta = timeit([&] { vA<K><<<g, 256>>>(U, ld, x, y, n); });
            float tb = timeit([&] { vB<K><<<g, 256>>>(U, ld, x, y, n); });
            float tc = timeit([&] { vC<K><<<g, 256>>>(U, ld, x, y, n); });
            printf("n=%ld grid=%d  A %.1f GB/s (%.1f us)  B %.1f GB/s (%.1f us)  C %.1f GB/s (%.1f us)\n", n, g,
                   bytes / ta / 1e6, ta * 1e3, bytes / tb / 1e6, tb * 1e3, bytes / tc / 1e6, tc * 1e3);
        }
        const long n2 = ld * K / 2;
        float tcp = timeit([&] { vcopy<<<nsm * 8, 256>>>((double2*)U, (double2*)U + n2 / 2, n2 / 2); });
        printf("n=%ld copy %.1f GB/s\n", n, 2.0 * 16 * (n2 / 2) / tcp / 1e6);
        cudaFree(U);
        cudaFree(x);
        cudaFree(y);
    }
    return 0;
}
