// fp64 latency probes on B200 (tools/): dependent chains of DFMA, sqrt, div, rsqrt, and the
// Jacobi rotation-parameter formula, one warp.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include "../paper_1711_10128_b200/csrc/eig.cu"
using namespace trplk;
__global__ void probe(double* out, long long* cyc, double seed) {
    double x = seed + threadIdx.x * 1e-3, y = 1.5;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) x = fma(x, 0.999, 1e-3);
    long long t1 = clock64();
    for (int i = 0; i < 256; ++i) x = sqrt(x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < 256; ++i) x = 1.0 / (x + 0.5);
    long long t3 = clock64();
    for (int i = 0; i < 256; ++i) x = rsqrt(x + 0.25);
    long long t4 = clock64();
    double c, s, dp, dq;
    int act;
    for (int i = 0; i < 256; ++i) {
        jacobi_param(x + 2.0, y, 0.3 + 1e-3 * x, 1.0, c, s, dp, dq, act);
        x = c + dp * 1e-9;
        y = dq;
    }
    long long t5 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256;
        cyc[4] = (t5 - t4) / 256;
    }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    probe<<<1, 32>>>(o, c, 0.5); cudaDeviceSynchronize();
    probe<<<1, 32>>>(o, c, 0.5);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: DFMA %lld  sqrt %lld  div %lld  rsqrt %lld  jacobi_param %lld\n", h[0], h[1], h[2], h[3], h[4]);
}
