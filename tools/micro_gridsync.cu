// Cost of a cooperative-groups grid barrier on B200 (tools/, measurement).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(256, 2) ksync(double* part, double* red, int iters, int nv) {
    cg::grid_group g = cg::this_grid();
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x < nv) part[threadIdx.x * gridDim.x + blockIdx.x] = acc + i;
        g.sync();
        // every CTA sums value (threadIdx.x / 32) over all CTAs: warp w -> value w
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        double s = 0.0;
        if (w < 8 && nv > 0)
            for (int c = lane; c < (int)gridDim.x; c += 32) s += part[(w % nv) * gridDim.x + c];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        acc += s * 1e-30;
        g.sync();
    }
    if (threadIdx.x == 0) red[blockIdx.x] = acc;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *part, *red; cudaMalloc(&part, 8 * 64 * 4096); cudaMalloc(&red, 8 * 4096);
    for (int per : {1, 2}) for (int nv : {0, 64}) {
        int grid = nsm * per, iters = 2000;
        void* args[] = {&part, &red, &iters, &nv};
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)ksync, grid, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)ksync, grid, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("grid %d nv %d: %.2f us per iteration (2 grid syncs%s) %s\n", grid, nv, 1e3 * ms / iters,
               nv ? " + partial write + all-CTA read of 8 values" : "", cudaGetErrorString(cudaGetLastError()));
    }
}
