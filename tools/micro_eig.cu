// Per-role cycle trace of the one-CTA Jacobi (tools/, measurement):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DEIG_TRACE -I include -I paper_1711_10128_b200/csrc \
//        -o tools/micro_eig tools/micro_eig.cu
//   ./tools/micro_eig 30
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../paper_1711_10128_b200/csrc/eig.cu"

int main(int argc, char** argv) {
    using namespace trplk;
    const int k = argc > 1 ? atoi(argv[1]) : 30;
    std::vector<double> T(QMAX * QMAX, 0.0);
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    for (int j = 0; j < k; ++j)
        for (int i = 0; i <= j; ++i) T[i + j * QMAX] = T[j + i * QMAX] = nd(g);
    Ctl* ctl;
    double *Td, *Y;
    cudaMalloc(&ctl, sizeof(Ctl));
    cudaMalloc(&Td, 8 * QMAX * QMAX);
    cudaMalloc(&Y, 8 * QMAX * QMAX);
    Ctl h{};
    h.flags = ~0u;
    h.k = k;
    cudaMemcpy(ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice);
    cudaMemcpy(Td, T.data(), 8 * QMAX * QMAX, cudaMemcpyHostToDevice);
    launch_eig(ctl, Td, QMAX, Y, QMAX, 0, k, 0, 0);
    cudaDeviceSynchronize();
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(eig_trace, z, sizeof(z));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) launch_eig(ctl, Td, QMAX, Y, QMAX, 0, k, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[32];
    cudaMemcpyFromSymbol(t, eig_trace, sizeof(t));
    Ctl hh;
    cudaMemcpy(&hh, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost);
    const double rounds = (double)t[30];
    printf("k=%d  %.1f us/launch  sweeps %d  rounds/launch %.0f  cycles/round %.0f (%s)\n", k, 1e3 * ms / reps,
           hh.eig_sweeps, rounds / reps, t[31] / rounds, cudaGetErrorString(cudaGetLastError()));
    for (int w = 0; w < EIG1_THREADS / 32; ++w) printf("  warp %2d: %.0f cycles to barrier\n", w, t[w] / rounds);
    printf("  warp 0 lane 0: %.0f cycles to the pivot entry, %.0f in the rotation parameters\n", t[16] / rounds,
           t[17] / rounds);
    return 0;
}
