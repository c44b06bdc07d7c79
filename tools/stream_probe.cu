// stream_probe.cu -- standalone driver for K3c (k_minres_stream.cu) on a constant coefficient:
// a = 1 everywhere gives the 5-point Laplacian; prints status, iterations and Q per system.
#include "../paper_2503_05533_b200/csrc/k_minres_stream.cu"
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 128, nb = argc > 2 ? atoi(argv[2]) : 2;
    const int P = 2 * N * N;
    std::vector<double> a((size_t)P * nb, 1.0);
    double *da, *dout, *scr;
    unsigned* ctr;
    cudaMalloc(&da, a.size() * 8);
    cudaMemcpy(da, a.data(), a.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&dout, (size_t)nb * 8 * 8);
    cudaMemset(dout, 0, (size_t)nb * 64);
    cudaMalloc(&ctr, 16);
    cudaMemset(ctr, 0, 16);
    const int nct = nb < 148 ? nb : 148;
    cudaMalloc(&scr, mlmc::minres_stream_scratch_per_cta(N) * nct);
    cudaError_t e = mlmc::launch_minres_stream(N, da, nb, 1e-8, 4 * N * N, dout, 0, ctr, scr, nct, 0);
    printf("launch: %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("sync: %s\n", cudaGetErrorString(e));
    std::vector<double> o((size_t)nb * 8);
    cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
    for (int b = 0; b < nb; ++b) printf("sys %d: Q %.15g iters %g res %g status %g\n", b, o[8 * b], o[8 * b + 2], o[8 * b + 4], o[8 * b + 6]);
    return 0;
}
