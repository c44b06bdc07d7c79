// tma_probe.cu -- standalone check of the 4D TMA box load used by K3c (k_minres_stream.cu):
// loads one 68 x 36 box of plane 1 / slot 1 with a (-2, -2) origin and compares with the host.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, double* out, int variant) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nbox = (variant == 2 || variant == 3 || variant == 5) ? 4 : 1;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(nbox * 68 * 36 * 8) : "memory");
        if (variant == 4) {
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sd),
                         "l"(&map), "r"(-1), "r"(-1), "r"(1), "r"(1), "r"(sb) : "memory");
        } else if (variant >= 2) {
            for (int k = 0; k < 4; ++k)
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sd + k * 19584 + (variant == 3 ? 78336 : 0)),
                             "l"(&map), "r"(-1), "r"(-1), "r"(k), "r"(1), "r"(sb) : "memory");
        } else if (variant == 0)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sd),
                         "l"(&map), "r"(-2), "r"(-2), "r"(1), "r"(1), "r"(sb) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sd),
                         "l"(&map), "r"(-2), "r"(-2), "r"(1), "r"(1), "r"(sb) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(sb) : "memory");
    for (int i = threadIdx.x; i < 68 * 36; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    const int N = 128, GP = N + 2, G = N + 1, NPL = 5, NS = 2;
    std::vector<double> h((size_t)GP * G * NPL * NS);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 68 * 36 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    CUtensorMap map;
    cuuint64_t dims[4] = {(cuuint64_t)GP, (cuuint64_t)G, (cuuint64_t)NPL, (cuuint64_t)NS};
    cuuint64_t str[3] = {(cuuint64_t)GP * 8, (cuuint64_t)GP * G * 8, (cuuint64_t)GP * G * 8 * NPL};
    cuuint32_t box[4] = {68, 36, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    const int smem = (variant == 2 || variant == 3 || variant == 4) ? 175040 : (variant == 5 ? 4 * 19584 + 64 : 68 * 36 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(map, o, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    std::vector<double> ho(68 * 36);
    cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 36; ++y)
        for (int x = 0; x < 68; ++x) {
            const int gx = x - 2, gy = y - 2;
            const double ref = (gx < 0 || gy < 0) ? 0.0 : h[(((size_t)1 * NPL + 1) * G + gy) * GP + gx];
            if (ho[y * 68 + x] != ref) ++bad;
        }
    printf("mismatches %d\n", bad);
    return 0;
}
