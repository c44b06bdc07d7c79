// Round-trip latency between the two CTAs of a cluster (one thread each), three signalling schemes:
//  0: st.async (8 B) completing on the receiver's mbarrier, receiver try_wait.parity (K3b's exchange)
//  1: the same with test_wait.parity polling
//  2: plain st.shared::cluster of the value + remote mbarrier.arrive.release.cluster, try_wait.acquire.cluster
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pp tools/micro/dsmem_pingpong.cu && /tmp/pp
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
template <int MODE>
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
    if (MODE == 0)
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(bar), "r"(par) : "memory");
    else if (MODE == 1)
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(bar), "r"(par) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(bar), "r"(par) : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, long long* out) {
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) double box;
    auto cl = cg::this_cluster();
    const int rank = cl.block_rank();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();
    if (threadIdx.x == 0) {
        const uint32_t mybar = s32(&bar), peer = rank ^ 1;
        const uint32_t rbar = mapa(mybar, peer), rbox = mapa(s32(&box), peer);
        double v = 1.0;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t par = i & 1;
            if (MODE != 2) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" ::"r"(mybar) : "memory");
            if ((rank == 0) ? true : false) {
                if (MODE != 2) {
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rbox), "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
                } else {
                    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rbox), "d"(v) : "memory");
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
                }
                wait<MODE>(mybar, par);
                v = box + 1.0;
            } else {
                wait<MODE>(mybar, par);
                v = box + 1.0;
                if (MODE != 2) {
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rbox), "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
                } else {
                    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rbox), "d"(v) : "memory");
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
                }
            }
        }
        long long t1 = clock64();
        if (rank == 0) { out[0] = t1 - t0; out[1] = (long long)v; }
    }
    cl.sync();
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    const int iters = 20000;
    auto run = [&](auto kern, const char* name) {
        kern<<<2, 32>>>(100, d);
        kern<<<2, 32>>>(iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%s: %s, %.1f cycles per round trip (check %lld)\n", name, cudaGetErrorString(e), (double)h[0] / iters, h[1]);
    };
    run(pingpong<0>, "st.async + try_wait");
    run(pingpong<1>, "st.async + test_wait");
    run(pingpong<2>, "st.shared::cluster + remote arrive.release + try_wait.acquire.cluster");
    return 0;
}
