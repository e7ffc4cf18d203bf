// Microbenchmark: DSMEM bandwidth in a 4-CTA cluster: (a) st.shared::cluster.v4 by all threads,
// (b) cp.async.bulk.shared::cluster.shared::cta (TMA-engine copy) with mbarrier complete_tx.
#include <cstdio>
#include <cstdint>
#include "../../paper_2312_06635_b200/csrc/tc_common.cuh"
using namespace gla::tc;
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) { uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r; }
__device__ __forceinline__ void cluster_sync() { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 1) kst(long long* cyc, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];   // 3 x 32 KB receive slots + 32 KB source
    const uint32_t me = cluster_rank();
    cluster_sync();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int p = 1; p < 4; ++p) {
            const uint32_t peer = (me + p) & 3;
            const uint32_t slot = ((me - peer + 4) & 3) - 1;   // 0..2
            const uint32_t dst = mapa(smem_u32(sm + slot * 32768), peer);
            for (int off = threadIdx.x * 16; off < 32768; off += 256 * 16)
                asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(dst + off), "r"(it), "r"(off), "r"(p), "r"(me) : "memory");
        }
        cluster_sync();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 1) kbulk(long long* cyc, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    const uint32_t me = cluster_rank();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    cluster_sync();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) mbar_expect_tx(&bar, 3 * 32768);
        cluster_sync();   // every receiver armed before any copy lands
        if (threadIdx.x < 3) {
            const uint32_t p = threadIdx.x + 1, peer = (me + p) & 3;
            const uint32_t slot = ((me - peer + 4) & 3) - 1;
            const uint32_t dst = mapa(smem_u32(sm + slot * 32768), peer);
            const uint32_t rbar = mapa(smem_u32(&bar), peer);
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(dst), "r"(smem_u32(sm + 3 * 32768)), "r"(32768), "r"(rbar) : "memory");
        }
        mbar_wait(&bar, it & 1);
    }
    cluster_sync();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    const int smem = 4 * 32768;
    cudaFuncSetAttribute(kst, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kbulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int iters = 200;
    for (int rep = 0; rep < 2; ++rep) {
        kst<<<144, 256, smem>>>(cyc, iters);
        cudaError_t e = cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("st.shared::cluster: %lld cycles, out %.1f B/clk/SM (err %d)\n", c, 3.0 * 32768 * iters / c, (int)e);
        kbulk<<<144, 256, smem>>>(cyc, iters);
        e = cudaDeviceSynchronize();
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("cp.async.bulk cluster: %lld cycles, out %.1f B/clk/SM (err %d)\n", c, 3.0 * 32768 * iters / c, (int)e);
    }
}
