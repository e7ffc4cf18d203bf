// Microbenchmark: single-thread tcgen05.mma issue rate, with descriptors precomputed once (64-bit adds per
// K step) and no "memory" clobber on the MMA asm (variant 1) vs the library's mma_bf16 wrappers (variant 0).
#include <cstdio>
#include "../../paper_2312_06635_b200/csrc/tc_common.cuh"
using namespace gla::tc;
__device__ __forceinline__ void mma_nc(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ta_nc(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int N, int ts, int iters, int var) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&tb, 512);
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_bf16(128, N, 0, 0);
        const uint64_t ad = sdesc_sw128(smem_u32(sm), 16, 1024), bd = sdesc_sw128(smem_u32(sm + 16384), 16, 1024);
        const uint32_t t0_ = tb;
        for (int it = 0; it < iters; it += 16) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int kk = u & 3;
                if (var) {
                    if (ts) mma_ta_nc(t0_, t0_ + 256 + 8 * kk, bd + 2 * kk, id, 1);
                    else mma_nc(t0_, ad + 2 * kk, bd + 2 * kk, id, 1);
                } else {
                    if (ts) mma_bf16_ta(t0_, t0_ + 256 + 8 * kk, bd + 2 * kk, id, 1);
                    else mma_bf16(t0_, ad + 2 * kk, bd + 2 * kk, id, 1);
                }
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}
int main() {
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int var = 0; var < 2; ++var) for (int ts = 0; ts < 2; ++ts)
        for (int N : {64, 128, 256}) {
            const int iters = 1 << 16;
            k<<<148, 128, 65536>>>(cyc, N, ts, iters, var);
            k<<<148, 128, 65536>>>(cyc, N, ts, iters, var);
            cudaError_t e = cudaDeviceSynchronize();
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("var %d %s N=%3d: %6.1f cycles per M128xK16 MMA (ideal %d) err %d\n", var, ts ? "TS" : "SS", N,
                   (double)c / iters, 128 * N / 256, (int)e);
        }
}
