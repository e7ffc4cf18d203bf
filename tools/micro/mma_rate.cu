// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion time per instruction (M = 128, K = 16) for
// N in {64, 128, 256}, A from shared memory (SS) or TMEM (TS); 148 CTAs, one issuing thread each.
#include <cstdio>
#include "../../paper_2312_06635_b200/csrc/tc_common.cuh"
using namespace gla::tc;

__global__ void __launch_bounds__(128, 1) k(long long* cyc, int N, int ts, int iters, int nw) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&tb, 512);
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(&bar, nw); fence_mbar_init(); }
    fence_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    long long t0 = clock64();
    if (warp < nw) {
        const uint32_t id = idesc_bf16(128, N, 0, 0);
        const uint32_t a = smem_u32(sm), b = smem_u32(sm + 16384);
        for (int it = 0; it < iters; it += 16) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int kk = u & 3;
                const uint32_t d = tb + warp * N;
                if (ts) mma_bf16_ta_w(d, tb + 256 + 8 * kk, sdesc_sw128(b + kk * 32, 16, 1024), id, 1);
                else mma_bf16_w(d, sdesc_sw128(a + kk * 32, 16, 1024), sdesc_sw128(b + kk * 32, 16, 1024), id, 1);
            }
        }
        mma_commit_w(&bar);
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
    for (int ts = 0; ts < 2; ++ts)
        for (int N : {64, 128, 256}) for (int nd : {1, 2, 4}) {
            if (N * nd > 256) continue;
            const int iters = 1 << 16;
            k<<<148, 128, 65536>>>(cyc, N, ts, iters, nd);
            k<<<148, 128, 65536>>>(cyc, N, ts, iters, nd);
            cudaError_t e = cudaDeviceSynchronize();
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("%s N=%3d accumulators %d: %6.1f cycles per M128xK16 MMA (ideal %d) err %d\n", ts ? "TS" : "SS", N, nd,
                   (double)c / (iters * nd), 128 * N / 256, (int)e);
        }
}
