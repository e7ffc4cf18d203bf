// Microbenchmark: tcgen05.ld throughput (32x32b.x32) per SM, and st, with 4 or 8 warps.
#include <cstdio>
#include "../../paper_2312_06635_b200/csrc/tc_common.cuh"
using namespace gla::tc;
__global__ void __launch_bounds__(256, 1) k(float* out, long long* cyc, int iters, int do_store) {
    __shared__ uint32_t tb;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&tb, 512);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t base = tb + ((uint32_t)(32 * (warp & 3)) << 16) + 256 * (warp >> 2);
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
        tmem_ld32(base + (it & 7) * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
        if (do_store) { tmem_st32(base + (it & 7) * 32, r); }
    }
    if (do_store) tmem_wait_st();
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}
int main() {
    float* out; long long* cyc; cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&cyc, 148 * 8);
    for (int nw : {4, 8}) for (int st = 0; st < 2; ++st) {
        int iters = 4096;
        k<<<148, nw * 32>>>(out, cyc, iters, st);
        cudaDeviceSynchronize();
        k<<<148, nw * 32>>>(out, cyc, iters, st);
        cudaError_t e = cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double bytes = (double)iters * nw * 32 * 32 * 4;
        printf("warps %d store %d: %lld cycles, %.1f bytes/clk/SM read (err %d)\n", nw, st, c, bytes / c, (int)e);
    }
}
