// tc_probe.cu -- unit probe for the tcgen05 / UMMA descriptor / TMA conventions of tc_common.cuh.
// Built into libgla_probe.so (tests only): one CTA computes D[M x N] = A[M x K] . B[K x N] with A and B
// staged in the SW128 row layout as K-major or MN-major operands, optionally loading the MN-major A tile with
// TMA (SWIZZLE_128B), and writes D (fp32) back.  tests/test_tc_probe.py compares it with torch.matmul.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include "../tc_common.cuh"

using namespace gla::tc;

__global__ void __launch_bounds__(128) k_probe(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ B,
                                               float* __restrict__ D, int M, int N, int K, int a_mn, int b_mn,
                                               int use_tma, int a_tmem, const __grid_constant__ CUtensorMap tmapA) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;                       // up to 64 KB
    uint8_t* sB = smem + 65536;               // up to 128 KB
    __shared__ uint64_t bar_mma, bar_tma;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (warp == 0) tmem_alloc(&tbase, 512);
    if (tid == 0) {
        mbar_init(&bar_mma, 1);
        mbar_init(&bar_tma, 1);
        fence_mbar_init();
    }
    __syncthreads();
    tc_fence_after();
    // stage A
    if (use_tma && a_mn) {
        if (tid == 0) {
            mbar_expect_tx(&bar_tma, (uint32_t)(M * K * 2));
            for (int mb = 0; mb < M / 64; ++mb)
                tma_load_2d(sA + mb * (K * 128), &tmapA, &bar_tma, mb * 64, 0);   // box {64 (M), K rows}
        }
        mbar_wait(&bar_tma, 0);
    } else {
        for (int e = tid; e < M * K; e += 128) {
            const int m = e / K, k = e % K;
            uint32_t off = a_mn ? (m / 64) * (K * 128) + sw128_off(k, m % 64) : (k / 64) * (M * 128) + sw128_off(m, k % 64);
            *reinterpret_cast<__nv_bfloat16*>(sA + off) = A[(size_t)m * K + k];
        }
    }
    for (int e = tid; e < N * K; e += 128) {
        const int k = e / N, n = e % N;      // B is [K][N] row-major in global
        uint32_t off = b_mn ? (n / 64) * (K * 128) + sw128_off(k, n % 64) : (k / 64) * (N * 128) + sw128_off(n, k % 64);
        *reinterpret_cast<__nv_bfloat16*>(sB + off) = B[(size_t)k * N + n];
    }
    const uint32_t tA = tbase + 256;          // A in TMEM (M = 128): row m = lane m, bf16 pairs per column
    if (a_tmem) {
        for (int c0 = 0; c0 < K / 2; c0 += 32) {
            uint32_t r[32];
            const int m = 32 * warp + lane;
            for (int j = 0; j < 32; ++j)
                r[j] = pack_bf16(__bfloat162float(A[(size_t)m * K + 2 * (c0 + j)]),
                                 __bfloat162float(A[(size_t)m * K + 2 * (c0 + j) + 1]));
            tmem_st32(taddr(tA, 32 * warp, c0), r);
        }
        tmem_wait_st();
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (tid == 0 && a_tmem) {
        const uint32_t id = idesc_bf16(M, N, 0, b_mn);
        for (int kk = 0; kk < K / 16; ++kk) {
            uint64_t bd = b_mn ? sdesc_sw128(smem_u32(sB) + kk * 2048, K * 128, 1024)
                               : sdesc_sw128(smem_u32(sB) + (kk / 4) * (N * 128) + (kk % 4) * 32, 16, 1024);
            mma_bf16_ta(tmem, tA + kk * 8, bd, id, kk > 0);
        }
        mma_commit(&bar_mma);
    } else if (tid == 0) {
        const uint32_t id = idesc_bf16(M, N, a_mn, b_mn);
        for (int kk = 0; kk < K / 16; ++kk) {
            uint64_t ad = a_mn ? sdesc_sw128(smem_u32(sA) + kk * 2048, K * 128, 1024)
                               : sdesc_sw128(smem_u32(sA) + (kk / 4) * (M * 128) + (kk % 4) * 32, 16, 1024);
            uint64_t bd = b_mn ? sdesc_sw128(smem_u32(sB) + kk * 2048, K * 128, 1024)
                               : sdesc_sw128(smem_u32(sB) + (kk / 4) * (N * 128) + (kk % 4) * 32, 16, 1024);
            mma_bf16(tmem, ad, bd, id, kk > 0);
        }
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr(tmem, 32 * warp, c0), r);
        tmem_wait_ld();
        int row;
        if (M == 128) row = 32 * warp + lane;
        else row = lane < 16 ? 16 * warp + lane : -1;
        if (row >= 0)
            for (int j = 0; j < 32; ++j) D[(size_t)row * N + c0 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// D[128 x N] = A[128 x K] . B[K x N] in tf32: A (fp32) staged into TMEM one element per column, B (fp32) as a
// K-major SW128 tile (N rows of 32 fp32 per K block of 32).
__global__ void __launch_bounds__(128) k_probe_tf32(const float* __restrict__ A, const float* __restrict__ B,
                                                    float* __restrict__ D, int N, int K) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sB = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar_mma;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (warp == 0) tmem_alloc(&tbase, 512);
    if (tid == 0) {
        mbar_init(&bar_mma, 1);
        fence_mbar_init();
    }
    __syncthreads();
    tc_fence_after();
    for (int e = tid; e < N * K; e += 128) {
        const int k = e / N, n = e % N;
        const uint32_t off = (k / 32) * (N * 128) + sw128_off(n, 2 * (k % 32));
        *reinterpret_cast<float*>(sB + off) = B[(size_t)k * N + n];
    }
    const uint32_t tA = tbase + 256;
    for (int c0 = 0; c0 < K; c0 += 32) {
        uint32_t r[32];
        const int m = 32 * warp + lane;
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(A[(size_t)m * K + c0 + j]);
        tmem_st32(taddr(tA, 32 * warp, c0), r);
    }
    tmem_wait_st();
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint32_t id = idesc_tf32(128, N, 0);
        for (int kk = 0; kk < K / 8; ++kk)
            mma_tf32_ta(tbase, tA + kk * 8, sdesc_sw128(smem_u32(sB) + (kk / 4) * (N * 128) + (kk % 4) * 32, 16, 1024),
                        id, kk > 0);
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr(tbase, 32 * warp, c0), r);
        tmem_wait_ld();
        for (int j = 0; j < 32; ++j) D[(size_t)(32 * warp + lane) * N + c0 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

extern "C" int probe_gemm_tf32(const float* A, const float* B, float* D, int N, int K) {
    const int smem = 131072 + 1024;
    cudaFuncSetAttribute(k_probe_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_probe_tf32<<<1, 128, smem>>>(A, B, D, N, K);
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 1000 + (int)e;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int probe_gemm(const void* A, const void* At, const void* B, float* D, int M, int N, int K, int a_mn,
                          int b_mn, int use_tma, int a_tmem) {
    CUtensorMap map{};
    if (use_tma) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 100;
        cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};           // At is [K][M] row-major
        cuuint64_t strides[1] = {(cuuint64_t)M * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)K};
        cuuint32_t es[2] = {1, 1};
        CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)At, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return 200 + (int)r;
    }
    const int smem = 65536 + 131072 + 1024;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_probe<<<1, 128, smem>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, M, N, K, a_mn, b_mn, use_tma, a_tmem, map);
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 1000 + (int)e;
}
