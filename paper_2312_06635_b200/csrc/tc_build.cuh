// tc_build.cuh -- per-chunk operand construction shared by the tensor-core kernels.
//
// Thread mapping (256 threads): thread = (channel octet oc, row group rg); it owns channels [8 oc, 8 oc + 8)
// of rows [rg RPG, (rg+1) RPG) of the 64-token chunk.  Its q / k / log alpha are loaded with 16-byte
// vector loads into registers one chunk ahead (the prefetch hides HBM latency behind the current chunk).
// The chunk-local inclusive cumsum b is a per-thread running sum plus an exchange of
// row-group totals through shared memory; it also yields r = b at row 31 (the per-channel normaliser) and
// Gamma = b at row 63 (the chunk's total log decay).  Arithmetic on channel pairs uses the sm_100a packed
// f32x2 FMUL2 / FFMA2 instructions.
#pragma once
#include "tc_common.cuh"

namespace gla {
namespace tc {

constexpr float kL2E = 1.4426950408889634f;

// ---- packed fp32x2 arithmetic (FMUL2 / FFMA2 / FADD2) -----------------------------------------------------------
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, {%6,%7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return add2(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 ex2_2(float2 a) { return make_float2(ex2f(a.x), ex2f(a.y)); }
__device__ __forceinline__ float2 unpack2(uint32_t u) { return make_float2(bf16lo(u), bf16hi(u)); }
__device__ __forceinline__ uint32_t pack2(float2 a) { return pack_bf16(a.x, a.y); }
__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

template <int K, int NT = 256>
struct Tile {
    static constexpr int NOCT = K / 8;          // threads per row
    static constexpr int RG = NT / NOCT;        // row groups
    static constexpr int RPG = 64 / RG;         // rows per thread
};

// Raw inputs of one chunk for one thread.
template <int K, int NT = 256>
struct ChunkRegs {
    uint4 q[Tile<K, NT>::RPG], k[Tile<K, NT>::RPG];
    float2 g[Tile<K, NT>::RPG][4];              // log alpha, then the thread-local inclusive prefix
};

template <typename TG>
__device__ __forceinline__ void load_g8(const TG* p, float2 (&d)[4]);
template <>
__device__ __forceinline__ void load_g8<float>(const float* p, float2 (&d)[4]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    d[0] = make_float2(a.x, a.y); d[1] = make_float2(a.z, a.w);
    d[2] = make_float2(b.x, b.y); d[3] = make_float2(b.z, b.w);
}
template <>
__device__ __forceinline__ void load_g8<__nv_bfloat16>(const __nv_bfloat16* p, float2 (&d)[4]) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    d[0] = unpack2(a.x); d[1] = unpack2(a.y); d[2] = unpack2(a.z); d[3] = unpack2(a.w);
}

// Load rows [row0, row0 + RPG) of chunk starting at global row `crow` (row index into [B*H*T, K]).
template <int K, typename TG, bool LQ, bool LK, int NT = 256>
__device__ __forceinline__ void load_chunk(ChunkRegs<K, NT>& R, const __nv_bfloat16* q, const __nv_bfloat16* k,
                                           const TG* g, size_t crow, int row0, int ch0) {
#pragma unroll
    for (int r = 0; r < Tile<K, NT>::RPG; ++r) {
        const size_t off = (crow + row0 + r) * K + ch0;
        if (LQ) R.q[r] = __ldg(reinterpret_cast<const uint4*>(q + off));
        if (LK) R.k[r] = __ldg(reinterpret_cast<const uint4*>(k + off));
        load_g8<TG>(g + off, R.g[r]);
    }
}

// Chunk-local cumsum.  After the call: R.g[r][p] = b at (row0 + r) minus `off` (the prefix of earlier row
// groups, returned in off[p]); rr = b at row 31; Gm = b at row 63 (all per channel pair).
// gtot: shared [RG][K] floats.  Contains one __syncthreads (the caller must not reuse gtot before the next one).
template <int K, int NT = 256>
__device__ __forceinline__ void chunk_cumsum(ChunkRegs<K, NT>& R, float* gtot, int rg, int ch0, float2 (&off)[4],
                                             float2 (&rr)[4], float2 (&Gm)[4]) {
    using Tl = Tile<K, NT>;
    float2 run[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int r = 0; r < Tl::RPG; ++r)
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            run[p] = add2(run[p], R.g[r][p]);
            R.g[r][p] = run[p];
        }
    float4* gt = reinterpret_cast<float4*>(gtot + rg * K + ch0);
    gt[0] = make_float4(run[0].x, run[0].y, run[1].x, run[1].y);
    gt[1] = make_float4(run[2].x, run[2].y, run[3].x, run[3].y);
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        off[p] = make_float2(0.f, 0.f);
        rr[p] = make_float2(0.f, 0.f);
        Gm[p] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int r2 = 0; r2 < Tl::RG; ++r2) {
        const float4* s = reinterpret_cast<const float4*>(gtot + r2 * K + ch0);
        const float4 a = s[0], b = s[1];
        const float2 v[4] = {make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y), make_float2(b.z, b.w)};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            if (r2 < rg) off[p] = add2(off[p], v[p]);
            if ((r2 + 1) * Tl::RPG <= 32) rr[p] = add2(rr[p], v[p]);
            Gm[p] = add2(Gm[p], v[p]);
        }
    }
}

// Factorised operand row: x (.) e^{(b - ref)} for one thread-row of 8 channels.
//   sign = +1: factor e^{b - ref} (Q side); sign = -1: factor e^{ref - b} (K side).
// Writes the bf16 hi row (and, if lo != nullptr, the bf16 residual row) as 16-byte stores.
__device__ __forceinline__ void scaled_row(const uint4& x, const float2 (&b)[4], const float2 (&refL)[4], float sign,
                                           uint8_t* hi, uint8_t* lo) {
    const float2 s2 = make_float2(sign * kL2E, sign * kL2E);
    uint32_t h[4], l[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 e = ex2_2(fma2(b[p], s2, refL[p]));     // exp(sign (b - ref))
        const float2 v = mul2(unpack2(word(x, p)), e);
        h[p] = pack2(v);
        l[p] = pack2(sub2(v, unpack2(h[p])));
    }
    *reinterpret_cast<uint4*>(hi) = make_uint4(h[0], h[1], h[2], h[3]);
    if (lo) *reinterpret_cast<uint4*>(lo) = make_uint4(l[0], l[1], l[2], l[3]);
}

// TMEM state pass over this thread's columns: SB <- bf16(Y * fsb), Y <- Y * fy (fsb, fy per channel, smem).
// Warp w handles TMEM lanes 32 (w%4) + [0,32) (one v per thread) and column half w/4.
template <int NL>
__device__ __forceinline__ void state_pass_cols(uint32_t tS, uint32_t lane_base, int c0, int vrow, const float* fsb,
                                                const float* fy, uint8_t* sSB, __nv_bfloat16* anch_row) {
    // NL 32-column TMEM loads in flight (tcgen05.ld is latency-bound, ~150 cycles per x32)
    uint32_t r[NL][32];
#pragma unroll
    for (int h = 0; h < NL; ++h) tmem_ld32(tS + lane_base + c0 + 32 * h, r[h]);
    tmem_wait_ld();
#pragma unroll
    for (int h = 0; h < NL; ++h) {
        const int cb = c0 + 32 * h;
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            const float4 fs = *reinterpret_cast<const float4*>(fsb + cb + j);
            const float4 fyv = *reinterpret_cast<const float4*>(fy + cb + j);
            const float2 y0 = make_float2(__uint_as_float(r[h][j]), __uint_as_float(r[h][j + 1]));
            const float2 y1 = make_float2(__uint_as_float(r[h][j + 2]), __uint_as_float(r[h][j + 3]));
            pk[j / 2] = pack2(mul2(y0, make_float2(fs.x, fs.y)));
            pk[j / 2 + 1] = pack2(mul2(y1, make_float2(fs.z, fs.w)));
            const float2 z0 = mul2(y0, make_float2(fyv.x, fyv.y)), z1 = mul2(y1, make_float2(fyv.z, fyv.w));
            r[h][j] = __float_as_uint(z0.x); r[h][j + 1] = __float_as_uint(z0.y);
            r[h][j + 2] = __float_as_uint(z1.x); r[h][j + 3] = __float_as_uint(z1.y);
        }
        tmem_st32(tS + lane_base + cb, r[h]);
        uint8_t* dst = sSB + (cb >> 6) * 16384;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int cc = (cb & 63) + 8 * u;
            const uint4 w = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            *reinterpret_cast<uint4*>(dst + sw128_off(vrow, cc)) = w;
            if (anch_row) *reinterpret_cast<uint4*>(anch_row + cb + 8 * u) = w;   // checkpoint copy (bwd anchors)
        }
    }
}

}  // namespace tc
}  // namespace gla
