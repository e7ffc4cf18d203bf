// tc.cu -- dispatch for the tensor-core path (tcgen05 kernels in tc_fwd2.cu / tc_bwd.cu), segment choice.
#include <cstdlib>

#include "tc.h"

namespace gla {
namespace tc {

cudaError_t fwd2_tc(const Problem& p, cudaStream_t st);    // prep + state kernels (tc_fwd2.cu), the default
size_t fwd2_ws(int B, int H, int T, int K, int V);

cudaError_t bwd_tc(const BwdProblem& p, cudaStream_t st);
size_t bwd_tc_ws(int B, int H, int T, int K, int V, int C);
bool bwd_tc_supported(int K, int V);

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

int fwd_segments(int BH, int V, int NC) {
    static int force = -1;   // GLA_SEGMENTS=1: never split; GLA_SEGMENTS=N (a power of two): N where valid
    if (force < 0) {
        const char* e = getenv("GLA_SEGMENTS");
        force = e ? atoi(e) : 0;
    }
    int S = 1;
    if (force == 1) return S;
    if (force > 1) return (NC % force == 0 && NC / force >= 8) ? force : 1;
    // The summaries cost a fixed share of a segment, so splitting pays when the unsplit walk would use at most a
    // quarter of the SMs (S = 4 at 32 CTAs 1.5x faster end to end), or half of them with long segments (below).
    const int nvt = V / 128 > 0 ? V / 128 : 1, ctas = BH * nvt;
    // Long walks that fill at most half of the SMs split in two (T = 8K at 1.3B: 1,040 vs 1,081 us per step); short
    // ones do not (340M, 32 chunks: S = 2 at 304 vs 253 us): the summaries and the chain are a fixed cost per segment.
    if ((long)ctas * 4 > num_sms())
        return ((long)ctas * 2 <= num_sms() && NC % 2 == 0 && NC / 2 >= 32) ? 2 : 1;
    while ((long)ctas * 2 * S <= num_sms() && NC % (2 * S) == 0 && NC / (2 * S) >= 8) S *= 2;
    return S >= 4 ? S : 1;
}

int seg_parts(int BH, int K, int V, int NC, int S) {
    if (S <= 1) return 1;
    static int force = -1;   // GLA_SEG_PARTS=P (a power of two <= 8) where it divides the segment's blocks
    if (force < 0) {
        const char* e = getenv("GLA_SEG_PARTS");
        force = e ? atoi(e) : 0;
    }
    if (force > 0) return ((NC / S) % force == 0 && NC / S / force >= 4 && force <= 8) ? force : 1;
    // The split summaries run one CTA per (128 channels, 256 values, segment, part).  One CTA streams a block in
    // ~0.86 us (latency-bound) and all CTAs together ~110 blocks/us (the L2 -> SM load rate), so parts pay only
    // while they stay within one wave (T = 8K at 1.3B: 64 -> 128 CTAs, 55 -> 41 us; two waves were slower at
    // every measured shape, profiles/r2_seg_parts.md).
    const long ctas = (long)(K / 128) * (V / 256) * BH * (S - 1);
    const int nb = NC / S;
    int P = 1;
    while (P < 8 && ctas * 2 * P <= num_sms() && nb % (2 * P) == 0 && nb / (2 * P) >= 4) P *= 2;
    return P;
}

bool supported(int B, int H, int T, int K, int V, int C, int c, int qkv_dtype, int gate_dtype) {
    (void)B; (void)H; (void)T; (void)gate_dtype;
    return qkv_dtype == 0 && (K == 64 || K == 128 || K == 256) && V % 128 == 0 && C == 64 && c > 0 && 64 % c == 0;
}

bool fwd_is_split() { return true; }

bool saved_anchors() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("GLA_SERIAL_WALKS");
        v = (s && s[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

cudaError_t fwd(const Problem& p, cudaStream_t st) {
    if (p.mode != 0) return simt::fwd(p, st);
    return fwd2_tc(p, st);
}

// Backward: tcgen05 kernels for K in {128, 256}; K = 64 (and dstate summaries) run the CUDA-core kernels.
cudaError_t bwd(const BwdProblem& p, cudaStream_t st) {
    if (p.mode == 0 && bwd_tc_supported(p.K, p.V)) return bwd_tc(p, st);
    return simt::bwd(p, st);
}

size_t fwd_ws(int B, int H, int T, int K, int V, int C) {
    return fwd2_ws(B, H, T, K, V);
}
size_t bwd_ws(int B, int H, int T, int K, int V, int C) {
    return bwd_tc_supported(K, V) ? bwd_tc_ws(B, H, T, K, V, C) : simt::bwd_ws(B, H, T, K, V, C);
}

}  // namespace tc
}  // namespace gla
