// tc.cu -- dispatch for the tensor-core path (tcgen05 kernels in tc_fwd.cu / tc_bwd.cu).
#include "tc.h"

namespace gla {
namespace tc {

cudaError_t fwd_tc(const Problem& p, cudaStream_t st);
size_t fwd_tc_ws(int B, int H, int T, int K, int V);

bool supported(int B, int H, int T, int K, int V, int C, int c, int qkv_dtype, int gate_dtype) {
    (void)B; (void)H; (void)T; (void)gate_dtype;
    return qkv_dtype == 0 && (K == 64 || K == 128 || K == 256) && V % 128 == 0 && C == 64 && c > 0 && 64 % c == 0;
}

cudaError_t fwd(const Problem& p, cudaStream_t st) {
    if (p.mode != 0) return simt::fwd(p, st);
    return fwd_tc(p, st);
}

// Backward: the tcgen05 backward kernels are not in this build yet; the fp32 CUDA-core kernels run it.
cudaError_t bwd(const BwdProblem& p, cudaStream_t st) { return simt::bwd(p, st); }

size_t fwd_ws(int B, int H, int T, int K, int V, int C) { return fwd_tc_ws(B, H, T, K, V); }
size_t bwd_ws(int B, int H, int T, int K, int V, int C) { return simt::bwd_ws(B, H, T, K, V, C); }

}  // namespace tc
}  // namespace gla
