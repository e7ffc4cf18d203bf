// tc_stub.cu -- placeholder until the tcgen05 kernels land: the TC path reports "unsupported".
#include "tc.h"
namespace gla {
namespace tc {
bool supported(int, int, int, int, int, int, int, int, int) { return false; }
cudaError_t fwd(const Problem&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t bwd(const BwdProblem&, cudaStream_t) { return cudaErrorNotSupported; }
size_t fwd_ws(int, int, int, int, int, int) { return 0; }
size_t bwd_ws(int, int, int, int, int, int) { return 0; }
}  // namespace tc
}  // namespace gla
