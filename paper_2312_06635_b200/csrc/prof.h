// prof.h -- optional per-launch CUDA-event tracing inside libgla (gla_profile_* in gla.h).
// When enabled, every kernel launch of the library is bracketed by two cudaEvents recorded on the
// launching stream; gla_profile_get() reports per-kernel total device time and launch count.
#pragma once
#include <cuda_runtime.h>

namespace gla {
namespace prof {
bool enabled();
void begin(const char* name, cudaStream_t st);   // record the start event of the next launch
void end(cudaStream_t st);                       // record the end event of that launch
struct Scope {
    cudaStream_t st;
    bool on;
    Scope(const char* name, cudaStream_t s) : st(s), on(enabled()) { if (on) begin(name, s); }
    ~Scope() { if (on) end(st); }
};
}  // namespace prof
}  // namespace gla
#define GLA_PROF(name, st) ::gla::prof::Scope _gla_prof_scope_##__LINE__(name, st)
