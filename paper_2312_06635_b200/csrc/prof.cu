// prof.cu -- see prof.h.
#include <mutex>
#include <string>
#include <vector>

#include <string.h>

#include "../../include/gla.h"
#include "prof.h"

namespace gla {
namespace prof {
namespace {
struct Rec { std::string name; cudaEvent_t a, b; };
std::mutex mu;
bool on = false;
std::vector<Rec> recs;
std::vector<cudaEvent_t> pool;
Rec* open_rec = nullptr;

cudaEvent_t get_event() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

bool enabled() { return on; }

void begin(const char* name, cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu);
    recs.push_back(Rec{name, get_event(), get_event()});
    cudaEventRecord(recs.back().a, st);
}

void end(cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu);
    if (!recs.empty()) cudaEventRecord(recs.back().b, st);
}
}  // namespace prof
}  // namespace gla

using namespace gla::prof;

extern "C" {

void gla_profile_enable(int enable) {
    std::lock_guard<std::mutex> g(mu);
    on = enable != 0;
}

void gla_profile_reset(void) {
    std::lock_guard<std::mutex> g(mu);
    for (auto& r : recs) { pool.push_back(r.a); pool.push_back(r.b); }
    recs.clear();
}

int gla_profile_count(void) {
    std::lock_guard<std::mutex> g(mu);
    return (int)recs.size();
}

// Aggregate by kernel name.  Fills up to `cap` entries; returns the number of distinct kernels.
// Synchronizes on the recorded events.
int gla_profile_get(int cap, char* names /* cap x 64 bytes */, float* total_ms, int* launches) {
    std::lock_guard<std::mutex> g(mu);
    std::vector<std::string> keys;
    std::vector<float> ms;
    std::vector<int> n;
    for (auto& r : recs) {
        cudaEventSynchronize(r.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        size_t i = 0;
        for (; i < keys.size(); ++i) if (keys[i] == r.name) break;
        if (i == keys.size()) { keys.push_back(r.name); ms.push_back(0.f); n.push_back(0); }
        ms[i] += t;
        n[i] += 1;
    }
    for (size_t i = 0; i < keys.size() && (int)i < cap; ++i) {
        strncpy(names + 64 * i, keys[i].c_str(), 63);
        names[64 * i + 63] = 0;
        total_ms[i] = ms[i];
        launches[i] = n[i];
    }
    return (int)keys.size();
}
}
