// Small host helpers shared by the engine translation units.
#pragma once

#include "engine.hpp"

#include <cstdint>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

namespace snb {

// host_pool.cpp: f(0..n-1) on a persistent pool of host threads (and the caller)
int host_threads();
void host_parallel(int n, const std::function<void(int)>& f);

namespace {

// NVTX range for the host phases of the engine (setup, simulate, graph
// capture / replay, per-phase launches, raster decode): visible in
// Nsight timelines, a no-op costing a few ns when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};


inline std::string fmt_double(double v) {  // model.cpp:26-30
    std::ostringstream os;
    os << v;
    return os.str();
}

inline void throw_first(const char* where, const std::vector<std::string>& v) {  // mat_engine.cpp:15-21
    if (v.empty()) return;
    std::string msg = std::string(where) + ": " + v.front();
    if (v.size() > 1) msg += " (+" + std::to_string(v.size() - 1) + " more)";
    throw InvalidArgument(msg);
}

// Host-to-device copy that is complete on return, ordered on the engine's
// stream: after every engine kernel queued before it, before every kernel
// queued after it, and independent of the legacy default stream (a plain
// pageable cudaMemcpy may return with its DMA still queued there, and the
// engine's non-blocking stream does not wait for it).
inline void h2d_sync(cudaStream_t s, void* dst, const void* src, size_t bytes, const char* what) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), what);
    cuda_check(cudaStreamSynchronize(s), what);
}

template <typename T>
inline void upload(cudaStream_t s, DevBuf& d, const std::vector<T>& h) {
    d.alloc(h.size() * sizeof(T));
    if (!h.empty()) h2d_sync(s, d.p, h.data(), h.size() * sizeof(T), "upload");
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

inline uint64_t host_mix64(uint64_t z) {  // rng.hpp:8-12
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}


}  // namespace
}  // namespace snb
