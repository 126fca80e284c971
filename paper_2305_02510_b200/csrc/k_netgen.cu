// On-device erdos_renyi generation (bit-identical to netgen.cpp) and the
// RandomStream key derivation.
#include "kernels_common.cuh"

namespace snb {

namespace {

// ---------------------------------------------------------------------------
// On-device erdos_renyi (netgen.cpp:36-51): pair (i, j), i != j, exists iff
// unit_at(i*n + j) < p on stream 1 -- bit-identical draws.
__device__ __forceinline__ bool er_edge(const ErArgs& e, int i, int j) {
    if (i == j || !(e.p > 0.0)) return false;
    if (e.p >= 1.0) return true;  // unit_at < 1 always
    const uint64_t pair = static_cast<uint64_t>(i) * static_cast<uint64_t>(e.n) + static_cast<uint64_t>(j);
    return unit_at(e.edge_key, pair) < e.p;
}
__device__ __forceinline__ int er_delay(const ErArgs& e, int i, int j) {
    if (e.delay_max <= 1) return 1;
    uint64_t key;
    if (e.delay_by_synapse_index)  // p == 1: synapse index of (i, j) in list order
        key = static_cast<uint64_t>(i) * static_cast<uint64_t>(e.n - 1) + static_cast<uint64_t>(j - (j > i ? 1 : 0));
    else
        key = static_cast<uint64_t>(i) * static_cast<uint64_t>(e.n) + static_cast<uint64_t>(j);
    return 1 + static_cast<int>(below_at(e.delay_key, key, static_cast<uint64_t>(e.delay_max)));
}

template <typename WT>
__global__ void k_er_dense(ErArgs e, WT* w, uint8_t* delay, uint32_t* mask, int first, int nl,
                           int64_t pitch) {
    const int i = blockIdx.x;
    const int64_t c = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x;  // < pitch
    if (c >= pitch) return;
    const int j = first + static_cast<int>(c);
    const bool present = c < nl && er_edge(e, i, j);
    const int64_t off = static_cast<int64_t>(i) * pitch + c;
    w[off] = present ? (sizeof(WT) == 4 ? WT(e.weight_f) : WT(e.weight_d)) : WT(0);
    if (delay) delay[off] = static_cast<uint8_t>(present ? er_delay(e, i, j) : 1);
    if (mask) {
        const uint32_t word = __ballot_sync(0xffffffffu, present && e.stdp);
        if ((threadIdx.x & 31) == 0) mask[static_cast<int64_t>(i) * (pitch >> 5) + (c >> 5)] = word;
    }
}

__global__ void k_er_sparse_count(ErArgs e, int first, int nl, int pb, int nblocks, int64_t* counts) {
    const int64_t tidg = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tidg >= static_cast<int64_t>(nl) * nblocks) return;
    const int b = static_cast<int>(tidg / nl);
    const int p = static_cast<int>(tidg - static_cast<int64_t>(b) * nl);
    const int j = first + p;
    const int i0 = b * pb, i1 = min(e.n, i0 + pb);
    int64_t cnt = 0;
    for (int i = i0; i < i1; ++i) cnt += er_edge(e, i, j) ? 1 : 0;
    counts[tidg] = cnt;
}

template <typename WT>
__global__ void k_er_sparse_fill(ErArgs e, int first, int nl, int pb, int nblocks, const int64_t* off,
                                 uint32_t* meta, WT* w) {
    const int64_t tidg = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tidg >= static_cast<int64_t>(nl) * nblocks) return;
    const int b = static_cast<int>(tidg / nl);
    const int p = static_cast<int>(tidg - static_cast<int64_t>(b) * nl);
    const int j = first + p;
    const int i0 = b * pb, i1 = min(e.n, i0 + pb);
    int64_t q = off[tidg];
    const int64_t end = off[tidg + 1];
    const WT wt = sizeof(WT) == 4 ? WT(e.weight_f) : WT(e.weight_d);
    for (int i = i0; i < i1; ++i) {
        if (!er_edge(e, i, j)) continue;
        const int d = er_delay(e, i, j);
        meta[q] = static_cast<uint32_t>(i - i0) | (static_cast<uint32_t>(d - 1) << 16) |
                  (e.stdp ? (1u << 22) : 0u);   // dictionary index 0 (bits 23..31) = e.weight
        if (w) w[q] = wt;
        ++q;
    }
    for (; q < end; ++q) {  // padding: never delivers, never plastic
        // dictionary mode: entry 1 (= 0.0) and pre slot pb, whose staged history is zero
        meta[q] = w ? 0u : ((1u << 23) | static_cast<uint32_t>(pb));
        if (w) w[q] = WT(0);
    }
}

}  // namespace

uint64_t stream_key(uint64_t seed, uint64_t stream) {
    // RandomStream(seed, stream, 0, 0) key derivation (rng.hpp:19-24)
    uint64_t k = mix64(seed + 0x9e3779b97f4a7c15ULL);
    k = mix64(k ^ stream);
    k = mix64(k ^ 0ull);
    return mix64(k ^ 0ull);
}

void launch_er_dense(const ErArgs& e, void* w, bool f64, uint8_t* delay, uint32_t* mask, int first,
                     int nl, int64_t pitch, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(e.n), static_cast<unsigned>((pitch + 255) / 256));
    if (f64) k_er_dense<double><<<grid, 256, 0, s>>>(e, static_cast<double*>(w), delay, mask, first, nl, pitch);
    else k_er_dense<float><<<grid, 256, 0, s>>>(e, static_cast<float*>(w), delay, mask, first, nl, pitch);
    check(cudaGetLastError(), "k_er_dense");
}

void launch_er_sparse_count(const ErArgs& e, int first, int nl, int pb, int nblocks, int64_t* counts,
                            cudaStream_t s) {
    const int64_t tot = static_cast<int64_t>(nl) * nblocks;
    k_er_sparse_count<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(e, first, nl, pb, nblocks, counts);
    check(cudaGetLastError(), "k_er_sparse_count");
}

void launch_er_sparse_fill(const ErArgs& e, int first, int nl, int pb, int nblocks, const int64_t* off,
                           uint32_t* meta, void* w, bool f64, cudaStream_t s) {
    const int64_t tot = static_cast<int64_t>(nl) * nblocks;
    const unsigned g = static_cast<unsigned>((tot + 255) / 256);
    if (f64) k_er_sparse_fill<double><<<g, 256, 0, s>>>(e, first, nl, pb, nblocks, off, meta, static_cast<double*>(w));
    else k_er_sparse_fill<float><<<g, 256, 0, s>>>(e, first, nl, pb, nblocks, off, meta, static_cast<float*>(w));
    check(cudaGetLastError(), "k_er_sparse_fill");
}

}  // namespace snb
