// Device-side inspection of the weight store (test/debug helpers that must not
// read the matrix back: cfg5's 36.9 GB of weights).
#include "kernels_common.cuh"

namespace snb {

namespace {

constexpr int kCensusMax = 8;

// counts[k] = cells of W[:, 0:nl] equal to vals[k] (k < nv, first match);
// counts[nv] = all other cells.  One CTA per row stripe, columns strided.
template <typename WT>
__global__ void __launch_bounds__(256) k_value_counts(const WT* W, int64_t pitch, int n, int nl, const WT* vals,
                                                      int nv, unsigned long long* counts) {
    __shared__ unsigned long long sc[kCensusMax + 1];
    if (threadIdx.x <= kCensusMax) sc[threadIdx.x] = 0;
    __syncthreads();
    WT v[kCensusMax];
#pragma unroll
    for (int k = 0; k < kCensusMax; ++k) v[k] = k < nv ? vals[k] : WT(0);
    unsigned long long c[kCensusMax + 1] = {};
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const WT* row = W + static_cast<int64_t>(i) * pitch;
        for (int j = threadIdx.x; j < nl; j += blockDim.x) {
            const WT w = __ldcs(row + j);
            int hit = nv;
#pragma unroll
            for (int k = kCensusMax - 1; k >= 0; --k)
                if (k < nv && w == v[k]) hit = k;
#pragma unroll
            for (int k = 0; k <= kCensusMax; ++k) c[k] += (hit == k) ? 1ull : 0ull;
        }
    }
#pragma unroll
    for (int k = 0; k <= kCensusMax; ++k)
        if (c[k]) atomicAdd(&sc[k], c[k]);
    __syncthreads();
    if (threadIdx.x <= nv && sc[threadIdx.x]) atomicAdd(counts + threadIdx.x, sc[threadIdx.x]);
}

}  // namespace

int census_max_values() { return kCensusMax; }

void launch_value_counts(const void* W, bool f64, int64_t pitch, int n, int nl, const void* vals, int nv,
                         unsigned long long* counts, int ctas, cudaStream_t s) {
    if (f64)
        k_value_counts<double><<<ctas, 256, 0, s>>>(static_cast<const double*>(W), pitch, n, nl,
                                                    static_cast<const double*>(vals), nv, counts);
    else
        k_value_counts<float><<<ctas, 256, 0, s>>>(static_cast<const float*>(W), pitch, n, nl,
                                                   static_cast<const float*>(vals), nv, counts);
    check(cudaGetLastError(), "k_value_counts");
}

}  // namespace snb
