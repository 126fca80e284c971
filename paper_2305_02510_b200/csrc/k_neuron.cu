// Neuron phase: LIF update + spike words + history/traces (k_neuron), the
// history kernel of partitioned runs (k_hist), and two helpers.
#include "kernels_common.cuh"

#include <cstdlib>

#ifndef SNB_NEURON_MINB
#define SNB_NEURON_MINB 4
#endif

namespace snb {

namespace {

template <bool EXACT, bool FUSED>
__global__ void __launch_bounds__(kThreads, SNB_NEURON_MINB) k_neuron(NeuronArgs a, HistArgs h) {
    const int t = *a.d_step;
    if (a.step_out && blockIdx.x == 0 && threadIdx.x == 0) *a.step_out = t;
    const uint32_t f = neuron_step<EXACT, FUSED, false>(a, h, blockIdx.x * kThreads + threadIdx.x, t);
    const int spikes = __syncthreads_count(f & 1u);
    const int active = FUSED ? __syncthreads_count(f & 2u) : 0;
    if (threadIdx.x == 0) {
        if (spikes) atomicAdd(a.spike_count, static_cast<unsigned long long>(spikes));
        if (active) atomicAdd(h.active_count, static_cast<unsigned long long>(active));
    }
    if (a.peer_bits) {
        // publish step t to every rank once all CTAs' words are out: each CTA
        // fences its peer stores system-wide and counts itself; the last CTA
        // releases flag[rank] = t + 1 in every rank's flag array
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t prev = atomicAdd(a.done, 1u);
            if (prev == gridDim.x - 1) {
                __threadfence_system();
                for (int q = 0; q < a.world; ++q) st_release_sys(a.peer_flags[q] + a.rank, t + 1);
                *a.done = 0;
            }
        }
    }
}

// Many partial rows (dense sweeps: 125 for cfg3, 334 per rank for an 8-way
// cfg5 partition): a CTA of kThreads threads takes kSplitPosts posts, its four
// thread quarters sum a quarter of the rows each (four times the loads in
// flight per post), and its first kSplitPosts threads combine the quarters in
// a fixed order and run the neuron step.
constexpr int kSplitPosts = kThreads / 4;
template <bool FUSED>
__global__ void __launch_bounds__(kThreads, SNB_NEURON_MINB) k_neuron_split(NeuronArgs a, HistArgs h) {
    __shared__ double quarter[4][kSplitPosts];
    const int t = *a.d_step;
    if (a.step_out && blockIdx.x == 0 && threadIdx.x == 0) *a.step_out = t;
    const int q = threadIdx.x / kSplitPosts, jl = threadIdx.x % kSplitPosts;
    const int j0 = blockIdx.x * kSplitPosts;
    if (j0 + jl < a.nl) {
        const int c0 = static_cast<int>((static_cast<int64_t>(a.nchunks) * q) / 4);
        const int c1 = static_cast<int>((static_cast<int64_t>(a.nchunks) * (q + 1)) / 4);
        quarter[q][jl] = partial_sum<false>(a, j0 + jl, c0, c1);
    }
    __syncthreads();
    uint32_t f = 0;
    if (threadIdx.x < kSplitPosts) {  // whole warps
        const double in = (quarter[0][jl] + quarter[1][jl]) + (quarter[2][jl] + quarter[3][jl]);
        f = neuron_step<false, FUSED, false, true>(a, h, j0 + jl, t, in);
    }
    const int spikes = __syncthreads_count(f & 1u);
    const int active = FUSED ? __syncthreads_count(f & 2u) : 0;
    if (threadIdx.x == 0) {
        if (spikes) atomicAdd(a.spike_count, static_cast<unsigned long long>(spikes));
        if (active) atomicAdd(h.active_count, static_cast<unsigned long long>(active));
    }
    if (a.peer_bits) {  // as k_neuron
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t prev = atomicAdd(a.done, 1u);
            if (prev == gridDim.x - 1) {
                __threadfence_system();
                for (int r = 0; r < a.world; ++r) st_release_sys(a.peer_flags[r] + a.rank, t + 1);
                *a.done = 0;
            }
        }
    }
}

// Partitioned runs: history/traces for all N from the all-gathered bitmask.
__global__ void __launch_bounds__(kThreads) k_hist(HistArgs h) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    const int t = *h.d_step;
    if (h.flags) {  // peer-to-peer exchange: wait for every rank's words of step t
        if (threadIdx.x == 0) {
            const uint64_t t0 = globaltimer_ns();
            for (int q = 0; q < h.world; ++q) {
                while (ld_acquire_sys(h.flags + q) <= t) {
                    if (globaltimer_ns() - t0 > 30ull * 1000000000ull) {  // 30 s: a peer died
                        atomicExch(h.error, 1);
                        break;
                    }
                    __nanosleep(200);
                }
            }
        }
        __syncthreads();
    }
    bool act = false;
    bool s = false;
    if (h.xbits) {
        // step t arrived in exchange buffer t & 1; a peer writes step t + 2 into
        // the same buffer only after its k_hist(t + 1) saw our flag t + 2, i.e.
        // after this kernel (and the sweep of step t) finished on this rank
        const uint32_t* src = h.xbits + static_cast<int64_t>(t & 1) * h.xstride;
        if (i < h.n) s = (src[i >> 5] >> (i & 31)) & 1u;
        const uint32_t word = __ballot_sync(0xffffffffu, s);
        if ((threadIdx.x & 31) == 0 && (i >> 5) < ((h.n + 31) >> 5)) h.bits[i >> 5] = word;
    } else if (i < h.n) {
        s = (h.bits[i >> 5] >> (i & 31)) & 1u;
    }
    if (i < h.n) act = hist_update(h, i, s, t);
    const uint32_t aw = __ballot_sync(0xffffffffu, act);
    if ((threadIdx.x & 31) == 0 && (i >> 5) < ((h.n + 31) >> 5)) h.active[i >> 5] = aw;
    const int active = __syncthreads_count(act);
    if (threadIdx.x == 0 && active) atomicAdd(h.active_count, static_cast<unsigned long long>(active));
}

__global__ void k_prologue(double* u, const double* v, const double* leak, const double* reset,
                           int nl, int abm) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nl) u[j] = abm ? 0.0 : leak_toward(v[j], leak[j], reset[j]);
}

__global__ void k_step_bump(int32_t* d_step) { *d_step += 1; }

}  // namespace

int neuron_split_min_rows() {
    static const int v = [] {
        const char* e = std::getenv("SNB_NEURON_SPLIT_ROWS");  // A/B knob; 0 disables the split kernel
        return e ? std::atoi(e) : 32;
    }();
    return v;
}

void launch_neuron(const NeuronArgs& a, bool exact, bool fused, const HistArgs& h, cudaStream_t s) {
    // the split grid is 4x the plain one: only while it fits one wave (cfg3 32k
    // posts: 22.4 -> 19.2 us; cfg5 96k posts: 29.5 -> 40 us, so no)
    static const int wave_posts = [] {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms * SNB_NEURON_MINB * kSplitPosts;
    }();
    const int split_rows = neuron_split_min_rows();
    if (!exact && !a.partial16 && split_rows > 0 && a.nchunks >= split_rows && a.nl <= wave_posts) {
        int grid = (a.nl + kSplitPosts - 1) / kSplitPosts;
        if (a.peer_bits && grid == 0) grid = 1;
        if (grid == 0) return;
        if (fused) k_neuron_split<true><<<grid, kThreads, 0, s>>>(a, h);
        else k_neuron_split<false><<<grid, kThreads, 0, s>>>(a, h);
        check(cudaGetLastError(), "k_neuron_split");
        return;
    }
    int grid = (a.nl + kThreads - 1) / kThreads;
    if (a.peer_bits && grid == 0) grid = 1;  // an empty partition still publishes its step
    if (grid == 0) return;
    if (exact) {
        if (fused) k_neuron<true, true><<<grid, kThreads, 0, s>>>(a, h);
        else k_neuron<true, false><<<grid, kThreads, 0, s>>>(a, h);
    } else {
        if (fused) k_neuron<false, true><<<grid, kThreads, 0, s>>>(a, h);
        else k_neuron<false, false><<<grid, kThreads, 0, s>>>(a, h);
    }
    check(cudaGetLastError(), "k_neuron");
}

void launch_hist(const HistArgs& h, cudaStream_t s) {
    const int grid = (h.n + kThreads - 1) / kThreads;
    k_hist<<<grid, kThreads, 0, s>>>(h);
    check(cudaGetLastError(), "k_hist");
}

void launch_prologue(double* u, const double* v, const double* leak, const double* reset, int nl,
                     bool abm, cudaStream_t s) {
    if (nl <= 0) return;
    k_prologue<<<(nl + 255) / 256, 256, 0, s>>>(u, v, leak, reset, nl, abm ? 1 : 0);
    check(cudaGetLastError(), "k_prologue");
}

void launch_step_bump(int32_t* d_step, cudaStream_t s) {
    k_step_bump<<<1, 1, 0, s>>>(d_step);
    check(cudaGetLastError(), "k_step_bump");
}

}  // namespace snb
