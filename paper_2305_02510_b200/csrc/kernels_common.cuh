// sm_100a kernels for the MAT-mode step (SuperNeuro MAT / spikeforge mat_engine).
//
// Per simulated step t the engine runs:
//   k_neuron   LIF update of the local posts          mat_engine.cpp:173-198, model.hpp:127-138
//              (+ history shift, STDP traces, active-row bitmask when single-partition)
//   [ncclAllGather of the spike bitmask, then k_hist over all N, when partitioned]
//   k_dense_sweep / k_sparse_pull
//              one pass over the weights: STDP update (mat_engine.cpp:242-249) fused
//              with the spike-gated propagation of step t+1 (mat_engine.cpp:79-93),
//              so every plastic weight is read and written exactly once per step.
//
// All kernels are HBM-streaming integer/fp32 work; no tensor cores (a batch-1
// binary-spike GEMV is not a dense contraction).
//
// This header holds the device helpers the kernel translation units share
// (k_neuron.cu, k_dense.cu, k_persistent.cu, k_sparse.cu, k_netgen.cu): the
// neuron step, the spike-history / STDP-trace update, the dense streaming
// sweep body, TMA / mbarrier wrappers, counter-based RNG and launch checks,
// in an anonymous namespace (each .cu gets its own copy).
#pragma once

#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cstdio>
#include <stdexcept>
#include <string>

// Checked builds (-DSNB_CHECKED, tools/build_variant.sh checked -DSNB_CHECKED):
// device-side bounds checks on the hot kernels' shared-memory and list
// indexing, and mbarrier waits that trap after ~2^31 polls instead of hanging
// -- the substitute for compute-sanitizer, which this GPU pool refuses
// (profiles/r02_compute_sanitizer_refused.txt).  Compiled out otherwise.
#ifdef SNB_CHECKED
#include <cstdio>
#define SNB_DCHECK(cond)                                                                    \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("SNB_DCHECK failed %s:%d block (%d,%d) thread %d: %s\n", __FILE__, __LINE__, \
                   blockIdx.x, blockIdx.y, threadIdx.x, #cond);                             \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define SNB_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace snb {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr int kSubRows = 1024;   // rows per active-list build in the dense sweep
constexpr int kHistWordsMax = 8; // history bits <= 512

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// RandomStream::u64_at / unit_at / below_at (rng.hpp:28-41)
__device__ __forceinline__ uint64_t u64_at(uint64_t key, uint64_t idx) {
    return mix64(key + idx * 0x9e3779b97f4a7c15ULL);
}
__device__ __forceinline__ double unit_at(uint64_t key, uint64_t idx) {
    return static_cast<double>(u64_at(key, idx) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ uint64_t below_at(uint64_t key, uint64_t idx, uint64_t n) {
    return __umul64hi(u64_at(key, idx), n);
}

// StochasticLifBehavior gate (abm_engine.cpp:34-39): the first unit draw of
// RandomStream(seed, agent stream, id, step); `key` = the stream key before
// the step mix (rng.hpp:19-24), precomputed per neuron on the host.
__device__ __forceinline__ bool agent_fires(uint64_t key, int t, double p) {
    const uint64_t k = mix64(key ^ static_cast<uint64_t>(t));
    return static_cast<double>(mix64(k) >> 11) * 0x1.0p-53 < p;
}

// leak_toward (model.hpp:127-138), literally.
__device__ __forceinline__ double leak_toward(double v, double leak, double reset) {
    const double d = v - reset;
    if (d > 0.0) {
        const double stepped = d - leak;
        return reset + (stepped > 0.0 ? stepped : 0.0);
    }
    if (d < 0.0) {
        const double stepped = d + leak;
        return reset + (stepped < 0.0 ? stepped : 0.0);
    }
    return v;
}

// std::clamp(v, lo, hi) (mat_engine.cpp:247) for both precisions.
template <typename T>
__device__ __forceinline__ T clamp_ref(T v, T lo, T hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}

// One plastic synapse (mat_engine.cpp:243-248): dw = 0; if s_post dw += pot_pre;
// if s_pre dw -= dep_post; w = clamp(w + dw, w_min, w_max), with the traces,
// dw and w + dw in fp64 like the reference.  dw: one subtraction of selected
// operands gives the reference's value in every case (0 + pot = pot,
// pot - dep rounded once, 0 - dep, +0).  fp32 storage rounds w + dw once;
// rounding is monotone, so RN(clamp(x, lo, hi)) == clamp(RN(x), RN(lo),
// RN(hi)) and the clamp runs in fp32 on bounds rounded the same way (min/max:
// identical to clamp_ref for the NaN-free values here, up to the sign of a
// zero weight).
__device__ __forceinline__ double stdp_dw(bool s_post, double pot, bool s_pre, double dep) {
    return (s_post ? pot : 0.0) - (s_pre ? dep : 0.0);
}
template <typename WT>
__device__ __forceinline__ WT stdp_apply(WT w, double dw, WT lo, WT hi);
template <>
__device__ __forceinline__ double stdp_apply<double>(double w, double dw, double lo, double hi) {
    return clamp_ref<double>(w + dw, lo, hi);
}
template <>
__device__ __forceinline__ float stdp_apply<float>(float w, double dw, float lo, float hi) {
    return fminf(fmaxf(__double2float_rn(static_cast<double>(w) + dw), lo), hi);
}

__device__ __forceinline__ uint32_t bit_of(const uint32_t* bits, int i) {
    return (__ldcg(bits + (i >> 5)) >> (i & 31)) & 1u;
}

// Amplitude of neuron j in one step's stimulus row [lo, hi) (neuron ids
// ascending, unique: the step's entries pre-summed in list order), 0 if absent.
// Rows of up to 16 entries (the paper protocol's few driven inputs) are read
// with all their loads in flight; longer rows are binary-searched.
__device__ __forceinline__ double stim_lookup(const int32_t* st_neuron, const double* st_amp, int64_t lo, int64_t hi,
                                              int j) {
    if (hi - lo <= 16) {
        int32_t nb[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) nb[k] = lo + k < hi ? __ldg(st_neuron + lo + k) : -1;
        int hit = -1;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (nb[k] == j) hit = k;
        return hit >= 0 ? __ldg(st_amp + lo + hit) : 0.0;
    }
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int nid = __ldg(st_neuron + mid);
        if (nid == j) return __ldg(st_amp + mid);
        if (nid < j) lo = mid + 1; else hi = mid;
    }
    return 0.0;
}

// ---------------------------------------------------------------------------
// History shift + windowed STDP traces for neuron i (mat_engine.cpp:200-240).
// hist bit k (across words) = s_i[t-k]; history before step 0 is zero, so the
// reference's `k > t` break (mat_engine.cpp:230) needs no special casing.
//   dep_i      = sum_{k=1..W} a_minus[k-1] s_i[t-k]           (k ascending, fp64)
//   pot_i^(d)  = sum_{k=1..W} a_plus[k-1]  s_i[t-k-d+1]       (lowered-net shift)
// Returns whether row i must be visited by the sweep this step.
//
// Windows + delay spans beyond 64 steps (any window >= 1 is valid,
// model.cpp:104-117) take hist_update_long: the same sums with the history
// words read back from global memory instead of one register.
__device__ __forceinline__ bool hist_update_long(const HistArgs& h, int i, bool s, int t) {
    uint64_t carry = s ? 1ull : 0ull, w0 = 0;
    for (int k = 0; k < h.hw; ++k) {
        uint64_t* p = h.hist + static_cast<int64_t>(k) * h.n + i;
        const uint64_t x = *p;
        const uint64_t nx = (x << 1) | carry;
        carry = x >> 63;
        *p = nx;
        if (k == 0) w0 = nx;
    }
    if (h.hist_lo) h.hist_lo[i] = static_cast<uint32_t>(w0);
    const uint64_t dmask = h.dmax >= 64 ? ~0ull : ((1ull << h.dmax) - 1ull);
    bool act = (w0 & dmask) != 0;
    if (h.stdp) {
        auto bit = [&](int b) { return (h.hist[static_cast<int64_t>(b >> 6) * h.n + i] >> (b & 63)) & 1ull; };
        double dep = 0.0;
        for (int k = 1; k <= h.window; ++k)
            if (bit(k)) dep += h.a_minus[k - 1];
        h.dep64[i] = dep;
        bool any_pot = false;
        for (int d = 1; d <= h.dp; ++d) {
            double pot = 0.0;
            for (int k = 1; k <= h.window; ++k)
                if (bit(k + d - 1)) pot += h.a_plus[k - 1];
            h.pot64[static_cast<int64_t>(i) * h.dp + (d - 1)] = pot;
            any_pot |= (pot != 0.0);
        }
        if (h.row_plastic[i] && (any_pot || t == h.clamp_step)) act = true;
    }
    return act;
}

__device__ __forceinline__ bool hist_update(const HistArgs& h, int i, bool s, int t) {
    // one history word (window + delay span <= 64) in registers; longer
    // histories (several words) go through hist_update_long, whose dynamic
    // bit indexing would otherwise put a word array in local memory on every path
    if (h.hw != 1) return hist_update_long(h, i, s, t);
    uint64_t* p = h.hist + i;
    const uint64_t w0 = (*p << 1) | (s ? 1ull : 0ull);
    *p = w0;
    if (h.hist_lo) h.hist_lo[i] = static_cast<uint32_t>(w0);
    const uint64_t dmask = h.dmax >= 64 ? ~0ull : ((1ull << h.dmax) - 1ull);
    bool act = (w0 & dmask) != 0;
    if (h.stdp) {
        // walk the set bits in ascending k, the order of the reference's sums
        // (mat_engine.cpp:226-240)
        const uint64_t wmask = h.window >= 63 ? ~0ull : ((1ull << (h.window + 1)) - 1ull);
        double dep = 0.0;
        for (uint64_t m = w0 & wmask & ~1ull; m; m &= m - 1) dep += h.a_minus[__ffsll(static_cast<long long>(m)) - 2];
        h.dep64[i] = dep;
        bool any_pot = false;
        for (int d = 1; d <= h.dp; ++d) {
            const uint64_t sh = w0 >> (d - 1);  // bit k of sh = s[t - k - d + 1]
            double pot = 0.0;
            for (uint64_t m = sh & wmask & ~1ull; m; m &= m - 1) pot += h.a_plus[__ffsll(static_cast<long long>(m)) - 2];
            h.pot64[static_cast<int64_t>(i) * h.dp + (d - 1)] = pot;
            any_pot |= (pot != 0.0);
        }
        // t == 0: apply_stdp clamps every plastic weight even when dw == 0
        // (mat_engine.cpp:243-249); afterwards weights stay inside the bounds,
        // so rows with no pairing and no delivery are provably unchanged.
        if (h.row_plastic[i] && (any_pot || t == h.clamp_step)) act = true;
    }
    return act;
}

// Sum of the synaptic input partials of local post j over chunk rows [c0, c1):
// acc[k] sums rows k, k+8, k+16, ... in order, then a fixed tree.
template <bool P16>  // rows are a.partial16 block counts (else fp64 a.partial)
__device__ __forceinline__ double partial_sum(const NeuronArgs& a, int j, int c0, int c1) {
    // 16 loads are issued before any add, so the rows arrive in a few memory
    // round trips
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int c = c0;
    if (P16) {
        // 16-bit block counts: 2 B per (block, post) instead of 8; the block's
        // value and the summation tree are the ones of the fp64 partials
        const float w0f = static_cast<float>(a.w0);
        auto val = [&](uint32_t k) {
            return a.w0_f32 ? static_cast<double>(static_cast<float>(k) * w0f) : static_cast<double>(k) * a.w0;
        };
        for (; c + 16 <= c1; c += 16) {
            uint32_t t[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = __ldcg(a.partial16 + static_cast<int64_t>(c + k) * a.nl + j);
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k & 7] += val(t[k]);
        }
        uint32_t t[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) t[k] = c + k < c1 ? __ldcg(a.partial16 + static_cast<int64_t>(c + k) * a.nl + j) : 0u;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (c + k < c1) acc[k & 7] += val(t[k]);
        c = c1;
    }
    for (; c + 16 <= c1; c += 16) {
        double t[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) t[k] = __ldcg(a.partial + static_cast<int64_t>(c + k) * a.nl + j);
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k & 7] += t[k];
    }
    for (; c + 8 <= c1; c += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += __ldcg(a.partial + static_cast<int64_t>(c + k) * a.nl + j);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)  // remainder; unrolled so acc stays in registers
        if (c + k < c1) acc[k] += __ldcg(a.partial + static_cast<int64_t>(c + k) * a.nl + j);
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// ---------------------------------------------------------------------------
// K1: LIF update of the local posts for step t (mat_engine.cpp:168-198).
// Called by full warps (j covers a multiple of 32); one neuron per thread.
// WARP_COUNT: lane 0 of each warp adds the warp's spike / active counts to the
// global counters; otherwise the caller aggregates the returned per-thread
// flags (bit 0 spiked, bit 1 active) per CTA - one same-address atomic per
// warp serialises at L2 once a step has ~10^4 warps.
template <bool EXACT, bool FUSED, bool WARP_COUNT = true, bool INPUT = false>
__device__ __forceinline__ uint32_t neuron_step(const NeuronArgs& a, const HistArgs& h, int j, int t,
                                                double given = 0.0) {
    const bool valid = j < a.nl;
    if (a.work && j == 0) *a.work = 0;  // the previous sweep has finished (stream / grid order)
    bool s = false;
    if (valid) {
        double v = a.v[j];
        const double reset = a.reset[j];
        double u;  // MAT: leak(v) + input; ABM: the synaptic input alone
        if (EXACT) {
            u = a.u_exact[j];  // (leak(v) +) sum in ascending pre order, from the sweep
        } else {
            // chunk partials: acc[k] sums chunks k, k+8, k+16, ... in order, then a
            // fixed tree (partial_sum); or the sum handed over by the split kernel
            const double in = INPUT ? given
                              : a.partial16 ? partial_sum<true>(a, j, 0, a.nchunks)
                                            : partial_sum<false>(a, j, 0, a.nchunks);
            u = a.abm ? in : leak_toward(v, a.leak[j], reset) + in;
        }
        // external stimulus: the step's entries pre-summed in list order
        // (mat_engine.cpp:271-275); u += ext only when the step has any (179-180)
        const int row = t - a.st_base;
        if (row >= 0 && row < a.st_steps) {
            int64_t lo = a.st_off[row], hi = a.st_off[row + 1];
            if (hi > lo) {
                const int gj = a.first + j;
                double ext = 0.0;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    const int nid = a.st_neuron[mid];
                    if (nid == gj) { ext = a.st_amp[mid]; break; }
                    if (nid < gj) lo = mid + 1; else hi = mid;
                }
                u += ext;
            }
        }
        // ABM: input = pending + ext, u = leak(v) + input (abm_engine.cpp:150-154, 24)
        if (a.abm) u = leak_toward(v, a.leak[j], reset) + u;
        s = u > a.thr[j];
        if (s && a.fire_p) {
            const double p = a.fire_p[j];
            if (p < 1.0) s = agent_fires(a.agent_key[j], t, p);
        }
        const int c = a.cnt[j];
        if (c > 0) {  // refractory: silent, held at reset (185-189)
            s = false;
            a.cnt[j] = c - 1;
            u = reset;
        }
        if (s) {
            v = reset;
            a.cnt[j] = a.refr[j];
        } else {
            v = u;
        }
        a.v[j] = v;
        if (a.trace && (t - a.t_base) < a.raster_rows)
            a.trace[static_cast<int64_t>(t - a.t_base) * a.nl + j] = v;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, s);
    const int lane = threadIdx.x & 31;
    const int wi = j >> 5;
    if (lane == 0 && wi < a.nl_words) {
        a.bits[(a.first >> 5) + wi] = word;
        if (a.peer_bits) {  // fused all-gather: store the word into every rank's exchange buffer t & 1 (NVLink)
            const int64_t o = static_cast<int64_t>(t & 1) * a.xstride + (a.first >> 5) + wi;
            for (int q = 0; q < a.world; ++q) a.peer_bits[q][o] = word;
        }
        if (a.raster && (t - a.t_base) < a.raster_rows)
            a.raster[static_cast<int64_t>(t - a.t_base) * a.nl_words + wi] = word;
        if (WARP_COUNT && word) atomicAdd(a.spike_count, static_cast<unsigned long long>(__popc(word)));
    }
    bool act = false;
    if (FUSED) {
        if (valid) act = hist_update(h, j, s, t);
        const uint32_t aw = __ballot_sync(0xffffffffu, act);
        if (lane == 0 && wi < a.nl_words) {
            h.active[wi] = aw;
            if (WARP_COUNT && aw) atomicAdd(h.active_count, static_cast<unsigned long long>(__popc(aw)));
        }
    }
    return (s ? 1u : 0u) | (act ? 2u : 0u);
}

__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}


// 128-bit weight vectors of the dense sweeps (fp32 x4, fp64 x2).
template <typename WT> struct VecT;
template <> struct VecT<float> {
    using V = float4;
    static constexpr int N = 4;
    __device__ static V load(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
    __device__ static void store(float* p, const V& v) { __stcs(reinterpret_cast<float4*>(p), v); }
    __device__ static float get(const V& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
    __device__ static void set(V& v, int k, float x) {
        if (k == 0) v.x = x; else if (k == 1) v.y = x; else if (k == 2) v.z = x; else v.w = x;
    }
};
template <> struct VecT<double> {
    using V = double2;
    static constexpr int N = 2;
    __device__ static V load(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }
    __device__ static void store(double* p, const V& v) { __stcs(reinterpret_cast<double2*>(p), v); }
    __device__ static double get(const V& v, int k) { return k == 0 ? v.x : v.y; }
    __device__ static void set(V& v, int k, double x) { if (k == 0) v.x = x; else v.y = x; }
};

// ---------------------------------------------------------------------------
// Streaming variant of the dense sweep (non-exact order), the hot kernel of
// the STDP configs.  Same arithmetic as k_dense_sweep but shaped for issue
// efficiency: one 16-byte shared record per active row (row|kind, history
// bits, pot), the active list padded to a multiple of U with inert rows so
// the U-row load batch has no bounds checks, 0/1 spike factors folded into
// FFMA (exact: the factors are 0 or 1), plasticity class dispatched once per
// row (warp-uniform), unconditional 128-bit streaming stores on plastic rows.
template <typename WT> struct RowRec;
template <> struct alignas(16) RowRec<float> {
    int32_t rowk;      // row | kind << 28
    uint32_t e_lo, e_hi;
    float pot;
};
template <> struct alignas(16) RowRec<double> {
    int32_t rowk;
    uint32_t e_lo, e_hi, pad;
    double pot;
    double pad2;
};

template <typename WT, bool STDP, bool DELAY>
__device__ __forceinline__ void dense_stream_body(const DenseArgs& a, int cta, int ncta) {
    using VT = VecT<WT>;
    using V = typename VT::V;
    constexpr int VEC = VT::N;
    constexpr int U = 8;
    using Rec = RowRec<double>;  // fp64 trace for both weight types (fp64 STDP math)
    __shared__ Rec s_rec[kSubRows + U];
    __shared__ uint32_t s_word[32];
    __shared__ int32_t s_wpref[33];

    const int tid = threadIdx.x;
    const int ntiles = (a.nl + a.tile_w - 1) / a.tile_w;
    const int items = ntiles * a.nchunks;
    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const double* pot = a.pot;
    const double* dep = a.dep;
    WT* W = static_cast<WT*>(a.w);
    const int64_t mpitch = a.pitch >> 5;

    // Items are claimed dynamically (a.work, reset by the neuron phase) so the
    // CTAs of a one-wave grid finish together; static striding otherwise.
    __shared__ int s_item;
    int item = cta;
    if (a.work) {
        __syncthreads();
        if (tid == 0) s_item = atomicAdd(a.work, 1);
        __syncthreads();
        item = s_item;
    }
    while (item < items) {
        const int chunk = item / ntiles;
        const int tile = item - chunk * ntiles;
        const int tcol = tid * VEC;
        const int c0 = tile * a.tile_w + tcol;
        const bool in_tile = tcol < a.tile_w && c0 < a.nl;
        const int gc0 = a.first + c0;
        const int r0 = chunk * a.rows_per_chunk;
        const int r1 = min(a.n, r0 + a.rows_per_chunk);

        bool sj[VEC];
        double depj[VEC];
        double acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const bool ok = in_tile && (c0 + k) < a.nl;
            sj[k] = ok && STDP && bit_of(a.bits, gc0 + k);
            depj[k] = (ok && STDP) ? __ldcg(dep + gc0 + k) : 0.0;
            acc[k] = 0.0;
        }

        // sub-chunks start at a 32-aligned base so <= 32 active words cover them
        for (int sa = r0, sb_next = r0; sa < r1; sa = sb_next) {
            const int base = sa & ~31;
            const int sb = min(r1, base + kSubRows);
            sb_next = sb;
            const int nwords = (sb - base + 31) >> 5;
            __syncthreads();
            if (tid < 32) {
                uint32_t wd = 0;
                if (tid < nwords) {
                    wd = __ldcg(a.active + (base >> 5) + tid);
                    const int lo = sa - (base + tid * 32);  // bits below sa
                    if (lo > 0) wd &= (lo >= 32) ? 0u : ~((1u << lo) - 1u);
                    const int rem = sb - (base + tid * 32);
                    if (rem < 32) wd &= (rem <= 0) ? 0u : ((1u << rem) - 1u);
                }
                const int c = __popc(wd);
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int x = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += x;
                }
                s_word[tid] = wd;
                s_wpref[tid] = incl - c;
                if (tid == 31) s_wpref[32] = incl;
            }
            __syncthreads();
            for (int r = sa + tid; r < sb; r += kThreads) {
                const int l = (r - base) >> 5, b = (r - base) & 31;
                const uint32_t wd = s_word[l];
                if ((wd >> b) & 1u) {
                    const int pos = s_wpref[l] + __popc(wd & ((1u << b) - 1u));
                    const uint64_t h = __ldcg(a.hist + r);
                    Rec rec;
                    const int kind = STDP ? static_cast<int>(__ldg(a.kind + r)) : 0;
                    rec.rowk = r | (kind << 28);
                    rec.e_lo = static_cast<uint32_t>(h);
                    rec.e_hi = static_cast<uint32_t>(h >> 32);
                    rec.pot = (STDP && !DELAY) ? __ldcg(pot + r) : 0.0;
                    s_rec[pos] = rec;
                }
            }
            const int cnt = s_wpref[32];
            if (tid < U && cnt > 0) {  // inert padding: re-reads row sa, no spike, no store
                Rec rec;
                rec.rowk = sa;
                rec.e_lo = rec.e_hi = 0;
                rec.pot = 0.0;
                s_rec[cnt + tid] = rec;
            }
            __syncthreads();
            if (!in_tile) continue;

            for (int gb = 0; gb < cnt; gb += U) {
                V wv[U];
                uint32_t dv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int row = s_rec[gb + u].rowk & 0x0fffffff;
                    const int64_t off = static_cast<int64_t>(row) * a.pitch + c0;
                    wv[u] = VT::load(W + off);
                    if (DELAY) {
                        if (VEC == 4) dv[u] = __ldg(reinterpret_cast<const uint32_t*>(a.delay + off));
                        else dv[u] = __ldg(reinterpret_cast<const uint16_t*>(a.delay + off));
                    }
                }
                WT grp[VEC];
#pragma unroll
                for (int k = 0; k < VEC; ++k) grp[k] = WT(0);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const Rec rec = s_rec[gb + u];
                    const int row = rec.rowk & 0x0fffffff;
                    const int kind = rec.rowk >> 28;
                    const uint64_t ebits = (static_cast<uint64_t>(rec.e_hi) << 32) | rec.e_lo;
                    WT w[VEC], ef[VEC];
#pragma unroll
                    for (int k = 0; k < VEC; ++k) {
                        w[k] = VT::get(wv[u], k);
                        const int d1 = DELAY ? static_cast<int>((dv[u] >> (8 * k)) & 0xffu) - 1 : 0;
                        ef[k] = ((ebits >> d1) & 1ull) ? WT(1) : WT(0);
                    }
                    if (STDP && a.plastic_on && kind != kRowNone) {
                        WT nw[VEC];
#pragma unroll
                        for (int k = 0; k < VEC; ++k) {
                            double p;
                            if (DELAY) {
                                const int d1 = static_cast<int>((dv[u] >> (8 * k)) & 0xffu) - 1;
                                p = __ldcg(pot + static_cast<int64_t>(row) * a.dp + d1);
                            } else {
                                p = rec.pot;
                            }
                            nw[k] = stdp_apply<WT>(w[k], stdp_dw(sj[k], p, ef[k] != WT(0), depj[k]), wmin, wmax);
                        }
                        if (kind == kRowAllButSelf) {
                            const int selfk = row - gc0;   // (i, i) is absent: keep it exactly
#pragma unroll
                            for (int k = 0; k < VEC; ++k) nw[k] = (selfk == k) ? w[k] : nw[k];
                        } else if (kind == kRowMixed) {
                            const uint32_t mv = __ldg(a.mask + static_cast<int64_t>(row) * mpitch + (c0 >> 5)) >> (c0 & 31);
#pragma unroll
                            for (int k = 0; k < VEC; ++k) nw[k] = ((mv >> k) & 1u) ? nw[k] : w[k];
                        }
                        V out;
#pragma unroll
                        for (int k = 0; k < VEC; ++k) {
                            VT::set(out, k, nw[k]);
                            w[k] = nw[k];
                        }
                        VT::store(W + static_cast<int64_t>(row) * a.pitch + c0, out);
                    }
#pragma unroll
                    for (int k = 0; k < VEC; ++k) grp[k] = fma(ef[k], w[k], grp[k]);
                }
#pragma unroll
                for (int k = 0; k < VEC; ++k) acc[k] += static_cast<double>(grp[k]);
            }
        }
        if (in_tile) {
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                if (c0 + k < a.nl) a.partial[static_cast<int64_t>(chunk) * a.nl + c0 + k] = acc[k];
        }
        if (a.work) {
            __syncthreads();
            if (tid == 0) s_item = atomicAdd(a.work, 1);
            __syncthreads();
            item = s_item;
        } else {
            item += ncta;
        }
    }
}


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef SNB_CHECKED
    uint32_t ok = 0;
    for (long long spins = 0; !ok; ++spins) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        SNB_DCHECK(spins < (1ll << 31));  // a lost arrival: trap instead of hanging the GPU
    }
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}


inline void check(cudaError_t err, const char* what) {
    if (err != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(err));
}


}  // namespace

}  // namespace snb
