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
#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cstdio>
#include <stdexcept>
#include <string>

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

__device__ __forceinline__ uint32_t bit_of(const uint32_t* bits, int i) {
    return (__ldcg(bits + (i >> 5)) >> (i & 31)) & 1u;
}

// ---------------------------------------------------------------------------
// History shift + windowed STDP traces for neuron i (mat_engine.cpp:200-240).
// hist bit k (across words) = s_i[t-k]; history before step 0 is zero, so the
// reference's `k > t` break (mat_engine.cpp:230) needs no special casing.
//   dep_i      = sum_{k=1..W} a_minus[k-1] s_i[t-k]           (k ascending, fp64)
//   pot_i^(d)  = sum_{k=1..W} a_plus[k-1]  s_i[t-k-d+1]       (lowered-net shift)
// Returns whether row i must be visited by the sweep this step.
__device__ __forceinline__ bool hist_update(const HistArgs& h, int i, bool s, int t) {
    uint64_t words[kHistWordsMax];
    uint64_t carry = s ? 1ull : 0ull;
#pragma unroll
    for (int k = 0; k < kHistWordsMax; ++k) {
        if (k < h.hw) {
            const uint64_t x = h.hist[static_cast<int64_t>(k) * h.n + i];
            const uint64_t nx = (x << 1) | carry;
            carry = x >> 63;
            h.hist[static_cast<int64_t>(k) * h.n + i] = nx;
            words[k] = nx;
        } else {
            words[k] = 0;
        }
    }
    if (h.hist_lo) h.hist_lo[i] = static_cast<uint32_t>(words[0]);
    const uint64_t dmask = h.dmax >= 64 ? ~0ull : ((1ull << h.dmax) - 1ull);
    bool act = (words[0] & dmask) != 0;
    if (h.stdp && h.hw == 1) {
        // one history word (window + delay span <= 64): walk the set bits in
        // ascending k, the order of the reference's sums (mat_engine.cpp:226-240)
        const uint64_t w0 = words[0];
        const uint64_t wmask = h.window >= 63 ? ~0ull : ((1ull << (h.window + 1)) - 1ull);
        double dep = 0.0;
        for (uint64_t m = w0 & wmask & ~1ull; m; m &= m - 1) dep += h.a_minus[__ffsll(static_cast<long long>(m)) - 2];
        h.dep64[i] = dep;
        h.dep32[i] = static_cast<float>(dep);
        bool any_pot = false;
        for (int d = 1; d <= h.dp; ++d) {
            const uint64_t sh = w0 >> (d - 1);  // bit k of sh = s[t - k - d + 1]
            double pot = 0.0;
            for (uint64_t m = sh & wmask & ~1ull; m; m &= m - 1) pot += h.a_plus[__ffsll(static_cast<long long>(m)) - 2];
            h.pot64[static_cast<int64_t>(i) * h.dp + (d - 1)] = pot;
            h.pot32[static_cast<int64_t>(i) * h.dp + (d - 1)] = static_cast<float>(pot);
            any_pot |= (pot != 0.0);
        }
        if (h.row_plastic[i] && (any_pot || t == 0)) act = true;
    } else if (h.stdp) {
        // dep: bits 1..W
        double dep = 0.0;
        for (int k = 1; k <= h.window; ++k) {
            const int b = k;
            if ((words[b >> 6] >> (b & 63)) & 1ull) dep += h.a_minus[k - 1];
        }
        h.dep64[i] = dep;
        h.dep32[i] = static_cast<float>(dep);
        bool any_pot = false;
        for (int d = 1; d <= h.dp; ++d) {
            double pot = 0.0;
            for (int k = 1; k <= h.window; ++k) {
                const int b = k + d - 1;
                if ((words[b >> 6] >> (b & 63)) & 1ull) pot += h.a_plus[k - 1];
            }
            h.pot64[static_cast<int64_t>(i) * h.dp + (d - 1)] = pot;
            h.pot32[static_cast<int64_t>(i) * h.dp + (d - 1)] = static_cast<float>(pot);
            any_pot |= (pot != 0.0);
        }
        // t == 0: apply_stdp clamps every plastic weight even when dw == 0
        // (mat_engine.cpp:243-249); afterwards weights stay inside the bounds,
        // so rows with no pairing and no delivery are provably unchanged.
        if (h.row_plastic[i] && (any_pot || t == 0)) act = true;
    }
    return act;
}

// ---------------------------------------------------------------------------
// K1: LIF update of the local posts for step t (mat_engine.cpp:168-198).
// Called by full warps (j covers a multiple of 32); one neuron per thread.
template <bool EXACT, bool FUSED>
__device__ __forceinline__ void neuron_step(const NeuronArgs& a, const HistArgs& h, int j, int t) {
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
            // fixed tree; 16 loads are issued before any add so a step's partials
            // arrive in a few memory round trips
            double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            int c = 0;
            for (; c + 16 <= a.nchunks; c += 16) {
                double t[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) t[k] = __ldcg(a.partial + static_cast<int64_t>(c + k) * a.nl + j);
#pragma unroll
                for (int k = 0; k < 16; ++k) acc[k & 7] += t[k];
            }
            for (; c + 8 <= a.nchunks; c += 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] += __ldcg(a.partial + static_cast<int64_t>(c + k) * a.nl + j);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)  // remainder; unrolled so acc stays in registers
                if (c + k < a.nchunks) acc[k] += __ldcg(a.partial + static_cast<int64_t>(c + k) * a.nl + j);
            const double in = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
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
        if (a.peer_bits)  // fused all-gather: store the word into every peer's bitmask (NVLink)
            for (int q = 0; q < a.world; ++q)
                if (q != a.rank) a.peer_bits[q][(a.first >> 5) + wi] = word;
        if (a.raster && (t - a.t_base) < a.raster_rows)
            a.raster[static_cast<int64_t>(t - a.t_base) * a.nl_words + wi] = word;
        if (word) atomicAdd(a.spike_count, static_cast<unsigned long long>(__popc(word)));
    }
    if (FUSED) {
        bool act = false;
        if (valid) act = hist_update(h, j, s, t);
        const uint32_t aw = __ballot_sync(0xffffffffu, act);
        if (lane == 0 && wi < a.nl_words) {
            h.active[wi] = aw;
            if (aw) atomicAdd(h.active_count, static_cast<unsigned long long>(__popc(aw)));
        }
    }
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

template <bool EXACT, bool FUSED>
__global__ void __launch_bounds__(kThreads) k_neuron(NeuronArgs a, HistArgs h) {
    const int t = *a.d_step;
    neuron_step<EXACT, FUSED>(a, h, blockIdx.x * kThreads + threadIdx.x, t);
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
    if (i < h.n) {
        const bool s = (h.bits[i >> 5] >> (i & 31)) & 1u;
        act = hist_update(h, i, s, t);
    }
    const uint32_t aw = __ballot_sync(0xffffffffu, act);
    if ((threadIdx.x & 31) == 0 && (i >> 5) < ((h.n + 31) >> 5)) {
        h.active[i >> 5] = aw;
        if (aw) atomicAdd(h.active_count, static_cast<unsigned long long>(__popc(aw)));
    }
}

__global__ void k_prologue(double* u, const double* v, const double* leak, const double* reset,
                           int nl, int abm) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nl) u[j] = abm ? 0.0 : leak_toward(v[j], leak[j], reset[j]);
}

__global__ void k_step_bump(int32_t* d_step) { *d_step += 1; }

// ---------------------------------------------------------------------------
// Dense sweep: W[pre][post] row-major (pre-major like mat_engine.cpp:34-38),
// column tiles x row chunks.  For each active row i (ascending) and each of the
// thread's VEC local columns j:
//   plastic: w' = clamp(w + s_j[t] pot_i^(d) - e_ij dep_j, w_min, w_max)
//   e_ij = s_i[t+1-d_ij] (history bit d-1): input to post j at step t+1
//   acc_j += e_ij * w'
// Non-exact: per-thread fp32 group sums of U rows promoted to fp64, partials
// per row chunk summed by k_neuron in chunk order (deterministic; exact for
// integer nets).  Exact: one chunk, fp64 accumulator seeded with leak(v_j)
// and rows added in ascending order exactly as mat_step does.
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

template <typename WT, bool STDP, bool DELAY, bool EXACT>
__global__ void __launch_bounds__(kThreads) k_dense_sweep(DenseArgs a) {
    using VT = VecT<WT>;
    using V = typename VT::V;
    constexpr int VEC = VT::N;
    constexpr int U = 8;  // rows in flight per thread

    __shared__ int32_t s_rows[kSubRows];
    __shared__ uint64_t s_e[kSubRows];
    __shared__ WT s_pot[STDP && !DELAY ? kSubRows : 1];
    __shared__ uint8_t s_kind[kSubRows];
    __shared__ uint32_t s_word[32];
    __shared__ int32_t s_wpref[33];

    const int tid = threadIdx.x;
    const int ntiles = (a.nl + a.tile_w - 1) / a.tile_w;
    const int items = ntiles * a.nchunks;
    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const WT* pot = static_cast<const WT*>(a.pot);
    const WT* dep = static_cast<const WT*>(a.dep);
    WT* W = static_cast<WT*>(a.w);
    const uint64_t dmask = DELAY ? ~0ull : 1ull;

    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int chunk = item / ntiles;
        const int tile = item - chunk * ntiles;
        const int tcol = tid * VEC;
        const int c0 = tile * a.tile_w + tcol;
        const bool in_tile = tcol < a.tile_w && c0 < a.nl;
        const int r0 = chunk * a.rows_per_chunk;
        const int r1 = min(a.n, r0 + a.rows_per_chunk);

        bool sj[VEC];
        WT depj[VEC];
        int gc[VEC];
        double acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            gc[k] = a.first + c0 + k;
            const bool ok = in_tile && (c0 + k) < a.nl;
            sj[k] = ok && STDP ? bit_of(a.bits, gc[k]) : false;
            depj[k] = ok && STDP ? dep[gc[k]] : WT(0);
            acc[k] = (EXACT && ok && !a.abm) ? leak_toward(a.v[c0 + k], a.leak[c0 + k], a.reset[c0 + k]) : 0.0;
        }

        for (int sa = r0; sa < r1; sa += kSubRows) {
            const int sb = min(r1, sa + kSubRows);
            const int nwords = (sb - sa + 31) >> 5;
            __syncthreads();  // previous sub-chunk fully consumed
            if (tid < 32) {
                uint32_t wd = 0;
                if (tid < nwords) {
                    wd = __ldcg(a.active + (sa >> 5) + tid);
                    const int rem = sb - (sa + tid * 32);
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
                const int l = (r - sa) >> 5, b = (r - sa) & 31;
                const uint32_t wd = s_word[l];
                if ((wd >> b) & 1u) {
                    const int pos = s_wpref[l] + __popc(wd & ((1u << b) - 1u));
                    s_rows[pos] = r;
                    s_e[pos] = __ldg(a.hist + r) & dmask;
                    if (STDP) s_kind[pos] = __ldg(a.kind + r);
                    if (STDP && !DELAY) s_pot[pos] = pot[r];
                }
            }
            __syncthreads();
            const int cnt = s_wpref[32];

            for (int gb = 0; gb < cnt; gb += U) {
                V wv[U];
                uint32_t dv[U];
                uint32_t mv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = gb + u;
                    dv[u] = 0x01010101u;
                    mv[u] = 0;
                    if (idx < cnt && in_tile) {
                        const int row = s_rows[idx];
                        const int64_t off = static_cast<int64_t>(row) * a.pitch + c0;
                        wv[u] = VT::load(W + off);
                        if (DELAY) {
                            if (VEC == 4) dv[u] = __ldg(reinterpret_cast<const uint32_t*>(a.delay + off));
                            else dv[u] = __ldg(reinterpret_cast<const uint16_t*>(a.delay + off));
                        }
                        if (STDP && s_kind[idx] == kRowMixed)
                            mv[u] = __ldg(a.mask + static_cast<int64_t>(row) * (a.pitch >> 5) + (c0 >> 5)) >> (c0 & 31);
                    } else {
#pragma unroll
                        for (int k = 0; k < VEC; ++k) VT::set(wv[u], k, WT(0));
                    }
                }
                WT grp[VEC];
#pragma unroll
                for (int k = 0; k < VEC; ++k) grp[k] = WT(0);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = gb + u;
                    if (idx >= cnt || !in_tile) continue;
                    const int row = s_rows[idx];
                    const uint64_t ebits = s_e[idx];
                    bool changed = false;
                    uint8_t kind = STDP ? s_kind[idx] : uint8_t(kRowNone);
#pragma unroll
                    for (int k = 0; k < VEC; ++k) {
                        WT w = VT::get(wv[u], k);
                        const int d1 = DELAY ? static_cast<int>((dv[u] >> (8 * k)) & 0xffu) - 1 : 0;
                        const bool e = (ebits >> d1) & 1ull;
                        if (STDP && kind != kRowNone) {
                            const bool pl = kind == kRowAll || (kind == kRowAllButSelf && gc[k] != row) ||
                                            (kind == kRowMixed && ((mv[u] >> k) & 1u));
                            if (pl) {
                                const WT p = DELAY ? pot[static_cast<int64_t>(row) * a.dp + d1] : s_pot[idx];
                                // dw = 0; if s_post: dw += pot; if s_pre: dw -= dep (243-246)
                                WT dw = WT(0);
                                if (sj[k]) dw += p;
                                if (e) dw -= depj[k];
                                const WT nw = clamp_ref<WT>(w + dw, wmin, wmax);
                                changed |= (nw != w);
                                w = nw;
                                VT::set(wv[u], k, nw);
                            }
                        }
                        if (e) {
                            if (EXACT) acc[k] += static_cast<double>(w);
                            else grp[k] += w;
                        }
                    }
                    if (STDP && changed) {
                        VT::store(W + static_cast<int64_t>(row) * a.pitch + c0, wv[u]);
                    }
                }
                if (!EXACT) {
#pragma unroll
                    for (int k = 0; k < VEC; ++k) acc[k] += static_cast<double>(grp[k]);
                }
            }
        }
        if (in_tile) {
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                if (c0 + k < a.nl) {
                    if (EXACT) a.u_exact[c0 + k] = acc[k];
                    else a.partial[static_cast<int64_t>(chunk) * a.nl + c0 + k] = acc[k];
                }
            }
        }
    }
    if (blockIdx.x == 0 && tid == 0) *a.d_step += 1;  // no other CTA reads it
}

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
    __shared__ RowRec<WT> s_rec[kSubRows + U];
    __shared__ uint32_t s_word[32];
    __shared__ int32_t s_wpref[33];

    const int tid = threadIdx.x;
    const int ntiles = (a.nl + a.tile_w - 1) / a.tile_w;
    const int items = ntiles * a.nchunks;
    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const WT* pot = static_cast<const WT*>(a.pot);
    const WT* dep = static_cast<const WT*>(a.dep);
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

        WT sjf[VEC], depj[VEC];
        double acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const bool ok = in_tile && (c0 + k) < a.nl;
            sjf[k] = (ok && STDP && bit_of(a.bits, gc0 + k)) ? WT(1) : WT(0);
            depj[k] = (ok && STDP) ? __ldcg(dep + gc0 + k) : WT(0);
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
                    RowRec<WT> rec;
                    const int kind = STDP ? static_cast<int>(__ldg(a.kind + r)) : 0;
                    rec.rowk = r | (kind << 28);
                    rec.e_lo = static_cast<uint32_t>(h);
                    rec.e_hi = static_cast<uint32_t>(h >> 32);
                    rec.pot = (STDP && !DELAY) ? __ldcg(pot + r) : WT(0);
                    s_rec[pos] = rec;
                }
            }
            const int cnt = s_wpref[32];
            if (tid < U && cnt > 0) {  // inert padding: re-reads row sa, no spike, no store
                RowRec<WT> rec;
                rec.rowk = sa;
                rec.e_lo = rec.e_hi = 0;
                rec.pot = WT(0);
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
                    const RowRec<WT> rec = s_rec[gb + u];
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
                    if (STDP && kind != kRowNone) {
                        WT nw[VEC];
#pragma unroll
                        for (int k = 0; k < VEC; ++k) {
                            WT p;
                            if (DELAY) {
                                const int d1 = static_cast<int>((dv[u] >> (8 * k)) & 0xffu) - 1;
                                p = __ldcg(pot + static_cast<int64_t>(row) * a.dp + d1);
                            } else {
                                p = rec.pot;
                            }
                            // dw = s_post*pot - s_pre*dep (mat_engine.cpp:243-246); 0/1 factors are exact
                            const WT dw = fma(sjf[k], p, -(ef[k] * depj[k]));
                            nw[k] = clamp_ref<WT>(w[k] + dw, wmin, wmax);
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

template <typename WT, bool STDP, bool DELAY>
__global__ void __launch_bounds__(kThreads, 2) k_dense_stream(DenseArgs a) {
    dense_stream_body<WT, STDP, DELAY>(a, blockIdx.x, gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_step += 1;  // no other CTA reads it
}

// ---------------------------------------------------------------------------
// TMA-staged dense sweep (fp32, unit delays): one CTA per SM, a producer warp
// streams the active rows' tile segments into a kTmaStages-deep shared-memory
// ring with cp.async.bulk (completion on mbarriers), 8 consumer warps apply
// the same per-element update as k_dense_stream from shared memory and write
// the new weights with 128-bit streaming stores.  Loads never occupy
// registers, so the in-flight window per SM is the whole ring.
constexpr int kTmaRows = 4;        // rows per stage
constexpr int kTmaStages = 8;      // ring depth
constexpr int kTmaListMax = 2048;  // rows per item (one list build per item)
constexpr int kTmaThreads = 288;   // 8 consumer warps + 1 producer warp

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
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <bool STDP>
__global__ void __launch_bounds__(kTmaThreads, 1) k_dense_tma(DenseArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool producer = warp == 8;
    const int ntiles = (a.nl + a.tile_w - 1) / a.tile_w;
    const int items = ntiles * a.nchunks;
    const uint32_t row_bytes = static_cast<uint32_t>(a.tile_w) * 4u;
    const size_t stage_bytes = static_cast<size_t>(kTmaRows) * row_bytes;
    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTmaStages * stage_bytes);
    uint64_t* empty = full + kTmaStages;
    RowRec<float>* s_rec = reinterpret_cast<RowRec<float>*>(empty + kTmaStages);
    __shared__ uint32_t s_word[32];
    __shared__ int32_t s_wpref[33];
    __shared__ int32_t s_cnt;
    __shared__ int s_item;

    const float wmin = static_cast<float>(a.w_min), wmax = static_cast<float>(a.w_max);
    const float* dep = static_cast<const float*>(a.dep);
    const float* pot = static_cast<const float*>(a.pot);
    float* W = static_cast<float*>(a.w);

    if (tid == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t it = 0;  // ring position, advanced identically by producer and consumers
    int item = blockIdx.x;
    if (a.work) {
        if (tid == 0) s_item = atomicAdd(a.work, 1);
        __syncthreads();
        item = s_item;
    }
    while (item < items) {
        const int chunk = item / ntiles;
        const int tile = item - chunk * ntiles;
        const int col0 = tile * a.tile_w;
        const int width = static_cast<int>(min(static_cast<int64_t>(a.tile_w), a.pitch - col0));
        const uint32_t copy_bytes = static_cast<uint32_t>(width) * 4u;
        const int r0 = chunk * a.rows_per_chunk;
        const int r1 = min(a.n, r0 + a.rows_per_chunk);

        // active-row list of [r0, r1) in <= 1024-row pieces (32-aligned bases)
        if (tid == 0) s_cnt = 0;
        __syncthreads();
        for (int sa = r0, sb_next = r0; sa < r1; sa = sb_next) {
            const int base = sa & ~31;
            const int sb = min(r1, base + kSubRows);
            sb_next = sb;
            const int nwords = (sb - base + 31) >> 5;
            const int cnt0 = s_cnt;
            if (tid < 32) {
                uint32_t wd = 0;
                if (tid < nwords) {
                    wd = __ldcg(a.active + (base >> 5) + tid);
                    const int lo = sa - (base + tid * 32);
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
                s_wpref[tid] = cnt0 + incl - c;
                if (tid == 31) s_wpref[32] = cnt0 + incl;
            }
            __syncthreads();
            for (int r = sa + tid; r < sb; r += kTmaThreads) {
                const int l = (r - base) >> 5, b = (r - base) & 31;
                const uint32_t wd = s_word[l];
                if ((wd >> b) & 1u) {
                    const int pos = s_wpref[l] + __popc(wd & ((1u << b) - 1u));
                    const uint64_t h = __ldcg(a.hist + r);
                    RowRec<float> rec;
                    const int kind = STDP ? static_cast<int>(__ldg(a.kind + r)) : 0;
                    rec.rowk = r | (kind << 28);
                    rec.e_lo = static_cast<uint32_t>(h);
                    rec.e_hi = static_cast<uint32_t>(h >> 32);
                    rec.pot = STDP ? __ldcg(pot + r) : 0.f;
                    s_rec[pos] = rec;
                }
            }
            __syncthreads();
            if (tid == 0) s_cnt = s_wpref[32];
            __syncthreads();
        }
        const int cnt = s_cnt;
        const int ngroups = (cnt + kTmaRows - 1) / kTmaRows;

        if (producer) {
            if (lane == 0) {
                for (int g = 0; g < ngroups; ++g, ++it) {
                    const int s = it % kTmaStages;
                    const uint32_t ph = (it / kTmaStages) & 1u;
                    mbar_wait(empty + s, ph ^ 1u);
                    const int nr = min(kTmaRows, cnt - g * kTmaRows);
                    mbar_arrive_expect_tx(full + s, static_cast<uint32_t>(nr) * copy_bytes);
                    for (int r = 0; r < nr; ++r) {
                        const int row = s_rec[g * kTmaRows + r].rowk & 0x0fffffff;
                        bulk_g2s(reinterpret_cast<uint8_t*>(ring) + s * stage_bytes + static_cast<size_t>(r) * row_bytes,
                                 W + static_cast<int64_t>(row) * a.pitch + col0, copy_bytes, full + s);
                    }
                }
            } else {
                it += ngroups;
            }
        } else {
            const int tcol = tid * 4;
            const int c0 = col0 + tcol;
            const bool in_tile = tcol < width && c0 < a.nl;
            const int gc0 = a.first + c0;
            float sjf[4], depj[4];
            double acc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool ok = in_tile && (c0 + k) < a.nl;
                sjf[k] = (ok && STDP && bit_of(a.bits, gc0 + k)) ? 1.f : 0.f;
                depj[k] = (ok && STDP) ? __ldcg(dep + gc0 + k) : 0.f;
                acc[k] = 0.0;
            }
            for (int g = 0; g < ngroups; ++g, ++it) {
                const int s = it % kTmaStages;
                const uint32_t ph = (it / kTmaStages) & 1u;
                mbar_wait(full + s, ph);
                const int nr = min(kTmaRows, cnt - g * kTmaRows);
                float grp[4] = {0.f, 0.f, 0.f, 0.f};
                if (in_tile) {
#pragma unroll
                    for (int r = 0; r < kTmaRows; ++r) {
                        if (r >= nr) break;
                        const RowRec<float> rec = s_rec[g * kTmaRows + r];
                        const int row = rec.rowk & 0x0fffffff;
                        const int kind = rec.rowk >> 28;
                        const float4 wv = *reinterpret_cast<const float4*>(
                            reinterpret_cast<const uint8_t*>(ring) + s * stage_bytes + static_cast<size_t>(r) * row_bytes + tcol * 4);
                        float w[4] = {wv.x, wv.y, wv.z, wv.w};
                        const float ef = (rec.e_lo & 1u) ? 1.f : 0.f;
                        if (STDP && kind != kRowNone) {
                            float nw[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float dw = fmaf(sjf[k], rec.pot, -(ef * depj[k]));
                                nw[k] = clamp_ref<float>(w[k] + dw, wmin, wmax);
                            }
                            if (kind == kRowAllButSelf) {
                                const int selfk = row - gc0;
#pragma unroll
                                for (int k = 0; k < 4; ++k) nw[k] = (selfk == k) ? w[k] : nw[k];
                            } else if (kind == kRowMixed) {
                                const uint32_t mv =
                                    __ldg(a.mask + static_cast<int64_t>(row) * (a.pitch >> 5) + (c0 >> 5)) >> (c0 & 31);
#pragma unroll
                                for (int k = 0; k < 4; ++k) nw[k] = ((mv >> k) & 1u) ? nw[k] : w[k];
                            }
                            __stcs(reinterpret_cast<float4*>(W + static_cast<int64_t>(row) * a.pitch + c0),
                                   make_float4(nw[0], nw[1], nw[2], nw[3]));
#pragma unroll
                            for (int k = 0; k < 4; ++k) w[k] = nw[k];
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k) grp[k] = fmaf(ef, w[k], grp[k]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[k] += static_cast<double>(grp[k]);
            }
            if (in_tile) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.nl) a.partial[static_cast<int64_t>(chunk) * a.nl + c0 + k] = acc[k];
            }
        }
        __syncthreads();  // ring drained for this item's rows; list may be rebuilt
        if (a.work) {
            if (tid == 0) s_item = atomicAdd(a.work, 1);
            __syncthreads();
            item = s_item;
        } else {
            item += gridDim.x;
        }
    }
    if (blockIdx.x == 0 && tid == 0) *a.d_step += 1;
}

size_t dense_tma_smem(int tile_w) {
    return static_cast<size_t>(kTmaStages) * kTmaRows * tile_w * 4 + 2 * kTmaStages * 8 +
           static_cast<size_t>(kTmaListMax + kTmaRows) * sizeof(RowRec<float>);
}

// ---------------------------------------------------------------------------
// Tiny nets: one CTA runs the whole call with every array in shared memory.
// Per step: (1) thread j integrates post j -- leak, its incoming list in
// ascending pre order (history bit d-1 of the pre = s_pre[t-d]), the step's
// stimulus, threshold/refractory/reset; (2) history shift, raster word (warp
// ballot), STDP traces; (3) thread j applies STDP to its own plastic synapses
// (mat_engine.cpp:242-249, every plastic synapse every step).  One CTA barrier
// per step (double-buffered history), no global memory on the critical path.
struct TinyLayout {
    size_t hist, pot, dep, off, meta, pidx, w, st_off, st_neuron, st_amp, ap, am, total;
};

__host__ __device__ inline size_t tiny_align(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

// Shared memory: history as 32-bit words, double-buffered (buffer b, word k,
// neuron j at [(b * 2hw + k) * np + j]) so one barrier per step separates the
// readers of step t from the writers of step t+1; STDP traces double-buffered
// the same way.  Per-neuron LIF state lives in the owning thread's registers.
__host__ __device__ inline TinyLayout tiny_layout(const TinyArgs& a) {
    TinyLayout L{};
    const size_t np = static_cast<size_t>((a.n + 31) / 32 * 32);
    size_t o = 0;
    L.hist = o; o = tiny_align(o + 2 * np * 8 * a.hw);
    L.pot = o; o = tiny_align(o + (a.stdp ? 2 * np * 8 * a.dp : 0));
    L.dep = o; o = tiny_align(o + (a.stdp ? 2 * np * 8 : 0));
    L.off = o; o = tiny_align(o + (static_cast<size_t>(a.n) + 1) * 4);
    L.meta = o; o = tiny_align(o + static_cast<size_t>(a.m) * 4);
    L.pidx = o; o = tiny_align(o + (a.stdp ? static_cast<size_t>(a.m) * 2 : 0));
    // weights in smem: as stored for STDP nets (the update runs in WT), as
    // double otherwise (no per-synapse conversion on the integration path)
    L.w = o; o = tiny_align(o + static_cast<size_t>(a.m) * ((a.f64 || !a.stdp) ? 8 : 4));
    L.st_off = o; o = tiny_align(o + (static_cast<size_t>(a.steps) + 1) * 4);
    L.st_neuron = o; o = tiny_align(o + static_cast<size_t>(a.st_count) * 4);
    L.st_amp = o; o = tiny_align(o + static_cast<size_t>(a.st_count) * 8);
    L.ap = o; o = tiny_align(o + (a.stdp ? static_cast<size_t>(a.window) * 8 : 0));
    L.am = o; o = tiny_align(o + (a.stdp ? static_cast<size_t>(a.window) * 8 : 0));
    L.total = o;
    return L;
}

// Bit test of one incoming synapse: meta = byte offset of the 32-bit history
// word within a buffer << 5 | bit; the funnel shift uses the low 5 bits.
__device__ __forceinline__ bool tiny_bit(const uint8_t* buf, uint32_t mq) {
    const uint32_t word = *reinterpret_cast<const uint32_t*>(buf + (mq >> 5));
    return __funnelshift_r(word, word, mq) & 1u;
}

template <typename WT, bool STDP>
__global__ void __launch_bounds__(1024, 1) k_tiny(TinyArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    const TinyLayout L = tiny_layout(a);
    const int tid = threadIdx.x;
    const int n = a.n;
    const int np = (n + 31) / 32 * 32;
    const int hw2 = 2 * a.hw;
    const size_t hbuf = static_cast<size_t>(hw2) * np * 4;  // bytes per history buffer
    uint32_t* hist = reinterpret_cast<uint32_t*>(sm + L.hist);
    double* pot = reinterpret_cast<double*>(sm + L.pot);
    double* dep = reinterpret_cast<double*>(sm + L.dep);
    uint32_t* off = reinterpret_cast<uint32_t*>(sm + L.off);
    uint32_t* meta = reinterpret_cast<uint32_t*>(sm + L.meta);
    uint16_t* pidx = reinterpret_cast<uint16_t*>(sm + L.pidx);
    using WS = typename std::conditional<STDP, WT, double>::type;  // smem weight type
    WS* w = reinterpret_cast<WS*>(sm + L.w);
    int32_t* st_off = reinterpret_cast<int32_t*>(sm + L.st_off);
    int32_t* st_neuron = reinterpret_cast<int32_t*>(sm + L.st_neuron);
    double* st_amp = reinterpret_cast<double*>(sm + L.st_amp);
    double* ap = reinterpret_cast<double*>(sm + L.ap);
    double* am = reinterpret_cast<double*>(sm + L.am);
    // ---- load: owned neuron state into registers, shared arrays ----
    const int j = tid;
    const bool own = j < n;
    double v = own ? a.v[j] : 0.0;
    const double thr = own ? a.thr[j] : 0.0;
    const double leak = own ? a.leak[j] : 0.0;
    const double rst = own ? a.reset[j] : 0.0;
    const int32_t refr = own ? a.refr[j] : 0;
    int32_t cnt = own ? a.cnt[j] : 0;
    const double fire_p = (own && a.fire_p) ? a.fire_p[j] : 1.0;
    const uint64_t akey = fire_p < 1.0 ? a.agent_key[j] : 0ull;
    for (int k = 0; k < a.hw; ++k) {
        const uint64_t x = own ? a.hist[static_cast<int64_t>(k) * n + j] : 0ull;
        hist[(2 * k) * np + j] = static_cast<uint32_t>(x);
        hist[(2 * k + 1) * np + j] = static_cast<uint32_t>(x >> 32);
    }
    const int nt = blockDim.x;
    for (int i = tid; i <= n; i += nt) off[i] = a.off[i];
    for (int q = tid; q < a.m; q += nt) {
        meta[q] = a.meta[q];
        w[q] = static_cast<WS>(static_cast<const WT*>(a.w)[q]);
        if (STDP) pidx[q] = a.pidx[q];
    }
    const int64_t sbase = a.st_rows > 0 ? a.st_off[0] : 0;
    for (int s = tid; s <= a.steps; s += nt)
        st_off[s] = a.st_rows > 0 ? static_cast<int32_t>(a.st_off[min(s, a.st_rows)] - sbase) : 0;
    for (int e = tid; e < a.st_count; e += nt) {
        st_neuron[e] = a.st_neuron[sbase + e];
        st_amp[e] = a.st_amp[sbase + e];
    }
    if (STDP)
        for (int k = tid; k < a.window; k += nt) {
            ap[k] = a.a_plus[k];
            am[k] = a.a_minus[k];
        }
    __syncthreads();
    const int t0 = *a.d_step;
    const int words = (n + 31) / 32;
    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const uint32_t q0 = own ? off[j] : 0u, q1 = own ? off[j + 1] : 0u;
    unsigned long long spikes = 0;
    for (int s = 0; s < a.steps; ++s) {
        const int cur = s & 1;
        const uint8_t* hc = sm + L.hist + cur * hbuf;        // history through t-1
        uint32_t* hn = reinterpret_cast<uint32_t*>(sm + L.hist + (cur ^ 1) * hbuf);  // through t
        bool fired = false;
        if (own) {
            // (1) leak, incoming list in ascending pre order (bit d-1 = s_pre[t-d]),
            // the step's stimulus, threshold, refractory (mat_engine.cpp:160-198)
            // MAT: u = leak(v) + w...; ABM: pending = 0.0 + w..., u = leak(v) + (pending + ext)
            double u = a.abm ? 0.0 : leak_toward(v, leak, rst);
#pragma unroll 4
            for (uint32_t q = q0; q < q1; ++q) {
                const uint32_t mq = meta[q];
                if (tiny_bit(hc, mq)) u += static_cast<double>(w[q]);  // WS = double unless STDP
            }
            int lo = st_off[s], hi = st_off[s + 1];
            if (hi > lo) {
                double ext = 0.0;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const int nm = st_neuron[mid];
                    if (nm == j) { ext = st_amp[mid]; break; }
                    if (nm < j) lo = mid + 1; else hi = mid;
                }
                u += ext;
            }
            if (a.abm) u = leak_toward(v, leak, rst) + u;
            fired = u > thr;
            if (fired && fire_p < 1.0) fired = agent_fires(akey, t0 + s, fire_p);
            if (cnt > 0) {
                fired = false;
                cnt -= 1;
                u = rst;
            }
            if (fired) {
                v = rst;
                cnt = refr;
            } else {
                v = u;
            }
            if (a.trace) a.trace[static_cast<int64_t>(s) * n + j] = v;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, fired);
        if ((tid & 31) == 0 && (tid >> 5) < words) {
            a.raster[static_cast<int64_t>(s) * words + (tid >> 5)] = word;
            spikes += __popc(word);
        }
        // (2) own history row into the other buffer (+ own STDP traces)
        if (j < np) {
            const uint32_t* hcw = reinterpret_cast<const uint32_t*>(hc);
            uint32_t carry = fired ? 1u : 0u;
            for (int k = 0; k < hw2; ++k) {
                const uint32_t x = hcw[k * np + j];
                hn[k * np + j] = (x << 1) | carry;
                carry = x >> 31;
            }
            if (STDP && own) {
                double* potn = pot + (cur ^ 1) * np * a.dp;
                double dsum = 0.0;
                for (int k = 1; k <= a.window; ++k)
                    if ((hn[(k >> 5) * np + j] >> (k & 31)) & 1u) dsum += am[k - 1];
                dep[(cur ^ 1) * np + j] = dsum;
                for (int d = 1; d <= a.dp; ++d) {
                    double psum = 0.0;
                    for (int k = 1; k <= a.window; ++k) {
                        const int b = k + d - 1;
                        if ((hn[(b >> 5) * np + j] >> (b & 31)) & 1u) psum += ap[k - 1];
                    }
                    potn[j * a.dp + (d - 1)] = psum;
                }
            }
        }
        __syncthreads();  // the new history (and traces) of step t are complete
        if (STDP && own) {
            // (3) STDP on post j's plastic synapses: dw = 0; if s_post dw += pot^(d)_pre;
            // if s_pre[t-d+1] dw -= dep_post; clamp (mat_engine.cpp:242-249)
            const uint8_t* hnb = reinterpret_cast<const uint8_t*>(hn);
            const double* potn = pot + (cur ^ 1) * np * a.dp;
            const double depj = dep[(cur ^ 1) * np + j];
            for (uint32_t q = q0; q < q1; ++q) {
                const uint16_t pq = pidx[q];
                if (pq == 0xffffu) continue;  // not plastic
                const uint32_t mq = meta[q];
                WT dw = WT(0);
                if (fired) dw += static_cast<WT>(potn[pq]);
                if (tiny_bit(hnb, mq)) dw -= static_cast<WT>(depj);
                w[q] = clamp_ref<WT>(w[q] + dw, wmin, wmax);
            }
        }
    }
    // ---- write back (the last step's history is in buffer steps & 1) ----
    const uint32_t* hl = reinterpret_cast<const uint32_t*>(sm + L.hist + (a.steps & 1) * hbuf);
    if (own) {
        a.v[j] = v;
        a.cnt[j] = cnt;
        for (int k = 0; k < a.hw; ++k)
            a.hist[static_cast<int64_t>(k) * n + j] =
                static_cast<uint64_t>(hl[(2 * k) * np + j]) | (static_cast<uint64_t>(hl[(2 * k + 1) * np + j]) << 32);
    }
    if (STDP) {
        __syncthreads();  // every owner's last-step weight update is done
        for (int q = tid; q < a.m; q += nt) static_cast<WT*>(a.w)[q] = static_cast<WT>(w[q]);
    }
    if (spikes) atomicAdd(a.spike_count, spikes);
    if (tid == 0) *a.d_step = t0 + a.steps;
}

// Persistent single-GPU step loop for small dense nets (launch-latency bound
// otherwise): one cooperative launch runs `steps` steps; neuron phase and
// sweep phase are separated by grid-wide barriers (cooperative groups).
template <typename WT, bool STDP, bool DELAY>
__global__ void __launch_bounds__(kThreads, 2) k_persistent_dense(NeuronArgs na, HistArgs h, DenseArgs da,
                                                                 int steps) {
    cg::grid_group grid = cg::this_grid();
    const bool single = gridDim.x == 1;
    int t = *na.d_step;
    const int span = ((na.nl + 31) / 32) * 32;
    for (int s = 0; s < steps; ++s, ++t) {
        for (int j = blockIdx.x * kThreads + threadIdx.x; j - static_cast<int>(threadIdx.x & 31) < span;
             j += gridDim.x * kThreads)
            neuron_step<false, true>(na, h, j, t);
        if (single) __syncthreads(); else grid.sync();
        dense_stream_body<WT, STDP, DELAY>(da, blockIdx.x, gridDim.x);
        if (single) __syncthreads(); else grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *na.d_step = t;
}

// ---------------------------------------------------------------------------
// Column-owner persistent loop: CTA c owns posts [W c, W c + W), W = 8 (the
// net must be small enough for every group to be co-resident).  Per step
// (1) warp 0 updates its 8 posts from the input its own sweep produced (LIF as
// neuron_step, history word, STDP traces, row activity) into the step's
// parity buffers; (2) one grid barrier; (3) 1024 threads sweep every active row
// of the CTA's 8 columns -- STDP of step t, then the delivery of step t + 1 --
// and reduce the row-lane partials in a fixed tree.  Groups share 32-bit
// words, so activity and raster words are OR-ed in (activity words
// triple-buffered: the buffer of step t + 2 is cleared during step t's sweep,
// after every reader of its previous use passed the barrier).  Used when the
// history fits one word.
constexpr int kColThreads = 1024;

template <typename WT, bool STDP, bool DELAY, int kColW>
__global__ void __launch_bounds__(kColThreads) k_persistent_cols(NeuronArgs na, DenseArgs da, ColArgs ca, int steps) {
    cg::grid_group grid = cg::this_grid();
    using VT = VecT<WT>;
    using V = typename VT::V;
    constexpr int VEC = VT::N;
    constexpr int CV = kColW / VEC;          // column vectors per CTA
    constexpr int RL = kColThreads / CV;     // row lanes
    __shared__ double s_red[RL][kColW + 1];
    __shared__ WT s_dep[kColW];
    __shared__ uint32_t s_spk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int j = c * kColW + lane;          // warp 0, lanes < 8: this lane's post
    const bool own = warp == 0 && lane < kColW && j < na.nl;
    const int cv = tid % CV, rl = tid / CV;
    const int j0 = c * kColW + cv * VEC;
    const int n = da.n;
    const int words = (n + 31) >> 5;
    const int64_t pitch = da.pitch, mpitch = pitch >> 5;
    const WT wmin = static_cast<WT>(da.w_min), wmax = static_cast<WT>(da.w_max);
    WT* W = static_cast<WT*>(da.w);
    WT* pot2 = static_cast<WT*>(ca.pot2);
    const uint64_t dmask = ca.dmax >= 64 ? ~0ull : ((1ull << ca.dmax) - 1ull);
    const uint64_t wmask = ca.window >= 63 ? ~0ull : ((1ull << (ca.window + 1)) - 1ull);
    double in = own ? na.partial[j] : 0.0;   // input of the call's first step
    int t = *na.d_step;
    // the owned neurons' state and parameters stay in warp 0's registers for
    // the whole call; only what other CTAs read goes through global memory
    double v = 0.0, thr = 0.0, leak = 0.0, rst = 0.0, fire_p = 1.0;
    int32_t cnt = 0, refr = 0;
    uint64_t hprev = 0, akey = 0;
    if (own) {
        v = na.v[j];
        thr = na.thr[j];
        leak = na.leak[j];
        rst = na.reset[j];
        cnt = na.cnt[j];
        refr = na.refr[j];
        hprev = ca.hist2[static_cast<int64_t>((t & 1) ^ 1) * n + j];
        if (na.fire_p) {
            fire_p = na.fire_p[j];
            akey = na.agent_key[j];
        }
    }
    // stimulus rows of the next step, fetched one step ahead
    auto stim_bounds = [&](int tt, int64_t& lo, int64_t& hi) {
        lo = hi = 0;
        const int row = tt - na.st_base;
        if (warp == 0 && row >= 0 && row < na.st_steps) {
            lo = __ldg(na.st_off + row);
            hi = __ldg(na.st_off + row + 1);
        }
    };
    int64_t slo, shi;
    stim_bounds(t, slo, shi);
    for (int s = 0; s < steps; ++s, ++t) {
        const int cur = t & 1;
        uint32_t* act_now = ca.act3 + (t % 3) * words;
        if (warp == 0) {
            bool fired = false, act = false;
            if (own) {
                double u = na.abm ? in : leak_toward(v, leak, rst) + in;
                if (shi > slo) {
                    int64_t lo = slo, hi = shi;
                    double ext = 0.0;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        const int nid = __ldg(na.st_neuron + mid);
                        if (nid == j) { ext = __ldg(na.st_amp + mid); break; }
                        if (nid < j) lo = mid + 1; else hi = mid;
                    }
                    u += ext;
                }
                if (na.abm) u = leak_toward(v, leak, rst) + u;
                fired = u > thr;
                if (fired && fire_p < 1.0) fired = agent_fires(akey, t, fire_p);
                if (cnt > 0) {
                    fired = false;
                    cnt -= 1;
                    u = rst;
                }
                if (fired) {
                    v = rst;
                    cnt = refr;
                } else {
                    v = u;
                }
                if (na.trace && (t - na.t_base) < na.raster_rows)
                    na.trace[static_cast<int64_t>(t - na.t_base) * na.nl + j] = v;
                const uint64_t hn = (hprev << 1) | (fired ? 1ull : 0ull);
                hprev = hn;
                ca.hist2[static_cast<int64_t>(cur) * n + j] = hn;
                act = (hn & dmask) != 0;
                if (STDP) {
                    // set bits in ascending k: the reference's order (mat_engine.cpp:226-240)
                    double dep = 0.0;
                    for (uint64_t m = hn & wmask & ~1ull; m; m &= m - 1) dep += ca.a_minus[__ffsll(static_cast<long long>(m)) - 2];
                    s_dep[lane] = static_cast<WT>(dep);
                    bool any_pot = false;
                    for (int d = 1; d <= da.dp; ++d) {
                        double pot = 0.0;
                        for (uint64_t m = (hn >> (d - 1)) & wmask & ~1ull; m; m &= m - 1)
                            pot += ca.a_plus[__ffsll(static_cast<long long>(m)) - 2];
                        pot2[(static_cast<int64_t>(cur) * n + j) * da.dp + (d - 1)] = static_cast<WT>(pot);
                        any_pot |= pot != 0.0;
                    }
                    if (ca.row_plastic[j] && (any_pot || t == 0)) act = true;
                }
            }
            const uint32_t word = __ballot_sync(0xffffffffu, fired);  // bits 0..W-1
            const uint32_t aw = __ballot_sync(0xffffffffu, act);
            if (lane == 0) {
                const int wi = (c * kColW) >> 5, sh = (c * kColW) & 31;
                if (aw) atomicOr(act_now + wi, aw << sh);
                if (word) {
                    if (na.raster && (t - na.t_base) < na.raster_rows)
                        atomicOr(na.raster + static_cast<int64_t>(t - na.t_base) * na.nl_words + wi, word << sh);
                    atomicAdd(na.spike_count, static_cast<unsigned long long>(__popc(word)));
                }
                s_spk = word;
            }
        }
        grid.sync();
        stim_bounds(t + 1, slo, shi);  // in flight during the sweep
        if (c == 0)  // clear the activity words of step t + 2 (last read by the sweep of step t - 1)
            for (int k = tid; k < words; k += kColThreads) ca.act3[((t + 2) % 3) * words + k] = 0u;
        // sweep of the CTA's columns: STDP of step t, delivery of step t + 1
        const uint32_t spk = s_spk;
        bool okc[VEC];
        WT sj[VEC], dj[VEC];
        double acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            okc[k] = j0 + k < na.nl;
            sj[k] = (STDP && okc[k] && ((spk >> (cv * VEC + k)) & 1u)) ? WT(1) : WT(0);
            dj[k] = STDP ? s_dep[cv * VEC + k] : WT(0);
            acc[k] = 0.0;
        }
        const uint64_t* hist = ca.hist2 + static_cast<int64_t>(cur) * n;
        const WT* potc = pot2 + static_cast<int64_t>(cur) * n * da.dp;
        // every load of a row is issued before its activity bit is tested: the
        // rows of a small net sit in L2 and one round trip per row pair is the
        // cost that matters here
#pragma unroll 2
        for (int i = rl; i < n; i += RL) {
            const uint32_t aword = __ldcg(act_now + (i >> 5));
            const uint64_t eb = __ldcg(hist + i);
            WT* wrow = W + static_cast<int64_t>(i) * pitch + j0;
            V wv = VT::load(wrow);
            uint32_t dv = 0;
            if (DELAY) {
                const uint8_t* dp8 = da.delay + static_cast<int64_t>(i) * pitch + j0;
                dv = VEC == 4 ? *reinterpret_cast<const uint32_t*>(dp8) : *reinterpret_cast<const uint16_t*>(dp8);
            }
            uint8_t kind = kRowNone;
            uint32_t mw = 0;
            if (STDP) {
                kind = da.kind[i];
                if (kind == kRowMixed) mw = da.mask[static_cast<int64_t>(i) * mpitch + (j0 >> 5)];
            }
            if (!((aword >> (i & 31)) & 1u)) continue;
            bool changed = false;
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                if (!okc[k]) continue;
                WT w = VT::get(wv, k);
                const int d1 = DELAY ? static_cast<int>((dv >> (8 * k)) & 0xffu) - 1 : 0;
                const bool e = (eb >> d1) & 1ull;
                if (STDP && kind != kRowNone) {
                    const bool pl = kind == kRowAll || (kind == kRowAllButSelf && j0 + k != i) ||
                                    (kind == kRowMixed && ((mw >> ((j0 & 31) + k)) & 1u));
                    if (pl) {
                        const WT p = __ldcg(potc + static_cast<int64_t>(i) * da.dp + d1);
                        WT dw = WT(0);  // dw = 0; if s_post dw += pot; if s_pre dw -= dep (mat_engine.cpp:243-246)
                        if (sj[k] != WT(0)) dw += p;
                        if (e) dw -= dj[k];
                        const WT nw = clamp_ref<WT>(w + dw, wmin, wmax);
                        changed |= nw != w;
                        w = nw;
                        VT::set(wv, k, nw);
                    }
                }
                if (e) acc[k] += static_cast<double>(w);
            }
            if (STDP && changed) VT::store(wrow, wv);
        }
        // fixed tree: 8-row groups, then 8 groups of 8, then the rest in order
#pragma unroll
        for (int k = 0; k < VEC; ++k) s_red[rl][cv * VEC + k] = acc[k];
        __syncthreads();
        for (int stride = 1; stride < RL; stride *= 8) {
            const int col = tid % kColW, g = tid / kColW;  // RL / 8 groups per level
            const int base = g * 8 * stride;
            if (base < RL) {
                double sum = 0.0;
                for (int r = 0; r < 8 && base + r * stride < RL; ++r) sum += s_red[base + r * stride][col];
                s_red[base][col] = sum;
            }
            __syncthreads();
        }
        if (warp == 0 && lane < kColW) in = s_red[0][lane];
        __syncthreads();
    }
    if (own) {
        da.partial[j] = in;  // (same buffer as na.partial) input of the next call's first step
        na.v[j] = v;
        na.cnt[j] = cnt;
    }
    if (blockIdx.x == 0 && tid == 0) *na.d_step = t;
}

// ---------------------------------------------------------------------------
// Sparse pull: blocked CSC.  CTA (post group, pre block b) stages the spike
// history of the block's pres in shared memory, then SUB lanes per post walk
// the post's incoming list (pre ascending, padded to 4) with 128-bit loads:
//   e = s_pre[t+1-d]  (history bit d-1)    acc += e * w'
// Replaces the CSR branch of WeightMatrix::propagate (mat_engine.cpp:88-92)
// and the oracle's delivery queue (oracle.cpp:91-95) without atomics.
template <int HB> struct HistT { using T = uint64_t; };
template <> struct HistT<16> { using T = uint16_t; };
template <> struct HistT<32> { using T = uint32_t; };

__host__ __device__ inline size_t sp_hist_bytes(int pb, int hbits) {
    return hbits == 1 ? ((static_cast<size_t>(pb) / 32 + 1) * 4 + 15) & ~static_cast<size_t>(15)
                      : ((static_cast<size_t>(pb) + 1) * (hbits / 8) + 15) & ~static_cast<size_t>(15);
}

// Shared-memory image of a pre block's spike history: pcount entries from
// global memory, then zeros up to and including slot pb (the inert padding
// pre of dictionary-encoded lists).  Returns the 16-aligned byte size.
template <int HB>
__device__ __forceinline__ size_t stage_history(const SparseArgs& a, int pre0, int pcount, uint8_t* smem) {
    using HT = typename HistT<HB>::T;
    const int tid = threadIdx.x;
    if (HB == 1) {
        uint32_t* sb = reinterpret_cast<uint32_t*>(smem);
        const int nw = (pcount + 31) >> 5;
        const int nw_all = a.pb / 32 + 1;
        for (int k = tid; k < nw_all; k += blockDim.x) sb[k] = k < nw ? __ldcg(a.bits + (pre0 >> 5) + k) : 0u;
        return (static_cast<size_t>(nw_all) * 4 + 15) & ~static_cast<size_t>(15);
    }
    HT* sh = reinterpret_cast<HT*>(smem);
    for (int k = tid; k <= a.pb; k += blockDim.x) {
        HT v = 0;
        if (k < pcount) v = static_cast<HT>(HB == 64 ? __ldcg(a.hist + pre0 + k) : __ldcg(a.hist_lo + pre0 + k));
        sh[k] = v;
    }
    return (static_cast<size_t>(a.pb + 1) * sizeof(HT) + 15) & ~static_cast<size_t>(15);
}

template <typename WT, bool STDP, int HB, int SUB, bool DICT>
#ifndef SNB_SPARSE_MINB
#define SNB_SPARSE_MINB 4  // <= 64 regs: 4 CTAs/SM (5 spills; cfg4 0.562 ms vs 0.652 unbounded)
#endif
__global__ void __launch_bounds__(kThreads, SNB_SPARSE_MINB) k_sparse_pull(SparseArgs a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    using HT = typename HistT<HB>::T;
    const int b = blockIdx.y;
    const int pre0 = b * a.pb;
    const int pcount = min(a.pb, a.n - pre0);
    const int tid = threadIdx.x;
    const size_t hbytes = stage_history<HB>(a, pre0, pcount, smem_raw);
    // weight dictionary (non-plastic nets with <= 511 distinct weights): the
    // meta word carries the index, so the weight stream disappears (4 B/synapse)
    WT* s_wd = reinterpret_cast<WT*>(smem_raw + hbytes);
    if (DICT)
        for (int k = tid; k < a.dict_size; k += kThreads) s_wd[k] = static_cast<const WT*>(a.wdict)[k];
    __syncthreads();
    const uint32_t* sbits = reinterpret_cast<const uint32_t*>(smem_raw);
    const HT* shist = reinterpret_cast<const HT*>(smem_raw);
    const bool uniform = DICT && a.dict_size == 2;  // {w, 0.0 padding}: every synapse carries w

    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const WT* pot = static_cast<const WT*>(a.pot);
    const WT* dep = static_cast<const WT*>(a.dep);
    WT* W = static_cast<WT*>(a.w);

    const int p0 = blockIdx.x * a.posts_per_cta;
    const int p1 = min(a.nl, p0 + a.posts_per_cta);
    constexpr int PER_WARP = 32 / SUB;
    const int warp = tid >> 5, lane = tid & 31;
    const int sg = lane / SUB, sl = lane % SUB;
    // Software pipeline: the next post's list bounds are loaded while the
    // current post streams, and each post's chunks are fetched UL at a time
    // (all loads issued before any use) -- one memory round trip per post.
    // chunk loads per lane per batch: cover a typical list in one round trip
#ifndef SNB_SPARSE_UL
#define SNB_SPARSE_UL 8
#endif
    constexpr int UL = DICT ? (SUB <= 8 ? SNB_SPARSE_UL : 4) : 2;
    const int stride = (kThreads / 32) * PER_WARP;
    const int64_t* offb = a.off + static_cast<int64_t>(b) * a.nl;
    int p = p0 + warp * PER_WARP + sg;
    int64_t beg = 0, end = 0;
    if (p < p1) {
        beg = __ldg(offb + p);
        end = __ldg(offb + p + 1);
    }
    for (int pbase = p0 + warp * PER_WARP; pbase < p1; pbase += stride) {  // warp-uniform trip count
        const bool valid = p < p1;
        const int pn = p + stride;
        int64_t nbeg = 0, nend = 0;
        if (pn < p1) {
            nbeg = __ldg(offb + pn);
            nend = __ldg(offb + pn + 1);
        }
        WT sum = WT(0);
        int cnt = 0;
        if (valid) {
            const int gp = a.first + p;
            bool sp = false;
            WT depp = WT(0);
            if (STDP) {
                sp = bit_of(a.bits, gp);
                depp = dep[gp];
            }
            for (int64_t q0 = beg + sl * 4; q0 < end; q0 += SUB * 4 * UL) {
                uint4 m4[UL];
                WT wv[UL][4];
#pragma unroll
                for (int u = 0; u < UL; ++u) {
                    const int64_t q = q0 + static_cast<int64_t>(u) * SUB * 4;
                    if (q < end) {
                        m4[u] = __ldcs(reinterpret_cast<const uint4*>(a.meta + q));
                        if (!DICT) {
                            if (sizeof(WT) == 4) {
                                const float4 f = __ldcs(reinterpret_cast<const float4*>(W + q));
                                wv[u][0] = f.x; wv[u][1] = f.y; wv[u][2] = f.z; wv[u][3] = f.w;
                            } else {
                                const double2 f0 = __ldcs(reinterpret_cast<const double2*>(W + q));
                                const double2 f1 = __ldcs(reinterpret_cast<const double2*>(W + q + 2));
                                wv[u][0] = f0.x; wv[u][1] = f0.y; wv[u][2] = f1.x; wv[u][3] = f1.y;
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < UL; ++u) {
                    const int64_t q = q0 + static_cast<int64_t>(u) * SUB * 4;
                    if (q >= end) continue;
                    if (DICT && uniform) {
                        // one weight for every synapse: count the delivering pres
                        // (padding points at the zero-history slot pb)
                        const uint32_t ms[4] = {m4[u].x, m4[u].y, m4[u].z, m4[u].w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int pl = static_cast<int>(ms[k] & 0xffffu);
                            if (HB == 1) cnt += static_cast<int>((sbits[pl >> 5] >> (pl & 31)) & 1u);
                            else cnt += static_cast<int>((shist[pl] >> ((ms[k] >> 16) & 63u)) & 1u);
                        }
                        continue;
                    }
                    if (DICT) {
                        wv[u][0] = s_wd[m4[u].x >> 23]; wv[u][1] = s_wd[m4[u].y >> 23];
                        wv[u][2] = s_wd[m4[u].z >> 23]; wv[u][3] = s_wd[m4[u].w >> 23];
                    }
                    const uint32_t ms[4] = {m4[u].x, m4[u].y, m4[u].z, m4[u].w};
                    bool changed = false;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t m = ms[k];
                        const int pl = static_cast<int>(m & 0xffffu);
                        const int d1 = static_cast<int>((m >> 16) & 63u);
                        uint32_t e;
                        if (HB == 1) e = (sbits[pl >> 5] >> (pl & 31)) & 1u;
                        else e = static_cast<uint32_t>((shist[pl] >> d1) & 1u);
                        WT w = wv[u][k];
                        if (!DICT && STDP && ((m >> 22) & 1u)) {
                            const WT pt = pot[static_cast<int64_t>(pre0 + pl) * a.dp + d1];
                            WT dw = WT(0);
                            if (sp) dw += pt;
                            if (e) dw -= depp;
                            const WT nw = clamp_ref<WT>(w + dw, wmin, wmax);
                            changed |= (nw != w);
                            w = nw;
                            wv[u][k] = nw;
                        }
                        if (e) sum += w;
                    }
                    if (!DICT && STDP && changed) {
                        if (sizeof(WT) == 4) {
                            __stcs(reinterpret_cast<float4*>(W + q),
                                   make_float4(float(wv[u][0]), float(wv[u][1]), float(wv[u][2]), float(wv[u][3])));
                        } else {
                            __stcs(reinterpret_cast<double2*>(W + q), make_double2(double(wv[u][0]), double(wv[u][1])));
                            __stcs(reinterpret_cast<double2*>(W + q + 2), make_double2(double(wv[u][2]), double(wv[u][3])));
                        }
                    }
                }
            }
        }
        if (DICT && uniform) {
#pragma unroll
            for (int o = SUB / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            sum = static_cast<WT>(cnt) * s_wd[0];
        } else {
#pragma unroll
            for (int o = SUB / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        }
        if (valid && sl == 0) a.partial[static_cast<int64_t>(b) * a.nl + p] = static_cast<double>(sum);
        p = pn;
        beg = nbeg;
        end = nend;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *a.d_step += 1;
}

// Sparse count: k_sparse_pull specialised for static lists that carry one
// weight w (dictionary {w, 0}: the ER generator's nets, cfg4).  Same CTA
// tiling and pipelining; per post the lanes count the delivering entries and
// one lane writes count * w.  Loads are predicated on the 32-bit number of
// remaining entries and the bit test is one funnel shift, so an entry costs
// address + LDS + SHF.W + AND (padding entries point at the zero-history slot pb).
template <typename WT, int HB, int SUB>
__global__ void __launch_bounds__(kThreads, SNB_SPARSE_MINB) k_sparse_count(SparseArgs a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    using HT = typename HistT<HB>::T;
    static_assert(HB != 64, "64-step histories use k_sparse_pull");
    const int b = blockIdx.y;
    const int pre0 = b * a.pb;
    const int pcount = min(a.pb, a.n - pre0);
    const int tid = threadIdx.x;
    stage_history<HB>(a, pre0, pcount, smem_raw);
    __syncthreads();
    const uint32_t* sbits = reinterpret_cast<const uint32_t*>(smem_raw);
    const HT* shist = reinterpret_cast<const HT*>(smem_raw);
    const WT w0 = static_cast<const WT*>(a.wdict)[0];
    const int p0 = blockIdx.x * a.posts_per_cta;
    const int p1 = min(a.nl, p0 + a.posts_per_cta);
    constexpr int PER_WARP = 32 / SUB;
#ifndef SNB_SPARSE_COUNT_UL
#define SNB_SPARSE_COUNT_UL 6  // cfg4 (tools/ab_sparse.sh): UL 4 0.579, 5 0.561, 6 0.514, 7 0.532, 8 0.541, 12 0.689 ms at SUB 8
#endif
    constexpr int UL = SUB <= 8 ? SNB_SPARSE_COUNT_UL : 4;
    constexpr int STEP = SUB * 4 * UL;  // entries one lane group covers per batch
    const int warp = tid >> 5, lane = tid & 31;
    const int sg = lane / SUB, sl = lane % SUB;
    const int stride = (kThreads / 32) * PER_WARP;
    const int64_t* offb = a.off + static_cast<int64_t>(b) * a.nl;
    int p = p0 + warp * PER_WARP + sg;
    int64_t beg = 0, end = 0;
    if (p < p1) {
        beg = __ldg(offb + p);
        end = __ldg(offb + p + 1);
    }
    for (int pbase = p0 + warp * PER_WARP; pbase < p1; pbase += stride) {  // warp-uniform trip count
        const bool valid = p < p1;
        const int pn = p + stride;
        int64_t nbeg = 0, nend = 0;
        if (pn < p1) {
            nbeg = __ldg(offb + pn);
            nend = __ldg(offb + pn + 1);
        }
        int cnt = 0;
        if (valid) {
            for (int64_t q0 = beg + sl * 4; q0 < end; q0 += STEP) {
                const int rem = static_cast<int>(min(end - q0, static_cast<int64_t>(STEP)));
                const uint4* src = reinterpret_cast<const uint4*>(a.meta + q0);
                uint4 m4[UL];
#pragma unroll
                for (int u = 0; u < UL; ++u)
                    if (u * SUB * 4 < rem) m4[u] = __ldcs(src + u * SUB);
#pragma unroll
                for (int u = 0; u < UL; ++u) {
                    if (u * SUB * 4 < rem) {
                        const uint32_t ms[4] = {m4[u].x, m4[u].y, m4[u].z, m4[u].w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t mk = ms[k];
                            if (HB == 1) {
                                const uint32_t h = sbits[(mk & 0xffffu) >> 5];
                                cnt += static_cast<int>(__funnelshift_r(h, h, mk) & 1u);  // bit pl & 31
                            } else {
                                const uint32_t h = static_cast<uint32_t>(shist[mk & 0xffffu]);
                                cnt += static_cast<int>(__funnelshift_r(h, h, mk >> 16) & 1u);  // bit d-1 < 32
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int o = SUB / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (valid && sl == 0)
            a.partial[static_cast<int64_t>(b) * a.nl + p] = static_cast<double>(static_cast<WT>(cnt) * w0);
        p = pn;
        beg = nbeg;
        end = nend;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *a.d_step += 1;
}

// ---------------------------------------------------------------------------
// Bank-aware order of one-weight lists (setup, k_sparse_count only: a count
// does not depend on the order of a list).  In k_sparse_count one warp-wide
// LDS of the staged history serves 32/SUB posts x SUB lanes, lane sl of a post
// reading entry 4*SUB*r + 4*sl + k of its list.  Each list is bucket-sorted by
// the shared-memory bank of its history word, rotated by the post's slot in
// the warp (p mod 32/SUB), and dealt lane-major: the SUB entries one LDS
// touches come from evenly spaced buckets, so the warp's 32 reads spread over
// the banks instead of colliding at random (3.9 wavefronts per LDS before).
__device__ __forceinline__ int sp_bank(uint32_t m, int hbits) {
    const int pl = static_cast<int>(m & 0xffffu);
    return hbits == 1 ? (pl >> 5) & 31 : hbits == 16 ? (pl >> 1) & 31 : pl & 31;
}

__global__ void k_sparse_bank_order(const uint32_t* in, uint32_t* out, const int64_t* off, int64_t lists,
                                    int nl, int sub, int hbits) {
    const int64_t L = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (L >= lists) return;
    const int64_t beg = off[L];
    const int len = static_cast<int>(off[L + 1] - beg);
    if (len == 0) return;
    const int per_warp = 32 / sub;
    const int phase = static_cast<int>((L % nl) % per_warp);
    int start[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) start[b] = 0;
    for (int j = 0; j < len; ++j) start[(sp_bank(in[beg + j], hbits) - phase) & 31] += 1;
    int acc = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const int c = start[b];
        start[b] = acc;
        acc += c;
    }
    // dealing order: lane-major over the (row, k) slots of the list's rows of
    // 4*sub entries; only the last row can be partial, and there whole lanes
    // drop out (len is a multiple of 4)
    const int row = 4 * sub;
    const int rows = (len + row - 1) / row;
    const int last = (len - row * (rows - 1)) / 4;  // lanes with a full last row
    const int full = 4 * rows, part = 4 * (rows - 1);
    for (int j = 0; j < len; ++j) {
        const uint32_t m = in[beg + j];
        const int si = start[(sp_bank(m, hbits) - phase) & 31]++;
        int sl, g;
        if (si < full * last) {
            sl = si / full;
            g = si - sl * full;
        } else {
            const int t = si - full * last;
            sl = last + t / part;  // part > 0 here: si < len = full * last + part * (sub - last)
            g = t - (sl - last) * part;
        }
        out[beg + (g >> 2) * row + 4 * sl + (g & 3)] = m;
    }
}


// ---------------------------------------------------------------------------
// Sparse TMA stream (static nets whose lists carry one weight w: the ER
// generator's networks, cfg4).  The blocked-CSC meta array is one contiguous
// stream in (block, post) order.  The host cuts it into stages of whole posts
// (<= kSpE entries, one pre block, <= kSpNbMax posts) and gives each CTA a
// contiguous run of stages inside one pre block (CTAs per block in proportion
// to its entries).  A producer warp
// streams every stage's meta words plus the stage-relative end position of each
// of its posts (uint16) into a kSpStages-deep ring with cp.async.bulk; each
// consumer warp takes whole stages (warp w: stages w, w + kSpConsumers, ...) and
// counts, 4 lanes per post, the entries whose pre delivers (e = s_pre[t+1-d])
// -> partial[b][p] = count * w, the value k_sparse_pull's uniform path writes.
// The loads never occupy registers; no CTA barrier per stage.
constexpr int kSpE = 2048;        // entries per stage (8 KB of meta)
constexpr int kSpStages = 20;     // ring depth: ~12 stages in flight beyond the ones being counted
constexpr int kSpNbMax = 256;     // posts per stage
constexpr int kSpConsumers = 8;   // consumer warps
constexpr int kSpThreads = 32 * (kSpConsumers + 1);

template <int HB>
__device__ __forceinline__ void sp_stage_history(const SparseArgs& a, int b, uint8_t* smem, int tid, int nt) {
    using HT = typename HistT<HB>::T;
    const int pre0 = b * a.pb;
    const int pcount = max(0, min(a.pb, a.n - pre0));
    if (HB == 1) {
        uint32_t* sb = reinterpret_cast<uint32_t*>(smem);
        const int nw = (pcount + 31) >> 5;
        const int nw_all = a.pb / 32 + 1;
        for (int k = tid; k < nw_all; k += nt) sb[k] = k < nw ? __ldcg(a.bits + (pre0 >> 5) + k) : 0u;
        return;
    }
    HT* sh = reinterpret_cast<HT*>(smem);
    for (int k = tid; k <= a.pb; k += nt) {
        HT v = 0;
        if (k < pcount) v = static_cast<HT>(HB == 64 ? __ldcg(a.hist + pre0 + k) : __ldcg(a.hist_lo + pre0 + k));
        sh[k] = v;
    }
}

template <int HB>
__device__ __forceinline__ uint32_t sp_hit(const uint8_t* hist, uint32_t m) {
    using HT = typename HistT<HB>::T;
    const int pl = static_cast<int>(m & 0xffffu);
    if (HB == 1) return (reinterpret_cast<const uint32_t*>(hist)[pl >> 5] >> (pl & 31)) & 1u;
    return static_cast<uint32_t>((reinterpret_cast<const HT*>(hist)[pl] >> ((m >> 16) & 63u)) & 1u);
}

template <typename WT, int HB>
__global__ void __launch_bounds__(kSpThreads, 1) k_sparse_tma(SparseArgs a, SpStagePlan plan) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    uint32_t* r_meta = reinterpret_cast<uint32_t*>(smem);
    uint16_t* r_bnd = reinterpret_cast<uint16_t*>(smem + kSpStages * kSpE * 4);
    uint8_t* s_hist = smem + kSpStages * (kSpE * 4 + kSpNbMax * 2);
    const size_t hist_bytes = sp_hist_bytes(a.pb, HB);
    int4* s_hdr = reinterpret_cast<int4*>(s_hist + hist_bytes);  // [stages] {entries, k0, nb, block}
    uint64_t* full = reinterpret_cast<uint64_t*>(s_hdr + kSpStages);
    uint64_t* empty = full + kSpStages;
    const int s0 = plan.cta_first[blockIdx.x], s1 = plan.cta_first[blockIdx.x + 1];
    const int blk0 = plan.cta_block[blockIdx.x];
    if (tid == 0) {
        for (int s = 0; s < kSpStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the one pre block of this CTA's stages
    if (warp < kSpConsumers) sp_stage_history<HB>(a, blk0, s_hist, tid, 32 * kSpConsumers);
    __syncthreads();
    if (warp == kSpConsumers) {
        // ---- producer: stage records read 32 at a time (one per lane) ----
        SpStage cur{}, nxt{};
        if (s0 + lane < s1) cur = plan.stages[s0 + lane];
        if (s0 + 32 + lane < s1) nxt = plan.stages[s0 + 32 + lane];
        for (int s = s0, i = 0; s < s1; ++s, ++i) {
            const int w = (s - s0) & 31;
            if (w == 0 && s != s0) {
                cur = nxt;
                if (s + 32 + lane < s1) nxt = plan.stages[s + 32 + lane];
            }
            const int64_t q = __shfl_sync(0xffffffffu, cur.q, w);
            const int64_t bo = __shfl_sync(0xffffffffu, cur.bnd_off, w);
            const int entries = __shfl_sync(0xffffffffu, cur.entries, w);
            const int k0 = __shfl_sync(0xffffffffu, cur.k0, w);
            const int nb = __shfl_sync(0xffffffffu, cur.nb, w);
            const int blk = __shfl_sync(0xffffffffu, cur.block, w);
            const int slot = i % kSpStages;
            if (lane == 0) {
                mbar_wait(empty + slot, ((i / kSpStages) & 1u) ^ 1u);
                s_hdr[slot] = make_int4(entries, k0, nb, blk);
                const uint32_t mbytes = static_cast<uint32_t>(entries) * 4u;
                const uint32_t bbytes = static_cast<uint32_t>((nb * 2 + 15) & ~15);
                mbar_arrive_expect_tx(full + slot, mbytes + bbytes);
                if (mbytes) bulk_g2s(r_meta + slot * kSpE, a.meta + q, mbytes, full + slot);
                if (bbytes) bulk_g2s(r_bnd + slot * kSpNbMax, plan.bnd + bo, bbytes, full + slot);
            }
            __syncwarp();
        }
        return;
    }
    // ---- consumer warp: stages warp, warp + kSpConsumers, ... of the CTA's run;
    // 4 lanes per post count the delivering entries of its list (16 B per lane-step) ----
    const WT w0 = static_cast<const WT*>(a.wdict)[0];
    const int sg = lane >> 2, sl = lane & 3;
    for (int i = warp; s0 + i < s1; i += kSpConsumers) {
        const int slot = i % kSpStages;
        mbar_wait(full + slot, (i / kSpStages) & 1u);
        const int4 hdr = s_hdr[slot];
        const int k0 = hdr.y, nb = hdr.z;
        const uint8_t* hist = s_hist;
        const uint32_t* m = r_meta + slot * kSpE;
        const uint16_t* bp = r_bnd + slot * kSpNbMax;
        for (int j0 = 0; j0 < nb; j0 += 8) {
            const int j = j0 + sg;
            int beg = 0, end = 0;
            if (j < nb) {
                end = bp[j];
                beg = j > 0 ? bp[j - 1] : 0;
            }
            int cnt = 0;
#pragma unroll 4
            for (int q = beg + sl * 4; q < end; q += 16) {
                const uint4 mm = *reinterpret_cast<const uint4*>(m + q);
                cnt += static_cast<int>(sp_hit<HB>(hist, mm.x) + sp_hit<HB>(hist, mm.y) + sp_hit<HB>(hist, mm.z) +
                                        sp_hit<HB>(hist, mm.w));
            }
            cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
            cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
            if (sl == 0 && j < nb) a.partial[k0 + j - 1] = static_cast<double>(static_cast<WT>(cnt) * w0);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
    }
    if (blockIdx.x == 0 && tid == 0) *a.d_step += 1;
}

// Sparse stream: the same blocked-CSC pull, but each warp streams a contiguous
// run of its CTA's posts as one flat array of 4-entry chunks (lists are padded
// to 4, so a chunk never straddles two posts): every lane issues U 128-bit
// meta + weight loads back to back (no per-post tail waste), a fixed
// segmented suffix-reduction over lanes folds chunks into per-post sums, and
// the last segment's sum is carried into the next iteration.  The order of
// additions is fixed by the data layout, so results are deterministic.
template <typename WT, bool STDP, int HB, bool DICT>
__global__ void __launch_bounds__(kThreads) k_sparse_stream(SparseArgs a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    using HT = typename HistT<HB>::T;
    constexpr int U = DICT ? 8 : 4;
    const int b = blockIdx.y;
    const int pre0 = b * a.pb;
    const int pcount = min(a.pb, a.n - pre0);
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *a.d_step += 1;  // nobody reads it here
    const size_t hbytes = stage_history<HB>(a, pre0, pcount, smem_raw);
    WT* s_wd = reinterpret_cast<WT*>(smem_raw + hbytes);
    if (DICT)
        for (int k = tid; k < a.dict_size; k += kThreads) s_wd[k] = static_cast<const WT*>(a.wdict)[k];
    __syncthreads();
    const uint32_t* sbits = reinterpret_cast<const uint32_t*>(smem_raw);
    const HT* shist = reinterpret_cast<const HT*>(smem_raw);
    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const WT* pot = static_cast<const WT*>(a.pot);
    const WT* dep = static_cast<const WT*>(a.dep);
    WT* W = static_cast<WT*>(a.w);
    const int64_t* off = a.off + static_cast<int64_t>(b) * a.nl;  // off[p], p in [0, nl]
    double* part = a.partial + static_cast<int64_t>(b) * a.nl;

    const int warp = tid >> 5, lane = tid & 31;
    const int p0 = blockIdx.x * a.posts_per_cta;
    const int p1 = min(a.nl, p0 + a.posts_per_cta);
    if (p0 >= p1) return;
    // split [p0, p1) among the 8 warps by entry count (boundaries at post starts)
    const int64_t e0 = __ldg(off + p0), e1 = __ldg(off + p1);
    auto lower_post = [&](int64_t target) {  // first p in [p0, p1] with off[p] >= target
        int lo = p0, hi = p1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(off + mid) < target) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    const int nwarps = kThreads / 32;
    const int pa = lower_post(e0 + (e1 - e0) * warp / nwarps);
    const int pb = warp == nwarps - 1 ? p1 : lower_post(e0 + (e1 - e0) * (warp + 1) / nwarps);
    if (pa >= pb) return;
    // empty lists never appear in the stream: their partial is 0
    for (int q = pa + lane; q < pb; q += 32)
        if (__ldg(off + q) == __ldg(off + q + 1)) part[q] = 0.0;

    int64_t e = __ldg(off + pa);
    const int64_t end = __ldg(off + pb);
    int carry_post = pa;
    WT carry = WT(0);
    int lp = pa;  // this lane's current post (monotone)
    while (e < end) {
        uint4 m4[U];
        WT wv[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = e + static_cast<int64_t>(u * 32 + lane) * 4;
            if (q < end) {
                m4[u] = __ldcs(reinterpret_cast<const uint4*>(a.meta + q));
                if (DICT) {
                    // resolved after the loads (smem), see below
                } else if (sizeof(WT) == 4) {
                    const float4 f = __ldcs(reinterpret_cast<const float4*>(W + q));
                    wv[u][0] = f.x; wv[u][1] = f.y; wv[u][2] = f.z; wv[u][3] = f.w;
                } else {
                    const double2 f0 = __ldcs(reinterpret_cast<const double2*>(W + q));
                    const double2 f1 = __ldcs(reinterpret_cast<const double2*>(W + q + 2));
                    wv[u][0] = f0.x; wv[u][1] = f0.y; wv[u][2] = f1.x; wv[u][3] = f1.y;
                }
            } else {
                m4[u] = make_uint4(0, 0, 0, 0);
                wv[u][0] = wv[u][1] = wv[u][2] = wv[u][3] = WT(0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = e + static_cast<int64_t>(u * 32 + lane) * 4;
            const bool valid = q < end;
            if (DICT) {
                wv[u][0] = s_wd[m4[u].x >> 23]; wv[u][1] = s_wd[m4[u].y >> 23];
                wv[u][2] = s_wd[m4[u].z >> 23]; wv[u][3] = s_wd[m4[u].w >> 23];
                if (!valid) wv[u][0] = wv[u][1] = wv[u][2] = wv[u][3] = WT(0);
            }
            int p = pb;  // sentinel for lanes past the end
            if (valid) {
                while (__ldg(off + lp + 1) <= q) ++lp;
                p = lp;
            }
            WT csum = WT(0);
            if (valid) {
                const uint32_t ms[4] = {m4[u].x, m4[u].y, m4[u].z, m4[u].w};
                bool sp = false;
                WT depp = WT(0);
                if (STDP) {
                    sp = bit_of(a.bits, a.first + p);
                    depp = __ldcg(dep + a.first + p);
                }
                bool changed = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t m = ms[k];
                    const int pl = static_cast<int>(m & 0xffffu);
                    const int d1 = static_cast<int>((m >> 16) & 63u);
                    uint32_t ev;
                    if (HB == 1) ev = (sbits[pl >> 5] >> (pl & 31)) & 1u;
                    else ev = static_cast<uint32_t>((shist[pl] >> d1) & 1u);
                    WT w = wv[u][k];
                    if (STDP && ((m >> 22) & 1u)) {
                        const WT pt = __ldcg(pot + static_cast<int64_t>(pre0 + pl) * a.dp + d1);
                        const WT dw = fma(sp ? WT(1) : WT(0), pt, -((ev ? WT(1) : WT(0)) * depp));
                        const WT nw = clamp_ref<WT>(w + dw, wmin, wmax);
                        changed |= (nw != w);
                        w = nw;
                        wv[u][k] = nw;
                    }
                    csum = fma(ev ? WT(1) : WT(0), w, csum);
                }
                if (STDP && changed) {
                    if (sizeof(WT) == 4) {
                        __stcs(reinterpret_cast<float4*>(W + q),
                               make_float4(float(wv[u][0]), float(wv[u][1]), float(wv[u][2]), float(wv[u][3])));
                    } else {
                        __stcs(reinterpret_cast<double2*>(W + q), make_double2(double(wv[u][0]), double(wv[u][1])));
                        __stcs(reinterpret_cast<double2*>(W + q + 2), make_double2(double(wv[u][2]), double(wv[u][3])));
                    }
                }
            }
            // segmented suffix sum over lanes (posts are non-decreasing in lane)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const WT x = __shfl_down_sync(0xffffffffu, csum, o);
                const int px = __shfl_down_sync(0xffffffffu, p, o);
                if (lane + o < 32 && px == p) csum += x;
            }
            const int pprev = __shfl_up_sync(0xffffffffu, p, 1);
            const bool head = lane == 0 || pprev != p;
            const int plast = __shfl_sync(0xffffffffu, p, 31);
            const int first_post = __shfl_sync(0xffffffffu, p, 0);
            if (first_post != carry_post && lane == 0 && carry_post < pb) part[carry_post] = static_cast<double>(carry);
            WT total = csum;
            if (head && lane == 0 && p == carry_post) total += carry;
            if (head && p != plast && p < pb) part[p] = static_cast<double>(total);
            // the segment holding lane 31 continues into the next iteration;
            // its head total already includes the old carry when it began at lane 0
            const int head_last = __ffs(__ballot_sync(0xffffffffu, p == plast)) - 1;
            carry = __shfl_sync(0xffffffffu, total, head_last);
            carry_post = plast;
        }
        e += static_cast<int64_t>(U * 32) * 4;
    }
    if (lane == 0 && carry_post < pb) part[carry_post] = static_cast<double>(carry);
}

// Sparse exact: one thread per post, ascending pre, fp64 seeded with leak(v).
template <typename WT, bool STDP>
__global__ void __launch_bounds__(kThreads) k_sparse_exact(SparseArgs a) {
    const int p = blockIdx.x * kThreads + threadIdx.x;
    if (p < a.nl) {
        const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
        const WT* pot = static_cast<const WT*>(a.pot);
        const WT* dep = static_cast<const WT*>(a.dep);
        WT* W = static_cast<WT*>(a.w);
        const int gp = a.first + p;
        const bool sp = STDP ? bit_of(a.bits, gp) : false;
        const WT depp = STDP ? dep[gp] : WT(0);
        double acc = a.abm ? 0.0 : leak_toward(a.v[p], a.leak[p], a.reset[p]);
        for (int b = 0; b < a.nblocks; ++b) {
            const int64_t beg = a.off[static_cast<int64_t>(b) * a.nl + p];
            const int64_t end = a.off[static_cast<int64_t>(b) * a.nl + p + 1];
            for (int64_t q = beg; q < end; ++q) {
                const uint32_t m = a.meta[q];
                const int pre = b * a.pb + static_cast<int>(m & 0xffffu);
                const int d1 = static_cast<int>((m >> 16) & 63u);
                const bool e = (a.hist[pre] >> d1) & 1ull;
                WT w = W[q];
                if (STDP && ((m >> 22) & 1u)) {
                    const WT pt = pot[static_cast<int64_t>(pre) * a.dp + d1];
                    WT dw = WT(0);
                    if (sp) dw += pt;
                    if (e) dw -= depp;
                    w = clamp_ref<WT>(w + dw, wmin, wmax);
                    W[q] = w;
                }
                if (e) acc += static_cast<double>(w);
            }
        }
        a.u_exact[p] = acc;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_step += 1;
}

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

void check(cudaError_t err, const char* what) {
    if (err != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(err));
}

}  // namespace

uint64_t stream_key(uint64_t seed, uint64_t stream) {
    // RandomStream(seed, stream, 0, 0) key derivation (rng.hpp:19-24)
    uint64_t k = mix64(seed + 0x9e3779b97f4a7c15ULL);
    k = mix64(k ^ stream);
    k = mix64(k ^ 0ull);
    return mix64(k ^ 0ull);
}

int dense_vec(bool f64) { return f64 ? 2 : 4; }

int dense_tma_max_rows() { return kTmaListMax; }

size_t tiny_smem_bytes(const TinyArgs& a) { return tiny_layout(a).total; }

int tiny_max_smem() {
    int dev = 0, v = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    check(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
    return v;
}

void launch_tiny(const TinyArgs& a, cudaStream_t s) {
    const size_t smem = tiny_smem_bytes(a);
    const int threads = (a.n + 31) / 32 * 32;
    auto go = [&](auto kern) {
        check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
              "k_tiny smem attribute");
        kern<<<1, threads, smem, s>>>(a);
    };
    if (a.f64) {
        if (a.stdp) go(k_tiny<double, true>);
        else go(k_tiny<double, false>);
    } else {
        if (a.stdp) go(k_tiny<float, true>);
        else go(k_tiny<float, false>);
    }
    check(cudaGetLastError(), "k_tiny");
}

void launch_dense_tma(const DenseArgs& a, bool stdp, int grid, cudaStream_t s) {
    const size_t smem = dense_tma_smem(a.tile_w);
    static size_t configured[2] = {0, 0};
    auto kern = stdp ? k_dense_tma<true> : k_dense_tma<false>;
    if (configured[stdp ? 1 : 0] < smem) {
        check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
              "k_dense_tma smem attribute");
        configured[stdp ? 1 : 0] = smem;
    }
    kern<<<grid, kTmaThreads, smem, s>>>(a);
    check(cudaGetLastError(), "k_dense_tma");
}
int dense_threads() { return kThreads; }
int sparse_block_pres(int hbits) {
    // 32 KB of staged history per CTA (pre ids are 16-bit block-local)
    switch (hbits) {
        case 1: return 32768;   // pre_local == pb is the inert padding slot (16-bit field)
        case 16: return 16384;
        case 32: return 8192;
        default: return 4096;
    }
}

void launch_neuron(const NeuronArgs& a, bool exact, bool fused, const HistArgs& h, cudaStream_t s) {
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

template <typename WT, bool STDP, bool DELAY, bool EXACT>
static void dense_go(const DenseArgs& a, int grid, cudaStream_t s) {
    if (EXACT) k_dense_sweep<WT, STDP, DELAY, true><<<grid, kThreads, 0, s>>>(a);
    else k_dense_stream<WT, STDP, DELAY><<<grid, kThreads, 0, s>>>(a);
}

template <typename WT, bool STDP, bool DELAY>
static void persistent_go(NeuronArgs na, HistArgs h, DenseArgs da, int grid, int steps, cudaStream_t s,
                          int* max_ctas) {
    auto kern = k_persistent_dense<WT, STDP, DELAY>;
    if (max_ctas) {
        int dev = 0, sms = 0, occ = 0;
        check(cudaGetDevice(&dev), "cudaGetDevice");
        check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
        check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0), "occupancy");
        *max_ctas = occ * sms;
        return;
    }
    void* args[] = {&na, &h, &da, &steps};
    check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(kThreads), args, 0, s),
          "k_persistent_dense");
}

static void persistent_dispatch(const NeuronArgs& na, const HistArgs& h, const DenseArgs& da, bool f64,
                                bool stdp, bool delay, int grid, int steps, cudaStream_t s, int* max_ctas) {
#define SNB_P(WT)                                                                         \
    do {                                                                                  \
        if (stdp) {                                                                       \
            if (delay) persistent_go<WT, true, true>(na, h, da, grid, steps, s, max_ctas);   \
            else persistent_go<WT, true, false>(na, h, da, grid, steps, s, max_ctas);        \
        } else {                                                                          \
            if (delay) persistent_go<WT, false, true>(na, h, da, grid, steps, s, max_ctas);  \
            else persistent_go<WT, false, false>(na, h, da, grid, steps, s, max_ctas);       \
        }                                                                                 \
    } while (0)
    if (f64) SNB_P(double);
    else SNB_P(float);
#undef SNB_P
}

template <typename WT, bool STDP, bool DELAY>
static int stream_occ() {
    int dev = 0, sms = 0, occ = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dense_stream<WT, STDP, DELAY>, kThreads, 0),
          "occupancy");
    return occ * sms;
}

int dense_stream_max_ctas(bool f64, bool stdp, bool delay) {
    if (f64) {
        if (stdp) return delay ? stream_occ<double, true, true>() : stream_occ<double, true, false>();
        return delay ? stream_occ<double, false, true>() : stream_occ<double, false, false>();
    }
    if (stdp) return delay ? stream_occ<float, true, true>() : stream_occ<float, true, false>();
    return delay ? stream_occ<float, false, true>() : stream_occ<float, false, false>();
}

template <typename WT, bool STDP, bool DELAY>
static int cols_go(const NeuronArgs& na, const DenseArgs& da, const ColArgs& ca, int width, int grid, int steps,
                   cudaStream_t s) {
    // 16- and 32-post groups were slower than the row-chunk loop (2048-neuron
    // STDP net: 29k vs 41k steps/s): only 8-post groups are instantiated
    if (width != 8) throw std::runtime_error("k_persistent_cols: column groups of 8 posts only");
    auto kern = k_persistent_cols<WT, STDP, DELAY, 8>;
    if (grid <= 0) {
        int dev = 0, sms = 0, occ = 0;
        check(cudaGetDevice(&dev), "cudaGetDevice");
        check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
        check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kColThreads, 0), "occupancy");
        return occ * sms;
    }
    NeuronArgs a = na;
    DenseArgs d = da;
    ColArgs c = ca;
    void* args[] = {&a, &d, &c, &steps};
    check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(kColThreads), args, 0, s),
          "k_persistent_cols");
    return grid;
}

static int cols_dispatch(const NeuronArgs& na, const DenseArgs& da, const ColArgs& ca, bool f64, bool stdp,
                         bool delay, int width, int grid, int steps, cudaStream_t s) {
#define SNB_C(WT)                                                                                 \
    do {                                                                                          \
        if (stdp) return delay ? cols_go<WT, true, true>(na, da, ca, width, grid, steps, s)       \
                               : cols_go<WT, true, false>(na, da, ca, width, grid, steps, s);     \
        return delay ? cols_go<WT, false, true>(na, da, ca, width, grid, steps, s)                \
                     : cols_go<WT, false, false>(na, da, ca, width, grid, steps, s);              \
    } while (0)
    if (f64) SNB_C(double);
    SNB_C(float);
#undef SNB_C
}

int persistent_cols_max_ctas(bool f64, bool stdp, bool delay, int width) {
    return cols_dispatch(NeuronArgs{}, DenseArgs{}, ColArgs{}, f64, stdp, delay, width, 0, 0, nullptr);
}

void launch_persistent_cols(const NeuronArgs& na, const DenseArgs& da, const ColArgs& ca, bool f64, bool stdp,
                            bool delay, int width, int grid, int steps, cudaStream_t s) {
    cols_dispatch(na, da, ca, f64, stdp, delay, width, grid, steps, s);
}

int persistent_max_ctas(bool f64, bool stdp, bool delay) {
    int m = 0;
    persistent_dispatch(NeuronArgs{}, HistArgs{}, DenseArgs{}, f64, stdp, delay, 0, 0, nullptr, &m);
    return m;
}

void launch_persistent_dense(const NeuronArgs& na, const HistArgs& h, const DenseArgs& da, bool f64,
                             bool stdp, bool delay, int grid, int steps, cudaStream_t s) {
    persistent_dispatch(na, h, da, f64, stdp, delay, grid, steps, s, nullptr);
}

void launch_dense(const DenseArgs& a, bool f64, bool stdp, bool delay, bool exact, int grid,
                  cudaStream_t s) {
#define SNB_DENSE(WT)                                                            \
    do {                                                                         \
        if (stdp) {                                                              \
            if (delay) {                                                         \
                if (exact) dense_go<WT, true, true, true>(a, grid, s);           \
                else dense_go<WT, true, true, false>(a, grid, s);                \
            } else {                                                             \
                if (exact) dense_go<WT, true, false, true>(a, grid, s);          \
                else dense_go<WT, true, false, false>(a, grid, s);               \
            }                                                                    \
        } else {                                                                 \
            if (delay) {                                                         \
                if (exact) dense_go<WT, false, true, true>(a, grid, s);          \
                else dense_go<WT, false, true, false>(a, grid, s);               \
            } else {                                                             \
                if (exact) dense_go<WT, false, false, true>(a, grid, s);         \
                else dense_go<WT, false, false, false>(a, grid, s);              \
            }                                                                    \
        }                                                                        \
    } while (0)
    if (f64) SNB_DENSE(double);
    else SNB_DENSE(float);
#undef SNB_DENSE
    check(cudaGetLastError(), "k_dense_sweep");
}

template <typename WT, bool STDP, int HB>
static void sparse_go_sub(const SparseArgs& a, int sub, int gx, size_t smem, cudaStream_t s) {
    dim3 grid(gx, a.nblocks);
    if (a.dict_size > 0) smem = ((smem + 15) & ~static_cast<size_t>(15)) + static_cast<size_t>(a.dict_size) * sizeof(WT);
    if (a.dict_size == 2 && !STDP && sub != 0 && HB != 64) {  // one weight: count the delivering pres
        constexpr int HC = HB == 64 ? 32 : HB;  // (64 never reaches the launch)
        switch (sub) {
            case 1: k_sparse_count<WT, HC, 1><<<grid, kThreads, smem, s>>>(a); break;
            case 2: k_sparse_count<WT, HC, 2><<<grid, kThreads, smem, s>>>(a); break;
            case 4: k_sparse_count<WT, HC, 4><<<grid, kThreads, smem, s>>>(a); break;
            case 8: k_sparse_count<WT, HC, 8><<<grid, kThreads, smem, s>>>(a); break;
            case 16: k_sparse_count<WT, HC, 16><<<grid, kThreads, smem, s>>>(a); break;
            default: k_sparse_count<WT, HC, 32><<<grid, kThreads, smem, s>>>(a); break;
        }
        return;
    }
    if (a.dict_size > 0 && !STDP) {
        switch (sub) {
            case 0: k_sparse_stream<WT, false, HB, true><<<grid, kThreads, smem, s>>>(a); break;
            case 1: k_sparse_pull<WT, false, HB, 1, true><<<grid, kThreads, smem, s>>>(a); break;
            case 2: k_sparse_pull<WT, false, HB, 2, true><<<grid, kThreads, smem, s>>>(a); break;
            case 4: k_sparse_pull<WT, false, HB, 4, true><<<grid, kThreads, smem, s>>>(a); break;
            case 8: k_sparse_pull<WT, false, HB, 8, true><<<grid, kThreads, smem, s>>>(a); break;
            case 16: k_sparse_pull<WT, false, HB, 16, true><<<grid, kThreads, smem, s>>>(a); break;
            default: k_sparse_pull<WT, false, HB, 32, true><<<grid, kThreads, smem, s>>>(a); break;
        }
        return;
    }
    switch (sub) {
        case 0: k_sparse_stream<WT, STDP, HB, false><<<grid, kThreads, smem, s>>>(a); break;
        case 4: k_sparse_pull<WT, STDP, HB, 4, false><<<grid, kThreads, smem, s>>>(a); break;
        case 8: k_sparse_pull<WT, STDP, HB, 8, false><<<grid, kThreads, smem, s>>>(a); break;
        case 16: k_sparse_pull<WT, STDP, HB, 16, false><<<grid, kThreads, smem, s>>>(a); break;
        default: k_sparse_pull<WT, STDP, HB, 32, false><<<grid, kThreads, smem, s>>>(a); break;
    }
}

static size_t hist_smem_bytes(int pb, int hbits) {
    if (hbits == 1) return (static_cast<size_t>(pb / 32 + 1) * 4 + 15) & ~static_cast<size_t>(15);
    return (static_cast<size_t>(pb + 1) * (hbits / 8) + 15) & ~static_cast<size_t>(15);
}

template <typename WT, bool STDP>
static void sparse_go(const SparseArgs& a, int hbits, int sub, int gx, cudaStream_t s) {
    const size_t smem = hist_smem_bytes(a.pb, hbits);
    switch (hbits) {
        case 1: sparse_go_sub<WT, STDP, 1>(a, sub, gx, smem, s); break;
        case 16: sparse_go_sub<WT, STDP, 16>(a, sub, gx, smem, s); break;
        case 32: sparse_go_sub<WT, STDP, 32>(a, sub, gx, smem, s); break;
        default: sparse_go_sub<WT, STDP, 64>(a, sub, gx, smem, s); break;
    }
}

void launch_sparse(const SparseArgs& a, bool f64, bool stdp, int hbits, int sub, bool exact, int gx,
                   cudaStream_t s) {
    if (exact) {
        const int grid = (a.nl + kThreads - 1) / kThreads;
        if (grid == 0) {
            launch_step_bump(a.d_step, s);
            return;
        }
        if (f64) {
            if (stdp) k_sparse_exact<double, true><<<grid, kThreads, 0, s>>>(a);
            else k_sparse_exact<double, false><<<grid, kThreads, 0, s>>>(a);
        } else {
            if (stdp) k_sparse_exact<float, true><<<grid, kThreads, 0, s>>>(a);
            else k_sparse_exact<float, false><<<grid, kThreads, 0, s>>>(a);
        }
    } else {
        if (f64) {
            if (stdp) sparse_go<double, true>(a, hbits, sub, gx, s);
            else sparse_go<double, false>(a, hbits, sub, gx, s);
        } else {
            if (stdp) sparse_go<float, true>(a, hbits, sub, gx, s);
            else sparse_go<float, false>(a, hbits, sub, gx, s);
        }
    }
    check(cudaGetLastError(), "k_sparse");
}

void launch_sparse_bank_order(const uint32_t* in, uint32_t* out, const int64_t* off, int64_t lists, int nl,
                              int sub, int hbits, cudaStream_t s) {
    if (lists <= 0) return;
    k_sparse_bank_order<<<static_cast<unsigned>((lists + 127) / 128), 128, 0, s>>>(in, out, off, lists, nl, sub,
                                                                                  hbits);
    check(cudaGetLastError(), "k_sparse_bank_order");
}

size_t sparse_tma_smem(const SparseArgs& a, int hbits) {
    return static_cast<size_t>(kSpStages) * (kSpE * 4 + kSpNbMax * 2) + sp_hist_bytes(a.pb, hbits) +
           kSpStages * 16 + 2 * kSpStages * 8;
}

int sparse_tma_stage_entries() { return kSpE; }
int sparse_tma_max_boundaries() { return kSpNbMax; }

void launch_sparse_tma(const SparseArgs& a, const SpStagePlan& plan, int ctas, bool f64, int hbits, cudaStream_t s) {
    const size_t smem = sparse_tma_smem(a, hbits);
    auto go = [&](auto kern) {
        check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
              "k_sparse_tma smem attribute");
        kern<<<ctas, kSpThreads, smem, s>>>(a, plan);
    };
    if (f64) {
        switch (hbits) {
            case 1: go(k_sparse_tma<double, 1>); break;
            case 16: go(k_sparse_tma<double, 16>); break;
            case 32: go(k_sparse_tma<double, 32>); break;
            default: go(k_sparse_tma<double, 64>); break;
        }
    } else {
        switch (hbits) {
            case 1: go(k_sparse_tma<float, 1>); break;
            case 16: go(k_sparse_tma<float, 16>); break;
            case 32: go(k_sparse_tma<float, 32>); break;
            default: go(k_sparse_tma<float, 64>); break;
        }
    }
    check(cudaGetLastError(), "k_sparse_tma");
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
