// Whole-call step loops: k_tiny (one CTA, shared-memory state),
// k_persistent_dense (row chunks) and k_persistent_cols (column owners).
#include "kernels_common.cuh"

namespace snb {

namespace {

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
#ifndef SNB_TINY_HREGS
#define SNB_TINY_HREGS 4
#endif
// own history words kept in registers (hw <= 2): cfg1 1.15e6 -> 1.24e6 steps/s.
// Caching the first 4 / 8 incoming entries (meta + weight) in registers as
// well lost (1.15e6 / 0.69e6: the 64-register cap of a 1024-thread CTA
// spills), and so did batching the list walk 4 entries at a time (metas,
// weights, history words issued together): 0.91e6 with branches, 0.97e6
// with selects (every fp64 add executed)
constexpr int kTinyHistRegs = SNB_TINY_HREGS;
constexpr int kTinyCountWords = 8;  // count mode: nets of <= 256 neurons

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
    SNB_DCHECK(q0 <= q1 && q1 <= static_cast<uint32_t>(a.m));
    // own history words in registers (<= kTinyHistRegs 32-bit words)
    const bool hreg = kTinyHistRegs > 0 && hw2 <= kTinyHistRegs;
    uint32_t hr[kTinyHistRegs > 0 ? kTinyHistRegs : 1];
#pragma unroll
    for (int k = 0; k < kTinyHistRegs; ++k) hr[k] = (hreg && k < hw2 && j < np) ? hist[k * np + j] : 0u;
    unsigned long long spikes = 0;
    double lv = leak_toward(v, leak, rst);  // leak(v) of the coming step
    const bool w0_int = a.w0 == trunc(a.w0) && fabs(a.w0) <= 1048576.0;  // integer weight below 2^20
    // count mode: this post's in-list as a pre bitmask in registers, the previous
    // step's spike words double-buffered in shared memory
    __shared__ uint32_t s_spk[2][kTinyCountWords];
    const bool cmode = !STDP && a.count_words > 0;
    uint32_t cm[kTinyCountWords];
#pragma unroll
    for (int k = 0; k < kTinyCountWords; ++k) cm[k] = 0u;
    if (cmode) {
        if (own)
            for (uint32_t q = q0; q < q1; ++q) {
                const uint32_t i = (meta[q] >> 5) >> 2;  // byte offset of pre i's word 0 (delay 1: bit 0)
#pragma unroll
                for (int k = 0; k < kTinyCountWords; ++k)
                    if (static_cast<uint32_t>(k) == (i >> 5)) cm[k] |= 1u << (i & 31);
            }
        const uint32_t w0 = __ballot_sync(0xffffffffu, own && (hist[j] & 1u));  // spikes of step t0 - 1
        if ((tid & 31) == 0 && (tid >> 5) < kTinyCountWords) s_spk[0][tid >> 5] = w0;
        __syncthreads();
    }
#ifdef SNB_TINY_TRACE
    long long tt_sum[6] = {0, 0, 0, 0, 0, 0};
    long long tt_prev = clock64();
#define SNB_TT_MARK(k)                                   \
    if (tid == 0) {                                      \
        const long long now = clock64();                 \
        tt_sum[k] += now - tt_prev;                      \
        tt_prev = now;                                   \
    }
#else
#define SNB_TT_MARK(k)
#endif
    for (int s = 0; s < a.steps; ++s) {
        const int cur = s & 1;
        const uint8_t* hc = sm + L.hist + cur * hbuf;        // history through t-1
        uint32_t* hn = reinterpret_cast<uint32_t*>(sm + L.hist + (cur ^ 1) * hbuf);  // through t
        bool fired = false;
        if (own) {
            // (1) leak, incoming list in ascending pre order (bit d-1 = s_pre[t-d]),
            // the step's stimulus, threshold, refractory (mat_engine.cpp:160-198)
            // MAT: u = leak(v) + w...; ABM: pending = 0.0 + w..., u = leak(v) + (pending + ext)
            double u = a.abm ? 0.0 : lv;
            if (cmode) {
                int k = 0;
#pragma unroll
                for (int wd = 0; wd < kTinyCountWords; ++wd)
                    if (wd < a.count_words) k += __popc(cm[wd] & s_spk[cur][wd]);
                const double w0 = a.w0;
                if (k > 0 && w0_int && u == trunc(u) && fabs(u) <= 1099511627776.0) {
                    // integers below 2^40 plus at most 1024 integer weights below 2^20:
                    // every partial sum of the reference's k adds is exact, so one
                    // fma is the same double (the chain of dependent adds was the
                    // step's longest latency)
                    u = fma(static_cast<double>(k), w0, u);
                } else {
                    for (int c = 0; c < k; ++c) u += w0;  // ascending-pre sum of equal weights
                }
            } else {
#pragma unroll 4
                for (uint32_t q = q0; q < q1; ++q) {
                    const uint32_t mq = meta[q];
                    if (tiny_bit(hc, mq)) u += static_cast<double>(w[q]);  // WS = double unless STDP
                }
            }
            SNB_TT_MARK(3)
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
            SNB_TT_MARK(4)
            if (a.abm) u = lv + u;
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
            lv = leak_toward(v, leak, rst);  // next step's leak, off its critical path
            if (a.trace) a.trace[static_cast<int64_t>(s) * n + j] = v;
        }
        SNB_TT_MARK(0)
        const uint32_t word = __ballot_sync(0xffffffffu, fired);
        if ((tid & 31) == 0 && (tid >> 5) < words) {
            a.raster[static_cast<int64_t>(s) * words + (tid >> 5)] = word;
            spikes += __popc(word);
            if (cmode) s_spk[cur ^ 1][tid >> 5] = word;  // read after the step's __syncthreads
        }
        // (2) own history row into the other buffer (+ own STDP traces)
        if (j < np) {
            uint32_t carry = fired ? 1u : 0u;
            if (hreg) {
#pragma unroll
                for (int k = 0; k < kTinyHistRegs; ++k) {
                    if (k < hw2) {
                        const uint32_t x = hr[k];
                        hr[k] = (x << 1) | carry;
                        hn[k * np + j] = hr[k];
                        carry = x >> 31;
                    }
                }
            } else {
                const uint32_t* hcw = reinterpret_cast<const uint32_t*>(hc);
                for (int k = 0; k < hw2; ++k) {
                    const uint32_t x = hcw[k * np + j];
                    hn[k * np + j] = (x << 1) | carry;
                    carry = x >> 31;
                }
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
        SNB_TT_MARK(1)
        __syncthreads();  // the new history (and traces) of step t are complete
        SNB_TT_MARK(2)
        if (STDP && a.plastic_on && own) {
            // (3) STDP on post j's plastic synapses: dw = 0; if s_post dw += pot^(d)_pre;
            // if s_pre[t-d+1] dw -= dep_post; clamp (mat_engine.cpp:242-249)
            const uint8_t* hnb = reinterpret_cast<const uint8_t*>(hn);
            const double* potn = pot + (cur ^ 1) * np * a.dp;
            const double depj = dep[(cur ^ 1) * np + j];
            for (uint32_t q = q0; q < q1; ++q) {
                const uint16_t pq = pidx[q];
                if (pq == 0xffffu) continue;  // not plastic
                const uint32_t mq = meta[q];
                w[q] = stdp_apply<WT>(w[q], stdp_dw(fired, fired ? potn[pq] : 0.0, tiny_bit(hnb, mq), depj), wmin,
                                      wmax);
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
#ifdef SNB_TINY_TRACE
    if (tid == 0 && a.steps > 0)
        printf("tiny trace: %d steps, cycles per step: inputs %.0f, stimulus %.0f, lif rest %.0f, raster+history %.0f, "
               "syncthreads %.0f\n", a.steps, double(tt_sum[3]) / a.steps, double(tt_sum[4]) / a.steps,
               double(tt_sum[0]) / a.steps, double(tt_sum[1]) / a.steps, double(tt_sum[2]) / a.steps);
#endif
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
    __shared__ double s_dep[kColW];
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
    double* pot2 = static_cast<double*>(ca.pot2);  // fp64 traces (fp64 STDP math)
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
                if (shi > slo) u += stim_lookup(na.st_neuron, na.st_amp, slo, shi, j);
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
                    s_dep[lane] = dep;
                    bool any_pot = false;
                    for (int d = 1; d <= da.dp; ++d) {
                        double pot = 0.0;
                        for (uint64_t m = (hn >> (d - 1)) & wmask & ~1ull; m; m &= m - 1)
                            pot += ca.a_plus[__ffsll(static_cast<long long>(m)) - 2];
                        pot2[(static_cast<int64_t>(cur) * n + j) * da.dp + (d - 1)] = pot;
                        any_pot |= pot != 0.0;
                    }
                    if (ca.row_plastic[j] && (any_pot || t == ca.clamp_step)) act = true;
                }
            }
            const uint32_t word = __ballot_sync(0xffffffffu, fired);  // bits 0..W-1
            const uint32_t aw = __ballot_sync(0xffffffffu, act);
            if (lane == 0) {
                const int wi = (c * kColW) >> 5, sh = (c * kColW) & 31;
                if (aw) {
                    atomicOr(act_now + wi, aw << sh);
                    if (ca.active_count) atomicAdd(ca.active_count, static_cast<unsigned long long>(__popc(aw)));
                }
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
        bool sj[VEC];
        double dj[VEC];
        double acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            okc[k] = j0 + k < na.nl;
            sj[k] = STDP && okc[k] && ((spk >> (cv * VEC + k)) & 1u);
            dj[k] = STDP ? s_dep[cv * VEC + k] : 0.0;
            acc[k] = 0.0;
        }
        const uint64_t* hist = ca.hist2 + static_cast<int64_t>(cur) * n;
        const double* potc = pot2 + static_cast<int64_t>(cur) * n * da.dp;
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
                if (STDP && da.plastic_on && kind != kRowNone) {
                    const bool pl = kind == kRowAll || (kind == kRowAllButSelf && j0 + k != i) ||
                                    (kind == kRowMixed && ((mw >> ((j0 & 31) + k)) & 1u));
                    if (pl) {
                        const double p = __ldcg(potc + static_cast<int64_t>(i) * da.dp + d1);
                        const WT nw = stdp_apply<WT>(w, stdp_dw(sj[k], p, e, dj[k]), wmin, wmax);
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
// Cluster loop for small static one-weight nets without plasticity (cfg2: 1000
// neurons all-to-all, delays 1..8): ONE thread-block cluster of cs CTAs (16,
// non-portable, or 8) runs the whole call.  CTA r owns posts [r P, r P + P)
// (P a multiple of 32) and keeps, in its shared memory, one rotation code per
// (pre, owned post) -- (d + 1) & 31 for a synapse of delay d, 1 for none -- and
// a copy of every pre's history word h << 1 (double-buffered by step parity).
// Per step: (1) the owner threads run the LIF update of their posts (as
// k_persistent_cols) and store their new history word into EVERY CTA's copy
// with distributed-shared-memory stores; (2) one cluster barrier
// (barrier.cluster arrive.release / wait.acquire) -- instead of a grid barrier
// plus L2 round trips; (3) each CTA counts, for its posts, the pres whose bit
// d - 1 is set: rot_r(h << 1, code) >> 31 per (pre, post), integer counts
// reduced in shared memory, input = count * w.  No global memory on the step
// path except the raster words and the stimulus table.
constexpr int kClThreads = 1024;

// DSMEM store that completes 4 transaction bytes on the target CTA's mbarrier
__device__ __forceinline__ void st_async_u32(uint32_t remote_addr, uint32_t v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(remote_addr),
                 "r"(v), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, int rank) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(addr), "r"(rank));
    return d;
}


// Shared-memory layout of k_cluster_count (D = 0: rotation codes; D = 8 / 16:
// delay bit-planes).  With planes, the exchange buffer is a ring of
// cl_ring(D) = D + 2 spike-word rows: row t mod R holds s[t] of every pre, and
// plane d of step t is row (t - d) mod R, so a step exchanges one word per 32
// pres (not D) and only plane 0 waits for it.  D + 2 rows keep a writer's
// step t + 1 off every row a peer can still be reading (planes 0..D-1 of its
// step t - 1 or t).
__host__ __device__ constexpr int cl_ring(int D) { return D > 0 ? D + 2 : 2; }
// Words between ring rows: one 16-byte bank group more than a row, so the
// rows the (post, delay) threads of a warp read together start in different
// banks (with a 128-byte multiple every row began at bank 0: 8-way conflicts
// on each LDS.128 of the plane counts)
__host__ __device__ constexpr int cl_rstride(int wn4) { return wn4 + 4; }
struct ClLayout {
    size_t code, ex, red, in, bar, total;
};
__host__ __device__ inline ClLayout cl_layout(int n, int P, int D) {
    ClLayout L{};
    const int npad = (n + 3) & ~3;
    const int wn4 = ((n + 31) / 32 + 15) & ~15;
    size_t o = 0;
    L.code = o;
    o += D == 0 ? static_cast<size_t>(n) * P : static_cast<size_t>(P) * D * wn4 * 4;
    L.ex = o;
    o += D == 0 ? static_cast<size_t>(2) * npad * 4 : static_cast<size_t>(cl_ring(D)) * cl_rstride(wn4) * 4;
    L.red = o;
    o += D == 0 ? static_cast<size_t>(kClThreads) * 4 * 4 : 0;
    L.in = o;
    o += static_cast<size_t>(P) * 8;
    L.bar = o;
    o += static_cast<size_t>(cl_ring(D)) * 8;
    L.total = o;
    return L;
}

#ifndef SNB_CL_MREG
#define SNB_CL_MREG 1
#endif

constexpr int kClMregs = 4;  // uint4 mask registers per thread of a 1024-thread CTA (16 words)

template <typename WT, int P, int D, int NT>
__global__ void __launch_bounds__(NT, 1) k_cluster_count(NeuronArgs na, ClusterArgs ca, int steps) {
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr int MR = kClMregs * (kClThreads / NT);  // uint4 mask registers per thread
    cg::cluster_group cluster = cg::this_cluster();
    const int r = static_cast<int>(cluster.block_rank());
    const int cs = ca.cs, n = na.n;
    const int npad = (n + 3) & ~3;
    const int wn4 = ((n + 31) / 32 + 15) & ~15;  // history words per delay plane (padded)
    const int rs = cl_rstride(wn4);               // words between exchange ring rows
    const ClLayout L = cl_layout(n, P, D);
    uint8_t* s_code = smem + L.code;                                  // D = 0: [n][P] rotation codes
    const uint32_t* s_mask = reinterpret_cast<const uint32_t*>(smem + L.code);  // D > 0: [P][D][wn4]
    uint32_t* s_ex = reinterpret_cast<uint32_t*>(smem + L.ex);        // [2][npad] h << 1, or [2][D][wn4] planes
    int* s_red = reinterpret_cast<int*>(smem + L.red);                // D = 0: [1024 / (P/4)][P]
    double* s_in = reinterpret_cast<double*>(smem + L.in);            // [P]
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.bar);      // [R] exchange buffer full
    constexpr int R = cl_ring(D);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {   // this CTA's code / mask block, once per call; zero the exchange buffers (plane padding)
        const size_t bytes = L.ex - L.code;
        const uint4* src = reinterpret_cast<const uint4*>(ca.codes + static_cast<size_t>(r) * bytes);
        uint4* dst = reinterpret_cast<uint4*>(smem + L.code);
        for (size_t k = tid; k < bytes / 16; k += NT) dst[k] = __ldg(src + k);
        for (size_t k = tid; k < (L.red - L.ex) / 4; k += NT) s_ex[k] = 0u;
    }
    // exchange by st.async into every CTA's buffer, each store completing its
    // bytes on that CTA's mbarrier of the buffer: no cluster barrier and no
    // fence on the step path; double buffering keeps writers one step behind
    // readers (a CTA writes buffer t+1 only after every CTA's step-t words
    // reached it, i.e. after every CTA finished reading buffer t-1)
    if (tid == 0) {
        for (int k = 0; k < R; ++k) mbar_init(&s_bar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int t = *na.d_step;
    if (D > 0) {
        __syncthreads();  // the zeroing above is complete
        // ring rows of the D - 1 steps before the call, from the history words
        // the previous call left in hist2 (bit k - 1 of pre i's word = s_i[t - k])
        const uint64_t* hp = ca.hist2 + static_cast<int64_t>((t & 1) ^ 1) * n;
        for (int i0 = warp * 32; i0 < n; i0 += NT) {
            const int i = i0 + lane;
            const uint64_t h = i < n ? hp[i] : 0ull;
            for (int k = 1; k < D; ++k) {
                const uint32_t b = __ballot_sync(0xffffffffu, (h >> (k - 1)) & 1ull);
                if (lane == 0) s_ex[(((t - k) % R + R) % R) * rs + (i0 >> 5)] = b;
            }
        }
    }
    cluster.sync();
    uint32_t ph0 = 0, ph1 = 0, phr = 0;      // phr: bit k = parity of ring row k's barrier
    const uint32_t tx_bytes = D == 0 ? 4u * static_cast<uint32_t>(na.nl)
                                     : 4u * static_cast<uint32_t>((na.nl + 31) / 32);
    const int p = tid;                       // owner thread of post j (tid < P)
    const int j = r * P + p;
    const bool own = tid < P && j < na.nl;
    double v = 0.0, thr = 0.0, leak = 0.0, rst = 0.0, fire_p = 1.0, in = 0.0;
    int32_t cnt = 0, refr = 0;
    uint64_t hprev = 0, akey = 0;
    unsigned long long spikes = 0, active = 0;
    if (own) {
        v = na.v[j];
        thr = na.thr[j];
        leak = na.leak[j];
        rst = na.reset[j];
        cnt = na.cnt[j];
        refr = na.refr[j];
        in = na.partial[j];
        hprev = ca.hist2[static_cast<int64_t>((t & 1) ^ 1) * n + j];
        if (na.fire_p) {
            fire_p = na.fire_p[j];
            akey = na.agent_key[j];
        }
    }
    double lv = leak_toward(v, leak, rst);  // leak(v) of the coming step
    // exchange targets of this lane (owner warps, lane < cs): CTA `lane`'s ring
    // and barriers, as cluster addresses
    const uint32_t rem_ex = (D > 0 && lane < cs) ? mapa_u32(smem_u32(s_ex), lane) : 0u;
    const uint32_t rem_bar = (D > 0 && lane < cs) ? mapa_u32(smem_u32(s_bar), lane) : 0u;
    int64_t slo = 0, shi = 0;                // stimulus rows of the step, fetched a step ahead
    auto stim_bounds = [&](int tt) {
        slo = shi = 0;
        const int row = tt - na.st_base;
        if (own && row >= 0 && row < na.st_steps) {
            slo = __ldg(na.st_off + row);
            shi = __ldg(na.st_off + row + 1);
        }
    };
    stim_bounds(t);
    const WT w0 = static_cast<WT>(ca.w0);
    // delay planes: when a thread's slice is exactly MR uint4 (cfg2: 1000 pres,
    // 2 threads per (post, plane)), it stays in registers for the whole call
    uint4 mreg[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) mreg[k] = make_uint4(0u, 0u, 0u, 0u);
    if (D > 0 && SNB_CL_MREG) {
        constexpr int PAIRS = P * (D > 0 ? D : 1);
        constexpr int T = NT / PAIRS >= 4 ? 4 : NT / PAIRS >= 2 ? 2 : 1;
        if (tid < PAIRS * T && wn4 / T == 4 * MR) {
            const int pi = tid / T, part = tid % T;
            const int pp = pi / (D > 0 ? D : 1), d = pi % (D > 0 ? D : 1);
            const uint4* m4 = reinterpret_cast<const uint4*>(s_mask + (pp * D + d) * wn4 + part * (wn4 / T));
#pragma unroll
            for (int k = 0; k < MR; ++k) mreg[k] = m4[k];
        }
    }
    // plane 0 split over a post's D lanes (one thread per (post, delay), 32-word
    // planes): after the exchange every lane counts 4 words of plane 0 instead of
    // the delay-0 lane counting all 32 -- the count that follows the wait is the
    // step's critical path
    constexpr bool SPLIT0 = D == 8 && NT / (P * (D > 0 ? D : 1)) == 1 && SNB_CL_MREG;
    uint4 m0 = make_uint4(0u, 0u, 0u, 0u);
    const bool split0 = SPLIT0 && wn4 == 32 && tid < P * D;
    if (split0) {
        constexpr int DD = D > 0 ? D : 1;
        const int pp = tid / DD, d = tid % DD;
        m0 = reinterpret_cast<const uint4*>(s_mask + (pp * DD + 0) * wn4)[d];
    }
#ifdef SNB_CL_TRACE
    // phase clocks of thread 0 (CTA 0): LIF + exchange issue, wait, count, barrier
    long long tr_sum[7] = {0, 0, 0, 0, 0, 0, 0};
    long long tr_prev = clock64();
#define SNB_CL_MARK(k)                                       \
    if (tid == 0) {                                          \
        const long long now = clock64();                     \
        tr_sum[k] += now - tr_prev;                          \
        tr_prev = now;                                       \
    }
#else
#define SNB_CL_MARK(k)
#endif
    for (int s = 0; s < steps; ++s, ++t) {
        const int cur = D > 0 ? t % R : (t & 1);  // exchange row / buffer of this step
        if (tid == 0) mbar_arrive_expect_tx(&s_bar[cur], tx_bytes);
        SNB_CL_MARK(4)
        if (tid < P) {  // (1) LIF update of the owned posts (k_persistent_cols' neuron phase)
            bool fired = false;
            uint64_t hn = 0;
            if (own) {
                double u = na.abm ? in : lv + in;
                if (shi > slo) u += stim_lookup(na.st_neuron, na.st_amp, slo, shi, j);
                if (na.abm) u = lv + u;
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
                lv = leak_toward(v, leak, rst);  // next step's leak, off its critical path
                if (na.trace && (t - na.t_base) < na.raster_rows)
                    na.trace[static_cast<int64_t>(t - na.t_base) * na.nl + j] = v;
                hn = (hprev << 1) | (fired ? 1ull : 0ull);
                hprev = hn;
                spikes += fired ? 1 : 0;
                active += (hn & ca.dmask) != 0 ? 1 : 0;
                if (D == 0) {  // this pre's word h << 1 into every CTA's copy
                    const uint32_t la = smem_u32(s_ex + cur * npad + j), lb = smem_u32(&s_bar[cur]);
                    const uint32_t h2 = static_cast<uint32_t>(hn << 1);
                    for (int q = 0; q < cs; ++q) st_async_u32(mapa_u32(la, q), h2, mapa_u32(lb, q));
                }
            }
            SNB_CL_MARK(5)
            const bool live = (r * P + warp * 32) < na.nl;  // warp-uniform
            const uint32_t word = __ballot_sync(0xffffffffu, fired);
            if (D > 0 && live && lane < cs) {  // the warp's spike word of step t into ring row t of CTA `lane`
                const int w = (r * P) / 32 + warp;
                // CTA `lane`'s window, mapped once per call (offsets carry over)
                st_async_u32(rem_ex + static_cast<uint32_t>((cur * rs + w) * 4), word,
                             rem_bar + static_cast<uint32_t>(cur * 8));
            }
            if (lane == 0 && na.raster && (t - na.t_base) < na.raster_rows && live)
                na.raster[static_cast<int64_t>(t - na.t_base) * na.nl_words + ((r * P) >> 5) + warp] = word;
        }

        // (2) every owner's words of the step have landed in this CTA's buffer
        // (the async-proxy stores are tracked by complete_tx, so a CTA-scope wait
        // sees them, as for bulk copies; an acquire.cluster wait adds an L1
        // invalidation per step: 2.81e5 vs 2.86e5 steps/s on cfg2)
        SNB_CL_MARK(6)
        stim_bounds(t + 1);
        if (D == 0) {
            if (cur) { mbar_wait(&s_bar[1], ph1); ph1 ^= 1u; }
            else { mbar_wait(&s_bar[0], ph0); ph0 ^= 1u; }
        }
        // (3) counts of the delivering pres for this CTA's posts (integers: any order is exact)
        if (D > 0) {
            // thread (post, delay d, part): popc(mask[post][d] & plane[d]) over its words
            constexpr int PAIRS = P * (D > 0 ? D : 1);
            constexpr int T = NT / PAIRS >= 4 ? 4 : NT / PAIRS >= 2 ? 2 : 1;
            // (combinations with PAIRS > NT are compiled but never launched)
            static_assert(D == 0 || PAIRS > NT || D * T <= 32, "cluster plane tiling");
            int sum = 0;
            const int pi = tid / T, part = tid % T;
            const int pp = pi / (D > 0 ? D : 1), d = pi % (D > 0 ? D : 1);
            const int per_part = wn4 / T;  // multiple of 4
            const bool pair = tid < PAIRS * T;
            auto plane_count = [&]() {
                const int row = ((t - d) % R + R) % R;  // plane d of step t = s[t - d]
                const uint4* e4 = reinterpret_cast<const uint4*>(s_ex + row * rs + part * per_part);
                int c = 0;
                if (SNB_CL_MREG && per_part == 4 * MR) {  // mask words in registers for the call
#pragma unroll
                    for (int k = 0; k < MR; ++k) {
                        const uint4 m = mreg[k], e = e4[k];
                        c += __popc(m.x & e.x) + __popc(m.y & e.y) + __popc(m.z & e.z) + __popc(m.w & e.w);
                    }
                } else {
                    const uint4* m4 = reinterpret_cast<const uint4*>(s_mask + (pp * D + d) * wn4 + part * per_part);
                    for (int k = 0; k < per_part / 4; ++k) {
                        const uint4 m = m4[k], e = e4[k];
                        c += __popc(m.x & e.x) + __popc(m.y & e.y) + __popc(m.z & e.z) + __popc(m.w & e.w);
                    }
                }
                return c;
            };
            // planes 1..D-1 are rows of earlier steps, already here: counted while
            // this step's words are in flight; plane 0 after the row's barrier
            SNB_CL_MARK(0)
            if (pair && d > 0) sum = plane_count();
            mbar_wait(&s_bar[cur], (phr >> cur) & 1u);
            phr ^= 1u << cur;
            SNB_CL_MARK(1)
            if (split0) {
                const uint4 e = reinterpret_cast<const uint4*>(s_ex + (t % R) * rs)[d];
                sum += __popc(m0.x & e.x) + __popc(m0.y & e.y) + __popc(m0.z & e.z) + __popc(m0.w & e.w);
            } else if (pair && d == 0) {
                sum = plane_count();
            }
            if (pair) {
#pragma unroll
                for (int o = (D * T) / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if (d == 0 && part == 0) s_in[pp] = static_cast<double>(static_cast<WT>(sum) * w0);
            }
            SNB_CL_MARK(2)
            __syncthreads();
            SNB_CL_MARK(3)
        } else {
            constexpr int CG = P / 4, RL = NT / CG;  // threads tid >= RL * CG idle in the sweep
            constexpr int per = NT / P >= 32 ? 32 : NT / P >= 16 ? 16 : NT / P >= 8 ? 8 : 4;
            const int cg4 = tid % CG, rl = tid / CG;
            const uint32_t* h2c = s_ex + cur * npad;
            int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll 4
            for (int i = rl < RL ? rl : n; i < n; i += RL) {
                const uint32_t code = *reinterpret_cast<const uint32_t*>(s_code + static_cast<size_t>(i) * P + cg4 * 4);
                const uint32_t h = h2c[i];
                c0 += static_cast<int>(__funnelshift_r(h, h, code) >> 31);
                c1 += static_cast<int>(__funnelshift_r(h, h, code >> 8) >> 31);
                c2 += static_cast<int>(__funnelshift_r(h, h, code >> 16) >> 31);
                c3 += static_cast<int>(__funnelshift_r(h, h, code >> 24) >> 31);
            }
            if (rl < RL) {
                int* red = s_red + rl * P + cg4 * 4;
                red[0] = c0;
                red[1] = c1;
                red[2] = c2;
                red[3] = c3;
            }
            __syncthreads();
            if (tid < per * P) {  // RL / per partials per thread, then shuffles over `per` lanes
                const int pp = tid / per, q = tid % per;
                int sum = 0;
#pragma unroll
                for (int k = q; k < RL; k += per) sum += s_red[k * P + pp];
#pragma unroll
                for (int o = per / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if (q == 0) s_in[pp] = static_cast<double>(static_cast<WT>(sum) * w0);
            }
            __syncthreads();
        }
        if (tid < P) in = s_in[p];
    }
    if (own) {
        ca.partial[j] = in;  // (same buffer as na.partial) input of the next call's first step
        na.v[j] = v;
        na.cnt[j] = cnt;
        ca.hist2[static_cast<int64_t>((t & 1) ^ 1) * n + j] = hprev;
    }
    if (tid < P) {
        for (int o = 16; o > 0; o >>= 1) {
            spikes += __shfl_xor_sync(0xffffffffu, spikes, o);
            active += __shfl_xor_sync(0xffffffffu, active, o);
        }
        if (lane == 0) {
            if (spikes) atomicAdd(na.spike_count, spikes);
            if (active && ca.active_count) atomicAdd(ca.active_count, active);
        }
    }
    if (r == 0 && tid == 0) *na.d_step = t;
#ifdef SNB_CL_TRACE
    if (r == 0 && tid == 0 && steps > 0)
        printf("cluster trace: %d steps, cycles per step: top %.0f, lif %.0f, exchange issue %.0f, stim bounds %.0f, "
               "wait (planes 1..D-1 + barrier) %.0f, plane 0 + reduce %.0f, syncthreads %.0f\n",
               steps, double(tr_sum[4]) / steps, double(tr_sum[5]) / steps, double(tr_sum[6]) / steps,
               double(tr_sum[0]) / steps, double(tr_sum[1]) / steps, double(tr_sum[2]) / steps,
               double(tr_sum[3]) / steps);
#endif
    cluster.sync();  // no CTA leaves while a peer's last stores may target it
}

// Setup: delay bit-planes of the cluster loop, [cs][P][D][wn4]: bit b of word w
// of plane d is set when pre 32 w + b has a synapse of delay d + 1 onto post
// r P + p (one-weight nets: a synapse is a non-zero weight).
template <typename WT>
__global__ void k_cluster_masks(DenseArgs da, int nl, int P, int cs, int D, uint32_t* masks) {
    const int wn4 = ((da.n + 31) / 32 + 15) & ~15;
    const int64_t total = static_cast<int64_t>(cs) * P * D * wn4;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int w = static_cast<int>(k % wn4);
        const int64_t rest = k / wn4;
        const int d = static_cast<int>(rest % D);
        const int64_t rp = rest / D;
        const int pp = static_cast<int>(rp % P), r = static_cast<int>(rp / P);
        const int j = r * P + pp;
        uint32_t bits = 0;
        if (j < nl)
            for (int b = 0; b < 32; ++b) {
                const int i = 32 * w + b;
                if (i >= da.n) break;
                const int64_t e = static_cast<int64_t>(i) * da.pitch + j;
                if (static_cast<const WT*>(da.w)[e] != WT(0) && (da.delay ? da.delay[e] : 1) == d + 1) bits |= 1u << b;
            }
        masks[k] = bits;
    }
}

// Setup: rotation codes of the cluster loop, [cs][n][P]; a synapse is a
// non-zero weight (one-weight nets), its delay d from the dense delay bytes.
template <typename WT>
__global__ void k_cluster_codes(DenseArgs da, int nl, int P, int cs, uint8_t* codes) {
    const int64_t total = static_cast<int64_t>(cs) * da.n * P;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(k % P);
        const int64_t ri = k / P;
        const int i = static_cast<int>(ri % da.n), r = static_cast<int>(ri / da.n);
        const int j = r * P + p;
        uint8_t c = 1;
        if (j < nl) {
            const int64_t e = static_cast<int64_t>(i) * da.pitch + j;
            if (static_cast<const WT*>(da.w)[e] != WT(0)) {
                const int d = da.delay ? da.delay[e] : 1;
                c = static_cast<uint8_t>((d + 1) & 31);
            }
        }
        codes[k] = c;
    }
}

}  // namespace

size_t tiny_smem_bytes(const TinyArgs& a) { return tiny_layout(a).total; }

int tiny_count_words_max() { return kTinyCountWords; }

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


// Threads per CTA of the cluster loop: 512 when the (post, delay) pairs fit
// (cfg2, P = 64 x D = 8: 1.86 -> 1.69 us per step -- half the warps contend
// for the schedulers after each exchange), else 1024.
static int cl_threads(int P, int D) {
    const char* e = std::getenv("SNB_CLUSTER_THREADS");  // A/B knob: 1024 keeps the wide CTAs
    if (e && std::atoi(e) == 1024) return kClThreads;
    return D > 0 && P * D <= 512 ? 512 : kClThreads;
}

static const void* cluster_kernel(bool f64, int P, int D) {
#define SNB_CLK(WT, DD)                                                                  \
    switch (P) {                                                                         \
        case 32: return reinterpret_cast<const void*>(k_cluster_count<WT, 32, DD, kClThreads>);      \
        case 64: return reinterpret_cast<const void*>(k_cluster_count<WT, 64, DD, kClThreads>);      \
        case 96: return reinterpret_cast<const void*>(k_cluster_count<WT, 96, DD, kClThreads>);      \
        default: return reinterpret_cast<const void*>(k_cluster_count<WT, 128, DD, kClThreads>);     \
    }
    if (D == 16 && P > 64) return nullptr;  // P * D > 1024: not planned
    // 512-thread CTAs where the (post, delay) pairs fit (cl_threads)
    if (cl_threads(P, D) == 512) {
#define SNB_CL5(WT)                                                                               \
    if (D == 8) return P == 32 ? reinterpret_cast<const void*>(k_cluster_count<WT, 32, 8, 512>)   \
                               : reinterpret_cast<const void*>(k_cluster_count<WT, 64, 8, 512>);  \
    return reinterpret_cast<const void*>(k_cluster_count<WT, 32, 16, 512>);
        if (f64) { SNB_CL5(double) }
        SNB_CL5(float)
#undef SNB_CL5
    }
    if (f64) {
        if (D == 8) SNB_CLK(double, 8)
        if (D == 16) return P == 32 ? reinterpret_cast<const void*>(k_cluster_count<double, 32, 16, kClThreads>)
                                    : reinterpret_cast<const void*>(k_cluster_count<double, 64, 16, kClThreads>);
        SNB_CLK(double, 0)
    }
    if (D == 8) SNB_CLK(float, 8)
    if (D == 16) return P == 32 ? reinterpret_cast<const void*>(k_cluster_count<float, 32, 16, kClThreads>)
                                : reinterpret_cast<const void*>(k_cluster_count<float, 64, 16, kClThreads>);
    SNB_CLK(float, 0)
#undef SNB_CLK
}

// Cluster shape for a net of n posts: 16 CTAs (non-portable) when the device
// runs such a cluster, else 8; delay bit-planes (D = 8 / 16) when the delays
// and the planes fit, else rotation codes (D = 0, delays <= 31).  0: no fit.
int cluster_plan(int n, int nl, bool f64, int dmax, int* P_out, int* D_out) {
    int dev = 0, optin = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
    const char* ck = std::getenv("SNB_CLUSTER_CODES");  // A/B knob: 1 = rotation codes only
    for (int cs : {16, 8}) {
        const int P = ((nl + cs - 1) / cs + 31) / 32 * 32;
        if (P != 32 && P != 64 && P != 96 && P != 128) continue;  // instantiated widths
        int cands[3] = {dmax <= 8 ? 8 : 16, 0, -1};
        if (dmax > 16 || (ck && std::string(ck) == "1")) cands[0] = 0, cands[1] = -1;
        for (int D : cands) {
            if (D < 0) break;
            if (D > 0 && P * D > kClThreads) continue;
            const size_t smem = cl_layout(n, P, D).total;
            if (smem > static_cast<size_t>(optin)) continue;
            const void* kern = cluster_kernel(f64, P, D);
            if (cs > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                  "k_cluster_count smem attribute");
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(cl_threads(P, D));
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if (clusters < 1) continue;
            *P_out = P;
            *D_out = D;
            return cs;
        }
    }
    return 0;
}

size_t cluster_table_bytes(int n, int P, int D, int cs) {
    const ClLayout L = cl_layout(n, P, D);
    return (L.ex - L.code) * cs;
}

void launch_cluster_table(const DenseArgs& da, int nl, int P, int D, int cs, void* table, bool f64, cudaStream_t s) {
    const int64_t total = D == 0 ? static_cast<int64_t>(cs) * da.n * P
                                 : static_cast<int64_t>(cs) * P * D * ((((da.n + 31) / 32) + 15) & ~15);
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    if (D == 0) {
        if (f64) k_cluster_codes<double><<<grid, 256, 0, s>>>(da, nl, P, cs, static_cast<uint8_t*>(table));
        else k_cluster_codes<float><<<grid, 256, 0, s>>>(da, nl, P, cs, static_cast<uint8_t*>(table));
    } else {
        if (f64) k_cluster_masks<double><<<grid, 256, 0, s>>>(da, nl, P, cs, D, static_cast<uint32_t*>(table));
        else k_cluster_masks<float><<<grid, 256, 0, s>>>(da, nl, P, cs, D, static_cast<uint32_t*>(table));
    }
    check(cudaGetLastError(), "cluster table");
}

void launch_cluster_count(const NeuronArgs& na, const ClusterArgs& ca, bool f64, int steps, cudaStream_t s) {
    const void* kern = cluster_kernel(f64, ca.P, ca.D);
    const size_t smem = cl_layout(na.n, ca.P, ca.D).total;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ca.cs);
    cfg.blockDim = dim3(cl_threads(ca.P, ca.D));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = ca.cs;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    NeuronArgs a0 = na;
    ClusterArgs a1 = ca;
    int a2 = steps;
    void* args[] = {&a0, &a1, &a2};
    check(cudaLaunchKernelExC(&cfg, kern, args), "k_cluster_count");
}

}  // namespace snb
