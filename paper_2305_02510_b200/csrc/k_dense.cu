// Dense sweeps over W[pre][post]: exact-order k_dense_sweep, streaming
// k_dense_stream and the TMA-staged k_dense_tma (the cfg3 hot kernel).
#include "kernels_common.cuh"

namespace snb {

namespace {

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
template <typename WT, bool STDP, bool DELAY, bool EXACT>
__global__ void __launch_bounds__(kThreads) k_dense_sweep(DenseArgs a) {
    using VT = VecT<WT>;
    using V = typename VT::V;
    constexpr int VEC = VT::N;
    constexpr int U = 8;  // rows in flight per thread

    __shared__ int32_t s_rows[kSubRows];
    __shared__ uint64_t s_e[kSubRows];
    __shared__ double s_pot[STDP && !DELAY ? kSubRows : 1];
    __shared__ uint8_t s_kind[kSubRows];
    __shared__ uint32_t s_word[32];
    __shared__ int32_t s_wpref[33];

    const int tid = threadIdx.x;
    const int ntiles = (a.nl + a.tile_w - 1) / a.tile_w;
    const int items = ntiles * a.nchunks;
    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const double* pot = a.pot;
    const double* dep = a.dep;
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
        double depj[VEC];
        int gc[VEC];
        double acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            gc[k] = a.first + c0 + k;
            const bool ok = in_tile && (c0 + k) < a.nl;
            sj[k] = ok && STDP ? bit_of(a.bits, gc[k]) : false;
            depj[k] = ok && STDP ? dep[gc[k]] : 0.0;
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
                        if (STDP && a.plastic_on && kind != kRowNone) {
                            const bool pl = kind == kRowAll || (kind == kRowAllButSelf && gc[k] != row) ||
                                            (kind == kRowMixed && ((mv[u] >> k) & 1u));
                            if (pl) {
                                const double p = DELAY ? pot[static_cast<int64_t>(row) * a.dp + d1] : s_pot[idx];
                                const WT nw = stdp_apply<WT>(w, stdp_dw(sj[k], p, e, depj[k]), wmin, wmax);
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

template <typename WT, bool STDP, bool DELAY>
__global__ void __launch_bounds__(kThreads, 2) k_dense_stream(DenseArgs a) {
    dense_stream_body<WT, STDP, DELAY>(a, blockIdx.x, gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_step += 1;  // no other CTA reads it
}

// ---------------------------------------------------------------------------
// TMA-staged dense sweep (fp32 or fp64 weights; with synaptic delays the
// rows' delay bytes ride in the same stages): one CTA per SM, a producer warp
// streams the active rows' tile segments into a kTmaStages-deep shared-memory
// ring with cp.async.bulk (completion on mbarriers), 8 x kTmaHalves consumer
// warps apply the same per-element update as k_dense_stream from shared
// memory and write the new weights with 128-bit streaming stores.  Loads
// never occupy registers, so the in-flight window per SM is the whole ring.
// Consumer warp w owns column slot w & 7 of every row r = w >> 3 (mod
// kTmaHalves) of a stage: two halves give each scheduler 4 consumer warps to
// hide the fp64 STDP arithmetic's dependent latency (cfg3 sweep 1.47 ms with
// one half); at the end of an item half 1 hands its column
// sums to half 0 through shared memory (fixed order: half 0 + half 1), so
// the neuron phase still adds one partial row per row chunk.
#ifndef SNB_TMA_HALVES
#define SNB_TMA_HALVES 2
#endif
constexpr int kTmaRows = 4;        // rows per stage
constexpr int kTmaStages = 8;      // ring depth
constexpr int kTmaListMax = 1024;  // rows per item at most (one list per item, double-buffered)
constexpr int kTmaHalves = SNB_TMA_HALVES;
constexpr int kTmaConsumers = 8 * kTmaHalves;               // consumer warps
constexpr int kTmaThreads = 32 * (kTmaConsumers + 2);       // + 1 producer warp + 1 planner warp
static_assert(kTmaHalves == 1 || kTmaHalves == 2, "row halves");
constexpr int kTmaXchDoubles = kTmaHalves > 1 ? 8 * 32 * 4 : 0;  // half-1 column sums (VEC <= 4)

__device__ __forceinline__ void tma_consumer_bar() {  // the consumer warps only (named barrier 1)
    asm volatile("bar.sync 1, %0;" ::"r"(kTmaConsumers * 32) : "memory");
}
constexpr int kTmaDp = 4;          // delayed STDP: pot^(d) traces staged per listed row
// Row records of both weight types carry the fp64 trace (RowRec<double>):
// the STDP update is computed in fp64 for fp32 storage too.
using TmaRec = RowRec<double>;

// Roles: warp kTmaConsumers + 1 (planner) claims the next item and builds its
// active-row list into the other of two list buffers while warp kTmaConsumers
// (producer) streams the current item's rows and the consumer warps process
// them, so an item's
// list build (two dependent global round trips + a scan) no longer stalls the
// ring between items.  Buffers hand over on mbarriers: ready[b] (planner ->
// producer + consumers), freeb[b] (producer + consumer warps -> planner) and
// issued (producer -> planner: claim the next item now).
template <typename WT, bool STDP, bool DELAY>
__global__ void __launch_bounds__(kTmaThreads, 1) k_dense_tma(DenseArgs a) {
    using VT = VecT<WT>;
    using V = typename VT::V;
    constexpr int VEC = VT::N;
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntiles = (a.nl + a.tile_w - 1) / a.tile_w;
    const int items = ntiles * a.nchunks;
    const uint32_t row_bytes = static_cast<uint32_t>(a.tile_w) * static_cast<uint32_t>(sizeof(WT));
    const uint32_t drow_bytes = DELAY ? static_cast<uint32_t>(a.tile_w) : 0u;  // delay bytes per row segment
    const size_t stage_bytes = static_cast<size_t>(kTmaRows) * (row_bytes + drow_bytes);
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTmaStages * stage_bytes);
    uint64_t* empty = full + kTmaStages;
    uint64_t* ready = empty + kTmaStages;
    uint64_t* freeb = ready + 2;
    uint64_t* issued = freeb + 2;  // producer -> planner: the current item's last stage is issued
    // list buffers sized for this launch's items (rows_per_chunk rows + one stage of padding)
    const int rec_cap = a.rows_per_chunk + kTmaRows;
    TmaRec* s_recs = reinterpret_cast<TmaRec*>(issued + 2);
    // delayed STDP: fp64 pot^(d) of each listed row for d = 1..kTmaDp (a.dp <= kTmaDp)
    double* s_potds = reinterpret_cast<double*>(s_recs + 2 * rec_cap);
    double* s_xch = s_potds + ((DELAY && STDP) ? 2 * rec_cap * kTmaDp : 0);  // kTmaXchDoubles
    __shared__ int s_item[2];
    __shared__ int s_cnt[2];

    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const double* dep = a.dep;
    const double* pot = a.pot;
    WT* W = static_cast<WT*>(a.w);

    if (tid == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kTmaConsumers);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(ready + b, 1);
            mbar_init(freeb + b, kTmaConsumers + 1);
        }
        mbar_init(issued, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kTmaConsumers + 1) {
        // ---- planner ----
        for (int ki = 0;; ++ki) {
            const int b = ki & 1;
            // claim the next item only once the current one is fully issued: a
            // claim made earlier would hold work back from CTAs that finish
            // first (the step's tail); the list build then overlaps the ring's
            // last kTmaStages stages
            if (ki >= 1) mbar_wait(issued, static_cast<uint32_t>((ki - 1) & 1));
            if (ki >= 2) mbar_wait(freeb + b, static_cast<uint32_t>(((ki >> 1) - 1) & 1));
            int item = blockIdx.x + ki * static_cast<int>(gridDim.x);
            if (a.work) {
                int got = 0;
                if (lane == 0) got = atomicAdd(a.work, 1);
                item = __shfl_sync(0xffffffffu, got, 0);
            }
            TmaRec* rec = s_recs + b * rec_cap;
            double* potd = s_potds + b * rec_cap * kTmaDp;
            int cnt = 0;
            if (item < items) {
                const int chunk = item / ntiles;
                const int r0 = chunk * a.rows_per_chunk;
                const int r1 = min(a.n, r0 + a.rows_per_chunk);
                // (1) row ids of the active rows of [r0, r1), ascending, one word per lane
                for (int wb = r0 & ~31; wb < r1; wb += 32 * 32) {
                    const int wr = wb + lane * 32;
                    uint32_t wd = 0;
                    if (wr < r1) {
                        wd = __ldcg(a.active + (wr >> 5));
                        const int lo = r0 - wr;
                        if (lo > 0) wd &= (lo >= 32) ? 0u : ~((1u << lo) - 1u);
                        const int rem = r1 - wr;
                        if (rem < 32) wd &= (rem <= 0) ? 0u : ((1u << rem) - 1u);
                    }
                    const int c = __popc(wd);
                    int incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int x = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += x;
                    }
                    int pos = cnt + incl - c;
                    SNB_DCHECK(pos + c <= rec_cap - kTmaRows);
                    for (uint32_t m = wd; m; m &= m - 1) rec[pos++].rowk = wr + __ffs(static_cast<int>(m)) - 1;
                    cnt += __shfl_sync(0xffffffffu, incl, 31);
                }
                __syncwarp();
                // (2) the rows' history words, kinds and traces, 4 rows per lane in flight
                for (int p0 = 0; p0 < cnt; p0 += 4 * 32) {
                    uint64_t h[4];
                    int kd[4];
                    double pt[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int p = p0 + u * 32 + lane;
                        h[u] = 0;
                        kd[u] = 0;
                        pt[u] = 0.0;
                        if (p < cnt) {
                            const int r = rec[p].rowk;
                            h[u] = __ldcg(a.hist + r);
                            kd[u] = STDP ? static_cast<int>(__ldg(a.kind + r)) : 0;
                            pt[u] = (STDP && !DELAY) ? __ldcg(pot + r) : 0.0;
                            if (STDP && DELAY)
                                for (int d = 0; d < kTmaDp; ++d)
                                    potd[p * kTmaDp + d] =
                                        d < a.dp ? __ldcg(pot + static_cast<int64_t>(r) * a.dp + d) : 0.0;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int p = p0 + u * 32 + lane;
                        if (p < cnt) {
                            TmaRec x;
                            x.rowk = rec[p].rowk | (kd[u] << 28);
                            x.e_lo = static_cast<uint32_t>(h[u]);
                            x.e_hi = static_cast<uint32_t>(h[u] >> 32);
                            x.pot = pt[u];
                            rec[p] = x;
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                s_item[b] = item < items ? item : -1;
                s_cnt[b] = cnt;
                mbar_arrive(ready + b);  // release: the list and its count
            }
            if (item >= items) break;
        }
    } else if (warp == kTmaConsumers) {
        // ---- producer ----
        uint32_t it = 0;  // ring position, advanced identically by producer and consumers
        for (int ki = 0;; ++ki) {
            const int b = ki & 1;
            mbar_wait(ready + b, static_cast<uint32_t>((ki >> 1) & 1));
            const int item = s_item[b];
            if (item < 0) break;
            const int cnt = s_cnt[b];
            const TmaRec* rec = s_recs + b * rec_cap;
            const int chunk = item / ntiles;
            const int tile = item - chunk * ntiles;
            const int col0 = tile * a.tile_w;
            const int width = static_cast<int>(min(static_cast<int64_t>(a.tile_w), a.pitch - col0));
            const uint32_t copy_bytes = static_cast<uint32_t>(width) * static_cast<uint32_t>(sizeof(WT));
            const int ngroups = (cnt + kTmaRows - 1) / kTmaRows;
            if (lane == 0) {
                for (int g = 0; g < ngroups; ++g, ++it) {
                    const int s = it % kTmaStages;
                    const uint32_t ph = (it / kTmaStages) & 1u;
                    mbar_wait(empty + s, ph ^ 1u);
                    const int nr = min(kTmaRows, cnt - g * kTmaRows);
                    mbar_arrive_expect_tx(full + s, static_cast<uint32_t>(nr) * (copy_bytes + (DELAY ? width : 0)));
                    uint8_t* st = ring + s * stage_bytes;
                    for (int r = 0; r < nr; ++r) {
                        const int row = rec[g * kTmaRows + r].rowk & 0x0fffffff;
                        SNB_DCHECK(row < a.n && col0 + width <= a.pitch && g * kTmaRows + r < cnt);
                        bulk_g2s(st + static_cast<size_t>(r) * row_bytes, W + static_cast<int64_t>(row) * a.pitch + col0,
                                 copy_bytes, full + s);
                        if (DELAY)
                            bulk_g2s(st + static_cast<size_t>(kTmaRows) * row_bytes + static_cast<size_t>(r) * drow_bytes,
                                     a.delay + static_cast<int64_t>(row) * a.pitch + col0, static_cast<uint32_t>(width),
                                     full + s);
                    }
                }
                mbar_arrive(issued);
                mbar_arrive(freeb + b);
            } else {
                it += ngroups;
            }
        }
    } else {
        // ---- consumers ----
        uint32_t it = 0;
        for (int ki = 0;; ++ki) {
            const int b = ki & 1;
            mbar_wait(ready + b, static_cast<uint32_t>((ki >> 1) & 1));
            const int item = s_item[b];
            if (item < 0) break;
            const int cnt = s_cnt[b];
            const TmaRec* s_rec = s_recs + b * rec_cap;
            const double* s_potd = s_potds + b * rec_cap * kTmaDp;
            const int chunk = item / ntiles;
            const int tile = item - chunk * ntiles;
            const int col0 = tile * a.tile_w;
            const int width = static_cast<int>(min(static_cast<int64_t>(a.tile_w), a.pitch - col0));
            const int ngroups = (cnt + kTmaRows - 1) / kTmaRows;
            const int rh = warp >> 3;                 // row half
            const int tcol = ((warp & 7) * 32 + lane) * VEC;
            const int c0 = col0 + tcol;
            const bool in_tile = tcol < width && c0 < a.nl;
            const int gc0 = a.first + c0;
            bool sj[VEC];
            double depj[VEC], sjd[VEC], ndep[VEC];
            double acc[VEC];
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                const bool ok = in_tile && (c0 + k) < a.nl;
                sj[k] = ok && STDP && bit_of(a.bits, gc0 + k);
                depj[k] = (ok && STDP) ? __ldcg(dep + gc0 + k) : 0.0;
                sjd[k] = sj[k] ? 1.0 : 0.0;  // exact 0/1 factors for the unit-delay fma form
                ndep[k] = -depj[k];
                acc[k] = 0.0;
            }
            for (int g = 0; g < ngroups; ++g, ++it) {
                const int s = it % kTmaStages;
                const uint32_t ph = (it / kTmaStages) & 1u;
                mbar_wait(full + s, ph);
                const int nr = min(kTmaRows, cnt - g * kTmaRows);
                const uint8_t* st = ring + s * stage_bytes;
                WT grp[VEC];
#pragma unroll
                for (int k = 0; k < VEC; ++k) grp[k] = WT(0);
                if (in_tile) {
#pragma unroll
                    for (int r = rh; r < kTmaRows; r += kTmaHalves) {
                        if (r >= nr) break;
                        const TmaRec rec = s_rec[g * kTmaRows + r];
                        const int row = rec.rowk & 0x0fffffff;
                        const int kind = rec.rowk >> 28;
                        SNB_DCHECK(g * kTmaRows + r < cnt && row < a.n);
                        const V wv = *reinterpret_cast<const V*>(st + static_cast<size_t>(r) * row_bytes + tcol * sizeof(WT));
                        uint32_t dv = 0;
                        if (DELAY) {
                            const uint8_t* dp8 = st + static_cast<size_t>(kTmaRows) * row_bytes +
                                                 static_cast<size_t>(r) * drow_bytes + tcol;
                            dv = VEC == 4 ? *reinterpret_cast<const uint32_t*>(dp8) : *reinterpret_cast<const uint16_t*>(dp8);
                        }
                        const uint64_t h = (static_cast<uint64_t>(rec.e_hi) << 32) | rec.e_lo;
                        WT w[VEC], ef[VEC];
                        int d1[VEC];
#pragma unroll
                        for (int k = 0; k < VEC; ++k) {
                            w[k] = VT::get(wv, k);
                            d1[k] = DELAY ? static_cast<int>((dv >> (8 * k)) & 0xffu) - 1 : 0;
                            ef[k] = ((h >> d1[k]) & 1ull) ? WT(1) : WT(0);  // s_pre[t+1-d], exact 0/1 factor
                        }
                        if (STDP && a.plastic_on && kind != kRowNone) {
                            WT nw[VEC];
                            if (DELAY) {
#pragma unroll
                                for (int k = 0; k < VEC; ++k) {
                                    SNB_DCHECK(d1[k] >= 0 && d1[k] < a.dp);
                                    const double p = s_potd[(g * kTmaRows + r) * kTmaDp + d1[k]];
                                    nw[k] = stdp_apply<WT>(w[k], stdp_dw(sj[k], p, ef[k] != WT(0), depj[k]), wmin, wmax);
                                }
                            } else if (h & 1ull) {
                                // unit delay: s_pre is the row's bit (warp-uniform branch);
                                // dw = fma(s_post, pot, -dep) rounds pot - dep once like the
                                // reference's dw -= dep, and is exactly -dep when s_post = 0
#pragma unroll
                                for (int k = 0; k < VEC; ++k)
                                    nw[k] = stdp_apply<WT>(w[k], fma(sjd[k], rec.pot, ndep[k]), wmin, wmax);
                            } else {
#pragma unroll
                                for (int k = 0; k < VEC; ++k) nw[k] = stdp_apply<WT>(w[k], sjd[k] * rec.pot, wmin, wmax);
                            }
                            if (kind == kRowAllButSelf) {
                                const int selfk = row - gc0;
#pragma unroll
                                for (int k = 0; k < VEC; ++k) nw[k] = (selfk == k) ? w[k] : nw[k];
                            } else if (kind == kRowMixed) {
                                const uint32_t mv =
                                    __ldg(a.mask + static_cast<int64_t>(row) * (a.pitch >> 5) + (c0 >> 5)) >> (c0 & 31);
#pragma unroll
                                for (int k = 0; k < VEC; ++k) nw[k] = ((mv >> k) & 1u) ? nw[k] : w[k];
                            }
                            V out = wv;
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
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
#pragma unroll
                for (int k = 0; k < VEC; ++k) acc[k] += static_cast<double>(grp[k]);
            }
            if (kTmaHalves > 1) {
                double* x = s_xch + ((warp & 7) * 32 + lane) * VEC;
                if (rh == 1) {
#pragma unroll
                    for (int k = 0; k < VEC; ++k) x[k] = acc[k];
                }
                tma_consumer_bar();
                if (rh == 0 && in_tile) {
#pragma unroll
                    for (int k = 0; k < VEC; ++k)
                        if (c0 + k < a.nl) a.partial[static_cast<int64_t>(chunk) * a.nl + c0 + k] = acc[k] + x[k];
                }
                tma_consumer_bar();  // x is rewritten by the next item
            } else if (in_tile) {
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    if (c0 + k < a.nl) a.partial[static_cast<int64_t>(chunk) * a.nl + c0 + k] = acc[k];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(freeb + b);
        }
    }
    if (blockIdx.x == 0 && tid == 0) *a.d_step += 1;
}

size_t dense_tma_smem(int tile_w, bool f64, bool delay, bool stdp, int rows) {
    const size_t esz = f64 ? 8 : 4;
    return static_cast<size_t>(kTmaStages) * kTmaRows * tile_w * (esz + (delay ? 1 : 0)) + (2 * kTmaStages + 6) * 8 +
           2 * static_cast<size_t>(rows + kTmaRows) * (sizeof(TmaRec) + ((delay && stdp) ? kTmaDp * 8 : 0)) +
           static_cast<size_t>(kTmaXchDoubles) * 8;
}

int smem_optin() {
    int dev = 0, optin = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
    return optin;
}

}  // namespace

int dense_vec(bool f64) { return f64 ? 2 : 4; }

int dense_tma_max_dp() { return kTmaDp; }

// Longest item row list (a multiple of 32, <= kTmaListMax) whose two list
// buffers fit next to the ring in the opt-in shared memory; 0 if even 32 rows
// do not fit.
int dense_tma_max_rows(int tile_w, bool f64, bool delay, bool stdp) {
    const size_t optin = static_cast<size_t>(smem_optin());
    for (int rows = kTmaListMax; rows >= 32; rows -= 32)
        if (dense_tma_smem(tile_w, f64, delay, stdp, rows) + 1024 <= optin) return rows;  // + static smem
    return 0;
}

template <typename WT, bool STDP, bool DELAY>
static void dense_tma_go(const DenseArgs& a, int grid, cudaStream_t s) {
    const size_t smem = dense_tma_smem(a.tile_w, sizeof(WT) == 8, DELAY, STDP, a.rows_per_chunk);
    static size_t configured = 0;
    auto kern = k_dense_tma<WT, STDP, DELAY>;
    if (configured < smem) {
        check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
              "k_dense_tma smem attribute");
        configured = smem;
    }
    kern<<<grid, kTmaThreads, smem, s>>>(a);
}

void launch_dense_tma(const DenseArgs& a, bool f64, bool stdp, bool delay, int grid, cudaStream_t s) {
#define SNB_T(WT)                                                                   \
    do {                                                                            \
        if (stdp) {                                                                 \
            if (delay) dense_tma_go<WT, true, true>(a, grid, s);                    \
            else dense_tma_go<WT, true, false>(a, grid, s);                         \
        } else {                                                                    \
            if (delay) dense_tma_go<WT, false, true>(a, grid, s);                   \
            else dense_tma_go<WT, false, false>(a, grid, s);                        \
        }                                                                           \
    } while (0)
    if (f64) SNB_T(double);
    else SNB_T(float);
#undef SNB_T
    check(cudaGetLastError(), "k_dense_tma");
}
int dense_threads() { return kThreads; }
template <typename WT, bool STDP, bool DELAY, bool EXACT>
static void dense_go(const DenseArgs& a, int grid, cudaStream_t s) {
    if (EXACT) k_dense_sweep<WT, STDP, DELAY, true><<<grid, kThreads, 0, s>>>(a);
    else k_dense_stream<WT, STDP, DELAY><<<grid, kThreads, 0, s>>>(a);
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

}  // namespace snb
