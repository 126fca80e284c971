// Sparse (blocked CSC) sweeps: k_sparse_pull, k_sparse_count (+ its setup-time
// bank-aware list order), k_sparse_exact, k_sparse_stream and the opt-in k_sparse_tma.
#include "kernels_common.cuh"

#include <cstdlib>
#include <string>

namespace snb {

namespace {

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

// PS: the pre block's pot^(d) traces are staged in shared memory (a.pot_staged);
// a compile-time flag so their loads are LDS, free to move past the weight
// stores (through one generic pointer for both cases every pot load was an
// LD.E.64 ordered after the previous chunk's weight store)
template <typename WT, bool STDP, int HB, int SUB, bool DICT, bool PS = false>
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
    // STDP: the block's pot^(d) traces, [pcount][dp], staged next to the history
    // (the per-synapse lookup would otherwise be a random global gather)
    double* s_pot = reinterpret_cast<double*>(smem_raw + hbytes);
    if (STDP && PS) {
        const double* src = a.pot + static_cast<int64_t>(pre0) * a.dp;
        for (int k = tid; k < pcount * a.dp; k += kThreads) s_pot[k] = __ldcg(src + k);
    }
    __syncthreads();
    const uint32_t* sbits = reinterpret_cast<const uint32_t*>(smem_raw);
    const HT* shist = reinterpret_cast<const HT*>(smem_raw);
    const bool uniform = DICT && a.dict_size == 2;  // {w, 0.0 padding}: every synapse carries w

    const WT wmin = static_cast<WT>(a.w_min), wmax = static_cast<WT>(a.w_max);
    const double* pot = (STDP && PS) ? s_pot : a.pot + static_cast<int64_t>(pre0) * a.dp;
    const double* dep = a.dep;
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
    constexpr int UL = DICT ? (SUB <= 8 ? SNB_SPARSE_UL : 4) : (SUB <= 2 ? 4 : 2);
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
            double depp = 0.0;
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
                    // the 4 history bits and pot^(d) traces first (all loads in flight together)
                    uint32_t ev[4];
                    double ptv[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t m = ms[k];
                        const int pl = static_cast<int>(m & 0xffffu);
                        const int d1 = static_cast<int>((m >> 16) & 63u);
                        SNB_DCHECK(pl <= a.pb && (!STDP || !((m >> 22) & 1u) || (pl < pcount && d1 < a.dp)));
                        if (HB == 1) ev[k] = (sbits[pl >> 5] >> (pl & 31)) & 1u;
                        else ev[k] = static_cast<uint32_t>((shist[pl] >> d1) & 1u);
                        // only spiking posts read pot^(d), only plastic synapses index it
                        ptv[k] = (!DICT && STDP && sp && ((m >> 22) & 1u)) ? pot[pl * a.dp + d1] : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t m = ms[k];
                        const uint32_t e = ev[k];
                        WT w = wv[u][k];
                        if (!DICT && STDP && a.plastic_on && ((m >> 22) & 1u)) {
                            const double pt = ptv[k];
                            const WT nw = stdp_apply<WT>(w, stdp_dw(sp, pt, e != 0u, depp), wmin, wmax);
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


// Joint bank schedule of the 32/SUB lists one warp of k_sparse_count reads
// together (posts P*k .. P*k+P-1 of one pre block; SUB = 4, 8, 16).  The lists
// are scheduled LDS by LDS: for slot g (row g/4, word g%4) every active lane of
// every post (posts in rotating order) takes an entry of its own list from the
// bank with the lowest load in this LDS so far, ties broken by the bank's
// remaining entries over the whole group (drain the heavy banks early).  The
// per-list bank-sorted deal above leaves the 32/SUB posts of a warp colliding
// with each other (cfg4: 2.59 wavefronts per LDS, measured and simulated);
// the joint schedule simulates to 1.60 against a lower bound of ~1.5 set by
// the group's bank histogram.  In place: meta -> tmp (bucketed) -> meta.
template <int SUB>
__global__ void k_sparse_bank_joint(uint32_t* meta, uint32_t* tmp, const int64_t* off, int nblocks, int nl,
                                    int hbits) {
    constexpr int P = 32 / SUB, ROW = 4 * SUB;
    const int groups = (nl + P - 1) / P;
    const int64_t G = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (G >= static_cast<int64_t>(groups) * nblocks) return;
    const int b = static_cast<int>(G / groups), k = static_cast<int>(G % groups);
    const int np = min(P, nl - P * k);
    const int64_t* o = off + static_cast<int64_t>(b) * nl + P * k;
    int cnt[P][32], cur[P][32], tot[32], len[P], rows[P], last[P];
    for (int j = 0; j < 32; ++j) tot[j] = 0;
    int gmax = 0;
    for (int i = 0; i < P; ++i) {
        for (int j = 0; j < 32; ++j) cnt[i][j] = 0;
        len[i] = i < np ? static_cast<int>(o[i + 1] - o[i]) : 0;
        rows[i] = (len[i] + ROW - 1) / ROW;
        last[i] = len[i] > 0 ? (len[i] - ROW * (rows[i] - 1)) / 4 : 0;  // lanes with a full last row
        gmax = max(gmax, 4 * rows[i]);
        if (i >= np) continue;
        for (int64_t q = o[i]; q < o[i + 1]; ++q) cnt[i][sp_bank(meta[q], hbits)] += 1;
        int acc = 0;
        for (int j = 0; j < 32; ++j) {
            cur[i][j] = acc;
            acc += cnt[i][j];
            tot[j] += cnt[i][j];
        }
        for (int64_t q = o[i]; q < o[i + 1]; ++q) {  // bucket by bank into tmp
            const uint32_t m = meta[q];
            tmp[o[i] + cur[i][sp_bank(m, hbits)]++] = m;
        }
        for (int j = 0; j < 32; ++j) cur[i][j] -= cnt[i][j];  // back to the bucket starts
    }
    for (int g = 0; g < gmax; ++g) {
        int load[32];
        for (int j = 0; j < 32; ++j) load[j] = 0;
        for (int r = 0; r < P; ++r) {
            const int i = (g + r) % P;
            if (i >= np) continue;
            const int slots_full = 4 * rows[i], slots_part = 4 * (rows[i] - 1);
            for (int sl = 0; sl < SUB; ++sl) {
                if (g >= (sl < last[i] ? slots_full : slots_part)) continue;
                int best = -1;
                for (int j = 0; j < 32; ++j) {
                    if (cnt[i][j] == 0) continue;
                    if (best < 0 || load[j] < load[best] || (load[j] == load[best] &&
                        (tot[j] > tot[best] || (tot[j] == tot[best] && cnt[i][j] > cnt[i][best]))))
                        best = j;
                }
                const uint32_t m = tmp[o[i] + cur[i][best]++];
                cnt[i][best] -= 1;
                tot[best] -= 1;
                load[best] += 1;
                meta[o[i] + (g >> 2) * ROW + 4 * sl + (g & 3)] = m;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 16-bit one-weight lists (k_sparse_count16).  A pre block of kC16Pres = 4 x
// 4095 pres is cut into 4 segments; each (block, post) list is regrouped by
// segment, every segment padded to whole 16-byte chunks of 8 entries.  The
// staged history image (uint16 per pre) puts segment s at slots [4096 s,
// 4096 s + 4096) with one zero slot (c16_zero_slot).  An entry addresses the 32-bit
// PAIR of slots holding its pre and a rotation that brings the pre's bit d-1
// (bit j of the pair) to bit 31:
//   entry = (slot >> 1) << 5 | (j + 1) & 31,   j = 16 (slot & 1) + d - 1, d <= 16
// so the test is one wrap-mode funnel shift by the entry itself (the shift
// unit keeps its low 5 bits; no masking of the delay field) and one shift by
// 31 (the ALU pipe is the limit: 77% busy; moving the address arithmetic and
// the accumulation onto the FMA pipe as IMAD.HI with run-time multipliers
// measured 0.420 / 0.452 ms against 0.421).  Padding entries read the segment's
// zero slot.  A list descriptor {first
// chunk, E1 | E2 << 8 | E3 << 16 | C << 24} carries the cumulative chunk
// counts of the segments (C <= 255 chunks); a chunk's segment is (c >= E1) +
// (c >= E2) + (c >= E3).  Half the bytes of the 32-bit meta words the other
// count kernel streams; same counts.
constexpr int kC16SegPres = 4095;
constexpr int kC16Pres = 4 * kC16SegPres;

// Zero slot of segment s: 4095 - 16 s, so the padding of the 4 segments reads
// 4 different banks (31, 23, 15, 7); pre offset j of the segment sits in slot
// j + (j >= zero slot).
__host__ __device__ constexpr int c16_zero_slot(int s) { return 4095 - 16 * s; }

// Stage one pre block's history: put(k, h) for every slot k of NSEG segments
// (h = the pre's 16-bit delay history, 0 for the zero slots and past the end).
template <int NSEG, typename Put>
__device__ __forceinline__ void c16_stage_slots(const SparseArgs& a, int pre0, int pcount, Put&& put) {
    constexpr int K = NSEG * 4096;
    constexpr int R = 8;  // slots per thread per pass, all loads issued before any use
    if (a.hist16) {
        // folded history: h = (history after step t - 1) << 1 | s[t]; the first CTA
        // of the pre block commits it to the other parity buffer for step t + 1
        const int t = *a.step_in;
        const uint32_t* bits = a.bits;
        if (a.flags) {  // p2p: every rank's step-t words have landed in exchange buffer t & 1
            if (threadIdx.x == 0) {
                const uint64_t g0 = globaltimer_ns();
                for (int q = 0; q < a.world; ++q)
                    while (ld_acquire_sys(a.flags + q) <= t) {
                        if (globaltimer_ns() - g0 > 30ull * 1000000000ull) {  // 30 s: a peer died
                            atomicExch(a.error, 1);
                            break;
                        }
                        __nanosleep(200);
                    }
            }
            __syncthreads();
            bits = a.xbits + static_cast<int64_t>(t & 1) * a.xstride;
        }
        const uint16_t* hin = a.hist16 + static_cast<int64_t>(t & 1) * a.n;
        uint16_t* hout = a.hist16 + static_cast<int64_t>((t + 1) & 1) * a.n;
        const bool commit = blockIdx.x == 0;
        for (int k0 = threadIdx.x; k0 < K; k0 += R * blockDim.x) {
            uint32_t hv[R], bw[R];
            int gs[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int k = k0 + r * blockDim.x;
                const int s = k >> 12, slot = k & 4095, z = c16_zero_slot(s);
                const int pre = s * kC16SegPres + slot - (slot > z);
                gs[r] = (k < K && slot != z && pre < pcount) ? pre0 + pre : -1;
                hv[r] = gs[r] >= 0 ? __ldcg(hin + gs[r]) : 0u;
                bw[r] = gs[r] >= 0 ? __ldcg(bits + (gs[r] >> 5)) : 0u;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int k = k0 + r * blockDim.x;
                const uint16_t h = gs[r] >= 0 ? static_cast<uint16_t>((hv[r] << 1) | ((bw[r] >> (gs[r] & 31)) & 1u)) : 0;
                if (k < K) put(k, h);
                if (commit && gs[r] >= 0) hout[gs[r]] = h;
            }
        }
        return;
    }
    for (int k0 = threadIdx.x; k0 < K; k0 += R * blockDim.x) {
        uint32_t hv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int k = k0 + r * blockDim.x;
            const int s = k >> 12, slot = k & 4095, z = c16_zero_slot(s);
            const int pre = s * kC16SegPres + slot - (slot > z);
            hv[r] = (k < K && slot != z && pre < pcount) ? __ldcg(a.hist_lo + pre0 + pre) : 0u;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (k0 + r * blockDim.x < K) put(k0 + r * blockDim.x, static_cast<uint16_t>(hv[r]));
    }
}

__device__ __forceinline__ void c16_stage(const SparseArgs& a, int pre0, int pcount, uint16_t* sh) {
    c16_stage_slots<4>(a, pre0, pcount, [&](int k, uint16_t h) { sh[k] = h; });
}

#ifndef SNB_C16_MINB
#define SNB_C16_MINB 4
#endif
// chunk loads per lane per batch; cfg4 (tools/ab_c16.sh): SUB 8: UL 2 0.527 ms, 3 0.499,
// 4 0.486, 5 0.504; SUB 4: UL 5 0.474, 6 0.452, 7 0.458, 8 0.474; SUB 2: UL 6 0.568
#ifdef SNB_C16_UL
#define SNB_C16_UL_OF(SUB) SNB_C16_UL
#else
#define SNB_C16_UL_OF(SUB) ((SUB) <= 4 ? 6 : 4)
#endif
#ifndef SNB_C16_PIPE
#define SNB_C16_PIPE 0
#endif

// Count the delivering entries of one loaded batch (UL chunks of lane sl).
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

template <int SUB, int UL>
__device__ __forceinline__ uint32_t c16_count_batch(const uint4 (&m4)[UL], int c0, int C, int E1, int E2, int E3,
                                                    const uint16_t* shist) {
    uint32_t cnt = 0;
#pragma unroll
    for (int u = 0; u < UL; ++u) {
        const int c = c0 + u * SUB;
        if (c < C) {
            SNB_DCHECK(E1 <= E2 && E2 <= E3 && E3 <= C && C <= 255);
            const uint16_t* sh = shist + (((c >= E1) + (c >= E2) + (c >= E3)) << 12);
            const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sh));
            const uint32_t ws[4] = {m4[u].x, m4[u].y, m4[u].z, m4[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t x = ws[k];
                const uint32_t h0 = lds_u32(base + ((x >> 3) & 0x1ffcu));   // pair (x >> 5) & 0x7ff
                const uint32_t h1 = lds_u32(base + ((x >> 19) & 0x1ffcu));  // pair x >> 21
                cnt += (__funnelshift_r(h0, h0, x) >> 31) + (__funnelshift_r(h1, h1, x >> 16) >> 31);
            }
        }
    }
    return cnt;
}

template <int SUB, int UL>
__device__ __forceinline__ void c16_load_batch(uint4 (&m4)[UL], const uint4* src, int c0, int C) {
#pragma unroll
    for (int u = 0; u < UL; ++u)
        if (c0 + u * SUB < C) m4[u] = __ldcs(src + c0 + u * SUB);
}

// NT threads per CTA: a CTA stages its pre block's 32 KB history once for
// NT / SUB posts at a time; bigger CTAs amortise the stage over more posts
// (what a post partition, with a G-th of the posts per block, needs).
template <typename WT, int SUB, int NT = kThreads>
__global__ void __launch_bounds__(NT, NT == kThreads ? SNB_C16_MINB : 1024 / NT)
    k_sparse_count16(SparseArgs a, const uint2* desc, const uint4* ent) {
    __shared__ __align__(16) uint16_t shist[4 * 4096];
    const int b = blockIdx.y;
    const int pre0 = b * kC16Pres;
    const int pcount = min(kC16Pres, a.n - pre0);
    const int tid = threadIdx.x;
    c16_stage(a, pre0, pcount, shist);
    __syncthreads();
    const WT w0 = static_cast<const WT*>(a.wdict)[0];
    const int p0 = blockIdx.x * a.posts_per_cta;
    const int p1 = min(a.nl, p0 + a.posts_per_cta);
    constexpr int PER_WARP = 32 / SUB;
    constexpr int UL = SNB_C16_UL_OF(SUB);
    constexpr int STEP = SUB * UL;
    const int warp = tid >> 5, lane = tid & 31;
    const int sg = lane / SUB, sl = lane % SUB;
    const int stride = (NT / 32) * PER_WARP;
    const uint2* db = desc + static_cast<int64_t>(b) * a.nl;
    int p = p0 + warp * PER_WARP + sg;
    uint2 d = make_uint2(0u, 0u);
    if (p < p1) d = __ldg(db + p);
#if SNB_C16_PIPE
    // software pipeline across posts: the next post's first batch is in flight
    // while the current one is counted
    uint4 mc[UL];
    c16_load_batch<SUB, UL>(mc, ent + d.x, sl, static_cast<int>(d.y >> 24));
    uint2 dn = make_uint2(0u, 0u);
    if (p + stride < p1) dn = __ldg(db + p + stride);
#endif
    for (int pbase = p0 + warp * PER_WARP; pbase < p1; pbase += stride) {  // warp-uniform trip count
        const bool valid = p < p1;
        const int pn = p + stride;
#if SNB_C16_PIPE
        uint4 mn[UL];
        c16_load_batch<SUB, UL>(mn, ent + dn.x, sl, static_cast<int>(dn.y >> 24));
        uint2 dnn = make_uint2(0u, 0u);
        if (pn + stride < p1) dnn = __ldg(db + pn + stride);
#else
        uint2 dn = make_uint2(0u, 0u);
        if (pn < p1) dn = __ldg(db + pn);
#endif
        int cnt = 0;
        if (valid) {
            const int C = static_cast<int>(d.y >> 24);
            const int E1 = static_cast<int>(d.y & 255u), E2 = static_cast<int>((d.y >> 8) & 255u),
                      E3 = static_cast<int>((d.y >> 16) & 255u);
            const uint4* src = ent + d.x;
#if SNB_C16_PIPE
            cnt = static_cast<int>(c16_count_batch<SUB, UL>(mc, sl, C, E1, E2, E3, shist));
            for (int c0 = sl + STEP; c0 < C; c0 += STEP) {
#else
            for (int c0 = sl; c0 < C; c0 += STEP) {
#endif
                uint4 m4[UL];
                c16_load_batch<SUB, UL>(m4, src, c0, C);
                cnt += static_cast<int>(c16_count_batch<SUB, UL>(m4, c0, C, E1, E2, E3, shist));
            }
        }
#pragma unroll
        for (int o = SUB / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (valid && sl == 0)
            a.partial16[static_cast<int64_t>(b) * a.nl + p] = static_cast<uint16_t>(cnt);
        p = pn;
        d = dn;
#if SNB_C16_PIPE
        dn = dnn;
#pragma unroll
        for (int u = 0; u < UL; ++u) mc[u] = mn[u];
#endif
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *a.d_step += 1;
}

// Byte-image variant (k_sparse_count8): the same segmented lists over 3
// segments (a pre block of kC8Pres = 3 x 4095 pres), but the staged image
// holds one BYTE per (slot, delay) -- byte 16 slot + d - 1 of a segment's 64 KB
// is bit d - 1 of the slot's history -- and an entry is that byte offset:
//   entry = slot << 4 | (d - 1)
// so the test is one LDS.U8 whose value is added as is: per 32-bit word of two
// entries one mask, one shift-add (LEA.HI) and one 3-input add instead of the
// two address extractions, two funnel shifts and two shift-adds of the pair
// encoding.  192 KB of image: one CTA of 1024 threads per SM.
constexpr int kC8Segs = 3;
constexpr int kC8Pres = kC8Segs * kC16SegPres;
constexpr int kC8ImageBytes = kC8Segs * 65536;

// 4 history bits -> 4 bytes of 0/1 (bit i of n to byte i)
__device__ __forceinline__ uint32_t c8_spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

template <int SUB, int UL>
__device__ __forceinline__ uint32_t c8_count_batch(const uint4 (&m4)[UL], int c0, int C, int E1, int E2,
                                                   const uint8_t* img) {
    uint32_t cnt = 0;
#pragma unroll
    for (int u = 0; u < UL; ++u) {
        const int c = c0 + u * SUB;
        if (c < C) {
            SNB_DCHECK(E1 <= E2 && E2 <= C && C <= 255);
            const uint8_t* seg = img + (((c >= E1) + (c >= E2)) << 16);
            const uint32_t ws[4] = {m4[u].x, m4[u].y, m4[u].z, m4[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) cnt += seg[ws[k] & 0xffffu] + seg[ws[k] >> 16];
        }
    }
    return cnt;
}

template <typename WT, int SUB, int NT>
__global__ void __launch_bounds__(NT, 1) k_sparse_count8(SparseArgs a, const uint2* desc, const uint4* ent) {
    extern __shared__ __align__(16) uint8_t c8img[];
    const int b = blockIdx.y;
    const int pre0 = b * kC8Pres;
    const int pcount = min(kC8Pres, a.n - pre0);
    const int tid = threadIdx.x;
    c16_stage_slots<kC8Segs>(a, pre0, pcount, [&](int k, uint16_t h) {
        const uint32_t x = h;
        *reinterpret_cast<uint4*>(c8img + 16 * k) =
            make_uint4(c8_spread4(x & 15u), c8_spread4((x >> 4) & 15u), c8_spread4((x >> 8) & 15u), c8_spread4(x >> 12));
    });
    __syncthreads();
    const WT w0 = static_cast<const WT*>(a.wdict)[0];
    const int p0 = blockIdx.x * a.posts_per_cta;
    const int p1 = min(a.nl, p0 + a.posts_per_cta);
    constexpr int PER_WARP = 32 / SUB;
    constexpr int UL = SNB_C16_UL_OF(SUB);
    const int warp = tid >> 5, lane = tid & 31;
    const int sg = lane / SUB, sl = lane % SUB;
    const int stride = (NT / 32) * PER_WARP;
    const uint2* db = desc + static_cast<int64_t>(b) * a.nl;
    const uint32_t lt = (1u << lane) - 1u;  // lanes below this one
    int p = p0 + warp * PER_WARP + sg;
    uint2 d = make_uint2(0u, 0u);
    if (p < p1) d = __ldg(db + p);
    for (int pbase = p0 + warp * PER_WARP; pbase < p1; pbase += stride) {  // warp-uniform trip count
        const bool valid = p < p1;
        const int pn = p + stride;
        uint2 dn = make_uint2(0u, 0u);
        if (pn < p1) dn = __ldg(db + pn);
        // the warp's P posts share one chunk stream, row-major: row r holds chunks
        // SUB r .. SUB r + SUB - 1 of every post that has them, in post order, so a
        // row's loads are one contiguous run of up to 512 bytes
        const int C = valid ? static_cast<int>(d.y >> 24) : 0;
        const int E1 = static_cast<int>(d.y & 255u), E2 = static_cast<int>((d.y >> 8) & 255u);
        const int rows = (static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(C))) + SUB - 1) / SUB;
        uint32_t pos = __shfl_sync(0xffffffffu, d.x, 0);  // the group's first chunk
        uint32_t cnt = 0;
        for (int r0 = 0; r0 < rows; r0 += UL) {
            const int c0 = r0 * SUB + sl;
            uint4 m4[UL];
#pragma unroll
            for (int u = 0; u < UL; ++u) {
                const bool act = c0 + u * SUB < C;
                const uint32_t A = __ballot_sync(0xffffffffu, act);
                if (act) m4[u] = __ldcs(ent + pos + __popc(A & lt));
                pos += __popc(A);
            }
            cnt += c8_count_batch<SUB, UL>(m4, c0, C, E1, E2, c8img);
        }
#pragma unroll
        for (int o = SUB / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (valid && sl == 0)
            a.partial16[static_cast<int64_t>(b) * a.nl + p] = static_cast<uint16_t>(cnt);
        p = pn;
        d = dn;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *a.d_step += 1;
}

// Setup: entries per segment of every 32-bit one-weight list (padding, pre slot
// pb, skipped) -> cnt[list] = n0 | n1 << 16 (x) and n2 | n3 << 16 (y).
__global__ void k_c16_count(const uint32_t* meta, const int64_t* off, int64_t lists, int pb, uint2* cnt) {
    const int64_t L = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (L >= lists) return;
    uint32_t n[4] = {0, 0, 0, 0};
    for (int64_t q = off[L]; q < off[L + 1]; ++q) {
        const uint32_t pl = meta[q] & 0xffffu;
        if (static_cast<int>(pl) == pb) continue;
        n[pl / kC16SegPres] += 1;
    }
    cnt[L] = make_uint2(n[0] | (n[1] << 16), n[2] | (n[3] << 16));
}

// Setup: the joint per-warp bank schedule of k_sparse_bank_joint, per segment:
// the P = 32/SUB lists one warp reads together are filled LDS by LDS (slot g =
// chunk row g/8, entry g%8); a lane takes, from its chunk's segment, an entry
// in the bank with the lowest load in this LDS so far (ties: most entries left
// in the group, then in the list), padding (the zero slot) once the segment is empty.
// host/device helpers of the fill (the fill also runs on the host in tools/c16_fill_check)
__host__ __device__ __forceinline__ int c16_popc(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __popc(x);
#else
    return __builtin_popcount(x);
#endif
}
__host__ __device__ __forceinline__ int c16_ffs(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __ffs(static_cast<int>(x));
#else
    return __builtin_ffs(static_cast<int>(x));
#endif
}
__host__ __device__ __forceinline__ int c16_min(int a, int b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int c16_max(int a, int b) { return a > b ? a : b; }

// BYTES: the byte-image encoding of k_sparse_count8 (slot << 4 | d - 1, bank
// (4 slot + (d - 1) / 4) mod 32) instead of the pair encoding.
__host__ __device__ __forceinline__ int c16_bank(bool bytes, int slot, int dm1) {
    return bytes ? ((slot << 2) + (dm1 >> 2)) & 31 : (slot >> 1) & 31;
}

template <int SUB, bool BYTES>
__host__ __device__ void c16_fill_group(int64_t G, const uint32_t* meta, uint32_t* tmp, const int64_t* off,
                                        const uint2* desc, int nl, int pb, uint16_t* out) {
    constexpr int P = 32 / SUB;
    const int groups = (nl + P - 1) / P;
    const int b = static_cast<int>(G / groups), k = static_cast<int>(G % groups);
    const int np = c16_min(P, nl - P * k);
    const int64_t L0 = static_cast<int64_t>(b) * nl + P * k;
    uint16_t cnt[P][4][32], cur[P][4][32];
    int tot[32], C[P], E[P][3];
    for (int j = 0; j < 32; ++j) tot[j] = 0;
    int gmax = 0;
    for (int i = 0; i < P; ++i) {
        for (int s = 0; s < 4; ++s)
            for (int j = 0; j < 32; ++j) cnt[i][s][j] = 0;
        C[i] = 0;
        E[i][0] = E[i][1] = E[i][2] = 0;
        if (i >= np) continue;
        const uint2 d = desc[L0 + i];
        C[i] = static_cast<int>(d.y >> 24);
        E[i][0] = static_cast<int>(d.y & 255u);
        E[i][1] = static_cast<int>((d.y >> 8) & 255u);
        E[i][2] = static_cast<int>((d.y >> 16) & 255u);
        gmax = c16_max(gmax, 8 * ((C[i] + SUB - 1) / SUB));
        const int64_t o0 = off[L0 + i], o1 = off[L0 + i + 1];
        for (int64_t q = o0; q < o1; ++q) {
            const int pl = static_cast<int>(meta[q] & 0xffffu);
            if (pl == pb) continue;
            const int s = pl / kC16SegPres;
            const int low = pl - s * kC16SegPres;
            cnt[i][s][c16_bank(BYTES, low + (low >= c16_zero_slot(s)), static_cast<int>((meta[q] >> 16) & 15u))] += 1;
        }
        int acc = 0;
        for (int s = 0; s < 4; ++s)
            for (int j = 0; j < 32; ++j) {
                cur[i][s][j] = static_cast<uint16_t>(acc);
                acc += cnt[i][s][j];
                tot[j] += cnt[i][s][j];
            }
        for (int64_t q = o0; q < o1; ++q) {  // bucket by (segment, bank) into tmp
            const uint32_t m = meta[q];
            const int pl = static_cast<int>(m & 0xffffu);
            if (pl == pb) continue;
            const int s = pl / kC16SegPres;
            const int slot = pl - s * kC16SegPres + (pl - s * kC16SegPres >= c16_zero_slot(s));
            const uint32_t dm1 = (m >> 16) & 15u;
            const uint32_t j = static_cast<uint32_t>(slot & 1) * 16u + dm1;  // bit of the pair
            tmp[o0 + cur[i][s][c16_bank(BYTES, slot, static_cast<int>(dm1))]++] =
                BYTES ? static_cast<uint32_t>(slot) << 4 | dm1 : static_cast<uint32_t>(slot >> 1) << 5 | ((j + 1u) & 31u);
        }
        for (int s = 0; s < 4; ++s)
            for (int j = 0; j < 32; ++j) cur[i][s][j] = static_cast<uint16_t>(cur[i][s][j] - cnt[i][s][j]);
    }
    for (int g = 0; g < gmax; ++g) {
        int load[32];
        for (int j = 0; j < 32; ++j) load[j] = 0;
        const int row = g >> 3, e = g & 7;
        // BYTES: chunks of row `row` start after the group's earlier rows, post i's
        // after the row's chunks of posts < i (k_sparse_count8's stream order)
        int64_t rbase = 0;
        int before[P];
        if (BYTES) {
            const int64_t g0 = desc[L0].x;
            int64_t prior = 0;
            for (int rr = 0; rr < row; ++rr)
                for (int i = 0; i < np; ++i) prior += c16_min(SUB, c16_max(0, C[i] - SUB * rr));
            int acc = 0;
            for (int i = 0; i < P; ++i) {
                before[i] = acc;
                if (i < np) acc += c16_min(SUB, c16_max(0, C[i] - SUB * row));
            }
            rbase = g0 + prior;
        }
        // BYTES: the LDS's lanes get pairwise different banks where their pools
        // allow it -- a maximum bipartite matching of lanes to banks (augmenting
        // paths, most constrained lanes first, abundant banks tried first), the
        // banks of padding lanes excluded; unmatched lanes fall back to the
        // least-loaded bank below
        int asg[P][SUB];
        if (BYTES) {
            int li[32], ls[32], order[32], matchB[32];
            uint32_t opt[32], fixed = 0;
            int nlanes = 0;
            for (int i = 0; i < P; ++i)
                for (int sl = 0; sl < SUB; ++sl) {
                    asg[i][sl] = -1;
                    const int c = row * SUB + sl;
                    if (i >= np || c >= C[i]) continue;
                    const int s = (c >= E[i][0]) + (c >= E[i][1]) + (c >= E[i][2]);
                    uint32_t m = 0;
                    for (int j = 0; j < 32; ++j)
                        if (cnt[i][s][j]) m |= 1u << j;
                    if (!m) {
                        fixed |= 1u << c16_bank(true, c16_zero_slot(s), 4 * s);
                        continue;
                    }
                    li[nlanes] = i;
                    ls[nlanes] = sl;
                    opt[nlanes] = m;
                    order[nlanes] = nlanes;
                    ++nlanes;
                }
            for (int l = 0; l < nlanes; ++l) {
                if (opt[l] & ~fixed) opt[l] &= ~fixed;
                for (int k = l; k > 0 && c16_popc(opt[order[k]]) < c16_popc(opt[order[k - 1]]); --k) {
                    const int t = order[k];
                    order[k] = order[k - 1];
                    order[k - 1] = t;
                }
            }
            for (int j = 0; j < 32; ++j) matchB[j] = -1;
            for (int q = 0; q < nlanes; ++q) {
                int stk[33], via[33], sp = 1;
                uint32_t rem[33], vis = 0;
                stk[0] = order[q];
                rem[0] = opt[order[q]];
                while (sp > 0) {
                    const uint32_t m = rem[sp - 1] & ~vis;
                    if (!m) {
                        --sp;
                        continue;
                    }
                    int b = -1;
                    for (uint32_t mm = m; mm; mm &= mm - 1) {
                        const int j = c16_ffs(mm) - 1;
                        if (b < 0 || tot[j] > tot[b]) b = j;
                    }
                    rem[sp - 1] = m & ~(1u << b);
                    vis |= 1u << b;
                    via[sp - 1] = b;
                    if (matchB[b] < 0) {
                        for (int k = 0; k < sp; ++k) matchB[via[k]] = stk[k];
                        break;
                    }
                    stk[sp] = matchB[b];
                    rem[sp] = opt[matchB[b]];
                    ++sp;
                }
            }
            for (int j = 0; j < 32; ++j) {
                if (matchB[j] >= 0) asg[li[matchB[j]]][ls[matchB[j]]] = j;
                load[j] += (matchB[j] >= 0) + static_cast<int>((fixed >> j) & 1u);
            }
        }
        // matched lanes take their entries first (pass 0), then the rest
        for (int pass = BYTES ? 0 : 1; pass < 2; ++pass)
        for (int r = 0; r < P; ++r) {
            const int i = (g + r) % P;
            if (i >= np) continue;
            const int64_t o0 = off[L0 + i];
            for (int sl = 0; sl < SUB; ++sl) {
                const int c = row * SUB + sl;
                if (c >= C[i]) continue;
                if (BYTES && (pass == 0) != (asg[i][sl] >= 0)) continue;
                const int64_t base = BYTES ? (rbase + before[i] + sl - c) * 8 : static_cast<int64_t>(desc[L0 + i].x) * 8;
                const int s = (c >= E[i][0]) + (c >= E[i][1]) + (c >= E[i][2]);
                int best = BYTES ? asg[i][sl] : -1;
                const bool matched = best >= 0;
                for (int j = 0; j < 32 && !matched; ++j) {
                    if (cnt[i][s][j] == 0) continue;
                    if (best < 0 || load[j] < load[best] ||
                        (load[j] == load[best] && (tot[j] > tot[best] ||
                                                   (tot[j] == tot[best] && cnt[i][s][j] > cnt[i][s][best]))))
                        best = j;
                }
                // padding: the segment's zero slot (pairs: upper half of its pair, bit 16;
                // bytes: byte 4 s, bank 28 + s)
                const int z = c16_zero_slot(s);
                uint16_t v = BYTES ? static_cast<uint16_t>(z << 4 | (4 * s)) : static_cast<uint16_t>((z >> 1) << 5 | 17);
                if (best >= 0) {
                    v = static_cast<uint16_t>(tmp[o0 + cur[i][s][best]]);
                    cur[i][s][best] += 1;
                    cnt[i][s][best] -= 1;
                    tot[best] -= 1;
                    if (!(BYTES && pass == 0)) load[best] += 1;
                } else if (!BYTES) {
                    load[c16_bank(BYTES, z, 4 * s)] += 1;
                }
                out[base + static_cast<int64_t>(c) * 8 + e] = v;
            }
        }
    }
}

template <int SUB, bool BYTES>
__global__ void k_c16_fill(const uint32_t* meta, uint32_t* tmp, const int64_t* off, const uint2* desc, int nblocks,
                           int nl, int pb, uint16_t* out) {
    constexpr int P = 32 / SUB;
    const int groups = (nl + P - 1) / P;
    const int64_t G = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (G >= static_cast<int64_t>(groups) * nblocks) return;
    c16_fill_group<SUB, BYTES>(G, meta, tmp, off, desc, nl, pb, out);
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
    const double* pot = a.pot;
    const double* dep = a.dep;
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
                double depp = 0.0;
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
                    if (STDP && a.plastic_on && ((m >> 22) & 1u)) {
                        const double pt = __ldcg(pot + static_cast<int64_t>(pre0 + pl) * a.dp + d1);
                        const WT nw = stdp_apply<WT>(w, stdp_dw(sp, pt, ev != 0u, depp), wmin, wmax);
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
        const double* pot = a.pot;
        const double* dep = a.dep;
        WT* W = static_cast<WT*>(a.w);
        const int gp = a.first + p;
        const bool sp = STDP ? bit_of(a.bits, gp) : false;
        const double depp = STDP ? dep[gp] : 0.0;
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
                if (STDP && a.plastic_on && ((m >> 22) & 1u)) {
                    const double pt = sp ? pot[static_cast<int64_t>(pre) * a.dp + d1] : 0.0;
                    const WT nw = stdp_apply<WT>(w, stdp_dw(sp, pt, e, depp), wmin, wmax);
                    if (nw != w) W[q] = nw;
                    w = nw;
                }
                if (e) acc += static_cast<double>(w);
            }
        }
        a.u_exact[p] = acc;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_step += 1;
}

}  // namespace

int sparse_pot_stage_bytes(int dp) { return (dp > 1 ? 64 : 24) * 1024; }

int sparse_block_pres(int hbits) {
    // 32 KB of staged history per CTA (pre ids are 16-bit block-local)
    switch (hbits) {
        case 1: return 32768;   // pre_local == pb is the inert padding slot (16-bit field)
        case 16: return 16384;
        case 32: return 8192;
        default: return 4096;
    }
}

template <typename WT, bool STDP, int HB>
static void sparse_go_sub(const SparseArgs& a, int sub, int gx, size_t smem, cudaStream_t s) {
    dim3 grid(gx, a.nblocks);
    if (a.dict_size > 0) smem = ((smem + 15) & ~static_cast<size_t>(15)) + static_cast<size_t>(a.dict_size) * sizeof(WT);
    if (STDP && a.pot_staged) smem += static_cast<size_t>(a.pb) * a.dp * sizeof(double);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024)
            check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                  "k_sparse smem attribute");
        kern<<<grid, kThreads, smem, s>>>(a);
    };
    if (a.dict_size == 2 && !STDP && sub != 0 && HB != 64) {  // one weight: count the delivering pres
        constexpr int HC = HB == 64 ? 32 : HB;  // (64 never reaches the launch)
        switch (sub) {
            case 1: go(k_sparse_count<WT, HC, 1>); break;
            case 2: go(k_sparse_count<WT, HC, 2>); break;
            case 4: go(k_sparse_count<WT, HC, 4>); break;
            case 8: go(k_sparse_count<WT, HC, 8>); break;
            case 16: go(k_sparse_count<WT, HC, 16>); break;
            default: go(k_sparse_count<WT, HC, 32>); break;
        }
        return;
    }
    if (a.dict_size > 0 && !STDP) {
        switch (sub) {
            case 0: go(k_sparse_stream<WT, false, HB, true>); break;
            case 1: go(k_sparse_pull<WT, false, HB, 1, true>); break;
            case 2: go(k_sparse_pull<WT, false, HB, 2, true>); break;
            case 4: go(k_sparse_pull<WT, false, HB, 4, true>); break;
            case 8: go(k_sparse_pull<WT, false, HB, 8, true>); break;
            case 16: go(k_sparse_pull<WT, false, HB, 16, true>); break;
            default: go(k_sparse_pull<WT, false, HB, 32, true>); break;
        }
        return;
    }
    if (STDP && a.pot_staged) {
        switch (sub) {
            case 2: go(k_sparse_pull<WT, STDP, HB, 2, false, true>); return;
            case 4: go(k_sparse_pull<WT, STDP, HB, 4, false, true>); return;
            case 8: go(k_sparse_pull<WT, STDP, HB, 8, false, true>); return;
            case 16: go(k_sparse_pull<WT, STDP, HB, 16, false, true>); return;
            case 32: go(k_sparse_pull<WT, STDP, HB, 32, false, true>); return;
            default: break;  // sub 0: the stream kernel reads a.pot_staged itself
        }
    }
    switch (sub) {
        case 0: go(k_sparse_stream<WT, STDP, HB, false>); break;
        case 4: go(k_sparse_pull<WT, STDP, HB, 4, false>); break;
        case 8: go(k_sparse_pull<WT, STDP, HB, 8, false>); break;
        case 16: go(k_sparse_pull<WT, STDP, HB, 16, false>); break;
        default: go(k_sparse_pull<WT, STDP, HB, 32, false>); break;
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

bool launch_sparse_bank_joint(uint32_t* meta, uint32_t* tmp, const int64_t* off, int nblocks, int nl, int sub,
                              int hbits, cudaStream_t s) {
    if (sub != 4 && sub != 8 && sub != 16) return false;
    const int P = 32 / sub;
    const int64_t groups = static_cast<int64_t>(nblocks) * ((nl + P - 1) / P);
    if (groups <= 0) return true;
    const unsigned grid = static_cast<unsigned>((groups + 63) / 64);
    switch (sub) {
        case 4: k_sparse_bank_joint<4><<<grid, 64, 0, s>>>(meta, tmp, off, nblocks, nl, hbits); break;
        case 8: k_sparse_bank_joint<8><<<grid, 64, 0, s>>>(meta, tmp, off, nblocks, nl, hbits); break;
        case 16: k_sparse_bank_joint<16><<<grid, 64, 0, s>>>(meta, tmp, off, nblocks, nl, hbits); break;
        default: return false;
    }
    check(cudaGetLastError(), "k_sparse_bank_joint");
    return true;
}

void launch_sparse_bank_order(const uint32_t* in, uint32_t* out, const int64_t* off, int64_t lists, int nl,
                              int sub, int hbits, cudaStream_t s) {
    if (lists <= 0) return;
    k_sparse_bank_order<<<static_cast<unsigned>((lists + 127) / 128), 128, 0, s>>>(in, out, off, lists, nl, sub,
                                                                                  hbits);
    check(cudaGetLastError(), "k_sparse_bank_order");
}

bool c16_bytes() {
    const char* e = std::getenv("SNB_C16_IMAGE");  // A/B knob: "bits" = the pair-encoded 16-bit image
    return !(e && std::string(e) == "bits");
}

int c16_block_pres() { return c16_bytes() ? kC8Pres : kC16Pres; }

void launch_c16_count(const uint32_t* meta, const int64_t* off, int64_t lists, int pb, uint2* cnt, cudaStream_t s) {
    if (lists <= 0) return;
    k_c16_count<<<static_cast<unsigned>((lists + 255) / 256), 256, 0, s>>>(meta, off, lists, pb, cnt);
    check(cudaGetLastError(), "k_c16_count");
}

bool launch_c16_fill(const uint32_t* meta, uint32_t* tmp, const int64_t* off, const uint2* desc, int nblocks, int nl,
                     int pb, int sub, uint16_t* out, cudaStream_t s) {
    const int P = 32 / sub;
    const int64_t groups = static_cast<int64_t>(nblocks) * ((nl + P - 1) / P);
    if (groups <= 0) return true;
    const unsigned grid = static_cast<unsigned>((groups + 63) / 64);
    const bool bytes = c16_bytes();
    auto go = [&](auto kb, auto kp) {
        (bytes ? kb : kp)<<<grid, 64, 0, s>>>(meta, tmp, off, desc, nblocks, nl, pb, out);
    };
    switch (sub) {
        case 2: go(k_c16_fill<2, true>, k_c16_fill<2, false>); break;
        case 4: go(k_c16_fill<4, true>, k_c16_fill<4, false>); break;
        case 8: go(k_c16_fill<8, true>, k_c16_fill<8, false>); break;
        case 16: go(k_c16_fill<16, true>, k_c16_fill<16, false>); break;
        default: return false;
    }
    check(cudaGetLastError(), "k_c16_fill");
    return true;
}

template <typename WT, int NT>
static void c16_go(const SparseArgs& a, const uint2* desc, const uint4* e, int sub, dim3 grid, cudaStream_t s) {
    static bool carveout = false;  // 33 KB of history per CTA: let the occupancy limit be registers
    if (!carveout) {
        for (auto k : {k_sparse_count16<WT, 2, NT>, k_sparse_count16<WT, 4, NT>, k_sparse_count16<WT, 8, NT>,
                       k_sparse_count16<WT, 16, NT>})
            check(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
        carveout = true;
    }
    switch (sub) {
        case 2: k_sparse_count16<WT, 2, NT><<<grid, NT, 0, s>>>(a, desc, e); break;
        case 4: k_sparse_count16<WT, 4, NT><<<grid, NT, 0, s>>>(a, desc, e); break;
        case 16: k_sparse_count16<WT, 16, NT><<<grid, NT, 0, s>>>(a, desc, e); break;
        default: k_sparse_count16<WT, 8, NT><<<grid, NT, 0, s>>>(a, desc, e); break;
    }
}

template <typename WT, int NT>
static void c8_go(const SparseArgs& a, const uint2* desc, const uint4* e, int sub, dim3 grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        for (auto k : {k_sparse_count8<WT, 2, NT>, k_sparse_count8<WT, 4, NT>, k_sparse_count8<WT, 8, NT>,
                       k_sparse_count8<WT, 16, NT>})
            check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kC8ImageBytes), "c8 smem");
        attr = true;
    }
    switch (sub) {
        case 2: k_sparse_count8<WT, 2, NT><<<grid, NT, kC8ImageBytes, s>>>(a, desc, e); break;
        case 4: k_sparse_count8<WT, 4, NT><<<grid, NT, kC8ImageBytes, s>>>(a, desc, e); break;
        case 16: k_sparse_count8<WT, 16, NT><<<grid, NT, kC8ImageBytes, s>>>(a, desc, e); break;
        default: k_sparse_count8<WT, 8, NT><<<grid, NT, kC8ImageBytes, s>>>(a, desc, e); break;
    }
}

int c16_threads(int nl) {
    if (c16_bytes()) {  // one CTA per SM (192 KB image): 1024 threads, or 512 (A/B knob)
        const char* t = std::getenv("SNB_C16_THREADS");
        return t && std::atoi(t) == 512 ? 512 : 1024;
    }
    // full-size lists: 256-thread CTAs (cfg4 0.4127 ms; 512: 0.4165, 1024: 0.419); post
    // partitions (an eighth of cfg4's posts per block): 1024 (65.8 us vs 70.4 at 512,
    // 79.1 at 256) -- a CTA stages its pre block once for 4x the posts
    int v = nl >= 131072 ? kThreads : 1024;
    if (const char* t = std::getenv("SNB_C16_THREADS")) v = std::atoi(t);  // A/B knob: 256, 512, 1024
    return (v == 512 || v == 1024) ? v : kThreads;
}

void launch_sparse_count16(const SparseArgs& a, const uint2* desc, const void* ent, bool f64, int sub, int gx,
                           int nt, cudaStream_t s) {
    dim3 grid(gx, a.nblocks);
    const uint4* e = static_cast<const uint4*>(ent);
    if (c16_bytes()) {
        if (f64) {
            if (nt == 512) c8_go<double, 512>(a, desc, e, sub, grid, s);
            else c8_go<double, 1024>(a, desc, e, sub, grid, s);
        } else {
            if (nt == 512) c8_go<float, 512>(a, desc, e, sub, grid, s);
            else c8_go<float, 1024>(a, desc, e, sub, grid, s);
        }
        check(cudaGetLastError(), "k_sparse_count8");
        return;
    }
    if (f64) {
        if (nt == 1024) c16_go<double, 1024>(a, desc, e, sub, grid, s);
        else if (nt == 512) c16_go<double, 512>(a, desc, e, sub, grid, s);
        else c16_go<double, kThreads>(a, desc, e, sub, grid, s);
    } else {
        if (nt == 1024) c16_go<float, 1024>(a, desc, e, sub, grid, s);
        else if (nt == 512) c16_go<float, 512>(a, desc, e, sub, grid, s);
        else c16_go<float, kThreads>(a, desc, e, sub, grid, s);
    }
    check(cudaGetLastError(), "k_sparse_count16");
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

}  // namespace snb
