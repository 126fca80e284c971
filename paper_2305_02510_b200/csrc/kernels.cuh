// Device-side parameter blocks and launcher declarations for the MAT step.
// Reference semantics: see DESIGN.md and the per-kernel comments in k_*.cu
// (shared device helpers in kernels_common.cuh).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace snb {

// Row (pre-neuron) plasticity classes for dense storage; computed per
// partition at setup so the sweep needs no mask loads for the common shapes.
enum RowKind : uint8_t {
    kRowNone = 0,     // no plastic synapse in this row's local columns
    kRowAll = 1,      // every local column is a plastic synapse
    kRowAllButSelf = 2,  // every local column but j == i plastic, (i,i) absent
    kRowMixed = 3     // consult the plastic bitmask
};

struct NeuronArgs {
    // local partition [first, first + nl)
    int32_t n;            // global neuron count
    int32_t first;
    int32_t nl;
    double* v;
    const double* thr;
    const double* leak;
    const double* reset;
    const int32_t* refr;
    int32_t* cnt;
    // synaptic input
    const double* partial;     // [nchunks][nl] (non-exact)
    int32_t nchunks;
    // or, from the 16-bit count-list sweeps: per-block delivery counts, a
    // block's input being (double)((WT)count * w0) as those sweeps computed it
    const uint16_t* partial16; // [nchunks][nl] or null
    double w0;
    int32_t w0_f32;            // WT = float
    const double* u_exact;     // [nl] (exact mode)
    // stimulus: per-step CSR over (neuron asc, amp)
    const int64_t* st_off;     // [st_steps + 1]
    const int32_t* st_neuron;
    const double* st_amp;
    int32_t st_steps;          // number of steps covered by the table
    int32_t st_base;           // step of table row 0 (row = t - st_base)
    // time
    int32_t* d_step;           // device step counter (read here; sweep increments)
    int32_t* step_out;         // or null: block 0 stores the step here for the sweep (folded history)
    int32_t* work;             // sweep work counter, reset here (null: static schedule)
    int32_t t_base;            // raster/trace row = t - t_base
    // outputs
    uint32_t* bits;            // full bitmask [words]; this kernel writes local words
    uint32_t* raster;          // [rows][nl_words] or null
    int32_t nl_words;
    int32_t raster_rows;
    double* trace;             // [rows][nl] or null
    unsigned long long* spike_count;
    // peer-to-peer spike exchange (fused into this kernel; null when unused):
    // every rank's exchange bitmask (two step-parity buffers of xstride
    // words: step t goes to buffer t & 1) and flag array, over NVLink
    uint32_t* const* peer_bits;   // [world] device pointers (peer or local)
    int32_t xstride;              // words per parity buffer
    int32_t* const* peer_flags;   // [world] -> int32[world]; flag[src] = last step src published
    uint32_t* done;               // CTA completion counter of this launch
    int32_t rank;
    int32_t world;
    // agent-based mode (abm_engine.cpp:146-189): u = leak(v) + (pending + ext),
    // where pending is the synaptic input summed from 0.0; stochastic firing
    // gate unit(seed, agent, step) < fire_p for fire_p < 1 (null: all "lif")
    int32_t abm;
    const double* fire_p;         // [nl] or null
    const uint64_t* agent_key;    // [nl] RandomStream(seed, agent stream, id) key before the step mix
};

struct HistArgs {
    int32_t n;
    uint32_t* bits;            // full spike bitmask of step t (k_hist rebuilds it from xbits in p2p mode)
    uint64_t* hist;            // [hw][n]; bit k of the concatenation = s[t-k]
    int32_t hw;
    int32_t dmax;              // propagation delay span (bits 0..dmax-1)
    // STDP traces
    int32_t stdp;
    int32_t window;
    int32_t dp;                // plastic delay span (pot per d = 1..dp)
    const double* a_plus;
    const double* a_minus;
    double* pot64;             // [n][dp]
    double* dep64;             // [n]
    const uint8_t* row_plastic;  // [n]
    uint32_t* active;          // [words] rows that the sweep must visit
    int32_t* d_step;
    uint32_t* hist_lo;         // [n] low 32 history bits (sparse pull staging)
    unsigned long long* active_count;  // running sum of active rows (algorithmic bytes)
    // peer-to-peer exchange: wait until every rank published step t (flags[q] > t)
    const int32_t* flags;              // this rank's int32[world] (written by peers) or null
    const uint32_t* xbits;             // this rank's exchange bitmask [2][xstride] (peers store step t into t & 1)
    int32_t xstride;
    int32_t world;
    int32_t* error;                    // set to 1 when the wait times out
    // first step that applies STDP: apply_stdp clamps every plastic weight on
    // its first call even when dw == 0 (mat_engine.cpp:243-249), so every
    // plastic row is visited then (0 unless plasticity was switched off first)
    int32_t clamp_step;
};

struct DenseArgs {
    int32_t n;                 // rows
    int32_t first;             // global id of local column 0
    int32_t nl;                // local columns
    int64_t pitch;             // elements per row
    void* w;                   // WT[n][pitch]
    const uint8_t* delay;      // [n][pitch] or null
    const uint32_t* mask;      // [n][pitch/32] plastic bits or null
    const uint8_t* kind;       // [n] RowKind
    const uint32_t* active;    // [words]
    const uint64_t* hist;      // word 0 of the history
    const uint32_t* bits;      // spike bitmask (column spikes s_j[t])
    const double* pot;         // [n][dp] fp64 traces (the STDP math is fp64 for every weight type)
    const double* dep;         // [n]
    int32_t dp;
    double w_min, w_max;
    int32_t tile_w;            // columns per CTA tile (multiple of VEC)
    int32_t rows_per_chunk;
    int32_t nchunks;
    double* partial;           // [nchunks][nl]
    // exact mode
    const double* v;           // local membrane (after this step)
    const double* leak;
    const double* reset;
    double* u_exact;           // [nl]
    int32_t* d_step;
    int32_t* work;             // dynamic item counter (null: static striding)
    int32_t abm;               // exact mode seeds the accumulator with 0.0 instead of leak(v)
    int32_t plastic_on;        // 0: steps without apply_stdp (sn_set_plasticity); weights untouched
};

struct SparseArgs {
    int32_t n;
    int32_t first;
    int32_t nl;
    int32_t pb;                // pres per block
    int32_t nblocks;
    const int64_t* off;        // [nblocks * nl + 1], lists padded to 4
    const uint32_t* meta;      // pre_local | (d-1) << 16 | plastic << 22
    void* w;                   // WT[]
    const uint32_t* bits;
    const uint32_t* hist_lo;
    const uint64_t* hist;
    const double* pot;         // [n][dp] fp64
    const double* dep;         // [n]
    int32_t dp;
    double w_min, w_max;
    int32_t posts_per_cta;
    const void* wdict;         // WT[dict_size] weight dictionary (meta bits 23..31) or null
    int32_t dict_size;         // 0: weights stream from w[]
    int32_t pot_staged;        // STDP: the block's pot^(d) traces are staged in shared memory
    double* partial;           // [nblocks][nl]
    uint16_t* partial16;       // [nblocks][nl] counts (k_sparse_count8 / count16)
    const double* v;
    const double* leak;
    const double* reset;
    double* u_exact;
    int32_t* d_step;
    int32_t abm;               // exact mode seeds the accumulator with 0.0 instead of leak(v)
    int32_t plastic_on;        // 0: steps without apply_stdp (sn_set_plasticity)
    // folded history (partitioned k_sparse_count16 runs, no k_hist): the sweep
    // shifts step t's spike bits into hist16[t & 1] -> hist16[(t + 1) & 1]
    // itself while staging; t comes from k_neuron via step_in (the sweep
    // bumps d_step, so it cannot read d_step safely)
    const int32_t* step_in;
    uint16_t* hist16;          // [2][n] or null
    // folded history over the p2p exchange: wait until every rank published
    // step t (flags[q] > t), then read the spike bits from exchange buffer t & 1
    const int32_t* flags;      // or null
    int32_t world;
    int32_t* error;            // set to 1 when the wait times out
    const uint32_t* xbits;
    int32_t xstride;
};

// Stage plan of k_sparse_tma (built on the host at setup from the CSC offsets):
// stage = <= sparse_tma_stage_entries() consecutive meta entries of one pre
// block plus the stage-relative positions of the post boundaries inside it.
struct SpStage {
    int64_t q;          // first meta entry
    int64_t bnd_off;    // first position in bnd (multiple of 8)
    int32_t entries;    // meta entries (multiple of 4)
    int32_t k0;         // 1 + the stage's first linear post b * nl + p (= partial row + 1)
    int32_t nb;         // whole posts in the stage (their end positions are in bnd)
    int32_t block;      // pre block of every entry of the stage
};
struct SpStagePlan {
    const SpStage* stages;
    const int32_t* cta_first;  // [ctas + 1] stage range per CTA
    const int32_t* cta_block;  // [ctas] first pre block of the CTA (its stages use it and the next)
    const uint16_t* bnd;       // end position of each post of a stage, stage-relative
};

// ---- launchers (k_neuron.cu, k_dense.cu, k_persistent.cu, k_sparse.cu, k_netgen.cu) ----
void launch_neuron(const NeuronArgs& a, bool exact, bool fused_hist, const HistArgs& h,
                   cudaStream_t s);
void launch_hist(const HistArgs& h, cudaStream_t s);
void launch_dense(const DenseArgs& a, bool f64, bool stdp, bool delay, bool exact, int grid_ctas,
                  cudaStream_t s);
int dense_vec(bool f64);
int dense_threads();
int dense_stream_max_ctas(bool f64, bool stdp, bool delay);  // occupancy x SMs
// TMA-staged sweep (fp32/fp64, optional delays): one CTA per SM, rows_per_chunk <= dense_tma_max_rows(...);
// with delays the tile width must be a multiple of 16 (the delay bytes are bulk-copied)
int dense_tma_max_dp();  // delayed STDP: plastic delay span the TMA sweep supports
// weight census of a dense block (k_inspect.cu): counts[k] = cells equal to vals[k], counts[nv] = others
int census_max_values();
void launch_value_counts(const void* W, bool f64, int64_t pitch, int n, int nl, const void* vals, int nv,
                         unsigned long long* counts, int ctas, cudaStream_t s);
int dense_tma_max_rows(int tile_w, bool f64, bool delay, bool stdp);  // longest row list whose buffers fit (0: none)
void launch_dense_tma(const DenseArgs& a, bool f64, bool stdp, bool delay, int grid, cudaStream_t s);
void launch_sparse(const SparseArgs& a, bool f64, bool stdp, int hbits, int sub, bool exact,
                   int grid_x, cudaStream_t s);
void launch_prologue(double* u_exact, const double* v, const double* leak, const double* reset,
                     int nl, bool abm, cudaStream_t s);
void launch_step_bump(int32_t* d_step, cudaStream_t s);
int sparse_block_pres(int hbits);
// STDP pull sweeps stage the pre block's pot^(d) traces in shared memory up to this many bytes
int sparse_pot_stage_bytes(int dp);
// setup: reorder one-weight lists for conflict-light history reads in k_sparse_count
// Joint per-warp bank schedule of one-weight lists, in place (tmp: scratch of
// the same size); false when SUB has no joint form (the per-list order applies).
bool launch_sparse_bank_joint(uint32_t* meta, uint32_t* tmp, const int64_t* off, int nblocks, int nl, int sub,
                              int hbits, cudaStream_t s);
void launch_sparse_bank_order(const uint32_t* in, uint32_t* out, const int64_t* off, int64_t lists, int nl,
                              int sub, int hbits, cudaStream_t s);
// 16-bit one-weight lists (k_sparse_count16): pres per block (4 segments of
// 4095), setup kernels (per-segment counts; joint bank-scheduled fill) and the sweep
int c16_block_pres();
bool c16_bytes();  // k_sparse_count8 byte image (default) vs the pair-encoded k_sparse_count16
void launch_c16_count(const uint32_t* meta, const int64_t* off, int64_t lists, int pb, uint2* cnt, cudaStream_t s);
bool launch_c16_fill(const uint32_t* meta, uint32_t* tmp, const int64_t* off, const uint2* desc, int nblocks, int nl,
                     int pb, int sub, uint16_t* out, cudaStream_t s);
void launch_sparse_count16(const SparseArgs& a, const uint2* desc, const void* ent, bool f64, int sub, int gx,
                           int nt, cudaStream_t s);
int c16_threads(int nl);  // threads per k_sparse_count16 CTA for nl local posts
// TMA-fed stream for static uniform-weight lists (dictionary {w, 0}), no exact order
size_t sparse_tma_smem(const SparseArgs& a, int hbits);
int sparse_tma_stage_entries();
int sparse_tma_max_boundaries();
void launch_sparse_tma(const SparseArgs& a, const SpStagePlan& plan, int ctas, bool f64, int hbits, cudaStream_t s);
// persistent cooperative step loop for small dense nets (single partition)
int persistent_max_ctas(bool f64, bool stdp, bool delay);
void launch_persistent_dense(const NeuronArgs& na, const HistArgs& h, const DenseArgs& da, bool f64,
                             bool stdp, bool delay, int grid, int steps, cudaStream_t s);

// ---- column-owner persistent loop (small dense nets, one history word) ----
// CTA c owns posts [w c, w c + w), w in {8, 16, 32}: it sweeps all rows for those columns and
// updates those neurons itself, so only one grid barrier per step is needed;
// the per-step state other CTAs read (history word, pot traces, row activity)
// is multi-buffered by step.
struct ColArgs {
    uint64_t* hist2;            // [2][n]   history word after step t in buffer t & 1
    void* pot2;                 // WT [2][n * dp]
    uint32_t* act3;             // [3][words] rows the sweep must visit (step t in t % 3; OR-ed)
    const uint8_t* row_plastic; // [n]
    const double* a_plus;
    const double* a_minus;
    int32_t window;
    int32_t dmax;
    unsigned long long* active_count;  // running sum of active rows (algorithmic bytes)
    int32_t clamp_step;                // HistArgs::clamp_step
};
// Cluster loop (k_cluster_count): static one-weight nets without STDP, delays <= 31
struct ClusterArgs {
    const uint8_t* codes;          // per-CTA table: [n][P] rotation codes (D = 0) or [P][D][wn4] delay planes
    int32_t P;                     // posts per CTA (32, 64, 96 or 128)
    int32_t D;                     // delay planes (8 / 16), 0 = rotation codes
    int32_t cs;                    // CTAs in the cluster
    double w0;                     // the one weight
    uint64_t* hist2;               // [2][n], ColArgs layout
    double* partial;               // [nl] input of the next step (= NeuronArgs::partial)
    unsigned long long* active_count;
    uint64_t dmask;
};
int cluster_plan(int n, int nl, bool f64, int dmax, int* P_out, int* D_out);
size_t cluster_table_bytes(int n, int P, int D, int cs);
void launch_cluster_table(const DenseArgs& da, int nl, int P, int D, int cs, void* table, bool f64, cudaStream_t s);
void launch_cluster_count(const NeuronArgs& na, const ClusterArgs& ca, bool f64, int steps, cudaStream_t s);
int persistent_cols_max_ctas(bool f64, bool stdp, bool delay, int width);
void launch_persistent_cols(const NeuronArgs& na, const DenseArgs& da, const ColArgs& ca, bool f64, bool stdp,
                            bool delay, int width, int grid, int steps, cudaStream_t s);

// ---- tiny nets: the whole T-step loop in one CTA, all state in shared memory ----
// Eligible when N <= 1024 and the incoming lists, the per-neuron state and the
// call's stimulus fit in shared memory.  Thread j owns post j: it sums its
// incoming list in ascending pre order starting from leak(v) (the order of
// mat_engine.cpp:173-180, so fp64 membranes are bit-exact) and applies STDP
// to its own plastic synapses.
struct TinyArgs {
    int32_t n;
    int32_t steps;
    int32_t hw;                // history words per neuron
    int32_t dmax;
    int32_t f64;               // weight precision of w
    // state (global, loaded at start and written back at the end)
    double* v;
    int32_t* cnt;
    uint64_t* hist;            // [hw][n]
    const double* thr;
    const double* leak;
    const double* reset;
    const int32_t* refr;
    // incoming lists, post-major, pre ascending
    const uint32_t* off;       // [n+1]
    const uint32_t* meta;      // history word byte offset << 5 | (d-1) & 31
    const uint16_t* pidx;      // STDP: pre * dp + (d-1), the pot^(d) trace of the pre; 0xffff = not plastic
    void* w;                   // float or double [m]
    int32_t m;
    // stimulus of this launch: rows of the per-step CSR (neuron ascending).
    // st_off points at the row of the launch's first step; entries are
    // st_neuron/st_amp[st_off[s]]; only the first st_rows rows exist.
    const int64_t* st_off;     // [st_rows + 1]
    const int32_t* st_neuron;
    const double* st_amp;
    int32_t st_rows;
    int32_t st_count;          // st_off[st_rows] - st_off[0]
    // STDP
    int32_t stdp;
    int32_t window;
    int32_t dp;
    const double* a_plus;
    const double* a_minus;
    double w_min, w_max;
    int32_t plastic_on;        // 0: steps without apply_stdp (sn_set_plasticity)
    // outputs (device or host-mapped pinned memory)
    uint32_t* raster;          // [steps][words]
    double* trace;             // [steps][n] or null
    unsigned long long* spike_count;
    int32_t* d_step;
    // agent-based mode (see NeuronArgs)
    int32_t abm;
    const double* fire_p;      // [n] or null
    const uint64_t* agent_key; // [n]
    // one-weight unit-delay nets without STDP: each post's in-list as a bitmask
    // over the pres (count_words words, <= kTinyCountWords), the input as
    // popc(mask & previous spike words) sequential additions of w0 (the
    // reference's ascending-pre sum of equal weights, bit for bit); 0 = off
    int32_t count_words;
    double w0;
};
size_t tiny_smem_bytes(const TinyArgs& a);
int tiny_max_smem();
int tiny_count_words_max();
void launch_tiny(const TinyArgs& a, cudaStream_t s);

// ---- on-device Erdos-Renyi generation (netgen.cpp:36-51 semantics) ----
struct ErArgs {
    int32_t n;
    double p;
    uint64_t edge_key;         // RandomStream(seed, 1) key
    uint64_t delay_key;        // RandomStream(seed, delay_stream) key
    int32_t delay_max;         // <= 1: unit delays
    int32_t delay_by_synapse_index;
    float weight_f;
    double weight_d;
    int32_t stdp;
};
// dense: fills W[n][pitch] for local columns [first, first+nl), delays, mask bits
void launch_er_dense(const ErArgs& e, void* w, bool f64, uint8_t* delay, uint32_t* mask,
                     int first, int nl, int64_t pitch, cudaStream_t s);
// sparse: pass 1 counts per (block, local post); pass 2 fills
void launch_er_sparse_count(const ErArgs& e, int first, int nl, int pb, int nblocks,
                            int64_t* counts, cudaStream_t s);
void launch_er_sparse_fill(const ErArgs& e, int first, int nl, int pb, int nblocks,
                           const int64_t* off, uint32_t* meta, void* w, bool f64,
                           cudaStream_t s);

uint64_t stream_key(uint64_t seed, uint64_t stream);

}  // namespace snb
