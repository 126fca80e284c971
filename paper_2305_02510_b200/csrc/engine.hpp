// Host engine behind the C ABI (include/superneuro_mat.h).
//
// Mirrors the state the reference keeps in MatState (mat_engine.hpp:56-80)
// but lays it out for HBM: SoA neuron state for the local post partition,
// spike history as bit words, weights dense pre-major or blocked CSC.
#pragma once

#include "../../include/superneuro_mat.h"
#include "kernels.cuh"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace snb {

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct LogicError : std::logic_error {
    using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t err, const char* what);

// Owning device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void alloc(size_t b);
    void release();
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

// Owning pinned host allocation.
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { release(); }
    void reserve(size_t b);
    void release();
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

struct RasterChunk {
    int32_t t0 = 0;
    int32_t rows = 0;
    std::vector<uint32_t> words;  // rows x nl_words
    bool stripped = false;        // relay neurons' bits cleared (Engine::strip_relays)
};

struct NcclComm;  // nccl_dl.cpp

class Engine {
public:
    explicit Engine(const sn_options& opt);
    ~Engine();

    void add_neurons(int64_t count, const double* thr, const double* leak, const double* reset,
                     const int32_t* refr, const int32_t* axonal, int64_t* first_id);
    void add_synapses(int64_t count, const int32_t* pre, const int32_t* post, const double* w,
                      const int32_t* delay, const uint8_t* stdp);
    void add_stimulus(int64_t count, const int32_t* step, const int32_t* neuron, const double* amp);
    void clear_stimulus();
    void set_stdp(int32_t window, const double* ap, const double* am, double wmin, double wmax);
    void generate_er(int32_t n, double p, uint64_t seed, double weight, int32_t delay_max,
                     uint64_t delay_stream, int32_t by_syn, int32_t stdp);
    void set_seed(uint64_t seed);
    void set_fire_probability(int64_t first, int64_t count, const double* p);
    void setup();
    void simulate(int32_t steps);
    // simulate + the raster of exactly these steps into the caller's arrays;
    // with stream_io and graphs, finished chunks are decoded while later ones run
    void simulate_raster(int32_t steps, int32_t* out_steps, int32_t* out_neurons, int64_t cap, int64_t* count);
    void synchronize();

    int64_t raster_size();
    void get_raster(int32_t* steps, int32_t* neurons, int64_t cap);
    void clear_raster();
    void get_membrane(double* out, int64_t count);
    int64_t trace_rows();
    void get_trace(double* out, int64_t count);
    void get_synapse_weights(double* out, int64_t count);
    void get_weight_matrix(double* out, int64_t count);
    void weight_value_counts(const double* values, int32_t count, int64_t* counts);
    void get_stats(sn_stats* out);
    void reset_stats();

    void comm_init(const uint8_t* id, int32_t rank, int32_t world);
    // peer-to-peer spike exchange fused into the neuron kernel (NVLink stores)
    static constexpr int kIpcHandleBytes = 64;
    void p2p_get_handles(uint8_t* out, int64_t cap);
    void p2p_open(const uint8_t* all_handles, int32_t world);
    static void p2p_connect_local(Engine* const* engines, int32_t world);
    // mat_step (mat_engine.cpp:168-208): one step whose external input is
    // exactly `ext` (n amplitudes, or none), returning its spikes ascending;
    // apply_stdp follows when plasticity is on (mat_run:277-279)
    void step(const double* ext, int64_t ext_len, int32_t* spikes, int64_t cap, int64_t* count);
    // whether steps apply STDP (mat_run with / without apply_stdp after mat_step)
    void set_plasticity(bool on);
    void step_local();
    void get_spike_words(uint32_t* out, int64_t words);
    void put_spike_words(int32_t first_word, const uint32_t* w, int64_t count);
    void step_finish();

    static void partition(int32_t n, int32_t rank, int32_t world, int32_t* first, int32_t* count);

private:
    void require_not_setup(const char* what) const;
    void require_setup(const char* what) const;
    void validate() const;
    void build_dense_from_lists();
    void build_sparse_from_lists();
    void build_generated();
    void alloc_state();
    void build_stimulus_table();
    void plan_launches();
    NeuronArgs neuron_args(int t_base, int rows, uint32_t* raster, double* trace,
                           const int64_t* st_off, const int32_t* st_neuron, const double* st_amp,
                           int32_t st_steps, int32_t st_base);
    HistArgs hist_args();
    void launch_sweep();
    void launch_sweep_only();  // no launch accounting (graph capture counts in bulk)
    double run_graph_chunks(const NeuronArgs& na, int steps);
    struct RasterSink {
        int32_t* steps = nullptr;
        int32_t* neurons = nullptr;
        int64_t cap = 0, count = 0;
        int32_t rows_done = 0;    // rows of the call already decoded into the arrays
    };
    RasterSink* sink_ = nullptr;  // set by simulate_raster for one call
    void sink_rows(const uint32_t* rows, int32_t nrows, int32_t t_first);
    static constexpr int kProfStride = 8;  // graph mode: time every 8th step's kernels
    int64_t steps_at_reset_ = 0;
    DenseArgs dense_args();
    void enqueue_step(const NeuronArgs& na, bool exchange);
    void flush_pending();
    void decode_raster();

    sn_options opt_;
    cudaStream_t stream_ = nullptr;
    // Device-to-host read ordered after all work queued on stream_ (a plain
    // cudaMemcpy runs on the legacy stream, which a non-blocking stream_ does
    // not synchronise with).
    void d2h(void* dst, const void* src, size_t bytes, const char* what) const;
    bool setup_done_ = false;

    // ---- model (host, as given) ----
    std::vector<double> thr_, leak_, reset_;
    std::vector<int32_t> refr_, axonal_;
    std::vector<int32_t> pre_, post_, delay_;
    std::vector<double> weight_;
    std::vector<uint8_t> plastic_;
    std::vector<int32_t> st_step_, st_neuron_;
    std::vector<double> st_amp_;
    bool stdp_on_ = false;
    int32_t window_ = 0;
    std::vector<double> a_plus_, a_minus_;
    double w_min_ = 0.0, w_max_ = 1.0;
    bool generated_ = false;
    ErArgs er_{};
    int32_t er_delay_max_ = 1;

    // agent-based mode (sn_options.mode == SN_MODE_ABM)
    bool abm_ = false;
    uint64_t seed_ = 0;
    std::vector<double> fire_p_;  // per neuron; empty = all "lif"
    bool any_stochastic_ = false;
    DevBuf d_firep_, d_akey_;
    static uint64_t agent_stream_key(uint64_t seed, uint64_t agent);
    std::string run_name() const { return abm_ ? "abm_run" : "mat_run"; }

    // ---- derived layout ----
    int32_t n_ = 0, first_ = 0, nl_ = 0, part_ = 0;
    int32_t words_ = 0, nl_words_ = 0;  // full bitmask words (world * part/32), local words
    bool dense_ = true, f64_ = false, exact_ = false, has_delay_ = false;
    int32_t dmax_ = 1, dp_ = 1, hw_ = 1, hbits_ = 1;
    int64_t pitch_ = 0;
    bool any_mixed_ = false;
    int64_t syn_local_ = 0;
    std::vector<int64_t> slot_;  // synapse list index -> storage element (-1 if not local)
    // sparse
    int32_t pb_ = 0, nblocks_ = 0, sub_ = 32, posts_per_cta_ = 0, sparse_gx_ = 1;
    int64_t sparse_elems_ = 0;
    std::vector<double> dict_;   // sparse weight dictionary (empty: weights stored per synapse)
    DevBuf d_wdict_;
    void upload_dict();
    int32_t sparse_pres_per_block() const;
    static bool c16_allowed();
    mutable bool pot_staged_ = false;  // STDP pull sweep stages the block's pot traces in smem
    bool sparse_tma_ = false;  // k_sparse_tma stage plan (static uniform-weight lists)
    bool bank_ordered_ = false;  // one-weight lists dealt bank-aware for k_sparse_count
    bool c16_ = false;           // 16-bit segmented one-weight lists (k_sparse_count16)
    int32_t c16_threads_ = 256;  // threads per k_sparse_count16 CTA (c16_threads)
    // partitioned k_sparse_count16 runs fold k_hist into the sweep's staging
    // (k_sparse.cu c16_stage): no history kernel on the step path
    bool fold_hist() const { return c16_ && (opt_.world > 1 || comm_ != nullptr); }
    DevBuf d_hist16_, d_step_copy_;
    DevBuf d_c16desc_, d_c16ent_;
    bool build_c16();
    DevBuf d_sp_stages_, d_sp_first_, d_sp_block_, d_sp_bnd_;
    int32_t sp_ctas_ = 0;
    bool build_sparse_tma_plan(int ctas);
    double sparse_weight(const std::vector<uint8_t>& host_w, const std::vector<uint32_t>& meta, int64_t q) const;
    // dense plan
    int32_t tile_w_ = 0, rows_per_chunk_ = 0, nchunks_ = 1, dense_grid_ = 1;
    bool persistent_ = false;     // small dense nets: one cooperative launch per simulate
    bool cols_ = false;           // ... as column owners (k_persistent_cols, one barrier per step)
    int32_t col_width_ = 8;       // posts per column group
    bool cluster_ = false;        // ... as one thread-block cluster (k_cluster_count: static one-weight nets)
    int32_t cl_cs_ = 0, cl_P_ = 0, cl_D_ = 0;
    double cl_w0_ = 0.0;
    DevBuf d_clcodes_;
    bool uniform_weight(double* w0) const;
    DevBuf d_hist2_, d_pot2_, d_act2_;
    bool dynamic_sched_ = false;  // dense sweep items claimed through an atomic counter
    bool tma_ = false;            // k_dense_tma (cp.async.bulk ring) instead of k_dense_stream
    // tiny nets: the whole call in one CTA with shared-memory state (k_tiny)
    static constexpr int kTinyMaxNeurons = 1024;
    bool tiny_ = false;
    DevBuf d_toff_, d_tpidx_;
    void materialize_er();
    bool build_tiny();
    void run_tiny(int t0, int steps, uint32_t* raster, double* trace, bool host_io);
    int32_t persist_grid_ = 1;
    double sweep_bytes_full_ = 0.0;  // algorithmic bytes of a sweep over every active row

    // ---- device ----
    DevBuf d_w_, d_delay_, d_mask_, d_kind_, d_row_plastic_;
    DevBuf d_off_, d_meta_;
    DevBuf d_v_, d_thr_, d_leak_, d_reset_, d_refr_, d_cnt_;
    DevBuf d_bits_, d_hist_, d_hist_lo_, d_active_;
    DevBuf d_pot64_, d_dep64_, d_ap_, d_am_;
    DevBuf d_partial_, d_uexact_;
    DevBuf d_step_, d_spikes_, d_work_;
    DevBuf d_st_off_, d_st_neuron_, d_st_amp_;
    int32_t st_steps_dev_ = 0;
    DevBuf d_stage_;
    DevBuf d_raster_, d_trace_;

    // ---- host results ----
    HostBuf h_stage_, h_raster_;
    std::vector<RasterChunk> raster_;
    std::vector<std::pair<const uint32_t*, int32_t>> dec_rows_;  // raster rows (words, step)
    std::vector<int64_t> dec_start_;                            // first event of each row
    bool events_valid_ = true;
    std::vector<double> trace_;
    int64_t trace_rows_ = 0;
    int32_t t_ = 0;  // host mirror of the device step counter

    // host stimulus CSR (per step, local neurons, summed in list order)
    std::vector<int64_t> hs_off_;
    std::vector<int32_t> hs_neuron_;
    std::vector<double> hs_amp_;
    bool stim_dirty_ = true;

    // ---- stats / profiling ----
    sn_stats stats_{};
    std::vector<cudaEvent_t> ev_pool_;
    struct Pending {
        cudaEvent_t a, b;
        int kind;  // 0 neuron, 1 sweep, 2 exchange, 3 whole
        double bytes;
    };
    std::vector<Pending> pending_;
    cudaEvent_t get_event();
    void record_begin(cudaEvent_t& e);

    NcclComm* comm_ = nullptr;
    bool p2p_ = false;
    DevBuf d_flags_, d_done_, d_err_, d_peer_bits_, d_peer_flags_, d_xbits_;
    std::vector<void*> ipc_opened_;  // peer allocations mapped with cudaIpcOpenMemHandle
    void set_peer_tables(const std::vector<uint32_t*>& bits, const std::vector<int32_t*>& flags);
    void check_exchange_error();
    bool host_exchange_ = false;
    // delay relays (effective delays > kMaxNativeDelay): relay neurons appended
    // after the user's, raster bits of ids >= n_user_ stripped on the host
    static constexpr int kMaxNativeDelay = 64;
    static constexpr int kMinGraphSteps = 4;  // shorter simulate calls launch without a graph
    void add_delay_relays();
    void strip_relays();
    bool relays_ = false;
    int32_t n_user_ = 0;          // neurons the caller added (== n_ without relays)
    int64_t m_user_ = 0;          // synapses the caller added
    std::vector<int32_t> pre_user_;
    int64_t relay_spikes_ = 0;    // relay spikes seen in stripped raster rows
    bool plasticity_ = true;      // sn_set_plasticity
    int32_t clamp_step_ = -1;     // first step that applied STDP (HistArgs::clamp_step), -1 = none yet
    void note_first_plastic_step() {
        if (stdp_on_ && plasticity_ && clamp_step_ < 0) clamp_step_ = t_;
    }
};

}  // namespace snb
