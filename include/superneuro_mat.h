/*
 * superneuro_mat.h -- C ABI of the B200-native MAT-mode simulation engine.
 *
 * Drop-in boundary for the reference's MAT path (SuperNeuro MAT mode as
 * implemented by spikeforge, /root/reference/proj).  Plain pointers and sizes
 * only; no exceptions cross this boundary.  Each entry point names the
 * reference interface it replaces.
 *
 *   reference (C++, proj/include/spikeforge/...)         this ABI
 *   ---------------------------------------------------  ----------------------------
 *   NeuronParams push (model.hpp:20-29)                   sn_add_neurons
 *   SynapseDef push (model.hpp:31-39)                     sn_add_synapses
 *   StimulusEntry push (model.hpp:53-63)                  sn_add_stimulus
 *   StdpConfig (model.hpp:67-78), defaults (model.cpp:10-22)
 *                                                         sn_set_stdp, sn_stdp_defaults
 *   WeightStorage Auto/Dense/Sparse (mat_engine.hpp:16)   sn_options.storage
 *   mat_init (mat_engine.hpp:89-90, mat_engine.cpp:109-166)
 *                                                         sn_setup
 *   mat_step + apply_stdp loop of mat_run
 *     (mat_engine.hpp:92-103, mat_engine.cpp:168-287)     sn_simulate
 *   RunResult.raster (model.hpp:87-104)                   sn_raster_size / sn_get_raster
 *   RunResult.membrane_trace                              sn_get_membrane_trace
 *   MatState.membrane (mat_engine.hpp:56-58)              sn_get_membrane
 *   WeightMatrix::slot_get(slot(s)) (mat_engine.hpp:37-39)
 *                                                         sn_get_synapse_weights
 *   erdos_renyi (netgen.hpp:31-34, netgen.cpp:19-54)      sn_generate_erdos_renyi
 *   AbmWorld / abm_run (abm_engine.hpp:70-121)            sn_options.mode = SN_MODE_ABM
 *   SimulationConfig::seed, StochasticLifBehavior
 *     (abm_engine.hpp:43-52, bindings.cpp:180-186)        sn_set_seed, sn_set_fire_probability
 *   std::invalid_argument / std::logic_error messages     sn_status + sn_last_error()
 *
 * Unlike mat_init (mat_engine.cpp:114-131), delays > 1 and axonal delays are
 * accepted and simulated natively (ring of spike-history bits) with the
 * timing of lower_delays + mat_run (lowering.cpp:22-59, oracle.cpp:91-95).
 *
 * Threading: one host thread drives one engine (MatState is not thread-safe
 * either); distinct engines are independent.
 */
#ifndef SUPERNEURO_MAT_H
#define SUPERNEURO_MAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SN_ABI_VERSION 2

#if defined(__GNUC__)
#define SN_API __attribute__((visibility("default")))
#else
#define SN_API
#endif

typedef struct sn_engine sn_engine;

typedef enum sn_status {
    SN_OK = 0,
    SN_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    SN_ERR_LOGIC = 2,            /* reference: std::logic_error (misuse/order) */
    SN_ERR_CUDA = 3,
    SN_ERR_NCCL = 4,
    SN_ERR_OOM = 5,
    SN_ERR_UNSUPPORTED = 6
} sn_status;

typedef enum sn_storage {
    SN_STORAGE_AUTO = 0,   /* dense when the N x N_local fp32 matrix is small or dense enough */
    SN_STORAGE_DENSE = 1,  /* row-major W[pre][post], pre-major like mat_engine.cpp:34-38 */
    SN_STORAGE_SPARSE = 2  /* post-major blocked CSC, spike-history pull */
} sn_storage;

typedef enum sn_precision {
    SN_WEIGHTS_F32 = 0,    /* fp32 weight storage (HBM traffic 4 B/synapse) */
    SN_WEIGHTS_F64 = 1     /* fp64 storage + fp64 STDP arithmetic (bit-exact weights) */
} sn_precision;

typedef enum sn_mode {
    SN_MODE_MAT = 0,  /* mat_run (mat_engine.cpp:168-287): u = leak(v) + W-sum [+ ext]; "lif" only */
    SN_MODE_ABM = 1   /* abm_run (abm_engine.cpp:146-243): u = leak(v) + (W-sum + ext), per-neuron
                         stochastic firing (sn_set_fire_probability), no plasticity */
} sn_mode;

typedef struct sn_options {
    int32_t abi_version;     /* = SN_ABI_VERSION */
    int32_t device;          /* CUDA ordinal */
    int32_t storage;         /* sn_storage */
    int32_t precision;       /* sn_precision */
    int32_t exact_order;     /* 1: each post accumulates its inputs sequentially in
                                ascending pre order starting from leak(v), as
                                mat_engine.cpp:173-180 does (bit-exact membranes on
                                float nets; slower).  0: fixed-order parallel
                                reduction (deterministic; exact on integer nets). */
    int32_t record_membrane; /* SimulationConfig::record_membrane */
    int32_t stream_io;       /* 1 (the end-to-end path): each sn_simulate copies its
                                steps' stimulus rows H2D from pinned memory in one
                                transfer, and the kernels store every step's spike
                                words straight into pinned (mapped) host memory.
                                0: stimulus table resident in HBM, raster staged in
                                HBM and copied once per call. */
    int32_t use_graphs;      /* 1: replay the per-step kernels as a CUDA graph */
    int32_t rank;            /* post-neuron partition index (0 when world == 1) */
    int32_t world;           /* number of partitions / GPUs (1 = single GPU) */
    int32_t profile;         /* 1: time every kernel with CUDA events (sn_get_stats) */
    int32_t persistent;      /* 0: auto (one cooperative launch per sn_simulate for small
                                dense single-GPU nets), -1: never */
    int32_t mode;            /* sn_mode: MAT (mat_run) or agent-based (abm_run) semantics */
    int32_t reserved[3];
} sn_options;

typedef struct sn_stats {
    int64_t steps_done;
    int64_t spike_count;        /* spikes of this partition since setup */
    int64_t kernel_launches;    /* kernels launched by the engine since setup */
    int64_t synapses_local;     /* synapses stored on this partition */
    int32_t dense;              /* 1 dense storage, 0 sparse */
    int32_t n_local;            /* posts owned by this partition */
    int32_t first_local;        /* first owned global id */
    int32_t max_delay;
    /* profile (opts.profile == 1): accumulated device time per kernel class */
    double sweep_ms;            /* propagation (+ STDP) sweep over the weights */
    int64_t sweep_launches;
    double neuron_ms;           /* LIF update (+ history/traces) */
    int64_t neuron_launches;
    double exchange_ms;         /* spike-bit all-gather */
    double last_simulate_ms;    /* device time of the last sn_simulate (events) */
    double sweep_bytes_per_launch_last; /* algorithmic bytes of the last sweep */
    double sweep_bytes_total;   /* algorithmic bytes of all sweeps since reset */
    int32_t sweep_kernel;       /* sn_sweep_kernel of the plan chosen at sn_setup */
    int32_t sweep_ctas;         /* grid size of that kernel */
    /* stream_io: host<->device bytes of the last sn_simulate (stimulus rows
       H2D, spike words D2H; 0 when the inputs are resident) */
    double h2d_bytes_last;
    double d2h_bytes_last;
} sn_stats;

typedef enum sn_sweep_kernel {
    SN_SWEEP_DENSE_STREAM = 1,  /* k_dense_stream: 128-bit LDG/STG streaming sweep */
    SN_SWEEP_DENSE_TMA = 2,     /* k_dense_tma: cp.async.bulk ring, one CTA per SM */
    SN_SWEEP_DENSE_EXACT = 3,   /* k_dense_sweep<EXACT>: ascending-pre fp64 order */
    SN_SWEEP_PERSISTENT = 4,    /* k_persistent_dense: whole step loop in one launch */
    SN_SWEEP_SPARSE_PULL = 5,   /* k_sparse_pull: SUB lanes per post, weights streamed */
    SN_SWEEP_SPARSE_DICT = 6,   /* k_sparse_pull with the weight dictionary (4 B/synapse) */
    SN_SWEEP_SPARSE_STREAM = 7, /* k_sparse_stream: flat chunk stream per warp */
    SN_SWEEP_SPARSE_EXACT = 8,  /* k_sparse_exact: one thread per post, ascending pre */
    SN_SWEEP_TINY = 9,          /* k_tiny: whole call in one CTA, state in shared memory
                                   (single partition, N <= 1024, lists fit in smem) */
    SN_SWEEP_SPARSE_TMA = 10,   /* k_sparse_tma: cp.async.bulk-fed stream of uniform-weight
                                   lists (opt-in, SNB_SPARSE_KERNEL=tma) */
    SN_SWEEP_SPARSE_COUNT = 11, /* k_sparse_count: k_sparse_pull specialised for one-weight
                                   static lists (counts the delivering pres) */
    SN_SWEEP_PERSISTENT_COLS = 12, /* k_persistent_cols: whole step loop in one launch, CTAs own
                                     32-post column groups, one grid barrier per step */
    SN_SWEEP_SPARSE_COUNT16 = 13, /* k_sparse_count16: one-weight lists as 16-bit entries in
                                     4095-pre segments (2 B/synapse), delays <= 16 */
    SN_SWEEP_CLUSTER = 14,        /* k_cluster_count: whole step loop in ONE thread-block cluster,
                                     history exchanged through distributed shared memory
                                     (small static one-weight nets, delays <= 31) */
    SN_SWEEP_SPARSE_COUNT8 = 15   /* k_sparse_count8: the 16-bit segmented lists of
                                     k_sparse_count16 over a byte-per-(pre, delay) shared
                                     image (3 x 4095-pre segments), default for them */
} sn_sweep_kernel;

/* ---- lifecycle ---------------------------------------------------------- */
SN_API sn_status sn_options_init(sn_options* opts);
SN_API sn_status sn_engine_create(const sn_options* opts, sn_engine** out);
SN_API void sn_engine_destroy(sn_engine* e);
/* Thread-local message of the last failing call on this thread ("" if none). */
SN_API const char* sn_last_error(void);
SN_API int32_t sn_abi_version(void);
SN_API int32_t sn_device_count(void);

/* ---- model building (before sn_setup) ----------------------------------- */
/* Appends `count` neurons; ids continue from the current count.  axonal_delay
 * may be NULL (all 0).  first_id may be NULL. */
SN_API sn_status sn_add_neurons(sn_engine* e, int64_t count, const double* threshold,
                         const double* leak, const double* reset,
                         const int32_t* refractory, const int32_t* axonal_delay,
                         int64_t* first_id);
/* Appends synapses in list order (the order sn_get_synapse_weights reports).
 * delay and stdp_enabled may be NULL (1 / not plastic). */
SN_API sn_status sn_add_synapses(sn_engine* e, int64_t count, const int32_t* pre,
                          const int32_t* post, const double* weight,
                          const int32_t* delay, const uint8_t* stdp_enabled);
/* Appends stimulus entries (any order; list order matters for float sums). */
SN_API sn_status sn_add_stimulus(sn_engine* e, int64_t count, const int32_t* step,
                          const int32_t* neuron, const double* amplitude);
/* Replaces the stimulus schedule (allowed after setup, between simulate calls). */
SN_API sn_status sn_clear_stimulus(sn_engine* e);
/* Enables windowed pairwise STDP (mat_engine.cpp:210-250). */
SN_API sn_status sn_set_stdp(sn_engine* e, int32_t window, const double* a_plus,
                      const double* a_minus, double w_min, double w_max);
/* StdpConfig::defaults() (model.cpp:10-22); a_plus/a_minus need `*window`
 * (20) slots; pass NULL to query the window only. */
SN_API sn_status sn_stdp_defaults(int32_t* window, double* a_plus, double* a_minus,
                           double* w_min, double* w_max);

/* On-device Erdos-Renyi network, bit-identical to erdos_renyi(n, p, seed)
 * (netgen.cpp:19-54: pair (i,j), i != j, exists iff unit_at(i*n+j) < p on
 * stream 1; thr 1, leak 0, reset 0, refr 0, weight 1, delay 1).  Replaces any
 * neurons/synapses added so far.  Optional variations:
 *   weight            weight of every synapse
 *   delay_max > 1     delay = 1 + RandomStream(seed, delay_stream).below_at(key, delay_max)
 *                     key = synapse list index when delay_by_synapse_index
 *                     (only for p == 1) else pair index i*n + j
 *   stdp_enabled      all synapses plastic
 * Synapse list order = the reference's (i ascending, j ascending). */
SN_API sn_status sn_generate_erdos_renyi(sn_engine* e, int32_t n, double p, uint64_t seed,
                                  double weight, int32_t delay_max,
                                  uint64_t delay_stream, int32_t delay_by_synapse_index,
                                  int32_t stdp_enabled);

/* ---- agent-based mode (sn_options.mode = SN_MODE_ABM) -------------------- */
/* SimulationConfig::seed (model.hpp:80-85): keys the per-(agent, step) random
 * streams of stochastic behaviours (abm_engine.cpp:163-164).  Before sn_setup. */
SN_API sn_status sn_set_seed(sn_engine* e, uint64_t seed);
/* Behaviour of neurons [first, first + count): the fire probability p of
 * StochasticLifBehavior (abm_engine.cpp:28-39) -- above threshold, the neuron
 * fires iff the first unit draw of RandomStream(seed, "abm-agen", id, step)
 * is < p.  p = 1 is "lif" (BehaviorRegistry's built-in, abm_engine.cpp:40),
 * 0.5 is "stochastic_lif" (:41), any p in [0, 1] is what
 * register_stochastic_lif(name, p) registers (bindings.cpp:180-186).
 * Neurons must already be added; p outside [0, 1] is SN_ERR_INVALID_ARGUMENT
 * ("stochastic lif: fire probability must be in [0, 1]").  In MAT mode any
 * p != 1 makes sn_setup fail like mat_init (mat_engine.cpp:116-119). */
SN_API sn_status sn_set_fire_probability(sn_engine* e, int64_t first, int64_t count,
                                         const double* fire_probability);

/* ---- mat_init / mat_run ------------------------------------------------- */
/* Validates (reference messages, model.cpp:34-117) and builds device state. */
SN_API sn_status sn_setup(sn_engine* e);
/* Advances `steps` steps (continuing from the current step). */
SN_API sn_status sn_simulate(sn_engine* e, int32_t steps);
/* Blocks until all queued device work of the engine is done. */
SN_API sn_status sn_synchronize(sn_engine* e);
/* sn_simulate plus the raster of exactly these steps, (step, neuron)
 * ascending, written into the caller's arrays -- the RunResult.raster of a
 * mat_run over these steps (mat_engine.cpp:252-287).  capacity must cover the
 * events (steps x neurons is always enough); *count receives their number.
 * With stream_io and graphs, finished 16-step chunks are expanded on the host
 * while later chunks run on the device.  The events also stay available to
 * sn_get_raster. */
SN_API sn_status sn_simulate_raster(sn_engine* e, int32_t steps, int32_t* out_steps, int32_t* out_neurons,
                                    int64_t capacity, int64_t* count);
/* One step of mat_step (mat_engine.cpp:168-208; the borrowed spike list of
 * mat_engine.hpp:92-94): the step's external input is exactly `ext` -- n
 * amplitudes, or ext_len = 0 for none (the stimulus schedule is not consulted
 * for this step) -- followed by apply_stdp when STDP is configured and
 * plasticity is on.  Writes the step's spiking ids ascending into `spikes`
 * (capacity `cap`; spikes = NULL only reports *count).  ext_len other than 0
 * or n: SN_ERR_INVALID_ARGUMENT "mat_step: ext must have one amplitude per
 * neuron" (mat_engine.cpp:170-171).  Single-partition engines. */
SN_API sn_status sn_step(sn_engine* e, const double* ext, int64_t ext_len, int32_t* spikes,
                         int64_t cap, int64_t* count);
/* Whether the following steps apply STDP (default on): off = mat_step
 * without apply_stdp (mat_engine.hpp:92-98 exposes them separately).  The
 * history and traces keep advancing, so re-enabling resumes exactly as the
 * reference's apply_stdp would, including its first-call clamp of every
 * plastic weight (mat_engine.cpp:243-249) on the first plastic step. */
SN_API sn_status sn_set_plasticity(sn_engine* e, int32_t enabled);

/* ---- results ------------------------------------------------------------ */
/* Spike events of this partition since setup, (step, neuron) ascending. */
SN_API sn_status sn_raster_size(sn_engine* e, int64_t* events);
SN_API sn_status sn_get_raster(sn_engine* e, int32_t* steps, int32_t* neurons, int64_t capacity);
/* Drops the host raster accumulated so far (long runs). */
SN_API sn_status sn_clear_raster(sn_engine* e);
/* Final membrane of this partition's neurons (n_local doubles, fp64). */
SN_API sn_status sn_get_membrane(sn_engine* e, double* out, int64_t count);
/* membrane_trace rows (one per simulated step) x n_local. */
SN_API sn_status sn_membrane_trace_rows(sn_engine* e, int64_t* rows);
SN_API sn_status sn_get_membrane_trace(sn_engine* e, double* out, int64_t count);
/* Current weight of every synapse added with sn_add_synapses, in list order
 * (fp64; fp32 storage is widened).  Partitioned engines report 0 for
 * synapses whose post they do not own. */
SN_API sn_status sn_get_synapse_weights(sn_engine* e, double* out, int64_t count);
/* Dense export of this partition's weight block W[pre][post_local]
 * (n x n_local doubles) -- absent synapses read 0 (test/debug helper). */
SN_API sn_status sn_get_weight_matrix(sn_engine* e, double* out, int64_t count);
/* Weight census on the device (dense storage; cfg5's 36.9 GB matrix cannot be
 * read back): counts[k] = stored weights of the n x n_local block equal to
 * values[k] rounded to the storage precision (k < count <= 8, first match),
 * counts[count] = every other cell, absent synapses (stored 0) included. */
SN_API sn_status sn_weight_value_counts(sn_engine* e, const double* values, int32_t count, int64_t* counts);
SN_API sn_status sn_get_stats(sn_engine* e, sn_stats* out);
SN_API sn_status sn_reset_stats(sn_engine* e);

/* ---- multi-GPU (post-neuron partitioning) -------------------------------- */
/* Size of an NCCL unique id (128). */
SN_API int32_t sn_comm_id_size(void);
/* rank 0 creates the id; the host broadcasts it (e.g. torch.distributed). */
SN_API sn_status sn_comm_create_id(uint8_t* id_out);
/* Joins the NCCL communicator; sn_simulate then all-gathers the spike
 * bitmask once per step (in-place ncclAllGather of n/8 bytes). */
SN_API sn_status sn_comm_init(sn_engine* e, const uint8_t* id, int32_t rank, int32_t world);
/* Host-driven exchange (used to emulate partitions on one GPU and by tests):
 * sn_step_local runs the LIF update of one step and leaves this partition's
 * spike words in its bitmask slice; the host copies every partition's slice
 * into every other partition's full bitmask with sn_put_spike_words, then
 * sn_step_finish runs history/traces and the sweep. */
SN_API sn_status sn_partition_range(int32_t n, int32_t rank, int32_t world, int32_t* first,
                             int32_t* count);
SN_API sn_status sn_step_local(sn_engine* e);
SN_API sn_status sn_get_spike_words(sn_engine* e, uint32_t* out, int64_t words);
SN_API sn_status sn_put_spike_words(sn_engine* e, int32_t first_word, const uint32_t* words,
                             int64_t count);
SN_API sn_status sn_step_finish(sn_engine* e);

/* Peer-to-peer exchange fused into the neuron kernel (alternative to NCCL):
 * every rank exports 128 bytes of CUDA IPC handles (its spike bitmask and its
 * per-rank flag array), the host all-gathers them (rank-major), each rank
 * opens its peers'; from then on the neuron kernel stores its spike words
 * directly into every peer's bitmask over NVLink and releases a step flag,
 * and the history kernel acquires all flags before reading.  One process per
 * GPU, all GPUs peer-capable (NVSwitch). */
SN_API int32_t sn_p2p_handle_size(void);
SN_API sn_status sn_p2p_get_handles(sn_engine* e, uint8_t* out, int64_t capacity);
SN_API sn_status sn_p2p_open(sn_engine* e, const uint8_t* all_handles, int32_t world);
/* Same protocol for `world` engines of ONE process on ONE device (partition
 * emulation; drive them with sn_step_local on all, then sn_step_finish). */
SN_API sn_status sn_p2p_connect_local(sn_engine* const* engines, int32_t world);

#ifdef __cplusplus
}
#endif

#endif /* SUPERNEURO_MAT_H */
