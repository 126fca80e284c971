// extern "C" boundary (include/superneuro_mat.h): exceptions never cross it;
// each call returns an sn_status and leaves a thread-local message, the way
// the reference surfaces std::invalid_argument / std::logic_error text
// (mat_engine.cpp:15-21, spikeforge_main.cpp:319-328).
#include "../../include/superneuro_mat.h"

#include "engine.hpp"
#include "nccl_dl.hpp"

#include <cmath>
#include <cstring>
#include <new>
#include <string>

using namespace snb;

struct sn_engine {
    Engine impl;
    explicit sn_engine(const sn_options& o) : impl(o) {}
};

namespace {

thread_local std::string g_error;

template <typename F>
sn_status guard(F&& f) {
    try {
        g_error.clear();
        f();
        return SN_OK;
    } catch (const InvalidArgument& e) {
        g_error = e.what();
        return SN_ERR_INVALID_ARGUMENT;
    } catch (const LogicError& e) {
        g_error = e.what();
        return SN_ERR_LOGIC;
    } catch (const OutOfMemory& e) {
        g_error = e.what();
        return SN_ERR_OOM;
    } catch (const CudaError& e) {
        g_error = e.what();
        return SN_ERR_CUDA;
    } catch (const NcclError& e) {
        g_error = e.what();
        return SN_ERR_NCCL;
    } catch (const Unsupported& e) {
        g_error = e.what();
        return SN_ERR_UNSUPPORTED;
    } catch (const std::bad_alloc&) {
        g_error = "out of host memory";
        return SN_ERR_OOM;
    } catch (const std::exception& e) {
        g_error = e.what();
        return SN_ERR_LOGIC;
    }
}

#define SN_NEED(e)                                                   \
    do {                                                             \
        if (!(e)) throw InvalidArgument("null sn_engine handle");    \
    } while (0)

}  // namespace

extern "C" {

int32_t sn_abi_version(void) { return SN_ABI_VERSION; }

const char* sn_last_error(void) { return g_error.c_str(); }

int32_t sn_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

sn_status sn_options_init(sn_options* o) {
    return guard([&] {
        if (!o) throw InvalidArgument("sn_options_init: null options");
        std::memset(o, 0, sizeof(*o));
        o->abi_version = SN_ABI_VERSION;
        o->storage = SN_STORAGE_AUTO;
        o->precision = SN_WEIGHTS_F32;
        o->use_graphs = 1;
        o->world = 1;
    });
}

sn_status sn_engine_create(const sn_options* o, sn_engine** out) {
    return guard([&] {
        if (!o || !out) throw InvalidArgument("sn_engine_create: null argument");
        if (o->abi_version != SN_ABI_VERSION)
            throw InvalidArgument("sn_engine_create: options ABI version mismatch");
        *out = nullptr;
        *out = new sn_engine(*o);
    });
}

void sn_engine_destroy(sn_engine* e) { delete e; }

sn_status sn_add_neurons(sn_engine* e, int64_t count, const double* threshold, const double* leak,
                         const double* reset, const int32_t* refractory, const int32_t* axonal_delay,
                         int64_t* first_id) {
    return guard([&] {
        SN_NEED(e);
        e->impl.add_neurons(count, threshold, leak, reset, refractory, axonal_delay, first_id);
    });
}

sn_status sn_add_synapses(sn_engine* e, int64_t count, const int32_t* pre, const int32_t* post,
                          const double* weight, const int32_t* delay, const uint8_t* stdp_enabled) {
    return guard([&] {
        SN_NEED(e);
        e->impl.add_synapses(count, pre, post, weight, delay, stdp_enabled);
    });
}

sn_status sn_add_stimulus(sn_engine* e, int64_t count, const int32_t* step, const int32_t* neuron,
                          const double* amplitude) {
    return guard([&] {
        SN_NEED(e);
        e->impl.add_stimulus(count, step, neuron, amplitude);
    });
}

sn_status sn_clear_stimulus(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.clear_stimulus();
    });
}

sn_status sn_set_stdp(sn_engine* e, int32_t window, const double* a_plus, const double* a_minus,
                      double w_min, double w_max) {
    return guard([&] {
        SN_NEED(e);
        e->impl.set_stdp(window, a_plus, a_minus, w_min, w_max);
    });
}

sn_status sn_stdp_defaults(int32_t* window, double* a_plus, double* a_minus, double* w_min,
                           double* w_max) {
    return guard([&] {
        // StdpConfig::defaults() (model.cpp:10-22): a[k-1] = A exp(-k/5), k = 1..20
        if (!window) throw InvalidArgument("sn_stdp_defaults: null window");
        *window = 20;
        for (int k = 1; k <= 20; ++k) {
            if (a_plus) a_plus[k - 1] = 0.01 * std::exp(-k / 5.0);
            if (a_minus) a_minus[k - 1] = 0.012 * std::exp(-k / 5.0);
        }
        if (w_min) *w_min = 0.0;
        if (w_max) *w_max = 1.0;
    });
}

sn_status sn_set_seed(sn_engine* e, uint64_t seed) {
    return guard([&] {
        SN_NEED(e);
        e->impl.set_seed(seed);
    });
}

sn_status sn_set_fire_probability(sn_engine* e, int64_t first, int64_t count, const double* p) {
    return guard([&] {
        SN_NEED(e);
        e->impl.set_fire_probability(first, count, p);
    });
}

sn_status sn_generate_erdos_renyi(sn_engine* e, int32_t n, double p, uint64_t seed, double weight,
                                  int32_t delay_max, uint64_t delay_stream, int32_t by_syn,
                                  int32_t stdp_enabled) {
    return guard([&] {
        SN_NEED(e);
        e->impl.generate_er(n, p, seed, weight, delay_max, delay_stream, by_syn, stdp_enabled);
    });
}

sn_status sn_setup(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.setup();
    });
}

sn_status sn_simulate(sn_engine* e, int32_t steps) {
    return guard([&] {
        SN_NEED(e);
        e->impl.simulate(steps);
    });
}

sn_status sn_synchronize(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.synchronize();
    });
}

sn_status sn_raster_size(sn_engine* e, int64_t* events) {
    return guard([&] {
        SN_NEED(e);
        if (!events) throw InvalidArgument("sn_raster_size: null output");
        *events = e->impl.raster_size();
    });
}

sn_status sn_get_raster(sn_engine* e, int32_t* steps, int32_t* neurons, int64_t capacity) {
    return guard([&] {
        SN_NEED(e);
        e->impl.get_raster(steps, neurons, capacity);
    });
}

sn_status sn_clear_raster(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.clear_raster();
    });
}

sn_status sn_get_membrane(sn_engine* e, double* out, int64_t count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.get_membrane(out, count);
    });
}

sn_status sn_membrane_trace_rows(sn_engine* e, int64_t* rows) {
    return guard([&] {
        SN_NEED(e);
        *rows = e->impl.trace_rows();
    });
}

sn_status sn_get_membrane_trace(sn_engine* e, double* out, int64_t count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.get_trace(out, count);
    });
}

sn_status sn_get_synapse_weights(sn_engine* e, double* out, int64_t count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.get_synapse_weights(out, count);
    });
}

sn_status sn_get_weight_matrix(sn_engine* e, double* out, int64_t count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.get_weight_matrix(out, count);
    });
}

sn_status sn_get_stats(sn_engine* e, sn_stats* out) {
    return guard([&] {
        SN_NEED(e);
        if (!out) throw InvalidArgument("sn_get_stats: null output");
        e->impl.get_stats(out);
    });
}

sn_status sn_reset_stats(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.reset_stats();
    });
}

int32_t sn_comm_id_size(void) { return NCCL_UNIQUE_ID_BYTES; }

sn_status sn_comm_create_id(uint8_t* id_out) {
    return guard([&] {
        if (!id_out) throw InvalidArgument("sn_comm_create_id: null output");
        nccl_unique_id(id_out);
    });
}

sn_status sn_comm_init(sn_engine* e, const uint8_t* id, int32_t rank, int32_t world) {
    return guard([&] {
        SN_NEED(e);
        if (!id) throw InvalidArgument("sn_comm_init: null id");
        e->impl.comm_init(id, rank, world);
    });
}

sn_status sn_partition_range(int32_t n, int32_t rank, int32_t world, int32_t* first, int32_t* count) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world || n < 0 || !first || !count)
            throw InvalidArgument("sn_partition_range: bad arguments");
        Engine::partition(n, rank, world, first, count);
    });
}

sn_status sn_weight_value_counts(sn_engine* e, const double* values, int32_t count, int64_t* counts) {
    return guard([&] {
        SN_NEED(e);
        e->impl.weight_value_counts(values, count, counts);
    });
}

sn_status sn_step(sn_engine* e, const double* ext, int64_t ext_len, int32_t* spikes, int64_t cap,
                  int64_t* count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.step(ext, ext_len, spikes, cap, count);
    });
}

sn_status sn_simulate_raster(sn_engine* e, int32_t steps, int32_t* out_steps, int32_t* out_neurons,
                             int64_t capacity, int64_t* count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.simulate_raster(steps, out_steps, out_neurons, capacity, count);
    });
}

sn_status sn_set_plasticity(sn_engine* e, int32_t enabled) {
    return guard([&] {
        SN_NEED(e);
        e->impl.set_plasticity(enabled != 0);
    });
}

sn_status sn_step_local(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.step_local();
    });
}

sn_status sn_get_spike_words(sn_engine* e, uint32_t* out, int64_t words) {
    return guard([&] {
        SN_NEED(e);
        e->impl.get_spike_words(out, words);
    });
}

sn_status sn_put_spike_words(sn_engine* e, int32_t first_word, const uint32_t* words, int64_t count) {
    return guard([&] {
        SN_NEED(e);
        e->impl.put_spike_words(first_word, words, count);
    });
}

int32_t sn_p2p_handle_size(void) { return 2 * Engine::kIpcHandleBytes; }

sn_status sn_p2p_get_handles(sn_engine* e, uint8_t* out, int64_t capacity) {
    return guard([&] {
        SN_NEED(e);
        if (!out) throw InvalidArgument("sn_p2p_get_handles: null output");
        e->impl.p2p_get_handles(out, capacity);
    });
}

sn_status sn_p2p_open(sn_engine* e, const uint8_t* all_handles, int32_t world) {
    return guard([&] {
        SN_NEED(e);
        if (!all_handles) throw InvalidArgument("sn_p2p_open: null handles");
        e->impl.p2p_open(all_handles, world);
    });
}

sn_status sn_p2p_connect_local(sn_engine* const* engines, int32_t world) {
    return guard([&] {
        if (!engines || world < 1) throw InvalidArgument("sn_p2p_connect_local: bad arguments");
        std::vector<Engine*> impls(static_cast<size_t>(world));
        for (int q = 0; q < world; ++q) {
            SN_NEED(engines[q]);
            impls[q] = &engines[q]->impl;
        }
        Engine::p2p_connect_local(impls.data(), world);
    });
}

sn_status sn_step_finish(sn_engine* e) {
    return guard([&] {
        SN_NEED(e);
        e->impl.step_finish();
    });
}

}  // extern "C"
