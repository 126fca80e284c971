// superneuro_mat.hpp -- header-only C++ facade over the C ABI
// (include/superneuro_mat.h) with SuperNeuro's MAT-mode model API
// (create_neuron / create_synapse / add_spike / setup / simulate) and a
// spikeforge-compatible mat_run (reference proj/include/spikeforge/mat_engine.hpp:100-103).
//
//   superneuro::Model m;
//   int a = m.create_neuron(1.0, 0.0, 0.0, 0);      // threshold, leak, reset, refractory
//   int b = m.create_neuron();
//   m.create_synapse(a, b, 2.0, 3, false);           // weight, delay, stdp
//   m.add_spike(0, a, 2.0);                          // step, neuron, amplitude
//   m.setup();
//   auto r = m.simulate(10);                         // r.events: (step, neuron) ascending
//
// Agent-based runs (abm_run, abm_engine.cpp:218-243): construct with
// SN_MODE_ABM, give stochastic neurons a fire probability (1 = "lif",
// 0.5 = "stochastic_lif") and set the run seed:
//
//   superneuro::Model m(0, SN_STORAGE_AUTO, SN_WEIGHTS_F64, SN_MODE_ABM);
//   m.set_exact_order(true);                        // bit-exact with the reference
//   int c = m.create_neuron(1.0, 0.0, 0.0, 0, 0, 0.5);
//   m.set_seed(9);
//
// Errors surface as std::invalid_argument / std::logic_error / std::runtime_error
// with the engine's message, the same exception types the reference throws.
#pragma once

#include "superneuro_mat.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace superneuro {

inline void check(sn_status st) {
    if (st == SN_OK) return;
    const std::string msg = sn_last_error();
    switch (st) {
        case SN_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SN_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

struct SpikeEvent {
    int32_t step = 0;
    int32_t neuron = 0;
};

struct Result {
    std::vector<SpikeEvent> events;     // (step, neuron) ascending, like SpikeRaster
    std::vector<double> membrane;       // final membrane per neuron
    std::vector<double> weights;        // final weight per synapse (create_synapse order)
};

struct StdpParams {                     // StdpConfig (model.hpp:67-78)
    int32_t window = 20;
    std::vector<double> a_plus, a_minus;
    double w_min = 0.0, w_max = 1.0;
    static StdpParams defaults() {
        StdpParams p;
        int32_t w = 0;
        check(sn_stdp_defaults(&w, nullptr, nullptr, nullptr, nullptr));
        p.window = w;
        p.a_plus.resize(w);
        p.a_minus.resize(w);
        check(sn_stdp_defaults(&w, p.a_plus.data(), p.a_minus.data(), &p.w_min, &p.w_max));
        return p;
    }
};

class Model {
public:
    explicit Model(int device = 0, sn_storage storage = SN_STORAGE_AUTO,
                   sn_precision precision = SN_WEIGHTS_F32, sn_mode mode = SN_MODE_MAT) {
        check(sn_options_init(&opts_));
        opts_.device = device;
        opts_.storage = storage;
        opts_.precision = precision;
        opts_.mode = mode;
    }
    // sequential ascending-pre accumulation (bit-exact membranes on float nets)
    void set_exact_order(bool on) { opts_.exact_order = on ? 1 : 0; }
    // SimulationConfig::seed: keys the stochastic behaviours of SN_MODE_ABM
    void set_seed(uint64_t seed) { seed_ = seed; }
    ~Model() {
        if (e_) sn_engine_destroy(e_);
    }
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;

    int create_neuron(double threshold = 1.0, double leak = 0.0, double reset_state = 0.0,
                      int refractory_period = 0, int axonal_delay = 0, double fire_probability = 1.0) {
        fire_p_.push_back(fire_probability);
        thr_.push_back(threshold);
        leak_.push_back(leak);
        reset_.push_back(reset_state);
        refr_.push_back(refractory_period);
        axonal_.push_back(axonal_delay);
        return static_cast<int>(thr_.size()) - 1;
    }
    int create_synapse(int pre, int post, double weight = 1.0, int delay = 1, bool enable_stdp = false) {
        pre_.push_back(pre);
        post_.push_back(post);
        w_.push_back(weight);
        d_.push_back(delay);
        stdp_.push_back(enable_stdp ? 1 : 0);
        return static_cast<int>(pre_.size()) - 1;
    }
    void add_spike(int step, int neuron, double amplitude = 1.0) {
        st_.push_back(step);
        sn_.push_back(neuron);
        sa_.push_back(amplitude);
    }
    void setup(const StdpParams* stdp = nullptr) {
        check(sn_engine_create(&opts_, &e_));
        const int64_t n = static_cast<int64_t>(thr_.size());
        check(sn_add_neurons(e_, n, thr_.data(), leak_.data(), reset_.data(), refr_.data(),
                             axonal_.data(), nullptr));
        check(sn_add_synapses(e_, static_cast<int64_t>(pre_.size()), pre_.data(), post_.data(),
                              w_.data(), d_.data(), stdp_.data()));
        if (stdp)
            check(sn_set_stdp(e_, stdp->window, stdp->a_plus.data(), stdp->a_minus.data(),
                              stdp->w_min, stdp->w_max));
        check(sn_set_seed(e_, seed_));
        for (double p : fire_p_)
            if (p != 1.0) {
                check(sn_set_fire_probability(e_, 0, n, fire_p_.data()));
                break;
            }
        check(sn_setup(e_));
    }
    Result simulate(int time_steps) {
        if (!e_) throw std::logic_error("simulate: call setup() first");
        if (pushed_ < st_.size()) {
            check(sn_add_stimulus(e_, static_cast<int64_t>(st_.size() - pushed_), st_.data() + pushed_,
                                  sn_.data() + pushed_, sa_.data() + pushed_));
            pushed_ = st_.size();
        }
        check(sn_clear_raster(e_));
        check(sn_simulate(e_, time_steps));
        Result r;
        int64_t ne = 0;
        check(sn_raster_size(e_, &ne));
        std::vector<int32_t> s(static_cast<size_t>(ne)), q(static_cast<size_t>(ne));
        check(sn_get_raster(e_, s.data(), q.data(), ne));
        r.events.resize(static_cast<size_t>(ne));
        for (int64_t i = 0; i < ne; ++i) r.events[i] = {s[i], q[i]};
        r.membrane.resize(thr_.size());
        check(sn_get_membrane(e_, r.membrane.data(), static_cast<int64_t>(r.membrane.size())));
        r.weights.resize(pre_.size());
        if (!pre_.empty())
            check(sn_get_synapse_weights(e_, r.weights.data(), static_cast<int64_t>(r.weights.size())));
        return r;
    }

    // mat_step (mat_engine.cpp:168-208): one step whose external input is
    // exactly `ext` (one amplitude per neuron, or empty); returns the step's
    // spiking neurons ascending -- the list mat_step lends (mat_engine.hpp:92-94).
    // apply_stdp follows when STDP is set up and plasticity is on.
    const std::vector<int>& step(const std::vector<double>& ext = {}) {
        if (!e_) throw std::logic_error("step: call setup() first");
        int64_t k = 0;
        step_spikes_.resize(thr_.size());
        static_assert(sizeof(int) == sizeof(int32_t), "int32 spike ids");
        check(sn_step(e_, ext.empty() ? nullptr : ext.data(), static_cast<int64_t>(ext.size()),
                      reinterpret_cast<int32_t*>(step_spikes_.data()), static_cast<int64_t>(step_spikes_.size()), &k));
        step_spikes_.resize(static_cast<size_t>(k));
        return step_spikes_;
    }
    // whether following steps run apply_stdp after mat_step (mat_engine.hpp:92-98)
    void set_plasticity(bool on) {
        if (!e_) throw std::logic_error("set_plasticity: call setup() first");
        check(sn_set_plasticity(e_, on ? 1 : 0));
    }

private:
    std::vector<int> step_spikes_;
    sn_options opts_{};
    sn_engine* e_ = nullptr;
    std::vector<double> thr_, leak_, reset_, w_, sa_, fire_p_;
    uint64_t seed_ = 0;
    std::vector<int32_t> refr_, axonal_, pre_, post_, d_, st_, sn_;
    std::vector<uint8_t> stdp_;
    size_t pushed_ = 0;
};

}  // namespace superneuro
