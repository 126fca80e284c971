// Reference-side binding: the pybind11 module a spikeforge maintainer adds to
// route the Python mat_run onto the B200 engine.  It sits
// next to the reference's own module spikeforge._core
// (proj/python/src/bindings.cpp), takes and returns the reference's own types
// (NetworkDef, SimulationConfig, StimulusSchedule, RunResult -- registered by
// _core) and calls this repo's C ABI (include/superneuro_mat.h, libsnmat.so).
//
//   import spikeforge as sf, spikeforge_gpu as g
//   sf.mat_run = g.mat_run_gpu            # drop-in: same arguments, same result
//
// Semantics follow mat_run (mat_engine.cpp:252-287): stimulus validated with
// the reference's messages (validate_stimulus, model.cpp:86-102), a raster of
// ascending (step, neuron) events, membrane_trace rows when
// cfg.record_membrane.  Deliberate difference: delays > 1 are simulated
// natively (mat_init asks for lower_delays first, mat_engine.cpp:127-131).
// Exceptions: SN_ERR_INVALID_ARGUMENT -> std::invalid_argument (ValueError),
// SN_ERR_LOGIC -> std::logic_error, anything else -> std::runtime_error.
#include "spikeforge/model.hpp"
#include "superneuro_mat.h"

#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace py = pybind11;
using namespace spikeforge;

namespace {

void check(sn_status st) {
    if (st == SN_OK) return;
    const std::string msg = sn_last_error();
    if (st == SN_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == SN_ERR_LOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

struct Engine {
    sn_engine* e = nullptr;
    explicit Engine(int device) {
        sn_options o;
        check(sn_options_init(&o));
        o.device = device;
        check(sn_engine_create(&o, &e));
    }
    ~Engine() { sn_engine_destroy(e); }
};

RunResult mat_run_gpu(const NetworkDef& net, const SimulationConfig& cfg, const StimulusSchedule& stim,
                      int device) {
    if (cfg.steps < 1) throw std::invalid_argument("mat_run: steps must be >= 1");
    const int n = net.neuron_count();
    {   // mat_run validates the stimulus against the network first (mat_engine.cpp:256-258)
        const auto bad = validate_stimulus(stim, n, cfg.steps);
        if (!bad.empty()) {
            std::string m = "mat_run: " + bad.front();
            if (bad.size() > 1) m += " (+" + std::to_string(bad.size() - 1) + " more)";
            throw std::invalid_argument(m);
        }
    }
    Engine g(device);
    for (int i = 0; i < n; ++i)
        if (net.neurons[i].behavior != "lif")
            throw std::invalid_argument("mat_init: homogeneous backend supports \"lif\" only; neuron " +
                                        std::to_string(i) + " has behavior \"" + net.neurons[i].behavior + "\"");
    std::vector<double> thr(n), leak(n), reset(n);
    std::vector<int32_t> refr(n), ax(n);
    for (int i = 0; i < n; ++i) {
        const NeuronParams& q = net.neurons[i];
        thr[i] = q.threshold;
        leak[i] = q.leak;
        reset[i] = q.reset;
        refr[i] = q.refractory;
        ax[i] = q.axonal_delay;
    }
    check(sn_add_neurons(g.e, n, thr.data(), leak.data(), reset.data(), refr.data(), ax.data(), nullptr));
    const size_t m = net.synapses.size();
    std::vector<int32_t> pre(m), post(m), delay(m);
    std::vector<double> w(m);
    std::vector<uint8_t> plastic(m);
    for (size_t s = 0; s < m; ++s) {
        const SynapseDef& y = net.synapses[s];
        pre[s] = y.pre;
        post[s] = y.post;
        w[s] = y.weight;
        delay[s] = y.delay;
        plastic[s] = y.stdp_enabled ? 1 : 0;
    }
    check(sn_add_synapses(g.e, static_cast<int64_t>(m), pre.data(), post.data(), w.data(), delay.data(),
                          plastic.data()));
    if (cfg.stdp)
        check(sn_set_stdp(g.e, cfg.stdp->window, cfg.stdp->a_plus.data(), cfg.stdp->a_minus.data(),
                          cfg.stdp->w_min, cfg.stdp->w_max));
    const size_t k = stim.entries.size();
    std::vector<int32_t> ss(k), sn(k);
    std::vector<double> sa(k);
    for (size_t i = 0; i < k; ++i) {
        ss[i] = stim.entries[i].step;
        sn[i] = stim.entries[i].neuron;
        sa[i] = stim.entries[i].amplitude;
    }
    check(sn_add_stimulus(g.e, static_cast<int64_t>(k), ss.data(), sn.data(), sa.data()));
    check(sn_setup(g.e));
    RunResult out;
    out.raster.neuron_count = n;
    out.raster.step_count = cfg.steps;
    if (cfg.record_membrane) {
        // one step per call so each row of the trace is read as it happens
        std::vector<double> row(static_cast<size_t>(n));
        for (int t = 0; t < cfg.steps; ++t) {
            check(sn_simulate(g.e, 1));
            check(sn_get_membrane(g.e, row.data(), n));
            out.membrane_trace.push_back(row);
        }
    } else {
        check(sn_simulate(g.e, cfg.steps));
    }
    int64_t ne = 0;
    check(sn_raster_size(g.e, &ne));
    std::vector<int32_t> es(static_cast<size_t>(ne)), en(static_cast<size_t>(ne));
    check(sn_get_raster(g.e, es.data(), en.data(), ne));
    out.raster.events.reserve(static_cast<size_t>(ne));
    for (int64_t i = 0; i < ne; ++i) out.raster.events.push_back({es[i], en[i]});
    return out;
}

}  // namespace

PYBIND11_MODULE(spikeforge_gpu, m) {
    m.doc() = "spikeforge.mat_run on the B200 engine (this repo's libsnmat.so)";
    py::module_::import("spikeforge._core");  // registers the reference's types
    m.def(
        "mat_run_gpu",
        [](const NetworkDef& net, const SimulationConfig& cfg, const StimulusSchedule& stim, int device) {
            py::gil_scoped_release release;
            return mat_run_gpu(net, cfg, stim, device);
        },
        py::arg("net"), py::arg("cfg"), py::arg("stim") = StimulusSchedule{}, py::arg("device") = 0);
    m.def("device_count", &sn_device_count);
}
