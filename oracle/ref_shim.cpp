// TEST INFRASTRUCTURE ONLY.  extern "C" shim over the reference's own C++
// library (spikeforge, /root/reference/proj/src), compiled from the read-only
// sources by oracle/Makefile into oracle/_ref/libspikeforge_ref.so.  Nothing
// here is shipped: tests/ use it to pin oracle/mat_oracle.c and to produce the
// golden fixtures; bench.py --impl reference uses ref_bench_scenario() to time
// the reference CPU path.
//
// Every entry point calls the reference's public API unchanged:
//   mat_init / mat_step / apply_stdp / mat_run   proj/src/mat_engine.cpp:109-287
//   oracle_run                                   proj/src/oracle.cpp:19-102
//   abm_run                                      proj/src/abm_engine.cpp:208-243
//   lower_delays / restrict_raster               proj/src/lowering.cpp:22-59, model.cpp:141-151
//   erdos_renyi / build_scenario                 proj/src/netgen.cpp:19-86
//   validate_network / StdpConfig::defaults      proj/src/model.cpp:10-117

#include "orc_problem.h"

#include "spikeforge/abm_engine.hpp"
#include "spikeforge/lowering.hpp"
#include "spikeforge/mat_engine.hpp"
#include "spikeforge/model.hpp"
#include "spikeforge/netgen.hpp"
#include "spikeforge/oracle.hpp"
#include "spikeforge/rng.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace spikeforge;

namespace {

double peak_rss_gb() {  // VmHWM of this process
    FILE* f = std::fopen("/proc/self/status", "r");
    if (!f) return -1.0;
    char line[256];
    double kb = -1.0;
    while (std::fgets(line, sizeof line, f))
        if (std::strncmp(line, "VmHWM:", 6) == 0) kb = std::atof(line + 6);
    std::fclose(f);
    return kb / (1024.0 * 1024.0);
}

NetworkDef to_net(const orc_problem* p) {
    NetworkDef net;
    net.neurons.resize(static_cast<std::size_t>(p->n));
    for (int i = 0; i < p->n; ++i) {
        NeuronParams& q = net.neurons[i];
        q.threshold = p->threshold[i];
        q.leak = p->leak[i];
        q.reset = p->reset[i];
        q.refractory = p->refractory[i];
        q.axonal_delay = p->axonal ? p->axonal[i] : 0;
        q.behavior = "lif";
    }
    net.synapses.resize(static_cast<std::size_t>(p->m));
    for (int64_t s = 0; s < p->m; ++s) {
        SynapseDef& y = net.synapses[s];
        y.pre = p->pre[s];
        y.post = p->post[s];
        y.weight = p->weight[s];
        y.delay = p->delay ? p->delay[s] : 1;
        y.stdp_enabled = p->stdp ? p->stdp[s] != 0 : false;
    }
    return net;
}

StimulusSchedule to_stim(const orc_problem* p) {
    StimulusSchedule stim;
    stim.entries.resize(static_cast<std::size_t>(p->k));
    for (int64_t i = 0; i < p->k; ++i)
        stim.entries[i] = StimulusEntry{p->st_step[i], p->st_neuron[i], p->st_amp[i]};
    return stim;
}

SimulationConfig to_cfg(const orc_problem* p) {
    SimulationConfig cfg;
    cfg.steps = p->steps;
    cfg.record_membrane = p->record_membrane != 0;
    if (p->stdp_on) {
        StdpConfig s;
        s.window = p->window;
        s.a_plus.assign(p->a_plus, p->a_plus + std::max(0, p->window));
        s.a_minus.assign(p->a_minus, p->a_minus + std::max(0, p->window));
        s.w_min = p->w_min;
        s.w_max = p->w_max;
        cfg.stdp = s;
    }
    return cfg;
}

template <typename T>
T* dup(const std::vector<T>& v) {
    T* out = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    if (!v.empty()) std::memcpy(out, v.data(), sizeof(T) * v.size());
    return out;
}

void put_raster(const SpikeRaster& r, orc_result* out) {
    out->n_events = static_cast<int64_t>(r.events.size());
    std::vector<int32_t> s(r.events.size()), n(r.events.size());
    for (std::size_t i = 0; i < r.events.size(); ++i) {
        s[i] = r.events[i].step;
        n[i] = r.events[i].neuron;
    }
    out->ev_step = dup(s);
    out->ev_neuron = dup(n);
    out->spike_count = out->n_events;
}

template <typename F>
int guarded(orc_result* out, F&& f) {
    std::memset(out, 0, sizeof(*out));
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        out->status = 1;
        std::snprintf(out->error, sizeof(out->error), "%s", e.what());
    } catch (const std::logic_error& e) {
        out->status = 2;
        std::snprintf(out->error, sizeof(out->error), "%s", e.what());
    } catch (const std::exception& e) {
        out->status = 3;
        std::snprintf(out->error, sizeof(out->error), "%s", e.what());
    }
    return out->status;
}

// The loop of mat_run (mat_engine.cpp:252-287) spelled out so the final
// MatState (membrane, weights) is observable; tests assert its raster equals
// mat_run's own.
struct MatOutcome {
    SpikeRaster raster;
    std::vector<std::vector<double>> trace;
    MatState st;
};

// plastic_steps (optional, one byte per step): apply_stdp only after the
// mat_step of steps with a non-zero byte -- the reference's public API driven
// like an engine whose plasticity is switched off for some steps.
MatOutcome mat_loop(const NetworkDef& net, const SimulationConfig& cfg,
                    const StimulusSchedule& stim, WeightStorage storage,
                    const uint8_t* plastic_steps = nullptr) {
    if (cfg.steps < 1) throw std::invalid_argument("mat_run: steps must be >= 1");
    MatOutcome o;
    o.st = mat_init(net, cfg, storage);
    {
        auto bad = validate_stimulus(stim, o.st.n, cfg.steps);
        if (!bad.empty()) throw std::invalid_argument("mat_run: " + bad.front());
    }
    std::vector<StimulusEntry> sorted = stim.entries;
    std::stable_sort(sorted.begin(), sorted.end(),
                     [](const StimulusEntry& a, const StimulusEntry& b) { return a.step < b.step; });
    o.raster.neuron_count = o.st.n;
    o.raster.step_count = cfg.steps;
    std::vector<double> ext(o.st.n, 0.0);
    std::size_t cursor = 0;
    for (int t = 0; t < cfg.steps; ++t) {
        const std::size_t first = cursor;
        bool any_ext = false;
        while (cursor < sorted.size() && sorted[cursor].step == t) {
            ext[sorted[cursor].neuron] += sorted[cursor].amplitude;
            any_ext = true;
            ++cursor;
        }
        const std::vector<int>& spiked =
            mat_step(o.st, any_ext ? std::span<const double>(ext) : std::span<const double>());
        if (cfg.stdp && (!plastic_steps || plastic_steps[t])) apply_stdp(o.st, *cfg.stdp);
        for (int j : spiked) o.raster.events.push_back({t, j});
        if (cfg.record_membrane) o.trace.push_back(o.st.membrane);
        for (std::size_t k = first; k < cursor; ++k) ext[sorted[k].neuron] = 0.0;
    }
    return o;
}

void put_state(const MatOutcome& o, int n_visible, const std::vector<int64_t>& slot_of,
               orc_result* out) {
    out->n = n_visible;
    std::vector<double> mem(o.st.membrane.begin(), o.st.membrane.begin() + n_visible);
    out->membrane = dup(mem);
    out->m = static_cast<int64_t>(slot_of.size());
    std::vector<double> w(slot_of.size());
    for (std::size_t s = 0; s < slot_of.size(); ++s)
        w[s] = o.st.weights.slot_get(o.st.weights.slot(static_cast<std::size_t>(slot_of[s])));
    out->weights = dup(w);
    if (!o.trace.empty()) {
        std::vector<double> tr;
        tr.reserve(o.trace.size() * n_visible);
        for (const auto& row : o.trace) tr.insert(tr.end(), row.begin(), row.begin() + n_visible);
        out->membrane_trace = dup(tr);
    }
}

WeightStorage to_storage(int s) {
    return s == 1 ? WeightStorage::Dense : s == 2 ? WeightStorage::Sparse : WeightStorage::Auto;
}

} // namespace

extern "C" {

void orc_result_free(orc_result* r) {
    if (!r) return;
    std::free(r->ev_step);
    std::free(r->ev_neuron);
    std::free(r->membrane);
    std::free(r->weights);
    std::free(r->membrane_trace);
    r->ev_step = r->ev_neuron = nullptr;
    r->membrane = r->weights = r->membrane_trace = nullptr;
}

// mat_run on the network as given (storage 0 Auto / 1 Dense / 2 Sparse).
// With lower != 0 the reference MAT path for delayed nets is used:
// lower_delays -> mat_run -> restrict_raster (spikeforge_main.cpp:44-64);
// final weights are read from each original synapse's last hop.
int ref_mat_run_masked(const orc_problem* p, int storage, int lower, const uint8_t* plastic_steps,
                       orc_result* out) {
    return guarded(out, [&] {
        const NetworkDef net = to_net(p);
        const SimulationConfig cfg = to_cfg(p);
        const StimulusSchedule stim = to_stim(p);
        if (!lower) {
            MatOutcome o = mat_loop(net, cfg, stim, to_storage(storage), plastic_steps);
            put_raster(o.raster, out);
            std::vector<int64_t> slot_of(net.synapses.size());
            for (std::size_t s = 0; s < slot_of.size(); ++s) slot_of[s] = static_cast<int64_t>(s);
            put_state(o, o.st.n, slot_of, out);
            return;
        }
        const LoweredNetwork lw = lower_delays(net);
        MatOutcome o = mat_loop(lw.net, cfg, stim, to_storage(storage), plastic_steps);
        put_raster(restrict_raster(o.raster, lw.original_count), out);
        // lower_delays emits, per original synapse in order, 1 synapse when the
        // effective delay is 1, else d (the last one carries weight + stdp).
        std::vector<int64_t> slot_of(net.synapses.size());
        int64_t cursor = 0;
        for (std::size_t s = 0; s < net.synapses.size(); ++s) {
            const int d = net.synapses[s].delay + net.neurons[net.synapses[s].pre].axonal_delay;
            cursor += d;
            slot_of[s] = cursor - 1;
        }
        put_state(o, lw.original_count, slot_of, out);
    });
}

int ref_mat_run(const orc_problem* p, int storage, int lower, orc_result* out) {
    return ref_mat_run_masked(p, storage, lower, nullptr, out);
}

// mat_run itself (raster only), to pin mat_loop above against the real thing.
int ref_mat_run_raster(const orc_problem* p, int storage, orc_result* out) {
    return guarded(out, [&] {
        const RunResult r = mat_run(to_net(p), to_cfg(p), to_stim(p), to_storage(storage));
        put_raster(r.raster, out);
    });
}

int ref_oracle_run(const orc_problem* p, orc_result* out) {
    return guarded(out, [&] { put_raster(oracle_run(to_net(p), to_cfg(p), to_stim(p)), out); });
}

int ref_abm_run(const orc_problem* p, orc_result* out) {
    return guarded(out, [&] {
        SimulationConfig cfg = to_cfg(p);
        cfg.stdp.reset();
        put_raster(abm_run(to_net(p), cfg, to_stim(p)).raster, out);
    });
}

// Scale golden of a generated scenario: build_scenario(n, p, seed) with a
// `steps`-step protocol, delays 1 + below_at(key, delay_max) on stream
// delay_stream (key = pair index i*n + j, or the synapse index when by_index),
// then the reference's native-delay path abm_run (== mat_run(lower_delays),
// pinned by the small goldens).  The network is built in place (no orc_problem
// copy): at N = 256,000, p = 0.01 it is 655 M synapses (~16 GB NetworkDef).
int ref_scenario_abm_raster(int n, double p, uint64_t seed, int steps, int delay_max, int by_index,
                            uint64_t delay_stream, double* info, orc_result* out) {
    return guarded(out, [&] {
        const auto s0 = std::chrono::steady_clock::now();
        BenchScenario sc;
        sc.neuron_count = n;
        sc.connection_probability = p;
        sc.steps = steps;
        sc.seed = seed;
        ScenarioBundle b = build_scenario(sc);
        if (delay_max > 1) {
            const RandomStream ds(seed, delay_stream);
            for (std::size_t s = 0; s < b.net.synapses.size(); ++s) {
                SynapseDef& y = b.net.synapses[s];
                const uint64_t key = by_index ? static_cast<uint64_t>(s)
                                              : static_cast<uint64_t>(y.pre) * static_cast<uint64_t>(n) + y.post;
                y.delay = 1 + static_cast<int>(ds.below_at(key, static_cast<uint64_t>(delay_max)));
            }
        }
        info[0] = static_cast<double>(b.net.synapses.size());
        const auto s1 = std::chrono::steady_clock::now();
        const RunResult r = abm_run(b.net, b.cfg, b.stim);
        info[1] = std::chrono::duration<double>(s1 - s0).count();
        info[2] = std::chrono::duration<double>(std::chrono::steady_clock::now() - s1).count();
        info[3] = peak_rss_gb();
        put_raster(r.raster, out);
    });
}

// Scale golden of the STDP scenario: build_scenario(n, p, seed) with every
// synapse plastic and StdpConfig::defaults(), mat_run for `steps` steps with
// the reference's Auto storage (CSR above 12,000 neurons).
int ref_scenario_stdp_raster(int n, double p, uint64_t seed, int steps, double* info, orc_result* out) {
    return guarded(out, [&] {
        const auto s0 = std::chrono::steady_clock::now();
        BenchScenario sc;
        sc.neuron_count = n;
        sc.connection_probability = p;
        sc.steps = steps;
        sc.seed = seed;
        ScenarioBundle b = build_scenario(sc);
        for (SynapseDef& s : b.net.synapses) s.stdp_enabled = true;
        b.cfg.stdp = StdpConfig::defaults();
        info[0] = static_cast<double>(b.net.synapses.size());
        const RunResult r = mat_run(b.net, b.cfg, b.stim);
        info[1] = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
        info[2] = peak_rss_gb();
        put_raster(r.raster, out);
    });
}

// abm_run with heterogeneous behaviours: fire_p[i] < 1 runs neuron i under a
// StochasticLifBehavior(fire_p[i]) registered through the reference's own
// registry (the register_stochastic_lif binding, bindings.cpp:180-186);
// "stochastic_lif" is used for 0.5 and "lif" for 1.  Always records the
// membrane trace: its last row is the final membrane.
int ref_abm_run_full(const orc_problem* p, orc_result* out) {
    return guarded(out, [&] {
        NetworkDef net = to_net(p);
        if (p->fire_p) {
            for (int i = 0; i < p->n; ++i) {
                const double fp = p->fire_p[i];
                if (fp == 1.0) continue;
                if (fp == 0.5) {
                    net.neurons[i].behavior = "stochastic_lif";
                    continue;
                }
                char name[64];
                std::snprintf(name, sizeof(name), "shim_stochastic_%a", fp);
                if (!BehaviorRegistry::global().find(name))
                    BehaviorRegistry::global().register_behavior(
                        name, std::make_shared<StochasticLifBehavior>(fp));
                net.neurons[i].behavior = name;
            }
        }
        SimulationConfig cfg = to_cfg(p);
        cfg.stdp.reset();
        cfg.seed = p->seed;
        cfg.record_membrane = true;
        const RunResult r = abm_run(net, cfg, to_stim(p));
        put_raster(r.raster, out);
        out->n = p->n;
        out->membrane = static_cast<double*>(std::malloc(sizeof(double) * std::max(1, p->n)));
        const auto& last = r.membrane_trace.back();
        std::copy(last.begin(), last.end(), out->membrane);
        if (p->record_membrane) {
            out->membrane_trace = static_cast<double*>(
                std::malloc(sizeof(double) * static_cast<std::size_t>(p->steps) * std::max(1, p->n)));
            for (int t = 0; t < p->steps; ++t)
                std::copy(r.membrane_trace[t].begin(), r.membrane_trace[t].end(),
                          out->membrane_trace + static_cast<std::size_t>(t) * p->n);
        }
    });
}

// validate_network + validate_stimulus + validate_stdp messages, '\n'-joined.
int ref_validate(const orc_problem* p, char* buf, int cap) {
    std::vector<std::string> all = validate_network(to_net(p));
    for (auto& s : validate_stimulus(to_stim(p), p->n, p->steps)) all.push_back(s);
    if (p->stdp_on)
        for (auto& s : validate_stdp(*to_cfg(p).stdp)) all.push_back(s);
    std::string joined;
    for (std::size_t i = 0; i < all.size(); ++i) {
        if (i) joined += '\n';
        joined += all[i];
    }
    if (cap > 0) std::snprintf(buf, static_cast<std::size_t>(cap), "%s", joined.c_str());
    return static_cast<int>(all.size());
}

// mat_init error text (e.g. "unit delays required"), empty when accepted.
int ref_mat_init_error(const orc_problem* p, char* buf, int cap) {
    orc_result r;
    const int rc = guarded(&r, [&] { (void)mat_init(to_net(p), to_cfg(p)); });
    if (cap > 0) std::snprintf(buf, static_cast<std::size_t>(cap), "%s", r.error);
    return rc;
}

int64_t ref_erdos_renyi(int n, double p, uint64_t seed, int32_t* pre, int32_t* post,
                        int64_t cap) {
    const NetworkDef net = erdos_renyi(n, p, seed);
    const int64_t m = static_cast<int64_t>(net.synapses.size());
    for (int64_t s = 0; s < m && s < cap; ++s) {
        pre[s] = net.synapses[s].pre;
        post[s] = net.synapses[s].post;
    }
    return m;
}

// build_scenario's input neuron picks (netgen.cpp:71-81), ascending.
int ref_scenario_inputs(int n, double p, int steps, uint64_t seed, int count, int32_t* out) {
    BenchScenario s;
    s.neuron_count = n;
    s.connection_probability = 0.0;  // edges are irrelevant to the picks
    (void)p;
    s.steps = steps;
    s.seed = seed;
    s.input_neuron_count = count;
    const ScenarioBundle b = build_scenario(s);
    for (std::size_t i = 0; i < b.input_neurons.size(); ++i) out[i] = b.input_neurons[i];
    return static_cast<int>(b.input_neurons.size());
}

void ref_stdp_defaults(int32_t* window, double* a_plus, double* a_minus, double* w_min,
                       double* w_max) {
    const StdpConfig c = StdpConfig::defaults();
    *window = c.window;
    for (int k = 0; k < c.window; ++k) {
        a_plus[k] = c.a_plus[k];
        a_minus[k] = c.a_minus[k];
    }
    *w_min = c.w_min;
    *w_max = c.w_max;
}

double ref_leak_toward(double v, double leak, double reset) { return leak_toward(v, leak, reset); }

uint64_t ref_mix64(uint64_t z) { return mix64(z); }

uint64_t ref_stream_u64(uint64_t seed, uint64_t stream, uint64_t index) {
    return RandomStream(seed, stream).u64_at(index);
}

double ref_stream_unit(uint64_t seed, uint64_t stream, uint64_t index) {
    return RandomStream(seed, stream).unit_at(index);
}

uint64_t ref_stream_below(uint64_t seed, uint64_t stream, uint64_t index, uint64_t n) {
    return RandomStream(seed, stream).below_at(index, n);
}

// CPU baseline: the reference bench cell methodology (bench.cpp:24-97) on
// build_scenario(n, p, seed) -- mat_init outside the clock, the step loop
// timed with steady_clock -- plus apply_stdp after every mat_step when
// stdp_on (all synapses plastic, StdpConfig::defaults()).  Times `steps`
// steps of a `horizon`-step protocol (stimulus every 10 steps, 3 inputs).
int ref_bench_scenario(int n, double p, uint64_t seed, int steps, int stdp_on, int storage,
                       orc_result* out) {
    return guarded(out, [&] {
        BenchScenario sc;
        sc.neuron_count = n;
        sc.connection_probability = p;
        sc.steps = steps;
        sc.seed = seed;
        ScenarioBundle b = build_scenario(sc);
        if (stdp_on) {
            for (SynapseDef& s : b.net.synapses) s.stdp_enabled = true;
            b.cfg.stdp = StdpConfig::defaults();
        }
        std::vector<std::vector<std::pair<int, double>>> per_step(static_cast<std::size_t>(steps));
        for (const StimulusEntry& e : b.stim.entries) per_step[e.step].emplace_back(e.neuron, e.amplitude);
        MatState st = mat_init(b.net, b.cfg, to_storage(storage));
        b.net = NetworkDef{};  // release the synapse list before timing
        std::vector<double> ext(static_cast<std::size_t>(n), 0.0);
        long long spikes = 0;
        const auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < steps; ++t) {
            for (const auto& [j, a] : per_step[t]) ext[j] += a;
            const std::vector<int>& spiked = mat_step(st, ext);
            if (b.cfg.stdp) apply_stdp(st, *b.cfg.stdp);
            spikes += static_cast<long long>(spiked.size());
            for (const auto& [j, a] : per_step[t]) ext[j] = 0.0;
        }
        out->seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out->spike_count = spikes;
    });
}

// CPU reference arm at the full workload size: build_scenario(n, p, seed)
// with a `horizon`-step protocol, mat_init with the reference's own storage
// choice (storage 0 = Auto: CSR above 12,000 neurons, mat_engine.cpp:13,
// 29-30) outside the clock; then `warmup` untimed steps (step 0 has no
// propagation) and `steps` timed steps of mat_step (+ apply_stdp), each timed
// with steady_clock (bench.cpp:24-50).  delay_max > 1 (delays
// 1 + below_at(key, delay_max) on stream delay_stream, key = i*n + j or the
// synapse index when by_index) runs the reference's native-delay path
// instead: AbmWorld built outside the clock, AbmWorld::step timed
// (abm_engine.cpp:146-206).  info[0..5] = {setup s, warm-up s, timed s,
// dense storage (1/0, -1 for abm), synapses, peak RSS GB}; step_s[k] = time
// of timed step k.
int ref_bench_run(int n, double p, uint64_t seed, int horizon, int warmup, int steps, int stdp_on,
                  int storage, int delay_max, int by_index, uint64_t delay_stream, double* info,
                  double* step_s, orc_result* out) {
    return guarded(out, [&] {
        using clk = std::chrono::steady_clock;
        const auto s0 = clk::now();
        BenchScenario sc;
        sc.neuron_count = n;
        sc.connection_probability = p;
        sc.steps = horizon;
        sc.seed = seed;
        ScenarioBundle b = build_scenario(sc);
        const int64_t m = static_cast<int64_t>(b.net.synapses.size());
        if (delay_max > 1) {
            const RandomStream ds(seed, delay_stream);
            for (std::size_t s = 0; s < b.net.synapses.size(); ++s) {
                SynapseDef& y = b.net.synapses[s];
                const uint64_t key = by_index ? static_cast<uint64_t>(s)
                                              : static_cast<uint64_t>(y.pre) * static_cast<uint64_t>(n) + y.post;
                y.delay = 1 + static_cast<int>(ds.below_at(key, static_cast<uint64_t>(delay_max)));
            }
        }
        if (stdp_on) {
            for (SynapseDef& s : b.net.synapses) s.stdp_enabled = true;
            b.cfg.stdp = StdpConfig::defaults();
        }
        std::vector<std::vector<std::pair<int, double>>> per_step(static_cast<std::size_t>(horizon));
        for (const StimulusEntry& e : b.stim.entries) per_step[e.step].emplace_back(e.neuron, e.amplitude);
        std::vector<double> ext(static_cast<std::size_t>(n), 0.0);
        long long spikes = 0;
        auto run = [&](auto&& step_fn) {
            info[0] = std::chrono::duration<double>(clk::now() - s0).count();
            auto one = [&](int t) {
                bool any = false;
                for (const auto& [j, a] : per_step[t]) { ext[j] += a; any = true; }
                const long long k = static_cast<long long>(step_fn(any).size());
                for (const auto& [j, a] : per_step[t]) ext[j] = 0.0;
                return k;
            };
            const auto w0 = clk::now();
            for (int t = 0; t < warmup; ++t) one(t);
            info[1] = std::chrono::duration<double>(clk::now() - w0).count();
            const auto t0 = clk::now();
            for (int k = 0; k < steps; ++k) {
                const auto a = clk::now();
                spikes += one(warmup + k);
                step_s[k] = std::chrono::duration<double>(clk::now() - a).count();
            }
            info[2] = std::chrono::duration<double>(clk::now() - t0).count();
        };
        if (delay_max > 1) {
            AbmWorld world(b.net, b.cfg);
            b.net = NetworkDef{};
            info[3] = -1;
            run([&](bool any) -> const std::vector<int>& {
                return world.step(any ? std::span<const double>(ext) : std::span<const double>());
            });
        } else {
            MatState st = mat_init(b.net, b.cfg, to_storage(storage));
            b.net = NetworkDef{};  // release the synapse list before timing
            info[3] = st.weights.dense() ? 1 : 0;
            run([&](bool) -> const std::vector<int>& {
                const std::vector<int>& spiked = mat_step(st, ext);
                if (b.cfg.stdp) apply_stdp(st, *b.cfg.stdp);
                return spiked;
            });
        }
        info[4] = static_cast<double>(m);
        info[5] = peak_rss_gb();
        out->seconds = info[2];
        out->spike_count = spikes;
    });
}

}  // extern "C"

// ---- wire formats (proj/src/io.cpp), for byte-identity tests of the Python io mirror ----
#ifdef SPIKEFORGE_WITH_IO
#include "spikeforge/io.hpp"

namespace {
char* dup_str(const std::string& s) {
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}
}  // namespace

extern "C" {

void ref_free_str(char* s) { std::free(s); }

char* ref_serialize_network(const orc_problem* p) { return dup_str(serialize_network(to_net(p))); }

char* ref_write_raster(const int32_t* steps, const int32_t* neurons, int64_t n) {
    SpikeRaster r;
    for (int64_t i = 0; i < n; ++i) r.events.push_back({steps[i], neurons[i]});
    return dup_str(write_raster(r));
}

char* ref_write_stimulus(const orc_problem* p) { return dup_str(write_stimulus(to_stim(p))); }

char* ref_serialize_stdp(const orc_problem* p) { return dup_str(serialize_stdp(*to_cfg(p).stdp)); }

// parse_network -> serialize_network round trip of a text (empty string on FormatError)
char* ref_roundtrip_network(const char* text) {
    try {
        return dup_str(serialize_network(parse_network(text)));
    } catch (const std::exception& e) {
        return dup_str(std::string("ERROR ") + e.what());
    }
}

}  // extern "C"
#endif
