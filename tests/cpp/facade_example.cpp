// Drop-in use of the C++ facade: the two-neuron delay-3 chain of the
// reference tests (test_oracle.cpp:47-51) -> {(0,0),(3,1)}; plus an STDP pair
// (test_stdp.cpp:46-57) -> weight 0.5 + 0.1 within fp32 storage tolerance;
// plus the mat_step KATs through Model::step (test_mat_engine.cpp:61-95);
// plus a seeded stochastic agent-based run.
#include "superneuro_mat.hpp"

#include <cmath>
#include <cstdio>
#include <vector>

int main() {
    try {
        superneuro::Model m;
        const int a = m.create_neuron(1.0, 0.0, 0.0, 0);
        const int b = m.create_neuron(1.0, 0.0, 0.0, 0);
        m.create_synapse(a, b, 2.0, 3, false);
        m.add_spike(0, a, 2.0);
        m.setup();
        const auto r = m.simulate(8);
        if (r.events.size() != 2 || r.events[0].step != 0 || r.events[0].neuron != 0 ||
            r.events[1].step != 3 || r.events[1].neuron != 1) {
            std::printf("FAIL raster\n");
            return 1;
        }
        superneuro::Model p(0, SN_STORAGE_DENSE, SN_WEIGHTS_F64);
        p.create_neuron();
        p.create_neuron();
        p.create_synapse(0, 1, 0.5, 1, true);
        p.add_spike(0, 0, 2.0);
        p.add_spike(2, 1, 2.0);
        superneuro::StdpParams s;
        s.window = 4;
        s.a_plus = {0.0, 0.1, 0.0, 0.0};
        s.a_minus = {0.0, 0.0, 0.0, 0.0};
        p.setup(&s);
        const auto q = p.simulate(3);
        if (q.weights.size() != 1 || q.weights[0] != 0.5 + 0.1) {
            std::printf("FAIL stdp %.17g\n", q.weights.empty() ? -1.0 : q.weights[0]);
            return 1;
        }
        // per-step API, the mat_step KATs of test_mat_engine.cpp:61-95: chain with
        // threshold 0.5 -> {0}, {1}, {}; refractory 3 -> {0}, {}, {}, {}, {0}
        {
            superneuro::Model c(0, SN_STORAGE_DENSE, SN_WEIGHTS_F64);
            c.create_neuron(0.5);
            c.create_neuron(0.5);
            c.create_synapse(0, 1, 1.0, 1, false);
            c.setup();
            const bool ok = c.step({1.0, 0.0}) == std::vector<int>{0} && c.step({0.0, 0.0}) == std::vector<int>{1} &&
                            c.step({0.0, 0.0}).empty();
            superneuro::Model r;
            r.create_neuron(1.0, 0.0, 0.0, 3);
            r.setup();
            std::vector<std::vector<int>> got;
            for (int t = 0; t < 5; ++t) got.push_back(r.step({2.0}));
            const std::vector<std::vector<int>> want{{0}, {}, {}, {}, {0}};
            if (!ok || got != want) {
                std::printf("FAIL step\n");
                return 1;
            }
        }
        // agent-based mode: stochastic_lif (p = 0.5) post, seeded -- deterministic
        // per seed, fires on some but not all of its above-threshold steps
        // (test_abm_engine.cpp:122-141)
        auto run_abm = [](uint64_t seed) {
            superneuro::Model g(0, SN_STORAGE_AUTO, SN_WEIGHTS_F64, SN_MODE_ABM);
            g.set_exact_order(true);
            g.create_neuron();
            g.create_neuron(1.0, 0.0, 0.0, 0, 0, 0.5);
            g.create_synapse(0, 1, 2.0, 1, false);
            for (int t = 0; t < 100; ++t) g.add_spike(t, 0, 2.0);
            g.set_seed(seed);
            g.setup();
            int fires = 0;
            for (const auto& ev : g.simulate(100).events) fires += ev.neuron == 1;
            return fires;
        };
        const int f9 = run_abm(9), f9b = run_abm(9);
        if (f9 != f9b || f9 <= 20 || f9 >= 80) {
            std::printf("FAIL abm %d %d\n", f9, f9b);
            return 1;
        }
        std::printf("facade ok\n");
        return 0;
    } catch (const std::exception& e) {
        std::printf("ERROR %s\n", e.what());
        return 2;
    }
}
