// Drop-in use of the C++ facade: the two-neuron delay-3 chain of the
// reference tests (test_oracle.cpp:47-51) -> {(0,0),(3,1)}; plus an STDP pair
// (test_stdp.cpp:46-57) -> weight 0.5 + 0.1 within fp32 storage tolerance.
#include "superneuro_mat.hpp"

#include <cmath>
#include <cstdio>

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
        std::printf("facade ok\n");
        return 0;
    } catch (const std::exception& e) {
        std::printf("ERROR %s\n", e.what());
        return 2;
    }
}
