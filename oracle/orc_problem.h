/*
 * TEST INFRASTRUCTURE ONLY -- shared problem/result structs for the two CPU
 * checkers under oracle/:
 *   - oracle/_ref/libspikeforge_ref.so : the reference's own C++ sources
 *     (the .cpp files under /root/reference/proj/src) compiled unmodified
 *     together with ref_shim.cpp
 *   - oracle/libmat_oracle.so          : mat_oracle.c, a plain-C restatement
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these.  The product path
 * (paper_2305_02510_b200/) never does.
 *
 * The fields mirror spikeforge::NetworkDef / StimulusSchedule / StdpConfig /
 * SimulationConfig (reference proj/include/spikeforge/model.hpp:20-85), as
 * flat structure-of-arrays so ctypes can fill them from numpy.
 */
#ifndef ORC_PROBLEM_H
#define ORC_PROBLEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_problem {
    /* neurons (model.hpp:20-29) */
    int32_t n;
    const double* threshold;
    const double* leak;        /* >= 0 or +inf */
    const double* reset;
    const int32_t* refractory;
    const int32_t* axonal;     /* may be NULL = all 0 */
    /* synapses (model.hpp:31-39), list order is significant */
    int64_t m;
    const int32_t* pre;
    const int32_t* post;
    const double* weight;
    const int32_t* delay;      /* may be NULL = all 1 */
    const uint8_t* stdp;       /* may be NULL = none plastic */
    /* stimulus (model.hpp:53-63), list order is significant */
    int64_t k;
    const int32_t* st_step;
    const int32_t* st_neuron;
    const double* st_amp;
    /* simulation (model.hpp:80-85) + StdpConfig (model.hpp:67-78) */
    int32_t steps;
    int32_t stdp_on;
    int32_t window;
    const double* a_plus;
    const double* a_minus;
    double w_min;
    double w_max;
    int32_t record_membrane;
    /* agent-based mode (abm_engine.hpp:70-121): SimulationConfig::seed and one
       fire probability per neuron (NULL = all "lif"; p < 1 = a StochasticLif
       behaviour with that probability, abm_engine.cpp:28-39) */
    uint64_t seed;
    const double* fire_p;
} orc_problem;

typedef struct orc_result {
    int32_t status;            /* 0 ok, 1 invalid_argument, 2 logic_error, 3 other */
    char error[1024];
    int64_t n_events;
    int32_t* ev_step;          /* malloc'd, (step, neuron) ascending */
    int32_t* ev_neuron;
    int32_t n;
    double* membrane;          /* malloc'd, final membrane, n entries */
    int64_t m;
    double* weights;           /* malloc'd, final weight of each synapse, list order */
    double* membrane_trace;    /* malloc'd steps*n when record_membrane, else NULL */
    int64_t spike_count;
    double seconds;            /* timed loop wall time where applicable */
} orc_result;

void orc_result_free(orc_result* r);

#ifdef __cplusplus
}
#endif

#endif
