/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's
 * agent-based (ABM) engine, the checker for the CUDA engine's ABM mode
 * (sn_options.mode = SN_MODE_ABM).  Never linked into, loaded by or called
 * from the product path.
 *
 * Parity pinning: tests/test_oracle_pinning.py runs this file and the
 * reference's own abm_run (oracle/_ref, proj/src/abm_engine.cpp) on the same
 * random nets, stochastic behaviours included, and requires identical rasters
 * and membrane traces.
 *
 * Semantics restated (reference file:line):
 *   world construction            proj/src/abm_engine.cpp:78-144
 *     membrane = reset, refractory counters 0, pending input 0; channels
 *     ordered by (pre, post); a delay-d channel is a d-slot register, an
 *     axonal delay a a-slot register per neuron.
 *   step, phase 1 (neurons)       abm_engine.cpp:146-189
 *     input = pending[i] + (step has stimulus ? ext[i] : 0.0); pending = 0;
 *     u = leak_toward(v, leak, reset) + input  (LifBehavior, :22-26);
 *     fired = u > thr, and for StochasticLifBehavior (:34-39) additionally
 *     unit_0 < p with unit_0 the first draw of RandomStream(seed,
 *     0x61626d2d6167656e, i, step) (:12, :163-164); refractory: fired = 0,
 *     cnt--, u = reset; a spike sets v = reset, cnt = refractory and loads the
 *     register heads (axon register when the axonal delay is > 0, else every
 *     outgoing channel); otherwise v = u.
 *   step, phase 2a (channels)     abm_engine.cpp:191-199: in channel order, a
 *     set tail adds the weight to pending[post]; registers shift by one.
 *   step, phase 2b (axons)        abm_engine.cpp:201-215: axon registers
 *     shift; a popped spike loads the heads of the (already shifted) outgoing
 *     channels.
 *   abm_run                       abm_engine.cpp:218-243: stimulus stable by
 *     step, ext[j] = 0.0 + a1 + a2 ... in list order; no plasticity.
 * A behaviour is a fire probability per neuron: "lif" = 1 (never draws),
 * "stochastic_lif" = 0.5, register_stochastic_lif(name, p) = p
 * (bindings.cpp:180-186).
 */
#include "orc_problem.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double abm_leak(double v, double leak, double reset) {  /* model.hpp:127-138 */
    const double d = v - reset;
    if (d > 0.0) return reset + (d - leak > 0.0 ? d - leak : 0.0);
    if (d < 0.0) return reset + (d + leak < 0.0 ? d + leak : 0.0);
    return v;
}

static uint64_t splitmix(uint64_t z) {  /* rng.hpp:8-12 */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* first unit draw of RandomStream(seed, stream, sub0, sub1) (rng.hpp:19-35) */
static double first_unit(uint64_t seed, uint64_t stream, uint64_t sub0, uint64_t sub1) {
    uint64_t k = splitmix(seed + 0x9e3779b97f4a7c15ULL);
    k = splitmix(k ^ stream);
    k = splitmix(k ^ sub0);
    k = splitmix(k ^ sub1);
    return (double)(splitmix(k) >> 11) * 0x1.0p-53;
}

static const orc_problem* g_abm_sort;
static int by_pre_post(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    const orc_problem* p = g_abm_sort;
    if (p->pre[x] != p->pre[y]) return p->pre[x] < p->pre[y] ? -1 : 1;
    if (p->post[x] != p->post[y]) return p->post[x] < p->post[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

int abm_oracle_run(const orc_problem* p, orc_result* out) {
    memset(out, 0, sizeof(*out));
    const int n = p->n, T = p->steps;
    const int64_t m = p->m;
    if (T < 1) {
        out->status = 1;
        snprintf(out->error, sizeof(out->error), "abm_run: steps must be >= 1");
        return 1;
    }
    /* channels in (pre, post) order; each owns `delay` register slots */
    int64_t* chan = malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    for (int64_t s = 0; s < m; ++s) chan[s] = s;
    g_abm_sort = p;
    qsort(chan, (size_t)m, sizeof(int64_t), by_pre_post);
    int64_t* slot0 = malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int64_t slots = 0;
    int64_t* first_out = calloc((size_t)n + 1, sizeof(int64_t));  /* channels of pre i: [first_out[i], first_out[i+1]) */
    for (int64_t c = 0; c < m; ++c) {
        slot0[c] = slots;
        slots += p->delay ? p->delay[chan[c]] : 1;
        first_out[p->pre[chan[c]] + 1] += 1;
    }
    for (int i = 0; i < n; ++i) first_out[i + 1] += first_out[i];
    unsigned char* reg = calloc((size_t)(slots ? slots : 1), 1);
    int64_t* axon0 = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t aslots = 0;
    for (int i = 0; i < n; ++i) {
        axon0[i] = aslots;
        aslots += p->axonal ? p->axonal[i] : 0;
    }
    unsigned char* areg = calloc((size_t)(aslots ? aslots : 1), 1);

    /* stimulus rows per step in list order */
    int64_t* srow = calloc((size_t)T + 1, sizeof(int64_t));
    int64_t* sidx = malloc(sizeof(int64_t) * (size_t)(p->k ? p->k : 1));
    for (int64_t e = 0; e < p->k; ++e) srow[p->st_step[e] + 1] += 1;
    for (int t = 0; t < T; ++t) srow[t + 1] += srow[t];
    {
        int64_t* fill = malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
        memcpy(fill, srow, sizeof(int64_t) * (size_t)T);
        for (int64_t e = 0; e < p->k; ++e) sidx[fill[p->st_step[e]]++] = e;
        free(fill);
    }

    double* v = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* pending = calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    double* ext = calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    int32_t* cnt = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    for (int i = 0; i < n; ++i) v[i] = p->reset[i];
    if (p->record_membrane) out->membrane_trace = malloc(sizeof(double) * (size_t)T * (size_t)(n > 0 ? n : 1));
    int64_t cap = 1024, nev = 0;
    int32_t* evs = malloc(sizeof(int32_t) * (size_t)cap);
    int32_t* evn = malloc(sizeof(int32_t) * (size_t)cap);

    for (int t = 0; t < T; ++t) {
        const int any = srow[t + 1] > srow[t];
        for (int64_t q = srow[t]; q < srow[t + 1]; ++q) ext[p->st_neuron[sidx[q]]] += p->st_amp[sidx[q]];
        /* phase 1: every neuron, ascending id */
        for (int i = 0; i < n; ++i) {
            const double input = pending[i] + (any ? ext[i] : 0.0);
            pending[i] = 0.0;
            double u = abm_leak(v[i], p->leak[i], p->reset[i]) + input;
            int fired = u > p->threshold[i];
            if (fired && p->fire_p && p->fire_p[i] < 1.0)
                fired = first_unit(p->seed, 0x61626d2d6167656eULL, (uint64_t)i, (uint64_t)t) < p->fire_p[i];
            if (cnt[i] > 0) {
                fired = 0;
                cnt[i] -= 1;
                u = p->reset[i];
            }
            if (!fired) {
                v[i] = u;
                continue;
            }
            v[i] = p->reset[i];
            cnt[i] = p->refractory[i];
            if (nev == cap) {
                cap *= 2;
                evs = realloc(evs, sizeof(int32_t) * (size_t)cap);
                evn = realloc(evn, sizeof(int32_t) * (size_t)cap);
            }
            evs[nev] = t;
            evn[nev++] = i;
            if (p->axonal && p->axonal[i] > 0)
                areg[axon0[i]] = 1;
            else
                for (int64_t c = first_out[i]; c < first_out[i + 1]; ++c) reg[slot0[c]] = 1;
        }
        /* phase 2a: channel tails deliver, registers shift */
        for (int64_t c = 0; c < m; ++c) {
            const int len = p->delay ? p->delay[chan[c]] : 1;
            unsigned char* r = reg + slot0[c];
            if (r[len - 1]) pending[p->post[chan[c]]] += p->weight[chan[c]];
            memmove(r + 1, r, (size_t)(len - 1));
            r[0] = 0;
        }
        /* phase 2b: axon registers shift; popped spikes load channel heads */
        for (int i = 0; i < n; ++i) {
            const int len = p->axonal ? p->axonal[i] : 0;
            if (len == 0) continue;
            unsigned char* r = areg + axon0[i];
            const unsigned char popped = r[len - 1];
            memmove(r + 1, r, (size_t)(len - 1));
            r[0] = 0;
            if (popped)
                for (int64_t c = first_out[i]; c < first_out[i + 1]; ++c) reg[slot0[c]] = 1;
        }
        for (int64_t q = srow[t]; q < srow[t + 1]; ++q) ext[p->st_neuron[sidx[q]]] = 0.0;
        if (p->record_membrane) memcpy(out->membrane_trace + (int64_t)t * n, v, sizeof(double) * (size_t)n);
    }

    out->n_events = nev;
    out->spike_count = nev;
    out->ev_step = evs;
    out->ev_neuron = evn;
    out->n = n;
    out->membrane = v;
    out->m = m;
    out->weights = malloc(sizeof(double) * (size_t)(m ? m : 1));  /* static: ABM has no plasticity */
    if (m) memcpy(out->weights, p->weight, sizeof(double) * (size_t)m);
    free(chan); free(slot0); free(first_out); free(reg); free(axon0); free(areg);
    free(srow); free(sidx); free(pending); free(ext); free(cnt);
    return 0;
}
