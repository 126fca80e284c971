/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference MAT step,
 * used by tests/ (and __graft_entry__.smoke()) as the checker for the CUDA
 * engine.  Never linked into, loaded by or called from the product path.
 *
 * Parity pinning: tests/test_oracle_pinning.py checks this file against the
 * reference's own compiled code (oracle/_ref/libspikeforge_ref.so built from
 * /root/reference/proj/src) and against the committed golden fixtures in
 * tests/golden/ (generated from that library by tests/golden/make_golden.py).
 *
 * Semantics restated (reference file:line):
 *   leak_toward                     proj/include/spikeforge/model.hpp:127-138
 *   mat_step order                  proj/src/mat_engine.cpp:168-208
 *     u = leak(v); u += sum_{i in S_prev, ascending} W[i][j]; u += ext (only
 *     when the step has stimulus); s = u > thr; refractory: s=0, cnt--, u=reset;
 *     spike: v=reset, cnt=R; else v=u
 *   propagate (ascending pre)       proj/src/mat_engine.cpp:79-93
 *   apply_stdp                      proj/src/mat_engine.cpp:210-250
 *     pot[i] = sum_{k=1..min(W,t)} a_plus[k-1] s_i[t-k]  (k ascending)
 *     dep[i] = sum_{k=1..min(W,t)} a_minus[k-1] s_i[t-k]
 *     per plastic synapse, list order: dw = 0; if s_post[t] dw += pot[pre];
 *     if s_pre[t] dw -= dep[post]; w = clamp(w + dw, w_min, w_max)
 *   mat_run stimulus handling       proj/src/mat_engine.cpp:256-285
 *     stable sort by step; ext[j] = 0.0 + a1 + a2 ... in list order
 *   delays (native, no proxies)     proj/src/oracle.cpp:91-95 (arrival =
 *     t + delay + axonal_delay) and proj/src/lowering.cpp:39-57: on a lowered
 *     net the stdp flag rides the last hop, whose source proxy fires at
 *     t_pre + d - 1, so STDP for a synapse of effective delay d pairs
 *     s_pre[t-d+1] (and pot shifted by d-1) with s_post[t].
 *   Propagation for delayed synapses uses the weight current at arrival
 *   (the final hop's weight at t-1 in the lowered net).
 */
#include "orc_problem.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double leak_toward(double v, double leak, double reset) {
    const double d = v - reset;
    if (d > 0.0) {
        const double stepped = d - leak;
        return reset + (stepped > 0.0 ? stepped : 0.0);
    }
    if (d < 0.0) {
        const double stepped = d + leak;
        return reset + (stepped < 0.0 ? stepped : 0.0);
    }
    return v;
}

typedef struct {
    int64_t syn;   /* index into the synapse list */
} edge_ref;

static int cmp_edge(const void* a, const void* b, void* ctx);

/* qsort_r is a GNU extension; use a file-static context instead. */
static const orc_problem* g_sort_problem;
static int cmp_edge_static(const void* a, const void* b) {
    return cmp_edge(a, b, (void*)g_sort_problem);
}
static int cmp_edge(const void* a, const void* b, void* ctx) {
    const orc_problem* p = (const orc_problem*)ctx;
    const int64_t x = ((const edge_ref*)a)->syn, y = ((const edge_ref*)b)->syn;
    if (p->pre[x] != p->pre[y]) return p->pre[x] < p->pre[y] ? -1 : 1;
    if (p->post[x] != p->post[y]) return p->post[x] < p->post[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

static void fail(orc_result* out, int status, const char* msg) {
    out->status = status;
    snprintf(out->error, sizeof(out->error), "%s", msg);
}

/* History lookup: s_i[tau], 0 for tau < 0 (nothing spiked before step 0). */
#define HIST(tau, i) ((tau) < 0 ? 0 : hist[((tau) % H) * (int64_t)n + (i)])

/* f32w = 1: the engine's default fp32 weight storage as a model of the same
 * algorithm -- every stored weight (initial and after each update) rounded to
 * float once, everything else (traces, dw, w + dw, clamp, input sums) in fp64
 * exactly as above.  Rounding is monotone, so RN(clamp(x)) = clamp(RN(x),
 * RN(lo), RN(hi)): the engine's fp32 clamp gives the same stored value. */
static int mat_oracle_impl(const orc_problem* p, orc_result* out, int f32w);

int mat_oracle_run(const orc_problem* p, orc_result* out) { return mat_oracle_impl(p, out, 0); }

int mat_oracle_run_f32w(const orc_problem* p, orc_result* out) { return mat_oracle_impl(p, out, 1); }

#define STORE_W(x) (f32w ? (double)(float)(x) : (x))

static int mat_oracle_impl(const orc_problem* p, orc_result* out, int f32w) {
    memset(out, 0, sizeof(*out));
    const int n = p->n;
    const int64_t m = p->m;
    const int T = p->steps;
    if (T < 1) { fail(out, 1, "mat_run: steps must be >= 1"); return out->status; }
    for (int64_t s = 0; s < m; ++s) {
        if (p->pre[s] < 0 || p->pre[s] >= n || p->post[s] < 0 || p->post[s] >= n) {
            fail(out, 1, "invalid synapse endpoint"); return out->status;
        }
        if (p->delay && p->delay[s] < 1) { fail(out, 1, "delay must be >= 1"); return out->status; }
    }
    for (int64_t e = 0; e < p->k; ++e)
        if (p->st_step[e] < 0 || p->st_step[e] >= T || p->st_neuron[e] < 0 || p->st_neuron[e] >= n) {
            fail(out, 1, "stimulus out of range"); return out->status;
        }

    /* effective delay and max */
    int dmax = 1;
    int32_t* deff = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    for (int64_t s = 0; s < m; ++s) {
        deff[s] = (p->delay ? p->delay[s] : 1) + (p->axonal ? p->axonal[p->pre[s]] : 0);
        if (deff[s] > dmax) dmax = deff[s];
    }
    const int W = p->stdp_on ? p->window : 0;
    const int H = dmax + W + 2; /* ring of spike vectors; covers t-k-d+1 */

    /* outgoing edges sorted by (pre, post): ascending-pre accumulation */
    edge_ref* order = (edge_ref*)malloc(sizeof(edge_ref) * (size_t)(m ? m : 1));
    for (int64_t s = 0; s < m; ++s) order[s].syn = s;
    g_sort_problem = p;
    qsort(order, (size_t)m, sizeof(edge_ref), cmp_edge_static);
    int64_t* row_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t s = 0; s < m; ++s) row_ptr[p->pre[s] + 1]++;
    for (int i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];

    /* stimulus: stable by step, summed in list order from 0.0 */
    double* ext = (double*)calloc((size_t)n, sizeof(double));
    int64_t* st_ptr = (int64_t*)calloc((size_t)T + 1, sizeof(int64_t));
    int64_t* st_ord = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p->k ? p->k : 1));
    for (int64_t e = 0; e < p->k; ++e) st_ptr[p->st_step[e] + 1]++;
    for (int t = 0; t < T; ++t) st_ptr[t + 1] += st_ptr[t];
    {
        int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)T);
        for (int t = 0; t < T; ++t) cur[t] = st_ptr[t];
        for (int64_t e = 0; e < p->k; ++e) st_ord[cur[p->st_step[e]]++] = e;
        free(cur);
    }

    double* v = (double*)malloc(sizeof(double) * (size_t)n);
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    int32_t* cnt = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    double* w = (double*)malloc(sizeof(double) * (size_t)(m ? m : 1));
    uint8_t* hist = (uint8_t*)calloc((size_t)H * (size_t)n, 1);
    double* dep = (double*)calloc((size_t)n, sizeof(double));
    double* potd = (double*)calloc((size_t)n * (size_t)dmax, sizeof(double));
    for (int i = 0; i < n; ++i) v[i] = p->reset[i];
    for (int64_t s = 0; s < m; ++s) w[s] = STORE_W(p->weight[s]);
    if (p->record_membrane)
        out->membrane_trace = (double*)malloc(sizeof(double) * (size_t)T * (size_t)n);

    int64_t ev_cap = 1024, nev = 0;
    int32_t* evs = (int32_t*)malloc(sizeof(int32_t) * (size_t)ev_cap);
    int32_t* evn = (int32_t*)malloc(sizeof(int32_t) * (size_t)ev_cap);

    for (int t = 0; t < T; ++t) {
        for (int j = 0; j < n; ++j) u[j] = leak_toward(v[j], p->leak[j], p->reset[j]);
        /* propagation: ascending pre; synapse (i->j, d) delivers s_i[t-d] */
        for (int i = 0; i < n; ++i) {
            for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
                const int64_t s = order[q].syn;
                if (HIST(t - deff[s], i)) u[p->post[s]] += w[s];
            }
        }
        if (st_ptr[t + 1] > st_ptr[t]) {
            for (int64_t q = st_ptr[t]; q < st_ptr[t + 1]; ++q) {
                const int64_t e = st_ord[q];
                ext[p->st_neuron[e]] += p->st_amp[e];
            }
            for (int j = 0; j < n; ++j) u[j] += ext[j];
            for (int64_t q = st_ptr[t]; q < st_ptr[t + 1]; ++q) ext[p->st_neuron[st_ord[q]]] = 0.0;
        }
        uint8_t* now = &hist[(int64_t)(t % H) * n];
        for (int j = 0; j < n; ++j) {
            int spiked = u[j] > p->threshold[j];
            if (cnt[j] > 0) {
                spiked = 0;
                cnt[j] -= 1;
                u[j] = p->reset[j];
            }
            if (spiked) {
                v[j] = p->reset[j];
                cnt[j] = p->refractory[j];
                if (nev == ev_cap) {
                    ev_cap *= 2;
                    evs = (int32_t*)realloc(evs, sizeof(int32_t) * (size_t)ev_cap);
                    evn = (int32_t*)realloc(evn, sizeof(int32_t) * (size_t)ev_cap);
                }
                evs[nev] = t;
                evn[nev] = j;
                ++nev;
            } else {
                v[j] = u[j];
            }
            now[j] = (uint8_t)spiked;
        }
        if (p->record_membrane) memcpy(out->membrane_trace + (int64_t)t * n, v, sizeof(double) * (size_t)n);

        if (p->stdp_on) {
            for (int j = 0; j < n; ++j) {
                double acc = 0.0;
                for (int k = 1; k <= W && k <= t; ++k)
                    if (HIST(t - k, j)) acc += p->a_minus[k - 1];
                dep[j] = acc;
            }
            /* pot[i][d-1]: effective pre train s_i shifted by d-1 (last proxy) */
            for (int i = 0; i < n; ++i)
                for (int d = 1; d <= dmax; ++d) {
                    double acc = 0.0;
                    for (int k = 1; k <= W && k <= t; ++k)
                        if (HIST(t - k - d + 1, i)) acc += p->a_plus[k - 1];
                    potd[(int64_t)i * dmax + (d - 1)] = acc;
                }
            for (int64_t s = 0; s < m; ++s) {
                if (!p->stdp || !p->stdp[s]) continue;
                const int i = p->pre[s], j = p->post[s], d = deff[s];
                const double pot = potd[(int64_t)i * dmax + (d - 1)];
                double dw = 0.0;
                if (now[j]) dw += pot;
                if (HIST(t - d + 1, i)) dw -= dep[j];
                double nw = w[s] + dw;
                /* std::clamp(v, lo, hi): v < lo ? lo : hi < v ? hi : v */
                nw = nw < p->w_min ? p->w_min : (p->w_max < nw ? p->w_max : nw);
                w[s] = STORE_W(nw);
            }
        }
    }

    out->n_events = nev;
    out->spike_count = nev;
    out->ev_step = evs;
    out->ev_neuron = evn;
    out->n = n;
    out->membrane = v;
    out->m = m;
    out->weights = w;
    free(u); free(cnt); free(hist); free(dep); free(potd); free(ext); free(st_ptr); free(st_ord);
    free(order); free(row_ptr); free(deff);
    return 0;
}

void orc_result_free(orc_result* r) {
    if (!r) return;
    free(r->ev_step); free(r->ev_neuron); free(r->membrane); free(r->weights);
    free(r->membrane_trace);
    r->ev_step = r->ev_neuron = NULL;
    r->membrane = r->weights = r->membrane_trace = NULL;
}
