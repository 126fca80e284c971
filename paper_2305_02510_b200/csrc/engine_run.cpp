// The per-step launch sequence: kernel argument blocks, graph-captured
// step chunks, persistent / tiny loops, stream I/O and the host-driven
// partition steps (sn_step_local / sn_step_finish).
#include "engine.hpp"

#include <chrono>
#include <cstdio>
#include "engine_util.hpp"
#include "nccl_dl.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>
#include <unordered_map>
#include <unordered_set>

namespace snb {

static int words_of(int n) { return (n + 31) / 32; }

// One k_tiny launch per chunk of steps whose stimulus fits next to the state.
void Engine::run_tiny(int t0, int steps, uint32_t* raster, double* trace, bool host_io) {
    TinyArgs a{};
    a.n = n_;
    a.hw = hw_;
    a.dmax = dmax_;
    a.f64 = f64_ ? 1 : 0;
    a.v = d_v_.as<double>();
    a.cnt = d_cnt_.as<int32_t>();
    a.hist = d_hist_.as<uint64_t>();
    a.thr = d_thr_.as<double>();
    a.leak = d_leak_.as<double>();
    a.reset = d_reset_.as<double>();
    a.refr = d_refr_.as<int32_t>();
    a.off = d_toff_.as<uint32_t>();
    a.meta = d_meta_.as<uint32_t>();
    a.pidx = d_tpidx_.as<uint16_t>();
    a.w = d_w_.p;
    a.m = static_cast<int32_t>(pre_.size());
    a.stdp = stdp_on_ ? 1 : 0;
    a.window = window_;
    a.dp = dp_;
    a.a_plus = d_ap_.as<double>();
    a.a_minus = d_am_.as<double>();
    a.w_min = w_min_;
    a.w_max = w_max_;
    a.plastic_on = plasticity_ ? 1 : 0;
    a.spike_count = d_spikes_.as<unsigned long long>();
    a.d_step = d_step_.as<int32_t>();
    a.abm = abm_ ? 1 : 0;
    a.fire_p = any_stochastic_ ? d_firep_.as<double>() : nullptr;
    a.agent_key = any_stochastic_ ? d_akey_.as<uint64_t>() : nullptr;
    {   // count mode: one weight, unit delays, no plasticity, <= 256 neurons
        double w0 = 0.0;
        const char* tc = std::getenv("SNB_TINY_COUNT");  // A/B knob: 0 walks the in-lists
        if (!stdp_on_ && dmax_ == 1 && words_of(n_) <= tiny_count_words_max() && !(tc && std::string(tc) == "0") &&
            uniform_weight(&w0)) {
            a.count_words = words_of(n_);
            a.w0 = f64_ ? w0 : static_cast<double>(static_cast<float>(w0));
        }
    }
    const size_t limit = static_cast<size_t>(tiny_max_smem());
    const int words = std::max(nl_words_, 1);
    const int table = static_cast<int>(hs_off_.size()) - 1;  // steps covered by the stimulus CSR
    for (int done = 0; done < steps;) {
        const int tt = t0 + done;
        int k = steps - done, rows = 0;
        int64_t lo = 0, hi = 0;
        for (;;) {  // shrink the launch until its stimulus fits next to the state
            rows = std::max(0, std::min(table - tt, k));
            lo = rows > 0 ? hs_off_[tt] : 0;
            hi = rows > 0 ? hs_off_[tt + rows] : 0;
            a.steps = k;
            a.st_rows = rows;
            a.st_count = static_cast<int32_t>(hi - lo);
            if (tiny_smem_bytes(a) <= limit || k == 1) break;
            k = std::max(1, k / 2);
        }
        if (rows == 0) {
            a.st_off = nullptr;
            a.st_neuron = nullptr;
            a.st_amp = nullptr;
        } else if (host_io) {
            // the kernel reads this launch's rows straight from pinned host memory
            const size_t cnt = static_cast<size_t>(hi - lo);
            const size_t ob = round_up((static_cast<int64_t>(rows) + 1) * 8, 16);
            h_stage_.reserve(ob + cnt * 12 + 16);
            uint8_t* base = h_stage_.as<uint8_t>();
            int64_t* soff = reinterpret_cast<int64_t*>(base);
            double* samp = reinterpret_cast<double*>(base + ob);
            int32_t* sneu = reinterpret_cast<int32_t*>(base + ob + cnt * 8);
            for (int s = 0; s <= rows; ++s) soff[s] = hs_off_[tt + s] - lo;
            std::memcpy(samp, hs_amp_.data() + lo, cnt * 8);
            std::memcpy(sneu, hs_neuron_.data() + lo, cnt * 4);
            a.st_off = soff;
            a.st_amp = samp;
            a.st_neuron = sneu;
            stats_.h2d_bytes_last += static_cast<double>(ob + cnt * 12);
        } else {  // device-resident table from build_stimulus_table
            a.st_off = d_st_off_.as<int64_t>() + tt;
            a.st_neuron = d_st_neuron_.as<int32_t>();
            a.st_amp = d_st_amp_.as<double>();
        }
        a.raster = raster + static_cast<size_t>(done) * words;
        a.trace = trace ? trace + static_cast<size_t>(done) * n_ : nullptr;
        launch_tiny(a, stream_);
        stats_.kernel_launches += 1;
        done += k;
        if (host_io && rows > 0 && done < steps)
            cuda_check(cudaStreamSynchronize(stream_), "tiny sync");  // staging is reused
    }
}

// ---- per-step launch sequence ----------------------------------------------
NeuronArgs Engine::neuron_args(int t_base, int rows, uint32_t* raster, double* trace, const int64_t* st_off,
                               const int32_t* st_neuron, const double* st_amp, int32_t st_steps,
                               int32_t st_base) {
    NeuronArgs a{};
    a.n = n_;
    a.first = first_;
    a.nl = nl_;
    a.v = d_v_.as<double>();
    a.thr = d_thr_.as<double>();
    a.leak = d_leak_.as<double>();
    a.reset = d_reset_.as<double>();
    a.refr = d_refr_.as<int32_t>();
    a.cnt = d_cnt_.as<int32_t>();
    a.partial = d_partial_.as<double>();
    a.nchunks = nchunks_;  // partial rows to sum
    a.partial16 = c16_ ? d_partial_.as<uint16_t>() : nullptr;
    a.w0 = dict_.empty() ? 0.0 : dict_[0];
    a.w0_f32 = f64_ ? 0 : 1;
    a.u_exact = d_uexact_.as<double>();
    a.st_off = st_off;
    a.st_neuron = st_neuron;
    a.st_amp = st_amp;
    a.st_steps = st_steps;
    a.st_base = st_base;
    a.d_step = d_step_.as<int32_t>();
    a.work = (dense_ && !exact_) ? d_work_.as<int32_t>() : nullptr;
    a.step_out = fold_hist() ? d_step_copy_.as<int32_t>() : nullptr;
    a.t_base = t_base;
    a.bits = d_bits_.as<uint32_t>();
    a.raster = raster;
    a.nl_words = nl_words_;
    a.raster_rows = rows;
    a.trace = trace;
    a.spike_count = d_spikes_.as<unsigned long long>();
    a.abm = abm_ ? 1 : 0;
    a.fire_p = any_stochastic_ ? d_firep_.as<double>() : nullptr;
    a.agent_key = any_stochastic_ ? d_akey_.as<uint64_t>() : nullptr;
    if (p2p_) {
        a.peer_bits = d_peer_bits_.as<uint32_t* const>();
        a.xstride = static_cast<int32_t>(d_xbits_.bytes / 8);
        a.peer_flags = d_peer_flags_.as<int32_t* const>();
        a.done = d_done_.as<uint32_t>();
        a.rank = opt_.rank;
        a.world = opt_.world;
    }
    return a;
}

HistArgs Engine::hist_args() {
    HistArgs h{};
    h.n = n_;
    h.bits = d_bits_.as<uint32_t>();
    h.hist = d_hist_.as<uint64_t>();
    h.hw = hw_;
    h.dmax = dmax_;
    h.stdp = stdp_on_ ? 1 : 0;
    h.window = window_;
    h.dp = stdp_on_ ? dp_ : 1;
    h.a_plus = d_ap_.as<double>();
    h.a_minus = d_am_.as<double>();
    h.pot64 = d_pot64_.as<double>();
    h.dep64 = d_dep64_.as<double>();
    h.row_plastic = d_row_plastic_.as<uint8_t>();
    h.active = d_active_.as<uint32_t>();
    h.d_step = d_step_.as<int32_t>();
    h.hist_lo = (!dense_ && (hbits_ == 16 || hbits_ == 32)) ? d_hist_lo_.as<uint32_t>() : nullptr;
    h.active_count = d_spikes_.as<unsigned long long>() + 1;
    h.clamp_step = clamp_step_;
    if (p2p_) {
        h.flags = d_flags_.as<int32_t>();
        h.xbits = d_xbits_.as<uint32_t>();
        h.xstride = static_cast<int32_t>(d_xbits_.bytes / 8);
        h.world = opt_.world;
        h.error = d_err_.as<int32_t>();
    }
    return h;
}

DenseArgs Engine::dense_args() {
    DenseArgs a{};
    a.n = n_;
    a.first = first_;
    a.nl = nl_;
    a.pitch = pitch_;
    a.w = d_w_.p;
    a.delay = has_delay_ ? d_delay_.as<uint8_t>() : nullptr;
    a.mask = any_mixed_ ? d_mask_.as<uint32_t>() : nullptr;
    a.kind = d_kind_.as<uint8_t>();
    a.active = d_active_.as<uint32_t>();
    a.hist = d_hist_.as<uint64_t>();
    a.bits = d_bits_.as<uint32_t>();
    a.pot = d_pot64_.as<double>();
    a.dep = d_dep64_.as<double>();
    a.dp = stdp_on_ ? dp_ : 1;
    a.w_min = w_min_;
    a.w_max = w_max_;
    a.tile_w = tile_w_;
    a.rows_per_chunk = rows_per_chunk_;
    a.nchunks = nchunks_;
    a.partial = d_partial_.as<double>();
    a.v = d_v_.as<double>();
    a.leak = d_leak_.as<double>();
    a.reset = d_reset_.as<double>();
    a.u_exact = d_uexact_.as<double>();
    a.d_step = d_step_.as<int32_t>();
    a.work = ((dynamic_sched_ || tma_) && !exact_ && !persistent_) ? d_work_.as<int32_t>() : nullptr;
    a.abm = abm_ ? 1 : 0;
    a.plastic_on = plasticity_ ? 1 : 0;
    return a;
}

void Engine::launch_sweep_only() {
    if (dense_) {
        DenseArgs a = dense_args();
        if (tma_) launch_dense_tma(a, f64_, stdp_on_, has_delay_, dense_grid_, stream_);
        else launch_dense(a, f64_, stdp_on_, has_delay_, exact_, dense_grid_, stream_);
    } else {
        SparseArgs a{};
        a.n = n_;
        a.first = first_;
        a.nl = nl_;
        a.pb = pb_;
        a.nblocks = nblocks_;
        a.off = d_off_.as<int64_t>();
        a.meta = d_meta_.as<uint32_t>();
        a.w = d_w_.p;
        a.bits = d_bits_.as<uint32_t>();
        a.hist_lo = d_hist_lo_.as<uint32_t>();
        a.hist = d_hist_.as<uint64_t>();
        a.pot = d_pot64_.as<double>();
        a.dep = d_dep64_.as<double>();
        a.dp = stdp_on_ ? dp_ : 1;
        a.w_min = w_min_;
        a.w_max = w_max_;
        a.posts_per_cta = posts_per_cta_;
        a.wdict = dict_.empty() ? nullptr : d_wdict_.p;
        a.dict_size = static_cast<int32_t>(dict_.size());
        a.pot_staged = pot_staged_ ? 1 : 0;
        a.partial = d_partial_.as<double>();
        a.partial16 = c16_ ? d_partial_.as<uint16_t>() : nullptr;
        a.v = d_v_.as<double>();
        a.leak = d_leak_.as<double>();
        a.reset = d_reset_.as<double>();
        a.u_exact = d_uexact_.as<double>();
        a.d_step = d_step_.as<int32_t>();
        a.abm = abm_ ? 1 : 0;
        a.plastic_on = plasticity_ ? 1 : 0;
        if (fold_hist()) {
            a.step_in = d_step_copy_.as<int32_t>();
            a.hist16 = d_hist16_.as<uint16_t>();
            if (p2p_) {  // the sweep itself waits for the peers' words of the step (no k_hist)
                a.flags = d_flags_.as<int32_t>();
                a.world = opt_.world;
                a.error = d_err_.as<int32_t>();
                a.xbits = d_xbits_.as<uint32_t>();
                a.xstride = static_cast<int32_t>(d_xbits_.bytes / 8);
            }
        }
        if (nl_ == 0) {
            launch_step_bump(a.d_step, stream_);
        } else if (sparse_tma_) {
            SpStagePlan plan{d_sp_stages_.as<SpStage>(), d_sp_first_.as<int32_t>(), d_sp_block_.as<int32_t>(),
                             d_sp_bnd_.as<uint16_t>()};
            launch_sparse_tma(a, plan, sp_ctas_, f64_, hbits_, stream_);
        } else if (c16_) {
            launch_sparse_count16(a, d_c16desc_.as<uint2>(), d_c16ent_.p, f64_, sub_, sparse_gx_, c16_threads_, stream_);
        } else {
            launch_sparse(a, f64_, stdp_on_, hbits_, sub_, exact_, sparse_gx_, stream_);
        }
    }
}

void Engine::launch_sweep() {
    launch_sweep_only();
    stats_.kernel_launches += 1;
}

cudaEvent_t Engine::get_event() {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void Engine::enqueue_step(const NeuronArgs& na, bool exchange) {
    const bool prof = opt_.profile != 0;
    const bool fused = opt_.world == 1 && !comm_;  // a 1-rank communicator runs the partitioned sequence
    const HistArgs h = hist_args();
    cudaEvent_t e0{}, e1{}, e2{}, e3{};
    if (prof) { e0 = get_event(); cuda_check(cudaEventRecord(e0, stream_), "rec"); }
    {
        NvtxRange nv("neuron phase");
        launch_neuron(na, exact_, fused, h, stream_);
    }
    stats_.kernel_launches += 1;
    if (prof) { e1 = get_event(); cuda_check(cudaEventRecord(e1, stream_), "rec"); pending_.push_back({e0, e1, 0, 0.0}); }
    if (!fused && exchange) {
        NvtxRange nv("spike exchange + history");
        if (prof) { e0 = get_event(); cuda_check(cudaEventRecord(e0, stream_), "rec"); }
        if (comm_ && !p2p_) comm_->all_gather_inplace(d_bits_.as<uint32_t>(), static_cast<size_t>(part_ / 32), stream_);
        if (!fold_hist()) {
            launch_hist(h, stream_);
            stats_.kernel_launches += 1;
        }
        if (prof) { e1 = get_event(); cuda_check(cudaEventRecord(e1, stream_), "rec"); pending_.push_back({e0, e1, 2, 0.0}); }
    }
    if (prof) { e2 = get_event(); cuda_check(cudaEventRecord(e2, stream_), "rec"); }
    {
        NvtxRange nv("sweep");
        launch_sweep();
    }
    if (prof) { e3 = get_event(); cuda_check(cudaEventRecord(e3, stream_), "rec"); pending_.push_back({e2, e3, 1, 0.0}); }
}

// The step loop as CUDA graphs of up to 64 steps (kernels read the step from
// d_step, so one graph serves every chunk of a simulate call).  With
// profiling, per-kernel CUDA events are captured into the graph (event record
// nodes) and read after each replay, so the timed loop keeps graph launch
// costs while reporting per-kernel device time.  Returns the summed device
// time of the chunks.
double Engine::run_graph_chunks(const NeuronArgs& na, int steps) {
    const bool prof = opt_.profile != 0;
    // a raster sink with stream_io decodes each finished chunk while the next
    // ones run: 16-step chunks leave only the last one's decode exposed
    const bool overlap = sink_ && opt_.stream_io && na.raster && !prof;
    const int chunk = std::min(steps, overlap ? 16 : 64);
    const bool fused = opt_.world == 1 && !comm_;  // a 1-rank communicator runs the partitioned sequence
    const int per = 6;
    std::vector<cudaEvent_t> ev(prof ? static_cast<size_t>(chunk) * per : 0);
    for (auto& e : ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    const HistArgs h = hist_args();
    auto capture = [&](int k) {
        NvtxRange nv("step graph capture");
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
        for (int s = 0; s < k; ++s) {
            // per-kernel events on every kProfStride-th step only: event nodes cost
            // ~1% of a 1.3 ms step when placed around every kernel
            cudaEvent_t* e = (prof && s % kProfStride == 0) ? &ev[static_cast<size_t>(s) * per] : nullptr;
            if (e) cuda_check(cudaEventRecordWithFlags(e[0], stream_, cudaEventRecordExternal), "rec");
            launch_neuron(na, exact_, fused, h, stream_);
            if (e) cuda_check(cudaEventRecordWithFlags(e[1], stream_, cudaEventRecordExternal), "rec");
            if (!fused) {
                if (e) cuda_check(cudaEventRecordWithFlags(e[2], stream_, cudaEventRecordExternal), "rec");
                if (comm_ && !p2p_) comm_->all_gather_inplace(d_bits_.as<uint32_t>(), static_cast<size_t>(part_ / 32), stream_);
                if (!fold_hist()) launch_hist(h, stream_);
                if (e) cuda_check(cudaEventRecordWithFlags(e[3], stream_, cudaEventRecordExternal), "rec");
            }
            if (e) cuda_check(cudaEventRecordWithFlags(e[4], stream_, cudaEventRecordExternal), "rec");
            launch_sweep_only();
            if (e) cuda_check(cudaEventRecordWithFlags(e[5], stream_, cudaEventRecordExternal), "rec");
        }
        cuda_check(cudaStreamEndCapture(stream_, &g), "end capture");
        cuda_check(cudaGraphInstantiate(&ge, g, 0), "instantiate");
        cudaGraphDestroy(g);
        return ge;
    };
#ifdef SNB_TIME_CAPTURE
    const auto c0 = std::chrono::steady_clock::now();
#endif
    cudaGraphExec_t full = capture(chunk);
    cudaGraphExec_t tail = (steps % chunk) ? capture(steps % chunk) : nullptr;
#ifdef SNB_TIME_CAPTURE
    std::fprintf(stderr, "graph capture+instantiate: %.1f us for %d + %d steps\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - c0).count(), chunk,
                 steps % chunk);
#endif
    const int per_step_kernels = (fused || fold_hist()) ? 2 : 3;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans;
    double total = 0.0;
    NvtxRange nv_replay("step graph replay");
    for (int done = 0; done < steps;) {
        const int k = std::min(chunk, steps - done);
        cudaEvent_t c0 = get_event(), c1 = get_event();
        cuda_check(cudaEventRecord(c0, stream_), "rec");
        cuda_check(cudaGraphLaunch(k == chunk ? full : tail, stream_), "graph launch");
        cuda_check(cudaEventRecord(c1, stream_), "rec");
        spans.emplace_back(c0, c1);
        stats_.kernel_launches += static_cast<int64_t>(per_step_kernels) * k;
        if (prof) {
            cuda_check(cudaStreamSynchronize(stream_), "profile sync");
            for (int s = 0; s < k; s += kProfStride) {
                const cudaEvent_t* e = &ev[static_cast<size_t>(s) * per];
                float a = 0.f, b = 0.f, c = 0.f;
                cuda_check(cudaEventElapsedTime(&a, e[0], e[1]), "elapsed");
                cuda_check(cudaEventElapsedTime(&c, e[4], e[5]), "elapsed");
                if (!fused) cuda_check(cudaEventElapsedTime(&b, e[2], e[3]), "elapsed");
                stats_.neuron_ms += a;
                stats_.neuron_launches += 1;
                stats_.exchange_ms += b;
                stats_.sweep_ms += c;
                stats_.sweep_launches += 1;
            }
        }
        done += k;
    }
    if (overlap) {  // every chunk is queued: decode each as its end event fires
        int row = 0;
        for (auto& sp : spans) {
#ifdef SNB_TIME_CAPTURE
            const auto w0 = std::chrono::steady_clock::now();
#endif
            cuda_check(cudaEventSynchronize(sp.second), "chunk sync");
#ifdef SNB_TIME_CAPTURE
            const auto w1 = std::chrono::steady_clock::now();
#endif
            const int k = std::min(chunk, steps - row);
            sink_rows(na.raster + static_cast<size_t>(row) * nl_words_, k, na.t_base + row);
#ifdef SNB_TIME_CAPTURE
            std::fprintf(stderr, "chunk %d rows: waited %.1f us, decoded in %.1f us\n", k,
                         std::chrono::duration<double, std::micro>(w1 - w0).count(),
                         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w1).count());
#endif
            row += k;
        }
    }
    cuda_check(cudaStreamSynchronize(stream_), "simulate sync");
    for (auto& sp : spans) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, sp.first, sp.second), "elapsed");
        total += ms;
        cudaEventDestroy(sp.first);
        cudaEventDestroy(sp.second);
    }
    cudaGraphExecDestroy(full);
    if (tail) cudaGraphExecDestroy(tail);
    for (auto& e : ev) cudaEventDestroy(e);
    return total;
}

void Engine::flush_pending() {
    if (pending_.empty()) return;
    cuda_check(cudaStreamSynchronize(stream_), "profile sync");
    for (auto& p : pending_) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, p.a, p.b), "elapsed");
        if (p.kind == 0) { stats_.neuron_ms += ms; stats_.neuron_launches += 1; }
        else if (p.kind == 1) { stats_.sweep_ms += ms; stats_.sweep_launches += 1; }
        else if (p.kind == 2) { stats_.exchange_ms += ms; }
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    pending_.clear();
}

void Engine::simulate(int32_t steps) {
    NvtxRange nv("sn_simulate");
    require_setup("sn_simulate");
    if (steps < 1) throw InvalidArgument(run_name() + ": steps must be >= 1");
    if (n_ == 0) {  // empty network: empty steps
        RasterChunk ch;
        ch.t0 = t_;
        ch.rows = steps;
        raster_.push_back(std::move(ch));
        if (opt_.record_membrane) trace_rows_ += steps;
        t_ += steps;
        stats_.steps_done = t_;
        stats_.last_simulate_ms = 0.0;
        events_valid_ = false;
        return;
    }
    if (opt_.world > 1 && !comm_ && !p2p_)
        throw LogicError("sn_simulate: partitioned engine needs sn_comm_init or sn_p2p_open "
                         "(or use sn_step_local/sn_step_finish)");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    note_first_plastic_step();
    build_stimulus_table();
    const int t0 = t_;
    double* trace = nullptr;
    if (opt_.record_membrane) {
        d_trace_.alloc(static_cast<size_t>(steps) * std::max(nl_, 1) * 8);
        trace = d_trace_.as<double>();
    }
    cudaEvent_t eb = get_event(), ee = get_event();
    double graph_ms = -1.0;  // device time summed over graph chunks (excludes host syncs)
    if (tiny_) {
        // one CTA runs the call; stream_io: stimulus read from and raster
        // written to pinned host memory by the kernel itself
        const size_t rwords = static_cast<size_t>(steps) * std::max(nl_words_, 1);
        uint32_t* raster;
        stats_.h2d_bytes_last = 0.0;
        if (opt_.stream_io) {
            h_raster_.reserve(rwords * 4);
            raster = h_raster_.as<uint32_t>();
        } else {
            if (d_raster_.bytes < rwords * 4) d_raster_.alloc(rwords * 4);
            raster = d_raster_.as<uint32_t>();
        }
        cuda_check(cudaEventRecord(eb, stream_), "rec");
        cudaEvent_t p0{}, p1{};
        if (opt_.profile) { p0 = get_event(); cuda_check(cudaEventRecord(p0, stream_), "rec"); }
        run_tiny(t0, steps, raster, trace, opt_.stream_io != 0);
        if (opt_.profile) {  // the call is one fused launch: accounted as the sweep
            p1 = get_event();
            cuda_check(cudaEventRecord(p1, stream_), "rec");
            pending_.push_back({p0, p1, 1, 0.0});
        }
        cuda_check(cudaEventRecord(ee, stream_), "rec");
        RasterChunk ch;
        ch.t0 = t0;
        ch.rows = steps;
        ch.words.resize(static_cast<size_t>(steps) * nl_words_);
        if (!opt_.stream_io && !ch.words.empty())
            cuda_check(cudaMemcpyAsync(ch.words.data(), raster, ch.words.size() * 4, cudaMemcpyDeviceToHost, stream_),
                       "raster D2H");
        cuda_check(cudaStreamSynchronize(stream_), "simulate sync");
        if (opt_.stream_io && !ch.words.empty()) std::memcpy(ch.words.data(), raster, ch.words.size() * 4);
        if (opt_.stream_io) stats_.d2h_bytes_last = static_cast<double>(ch.words.size()) * 4;
        raster_.push_back(std::move(ch));
    } else {
        // stream_io (the end-to-end path): this call's stimulus rows go H2D from
        // pinned memory in one copy inside the timed region, and the kernels
        // store every step's spike words straight into pinned host memory
        // (mapped), so each step's result crosses to the host as it is made.
        const size_t rwords = static_cast<size_t>(steps) * std::max(nl_words_, 1);
        uint32_t* raster = nullptr;
        const int64_t* st_off = d_st_off_.as<int64_t>();
        const int32_t* st_neuron = d_st_neuron_.as<int32_t>();
        const double* st_amp = d_st_amp_.as<double>();
        int32_t st_rows = st_steps_dev_, st_base = 0;
        cuda_check(cudaEventRecord(eb, stream_), "rec");
        if (opt_.stream_io) {
            h_raster_.reserve(rwords * 4);
            raster = h_raster_.as<uint32_t>();
            const int table = static_cast<int>(hs_off_.size()) - 1;
            st_rows = std::max(0, std::min(table - t0, steps));
            st_base = t0;
            const int64_t lo = st_rows > 0 ? hs_off_[t0] : 0, hi = st_rows > 0 ? hs_off_[t0 + st_rows] : 0;
            const size_t cnt = static_cast<size_t>(hi - lo);
            const size_t ob = round_up((static_cast<int64_t>(st_rows) + 1) * 8, 16);
            const size_t bytes = ob + cnt * 12 + 16;
            h_stage_.reserve(bytes);
            uint8_t* hb = h_stage_.as<uint8_t>();
            int64_t* soff = reinterpret_cast<int64_t*>(hb);
            for (int r = 0; r <= st_rows; ++r) soff[r] = (st_rows > 0 ? hs_off_[t0 + r] : 0) - lo;
            if (cnt) {
                std::memcpy(hb + ob, hs_amp_.data() + lo, cnt * 8);
                std::memcpy(hb + ob + cnt * 8, hs_neuron_.data() + lo, cnt * 4);
            }
            if (d_stage_.bytes < bytes) d_stage_.alloc(std::max(bytes, 2 * d_stage_.bytes));
            cuda_check(cudaMemcpyAsync(d_stage_.p, hb, bytes, cudaMemcpyHostToDevice, stream_), "stim H2D");
            uint8_t* db = d_stage_.as<uint8_t>();
            st_off = reinterpret_cast<const int64_t*>(db);
            st_amp = reinterpret_cast<const double*>(db + ob);
            st_neuron = reinterpret_cast<const int32_t*>(db + ob + cnt * 8);
            stats_.h2d_bytes_last = static_cast<double>(bytes);
        } else {
            if (d_raster_.bytes < rwords * 4) d_raster_.alloc(rwords * 4);
            raster = d_raster_.as<uint32_t>();
        }
        NeuronArgs na = neuron_args(t0, steps, raster, trace, st_off, st_neuron, st_amp, st_rows, st_base);
        if (persistent_) {
            cudaEvent_t p0{}, p1{};
            if (opt_.profile) { p0 = get_event(); cuda_check(cudaEventRecord(p0, stream_), "rec"); }
            if (cluster_) {
                ClusterArgs ka{};
                ka.codes = d_clcodes_.as<uint8_t>();
                ka.P = cl_P_;
                ka.D = cl_D_;
                ka.cs = cl_cs_;
                ka.w0 = cl_w0_;
                ka.hist2 = d_hist2_.as<uint64_t>();
                ka.partial = d_partial_.as<double>();
                ka.active_count = d_spikes_.as<unsigned long long>() + 1;
                ka.dmask = dmax_ >= 64 ? ~0ull : ((1ull << dmax_) - 1ull);
                // a raster sink with stream_io: the call runs as 4 launches (each
                // resumes from the state the previous one saved, like consecutive
                // calls) and the host expands each launch's rows while the next
                // runs (cfg2: 1M events per 1000 steps)
                const bool overlap = sink_ && opt_.stream_io && raster && !opt_.profile && steps >= 256;
                if (!overlap) {
                    launch_cluster_count(na, ka, f64_, steps, stream_);
                } else {
                    const int chunk = (steps + 3) / 4;
                    std::vector<std::pair<int, cudaEvent_t>> ends;
                    for (int done = 0; done < steps; done += chunk) {
                        const int k = std::min(chunk, steps - done);
                        launch_cluster_count(na, ka, f64_, k, stream_);
                        cudaEvent_t e = get_event();
                        cuda_check(cudaEventRecord(e, stream_), "rec");
                        ends.emplace_back(k, e);
                    }
                    stats_.kernel_launches += static_cast<int64_t>(ends.size()) - 1;
                    int row = 0;
                    for (auto& e : ends) {
                        cuda_check(cudaEventSynchronize(e.second), "chunk sync");
                        sink_rows(na.raster + static_cast<size_t>(row) * nl_words_, e.first, na.t_base + row);
                        row += e.first;
                        cudaEventDestroy(e.second);
                    }
                }
            } else if (cols_) {
                ColArgs ca{};
                ca.hist2 = d_hist2_.as<uint64_t>();
                ca.pot2 = d_pot2_.p;
                ca.act3 = d_act2_.as<uint32_t>();
                ca.row_plastic = d_row_plastic_.as<uint8_t>();
                ca.a_plus = d_ap_.as<double>();
                ca.a_minus = d_am_.as<double>();
                ca.window = window_;
                ca.dmax = dmax_;
                ca.active_count = d_spikes_.as<unsigned long long>() + 1;
                ca.clamp_step = clamp_step_;
                // activity and raster words are OR-ed by 8-post groups: start from
                // zero, and keep the OR targets in device memory (atomics on mapped
                // host memory would cross PCIe one by one); stream_io copies the
                // raster out once after the kernel
                cuda_check(cudaMemsetAsync(d_act2_.p, 0, d_act2_.bytes, stream_), "memset");
                const size_t rbytes = static_cast<size_t>(steps) * nl_words_ * 4;
                NeuronArgs nc = na;
                if (opt_.stream_io && raster) {
                    if (d_raster_.bytes < rbytes) d_raster_.alloc(rbytes);
                    nc.raster = d_raster_.as<uint32_t>();
                }
                if (nc.raster && rbytes) cuda_check(cudaMemsetAsync(nc.raster, 0, rbytes, stream_), "memset");
                launch_persistent_cols(nc, dense_args(), ca, f64_, stdp_on_, has_delay_, col_width_, persist_grid_,
                                       steps, stream_);
                if (opt_.stream_io && raster && rbytes)
                    cuda_check(cudaMemcpyAsync(raster, nc.raster, rbytes, cudaMemcpyDeviceToHost, stream_), "raster D2H");
            } else {
                launch_persistent_dense(na, hist_args(), dense_args(), f64_, stdp_on_, has_delay_, persist_grid_,
                                        steps, stream_);
            }
            stats_.kernel_launches += 1;
            if (opt_.profile) {
                p1 = get_event();
                cuda_check(cudaEventRecord(p1, stream_), "rec");
                pending_.push_back({p0, p1, 1, 0.0});
            }
            cuda_check(cudaEventRecord(ee, stream_), "rec");
        } else if (opt_.use_graphs && steps >= kMinGraphSteps) {
            // (a capture + instantiate costs ~1 ms: calls of a few steps, sn_step's
            // in particular, launch their kernels directly)
            graph_ms = run_graph_chunks(na, steps);
            cuda_check(cudaEventRecord(ee, stream_), "rec");
        } else {
            for (int s = 0; s < steps; ++s) enqueue_step(na, true);
            cuda_check(cudaEventRecord(ee, stream_), "rec");
        }
        RasterChunk ch;
        ch.t0 = t0;
        ch.rows = steps;
        ch.words.resize(static_cast<size_t>(steps) * nl_words_);
        if (!opt_.stream_io && !ch.words.empty())
            cuda_check(cudaMemcpyAsync(ch.words.data(), d_raster_.p, ch.words.size() * 4, cudaMemcpyDeviceToHost, stream_), "raster D2H");
        cuda_check(cudaStreamSynchronize(stream_), "simulate sync");
        if (opt_.stream_io && !ch.words.empty()) std::memcpy(ch.words.data(), raster, ch.words.size() * 4);
        if (opt_.stream_io) stats_.d2h_bytes_last = static_cast<double>(ch.words.size()) * 4;
        raster_.push_back(std::move(ch));
    }
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, eb, ee), "elapsed");
    cudaEventDestroy(eb);
    cudaEventDestroy(ee);
    stats_.last_simulate_ms = graph_ms >= 0.0 ? graph_ms : ms;
    flush_pending();
    check_exchange_error();
    if (opt_.record_membrane) {
        const size_t cnt = static_cast<size_t>(steps) * nl_;
        const size_t old = trace_.size();
        trace_.resize(old + cnt);
        if (cnt) d2h(trace_.data() + old, d_trace_.p, cnt * 8, "trace D2H");
        trace_rows_ += steps;
    }
    t_ += steps;
    stats_.steps_done = t_;
    events_valid_ = false;
}

void Engine::synchronize() { cuda_check(cudaStreamSynchronize(stream_), "sn_synchronize"); }

// Rows of spike words -> (step, neuron) events appended to the sink, rows in
// parallel (the same expansion as get_raster); relay neurons' bits skipped.
void Engine::sink_rows(const uint32_t* rows, int32_t nrows, int32_t t_first) {
    RasterSink& k = *sink_;
    const int lim = relays_ ? n_user_ - first_ : nl_;  // local ids below lim are the caller's
    auto word_of = [&](const uint32_t* row, int w) {
        const int lo = lim - w * 32;
        return lo >= 32 ? row[w] : lo <= 0 ? 0u : (row[w] & ((1u << lo) - 1u));
    };
    // work units: (row, word segment), enough of them for every thread even
    // when a chunk has few rows (the last chunk of a call is on the critical path)
    const unsigned hw = static_cast<unsigned>(host_threads());
    const int segs = std::max(1, std::min<int>(std::max(1, nl_words_ / 256),
                                                (static_cast<int>(hw) + nrows - 1) / std::max(1, nrows)));
    const int seg_words = (nl_words_ + segs - 1) / segs;
    const int units = nrows * segs;
    std::vector<int64_t> start(static_cast<size_t>(units) + 1, 0);
    for (int u = 0; u < units; ++u) {
        const uint32_t* row = rows + static_cast<size_t>(u / segs) * nl_words_;
        const int w0 = (u % segs) * seg_words, w1 = std::min(nl_words_, w0 + seg_words);
        int64_t c = 0;
        for (int w = w0; w < w1; ++w) c += __builtin_popcount(word_of(row, w));
        start[u + 1] = start[u] + c;
    }
    if (k.count + start[units] > k.cap)
        throw InvalidArgument("sn_simulate_raster: capacity " + std::to_string(k.cap) + " < " +
                              std::to_string(k.count + start[units]) + " events");
    auto expand = [&](int a, int b) {
        for (int u = a; u < b; ++u) {
            const int r = u / segs;
            const uint32_t* row = rows + static_cast<size_t>(r) * nl_words_;
            const int w0 = (u % segs) * seg_words, w1 = std::min(nl_words_, w0 + seg_words);
            int64_t o = k.count + start[u];
            for (int w = w0; w < w1; ++w)
                for (uint32_t x = word_of(row, w); x; x &= x - 1) {
                    k.steps[o] = t_first + r;
                    k.neurons[o] = first_ + w * 32 + __builtin_ctz(x);
                    ++o;
                }
        }
    };
    const int nthreads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({static_cast<int64_t>(hw),
                                                                               start[units] / 65536, units})));
    if (nthreads == 1) {
        expand(0, units);
    } else {
        // contiguous unit ranges of about equal event counts, on the host pool
        std::vector<int> cut(static_cast<size_t>(nthreads) + 1, units);
        cut[0] = 0;
        for (int i = 1; i < nthreads; ++i) {
            const int64_t target = start[units] * i / nthreads;
            int u1 = cut[i - 1];
            while (u1 < units && start[u1] < target) ++u1;
            cut[i] = u1;
        }
        host_parallel(nthreads, [&](int i) { expand(cut[i], cut[i + 1]); });
    }
    k.count += start[units];
    k.rows_done += nrows;
}

void Engine::simulate_raster(int32_t steps, int32_t* out_steps, int32_t* out_neurons, int64_t cap, int64_t* count) {
    require_setup("sn_simulate_raster");
    if (!count || (cap > 0 && (!out_steps || !out_neurons))) throw InvalidArgument("sn_simulate_raster: null parameter");
    RasterSink k;
    k.steps = out_steps;
    k.neurons = out_neurons;
    k.cap = cap;
    sink_ = &k;
    const int32_t t0 = t_;
    try {
        simulate(steps);
    } catch (...) {
        sink_ = nullptr;
        throw;
    }
    sink_ = nullptr;
    if (k.rows_done < steps) {  // no overlap on this path: decode the call's rows now
        const RasterChunk& ch = raster_.back();
        if (ch.t0 != t0 || ch.rows != steps) throw LogicError("sn_simulate_raster: the call's raster rows are missing");
        sink_ = &k;
        try {
            sink_rows(ch.words.data() + static_cast<size_t>(k.rows_done) * nl_words_, steps - k.rows_done,
                      t0 + k.rows_done);
        } catch (...) {
            sink_ = nullptr;
            throw;
        }
        sink_ = nullptr;
    }
    *count = k.count;
}

// ---- host-driven exchange (partition emulation / custom transports) ---------
void Engine::set_plasticity(bool on) {
    if (!stdp_on_ && on) {
        plasticity_ = true;  // nothing to apply; a no-op like calling mat_run without an StdpConfig
        return;
    }
    plasticity_ = on;
}

void Engine::step(const double* ext, int64_t ext_len, int32_t* spikes, int64_t cap, int64_t* count) {
    require_setup("sn_step");
    if (opt_.world > 1) throw LogicError("sn_step: partitioned engines step through sn_step_local / sn_step_finish");
    if (ext_len != 0 && ext_len != n_user_)  // mat_engine.cpp:170-171
        throw InvalidArgument("mat_step: ext must have one amplitude per neuron");
    if (ext_len && !ext) throw InvalidArgument("sn_step: null ext");
    if (!count) throw InvalidArgument("sn_step: null count");
    // the step's input is exactly ext: mat_step does not consult a schedule.
    // The schedule is swapped for one row holding ext's non-zero entries
    // (adding a zero amplitude leaves u unchanged) and restored afterwards.
    std::vector<int32_t> ss, sn;
    std::vector<double> sa;
    ss.swap(st_step_);
    sn.swap(st_neuron_);
    sa.swap(st_amp_);
    for (int64_t j = 0; j < ext_len; ++j) {
        if (!std::isfinite(ext[j])) {
            ss.swap(st_step_);
            sn.swap(st_neuron_);
            sa.swap(st_amp_);
            throw InvalidArgument("mat_step: ext[" + std::to_string(j) + "] must be finite");
        }
        if (ext[j] != 0.0) {
            st_step_.push_back(t_);
            st_neuron_.push_back(static_cast<int32_t>(j));
            st_amp_.push_back(ext[j]);
        }
    }
    stim_dirty_ = true;
    const int32_t t = t_;
    try {
        simulate(1);
    } catch (...) {
        st_step_.swap(ss);
        st_neuron_.swap(sn);
        st_amp_.swap(sa);
        stim_dirty_ = true;
        throw;
    }
    st_step_.swap(ss);
    st_neuron_.swap(sn);
    st_amp_.swap(sa);
    stim_dirty_ = true;
    // this step's spike words: the last row of the host raster
    strip_relays();
    const RasterChunk& ch = raster_.back();
    if (ch.t0 + ch.rows - 1 != t) throw LogicError("sn_step: raster row of the step is missing");
    const uint32_t* row = ch.words.data() + static_cast<size_t>(ch.rows - 1) * nl_words_;
    int64_t c = 0;
    for (int w = 0; w < nl_words_; ++w) c += __builtin_popcount(row[w]);
    *count = c;
    if (!spikes) return;  // size query
    if (cap < c) throw InvalidArgument("sn_step: capacity " + std::to_string(cap) + " < " + std::to_string(c) + " spikes");
    int64_t o = 0;
    for (int w = 0; w < nl_words_; ++w)
        for (uint32_t m = row[w]; m; m &= m - 1) spikes[o++] = first_ + w * 32 + __builtin_ctz(m);
}

void Engine::step_local() {
    NvtxRange nv("sn_step_local");
    require_setup("sn_step_local");
    if (n_ == 0) throw LogicError("sn_step_local: the network has no neurons");
    if (tiny_) throw LogicError("sn_step_local: single-partition engines run through sn_simulate");
    host_exchange_ = true;
    note_first_plastic_step();
    build_stimulus_table();
    if (d_raster_.bytes < static_cast<size_t>(std::max(nl_words_, 1)) * 4)
        d_raster_.alloc(static_cast<size_t>(std::max(nl_words_, 1)) * 4);
    double* trace = nullptr;
    if (opt_.record_membrane) {
        d_trace_.alloc(static_cast<size_t>(std::max(nl_, 1)) * 8);
        trace = d_trace_.as<double>();
    }
    if (opt_.stream_io) throw Unsupported("sn_step_local: stream_io engines use sn_simulate");
    NeuronArgs na = neuron_args(t_, 1, d_raster_.as<uint32_t>(), trace, d_st_off_.as<int64_t>(),
                                d_st_neuron_.as<int32_t>(), d_st_amp_.as<double>(), st_steps_dev_, 0);
    launch_neuron(na, exact_, opt_.world == 1, hist_args(), stream_);
    stats_.kernel_launches += 1;
    cuda_check(cudaStreamSynchronize(stream_), "step_local sync");
}

void Engine::get_spike_words(uint32_t* out, int64_t words) {
    require_setup("sn_get_spike_words");
    if (words > words_) throw InvalidArgument("sn_get_spike_words: more words than the bitmask holds");
    d2h(out, d_bits_.p, static_cast<size_t>(words) * 4, "bits D2H");
}

void Engine::put_spike_words(int32_t first_word, const uint32_t* w, int64_t count) {
    require_setup("sn_put_spike_words");
    if (first_word < 0 || first_word + count > words_) throw InvalidArgument("sn_put_spike_words: range outside the bitmask");
    h2d_sync(stream_, d_bits_.as<uint32_t>() + first_word, w, static_cast<size_t>(count) * 4, "bits H2D");
}

void Engine::step_finish() {
    NvtxRange nv("sn_step_finish");
    require_setup("sn_step_finish");
    if (n_ == 0) throw LogicError("sn_step_finish: the network has no neurons");
    if (tiny_) throw LogicError("sn_step_finish: single-partition engines run through sn_simulate");
    if (opt_.world > 1 && !fold_hist()) {
        launch_hist(hist_args(), stream_);
        stats_.kernel_launches += 1;
    }
    launch_sweep();
    RasterChunk ch;
    ch.t0 = t_;
    ch.rows = 1;
    ch.words.resize(static_cast<size_t>(nl_words_));
    if (nl_words_) cuda_check(cudaMemcpyAsync(ch.words.data(), d_raster_.p, ch.words.size() * 4, cudaMemcpyDeviceToHost, stream_), "raster D2H");
    cuda_check(cudaStreamSynchronize(stream_), "step_finish sync");
    check_exchange_error();
    raster_.push_back(std::move(ch));
    if (opt_.record_membrane) {
        const size_t old = trace_.size();
        trace_.resize(old + nl_);
        if (nl_) d2h(trace_.data() + old, d_trace_.p, static_cast<size_t>(nl_) * 8, "trace D2H");
        trace_rows_ += 1;
    }
    t_ += 1;
    stats_.steps_done = t_;
    events_valid_ = false;
}

}  // namespace snb
