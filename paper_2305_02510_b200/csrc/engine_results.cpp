// Results and statistics: raster decode, membranes, traces, weights, stats.
#include "engine.hpp"
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

// ---- results -------------------------------------------------------------------
// Bitmask raster -> (step, neuron) events, ascending: per-row popcounts, a
// prefix sum, then rows decoded in parallel straight into the two arrays.
void Engine::decode_raster() {
    if (events_valid_) return;
    NvtxRange nv("raster decode");
    strip_relays();
    std::vector<std::pair<const uint32_t*, int32_t>> rows;  // (words, step)
    for (const RasterChunk& ch : raster_)
        for (int r = 0; r < ch.rows; ++r)
            rows.emplace_back(ch.words.data() + static_cast<size_t>(r) * nl_words_, ch.t0 + r);
    std::vector<int64_t> start(rows.size() + 1, 0);
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    // a thread per ~64k words: spawning costs tens of microseconds
    const size_t nthreads = std::max<size_t>(1, std::min<size_t>(hw, rows.size() * nl_words_ / 65536));
    auto parallel = [&](auto&& fn) {
        if (nthreads == 1) return fn(size_t{0}, rows.size());
        std::vector<std::thread> pool;
        const size_t per = (rows.size() + nthreads - 1) / nthreads;
        for (size_t t = 0; t < nthreads; ++t) {
            const size_t a = t * per, b = std::min(rows.size(), a + per);
            if (a >= b) break;
            pool.emplace_back([&fn, a, b] { fn(a, b); });
        }
        for (auto& th : pool) th.join();
    };
    parallel([&](size_t a, size_t b) {
        for (size_t r = a; r < b; ++r) {
            int64_t c = 0;
            for (int w = 0; w < nl_words_; ++w) c += __builtin_popcount(rows[r].first[w]);
            start[r + 1] = c;
        }
    });
    for (size_t r = 0; r < rows.size(); ++r) start[r + 1] += start[r];
    dec_rows_ = std::move(rows);
    dec_start_ = std::move(start);
    events_valid_ = true;
}

int64_t Engine::raster_size() {
    require_setup("sn_raster_size");
    decode_raster();
    return dec_start_.empty() ? 0 : dec_start_.back();
}

// Rows are expanded in parallel straight into the caller's arrays (no
// intermediate copy: for 3.2 M events this is the bulk of the e2e overhead).
void Engine::get_raster(int32_t* steps, int32_t* neurons, int64_t cap) {
    require_setup("sn_get_raster");
    decode_raster();
    const int64_t ne = dec_start_.empty() ? 0 : dec_start_.back();
    if (cap < ne)
        throw InvalidArgument("sn_get_raster: capacity " + std::to_string(cap) + " < " + std::to_string(ne) + " events");
    const size_t nrows = dec_rows_.size();
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t nthreads = std::max<size_t>(1, std::min<size_t>(hw, static_cast<size_t>(ne / 131072)));
    const size_t per = (nrows + nthreads - 1) / std::max<size_t>(nthreads, 1);
    auto expand = [this, steps, neurons](size_t a, size_t b) {
        for (size_t r = a; r < b; ++r) {
            int64_t o = dec_start_[r];
            const uint32_t* row = dec_rows_[r].first;
            const int32_t step = dec_rows_[r].second;
            for (int w = 0; w < nl_words_; ++w) {
                uint32_t x = row[w];
                while (x) {
                    const int bit = __builtin_ctz(x);
                    x &= x - 1;
                    steps[o] = step;
                    neurons[o] = first_ + w * 32 + bit;
                    ++o;
                }
            }
        }
    };
    if (nthreads == 1) return expand(0, nrows);
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nthreads; ++t) {
        const size_t a = t * per, b = std::min(nrows, a + per);
        if (a >= b) break;
        pool.emplace_back(expand, a, b);
    }
    for (auto& th : pool) th.join();
}

void Engine::clear_raster() {
    strip_relays();  // count the relay spikes of the dropped rows first (stats)
    raster_.clear();
    dec_rows_.clear();
    dec_start_.clear();
    events_valid_ = true;
}

void Engine::get_membrane(double* out, int64_t count) {
    require_setup("sn_get_membrane");
    const int32_t nv = relays_ ? n_user_ : nl_;  // relay neurons are internal
    if (count < nv) throw InvalidArgument("sn_get_membrane: buffer smaller than the local neuron count");
    if (nv) d2h(out, d_v_.p, static_cast<size_t>(nv) * 8, "membrane D2H");
}

int64_t Engine::trace_rows() { return trace_rows_; }

void Engine::get_trace(double* out, int64_t count) {
    const int64_t nv = relays_ ? n_user_ : nl_;
    if (count < trace_rows_ * nv) throw InvalidArgument("sn_get_membrane_trace: buffer too small");
    if (nv == nl_) {
        std::memcpy(out, trace_.data(), trace_.size() * 8);
        return;
    }
    for (int64_t r = 0; r < trace_rows_; ++r)  // drop the relay columns
        std::memcpy(out + r * nv, trace_.data() + r * nl_, static_cast<size_t>(nv) * 8);
}

void Engine::get_synapse_weights(double* out, int64_t count) {
    require_setup("sn_get_synapse_weights");
    if (generated_) throw Unsupported("sn_get_synapse_weights: generated networks have no synapse list; use sn_get_weight_matrix");
    if (count < m_user_) throw InvalidArgument("sn_get_synapse_weights: buffer too small");
    if (m_user_ == 0) return;
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    const size_t esz = f64_ ? 8 : 4;
    std::vector<uint8_t> host(d_w_.bytes);
    d2h(host.data(), d_w_.p, d_w_.bytes, "weights D2H");
    std::vector<uint32_t> meta;
    if (!dense_ && !dict_.empty()) {
        meta.resize(static_cast<size_t>(sparse_elems_));
        if (!meta.empty()) d2h(meta.data(), d_meta_.p, meta.size() * 4, "meta D2H");
    }
    for (size_t s = 0; s < static_cast<size_t>(m_user_); ++s) {  // relay hops follow the caller's synapses
        if (slot_[s] < 0) { out[s] = 0.0; continue; }
        if (bank_ordered_) { out[s] = dict_[0]; continue; }  // lists reordered; one weight
        if (!meta.empty()) out[s] = dict_[meta[slot_[s]] >> 23];
        else if (esz == 8) out[s] = reinterpret_cast<const double*>(host.data())[slot_[s]];
        else out[s] = static_cast<double>(reinterpret_cast<const float*>(host.data())[slot_[s]]);
    }
}

// Census of the dense weight block W[0:n][0:n_local] on the device: how many
// stored weights equal each of `values` (rounded to the storage precision);
// counts[count] = every other cell, absent synapses (stored 0) included.
void Engine::weight_value_counts(const double* values, int32_t count, int64_t* counts) {
    require_setup("sn_weight_value_counts");
    if (!dense_ || tiny_ || relays_) throw Unsupported("sn_weight_value_counts: dense weight storage (no delay relays) only");
    if (count < 0 || count > census_max_values())
        throw InvalidArgument("sn_weight_value_counts: 0.." + std::to_string(census_max_values()) + " values");
    if ((count && !values) || !counts) throw InvalidArgument("sn_weight_value_counts: null parameter array");
    DevBuf dv, dc;
    if (f64_) {
        upload(stream_, dv, std::vector<double>(values, values + count));
    } else {
        std::vector<float> f(static_cast<size_t>(count));
        for (int k = 0; k < count; ++k) f[k] = static_cast<float>(values[k]);
        upload(stream_, dv, f);
    }
    dc.alloc(static_cast<size_t>(count + 1) * 8);
    cuda_check(cudaMemsetAsync(dc.p, 0, dc.bytes, stream_), "memset");
    int dev = 0, sms = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    launch_value_counts(d_w_.p, f64_, pitch_, n_, nl_, dv.p, count, dc.as<unsigned long long>(),
                        std::min(n_, sms * 8), stream_);
    d2h(counts, dc.p, dc.bytes, "counts D2H");
}

void Engine::get_weight_matrix(double* out, int64_t count) {
    require_setup("sn_get_weight_matrix");
    if (n_ == 0) return;
    if (relays_) {  // the caller's n x n matrix: each synapse at its own (pre, post), relays hidden
        if (count < static_cast<int64_t>(n_user_) * n_user_) throw InvalidArgument("sn_get_weight_matrix: buffer too small");
        std::vector<double> w(static_cast<size_t>(m_user_));
        get_synapse_weights(w.data(), m_user_);
        std::fill(out, out + static_cast<int64_t>(n_user_) * n_user_, 0.0);
        for (int64_t s = 0; s < m_user_; ++s) out[static_cast<int64_t>(pre_user_[s]) * n_user_ + post_[s]] = w[s];
        return;
    }
    if (count < static_cast<int64_t>(n_) * nl_) throw InvalidArgument("sn_get_weight_matrix: buffer too small");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    std::fill(out, out + static_cast<int64_t>(n_) * nl_, 0.0);
    const size_t esz = f64_ ? 8 : 4;
    std::vector<uint8_t> host(d_w_.bytes);
    d2h(host.data(), d_w_.p, d_w_.bytes, "weights D2H");
    auto get = [&](int64_t q) {
        return esz == 8 ? reinterpret_cast<const double*>(host.data())[q]
                        : static_cast<double>(reinterpret_cast<const float*>(host.data())[q]);
    };
    if (tiny_) {
        for (size_t s = 0; s < pre_.size(); ++s) out[static_cast<int64_t>(pre_[s]) * nl_ + post_[s]] = get(slot_[s]);
    } else if (dense_) {
        for (int i = 0; i < n_; ++i)
            for (int c = 0; c < nl_; ++c) out[static_cast<int64_t>(i) * nl_ + c] = get(static_cast<int64_t>(i) * pitch_ + c);
    } else {
        std::vector<int64_t> off(static_cast<size_t>(nblocks_) * nl_ + 1);
        std::vector<uint32_t> meta(static_cast<size_t>(sparse_elems_));
        d2h(off.data(), d_off_.p, off.size() * 8, "off D2H");
        if (!meta.empty()) d2h(meta.data(), d_meta_.p, meta.size() * 4, "meta D2H");
        for (int b = 0; b < nblocks_; ++b)
            for (int p = 0; p < nl_; ++p)
                for (int64_t q = off[static_cast<size_t>(b) * nl_ + p]; q < off[static_cast<size_t>(b) * nl_ + p + 1]; ++q) {
                    const double w = sparse_weight(host, meta, q);
                    const int i = b * pb_ + static_cast<int>(meta[q] & 0xffffu);
                    if (w != 0.0) out[static_cast<int64_t>(i) * nl_ + p] = w;
                }
    }
}

void Engine::get_stats(sn_stats* out) {
    if (setup_done_ && n_ > 0) {
        unsigned long long c[2] = {0, 0};
        d2h(c, d_spikes_.p, 16, "stats D2H");
        strip_relays();
        stats_.spike_count = static_cast<int64_t>(c[0]) - relay_spikes_;  // the caller's neurons only
        // algorithmic bytes: every visited row (dense) or every stored synapse (sparse pull)
        if (dense_) {
            const double per_row = static_cast<double>(nl_) * ((stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + (has_delay_ ? 1 : 0));
            stats_.sweep_bytes_total = static_cast<double>(c[1]) * per_row;
        } else {
            stats_.sweep_bytes_total = sweep_bytes_full_ * static_cast<double>(t_ - steps_at_reset_);
        }
        stats_.sweep_bytes_per_launch_last = sweep_bytes_full_;
        if (tiny_) {
            stats_.sweep_kernel = SN_SWEEP_TINY;
            stats_.sweep_ctas = 1;
        } else if (dense_) {
            stats_.sweep_kernel = persistent_ ? (cluster_ ? SN_SWEEP_CLUSTER : cols_ ? SN_SWEEP_PERSISTENT_COLS : SN_SWEEP_PERSISTENT)
                                  : exact_    ? SN_SWEEP_DENSE_EXACT
                                  : tma_      ? SN_SWEEP_DENSE_TMA
                                              : SN_SWEEP_DENSE_STREAM;
            stats_.sweep_ctas = persistent_ ? persist_grid_ : dense_grid_;
        } else {
            stats_.sweep_kernel = exact_ ? SN_SWEEP_SPARSE_EXACT
                                  : sparse_tma_ ? SN_SWEEP_SPARSE_TMA
                                  : c16_ ? (c16_bytes() ? SN_SWEEP_SPARSE_COUNT8 : SN_SWEEP_SPARSE_COUNT16)
                                  : (dict_.size() == 2 && !stdp_on_ && sub_ != 0 && hbits_ != 64) ? SN_SWEEP_SPARSE_COUNT
                                  : sub_ == 0 ? SN_SWEEP_SPARSE_STREAM
                                  : !dict_.empty() ? SN_SWEEP_SPARSE_DICT
                                                   : SN_SWEEP_SPARSE_PULL;
            stats_.sweep_ctas = sparse_tma_ ? sp_ctas_ : sparse_gx_ * nblocks_;
        }
    }
    *out = stats_;
}

void Engine::reset_stats() {
    stats_.sweep_ms = stats_.neuron_ms = stats_.exchange_ms = 0.0;
    stats_.sweep_launches = stats_.neuron_launches = 0;
    stats_.kernel_launches = 0;
    stats_.sweep_bytes_total = 0.0;
    steps_at_reset_ = t_;
    if (setup_done_ && n_ > 0) cuda_check(cudaMemsetAsync(d_spikes_.as<unsigned long long>() + 1, 0, 8, stream_), "reset");
}

}  // namespace snb
