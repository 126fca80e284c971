// Device layouts of the engine: the tiny-net in-lists, dense W[pre][post]
// with delays / plastic masks / row kinds, blocked CSC (with the weight
// dictionary and bank-aware list order), on-device generated nets, and the
// launch plans of every kernel family.
#include <cstdio>
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

// In-lists for k_tiny: post-major, pre ascending.  Returns false when the
// state and the lists would not leave room for a step's stimulus in shared memory.
bool Engine::build_tiny() {
    TinyArgs probe{};  // state + lists + one step with every neuron stimulated
    probe.n = n_;
    probe.steps = 1;
    probe.hw = hw_;
    probe.f64 = f64_ ? 1 : 0;
    probe.m = static_cast<int32_t>(pre_.size());
    probe.st_count = n_;
    probe.stdp = stdp_on_ ? 1 : 0;
    probe.window = window_;
    probe.dp = dp_;
    if (tiny_smem_bytes(probe) + 4096 > static_cast<size_t>(tiny_max_smem())) return false;
    if (stdp_on_ && static_cast<int64_t>(n_) * dp_ >= 0xffff) return false;  // pidx is 16-bit, 0xffff reserved

    std::vector<uint32_t> off(static_cast<size_t>(n_) + 1, 0);
    for (size_t s = 0; s < pre_.size(); ++s) ++off[post_[s] + 1];
    for (int j = 0; j < n_; ++j) off[j + 1] += off[j];
    std::vector<size_t> ord(pre_.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
        return post_[a] != post_[b] ? post_[a] < post_[b] : pre_[a] < pre_[b];
    });
    // meta: byte offset of the 32-bit history word of delay bit d-1 of pre
    // (word (d-1)/32 * np + pre) << 5 | bit; pidx 0xffff marks non-plastic
    const uint32_t np = static_cast<uint32_t>(round_up(n_, 32));
    std::vector<uint32_t> meta(pre_.size());
    std::vector<uint16_t> pidx(stdp_on_ ? pre_.size() : 0);
    std::vector<float> wf;
    std::vector<double> wd;
    if (f64_) wd.resize(pre_.size());
    else wf.resize(pre_.size());
    slot_.assign(pre_.size(), -1);
    for (size_t q = 0; q < ord.size(); ++q) {
        const size_t s = ord[q];
        const uint32_t d1 = static_cast<uint32_t>(delay_[s] + axonal_[pre_[s]] - 1);
        const uint32_t pre = static_cast<uint32_t>(pre_[s]);
        const bool pl = stdp_on_ && plastic_[s];
        meta[q] = ((((d1 >> 5) * np + pre) * 4u) << 5) | (d1 & 31u);
        if (stdp_on_) pidx[q] = pl ? static_cast<uint16_t>(pre * static_cast<uint32_t>(dp_) + d1) : uint16_t(0xffff);
        if (f64_) wd[q] = weight_[s];
        else wf[q] = static_cast<float>(weight_[s]);
        slot_[s] = static_cast<int64_t>(q);
    }
    upload(stream_, d_toff_, off);
    upload(stream_, d_meta_, meta);
    upload(stream_, d_tpidx_, pidx);
    if (f64_) upload(stream_, d_w_, wd);
    else upload(stream_, d_w_, wf);
    syn_local_ = static_cast<int64_t>(pre_.size());
    sweep_bytes_full_ = static_cast<double>(pre_.size()) * ((stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + 4.0);
    return true;
}

void Engine::build_dense_from_lists() {
    pitch_ = round_up(std::max(nl_, 1), 32);
    const int64_t elems = static_cast<int64_t>(n_) * pitch_;
    std::vector<float> wf;
    std::vector<double> wd;
    if (f64_) wd.assign(static_cast<size_t>(elems), 0.0);
    else wf.assign(static_cast<size_t>(elems), 0.0f);
    std::vector<uint8_t> dl;
    if (has_delay_) dl.assign(static_cast<size_t>(elems), 1);
    std::vector<int64_t> pl_count(n_, 0);
    std::vector<uint8_t> self_present(n_, 0);
    slot_.assign(pre_.size(), -1);
    syn_local_ = 0;
    for (size_t s = 0; s < pre_.size(); ++s) {
        const int j = post_[s];
        if (j < first_ || j >= first_ + nl_) continue;
        const int i = pre_[s];
        const int64_t off = static_cast<int64_t>(i) * pitch_ + (j - first_);
        if (f64_) wd[off] = weight_[s];
        else wf[off] = static_cast<float>(weight_[s]);
        if (has_delay_) dl[off] = static_cast<uint8_t>(delay_[s] + axonal_[i]);
        slot_[s] = off;
        ++syn_local_;
        if (stdp_on_ && plastic_[s]) ++pl_count[i];
        if (i == j) self_present[i] = 1;
    }
    std::vector<uint8_t> kind(n_, kRowNone), row_pl(n_, 0);
    any_mixed_ = false;
    for (int i = 0; i < n_; ++i) {
        const bool self_local = i >= first_ && i < first_ + nl_;
        if (pl_count[i] == 0) kind[i] = kRowNone;
        else if (pl_count[i] == nl_) kind[i] = kRowAll;
        else if (self_local && pl_count[i] == nl_ - 1 && !self_present[i]) kind[i] = kRowAllButSelf;
        else { kind[i] = kRowMixed; any_mixed_ = true; }
        row_pl[i] = kind[i] != kRowNone;
    }
    if (f64_) upload(stream_, d_w_, wd);
    else upload(stream_, d_w_, wf);
    if (has_delay_) upload(stream_, d_delay_, dl);
    if (any_mixed_) {
        std::vector<uint32_t> mask(static_cast<size_t>(n_) * (pitch_ / 32), 0u);
        for (size_t s = 0; s < pre_.size(); ++s) {
            if (slot_[s] < 0 || !plastic_[s]) continue;
            const int64_t off = slot_[s];
            const int64_t row = off / pitch_, c = off % pitch_;
            mask[row * (pitch_ / 32) + c / 32] |= 1u << (c % 32);
        }
        upload(stream_, d_mask_, mask);
    }
    upload(stream_, d_kind_, kind);
    upload(stream_, d_row_plastic_, row_pl);
    sweep_bytes_full_ = static_cast<double>(n_) * nl_ * ((stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + (has_delay_ ? 1 : 0));
}

// Pres per block: the history-width limit, and for STDP pull sweeps small
// enough that the block's pot^(d) traces fit the shared-memory stage.
int32_t Engine::sparse_pres_per_block() const {
    int pb = sparse_block_pres(hbits_);
    pot_staged_ = false;
    // static nets with delays <= 16: 4 x 4095-pre blocks, the layout k_sparse_count16's
    // 16-bit entries need (the other sparse kernels take any block size)
    if (hbits_ == 16 && !stdp_on_ && !exact_ && c16_allowed()) pb = c16_block_pres();
    if (stdp_on_ && !exact_) {
        const int esz = 8;  // fp64 traces for every weight type
        // 100k-neuron ER(p=0.01) STDP sweep: staged 0.314 ms vs 0.413 gathered at dp = 1;
        // at dp = 8 the 768-pre blocks of a 24 KB stage lost (0.672 vs 0.591 ms) while
        // 2048-pre blocks in 64 KB (3 CTAs/SM) won (0.532); blocks below 2048 pres
        // are never staged (list overhead), and dp = 1 keeps 24 KB (4 CTAs/SM:
        // 0.328 ms vs 0.347 at 48 KB, 0.408 at 64 KB)
        int budget = sparse_pot_stage_bytes(dp_);
        if (const char* kb = std::getenv("SNB_SPARSE_POT_KB")) budget = std::atoi(kb) * 1024;  // A/B knob
        const int fit = budget / (std::max(dp_, 1) * esz) / 32 * 32;
        if (fit >= 2048) {
            pb = std::min(pb, fit);
            pot_staged_ = true;
        }
    }
    return pb;
}

void Engine::build_sparse_from_lists() {
    pb_ = sparse_pres_per_block();
    nblocks_ = (n_ + pb_ - 1) / pb_;
    const int64_t nseg = static_cast<int64_t>(nblocks_) * nl_;
    std::vector<int64_t> cnt(static_cast<size_t>(nseg) + 1, 0);
    std::vector<int64_t> local;
    local.reserve(pre_.size());
    for (size_t s = 0; s < pre_.size(); ++s) {
        const int j = post_[s];
        if (j < first_ || j >= first_ + nl_) continue;
        local.push_back(static_cast<int64_t>(s));
        ++cnt[static_cast<int64_t>(pre_[s] / pb_) * nl_ + (j - first_)];
    }
    syn_local_ = static_cast<int64_t>(local.size());
    std::vector<int64_t> off(static_cast<size_t>(nseg) + 1, 0);
    for (int64_t g = 0; g < nseg; ++g) off[g + 1] = off[g] + round_up(cnt[g], 4);
    sparse_elems_ = off[nseg];
    // order within a segment: pre ascending (matches the CSR propagate order)
    std::sort(local.begin(), local.end(), [&](int64_t a, int64_t b) {
        const int64_t ga = static_cast<int64_t>(pre_[a] / pb_) * nl_ + (post_[a] - first_);
        const int64_t gb = static_cast<int64_t>(pre_[b] / pb_) * nl_ + (post_[b] - first_);
        if (ga != gb) return ga < gb;
        return pre_[a] < pre_[b];
    });
    // weight dictionary: a static (non-plastic) net with <= 511 distinct weights
    // keeps only the 4-byte meta word per synapse (index in bits 23..31)
    dict_.clear();
    if (!stdp_on_ && !exact_) {
        std::unordered_map<uint64_t, int> idx;
        bool fits = true;
        for (int64_t s : local) {
            uint64_t key;
            const double w = f64_ ? weight_[s] : static_cast<double>(static_cast<float>(weight_[s]));
            std::memcpy(&key, &w, 8);
            if (idx.emplace(key, static_cast<int>(dict_.size())).second) dict_.push_back(w);
            if (dict_.size() > 511) { fits = false; break; }
        }
        if (!fits) dict_.clear();
        else dict_.push_back(0.0);  // padding entry
    }
    const bool dict = !dict_.empty();
    std::unordered_map<uint64_t, int> dict_idx;
    for (size_t k = 0; k < dict_.size(); ++k) {
        uint64_t key;
        std::memcpy(&key, &dict_[k], 8);
        dict_idx.emplace(key, static_cast<int>(k));
    }
    // dictionary padding: value 0.0 and the inert pre slot pb (zero history)
    const uint32_t pad_meta = dict ? ((static_cast<uint32_t>(dict_.size() - 1) << 23) | static_cast<uint32_t>(pb_)) : 0u;
    std::vector<uint32_t> meta(static_cast<size_t>(sparse_elems_), pad_meta);
    std::vector<float> wf;
    std::vector<double> wd;
    if (!dict) {
        if (f64_) wd.assign(static_cast<size_t>(sparse_elems_), 0.0);
        else wf.assign(static_cast<size_t>(sparse_elems_), 0.0f);
    }
    std::vector<int64_t> cur(off.begin(), off.end() - 1);
    slot_.assign(pre_.size(), -1);
    std::vector<uint8_t> row_pl(n_, 0);
    for (int64_t s : local) {
        const int i = pre_[s];
        const int64_t g = static_cast<int64_t>(i / pb_) * nl_ + (post_[s] - first_);
        const int64_t q = cur[g]++;
        const int d = delay_[s] + axonal_[i];
        const bool pl = stdp_on_ && plastic_[s];
        meta[q] = static_cast<uint32_t>(i % pb_) | (static_cast<uint32_t>(d - 1) << 16) | (pl ? (1u << 22) : 0u);
        if (dict) {
            const double w = f64_ ? weight_[s] : static_cast<double>(static_cast<float>(weight_[s]));
            uint64_t key;
            std::memcpy(&key, &w, 8);
            meta[q] |= static_cast<uint32_t>(dict_idx.at(key)) << 23;
        } else if (f64_) {
            wd[q] = weight_[s];
        } else {
            wf[q] = static_cast<float>(weight_[s]);
        }
        slot_[s] = q;
        if (pl) row_pl[i] = 1;
    }
    upload(stream_, d_off_, off);
    upload(stream_, d_meta_, meta);
    if (dict) d_w_.alloc(16);
    else if (f64_) upload(stream_, d_w_, wd);
    else upload(stream_, d_w_, wf);
    upload_dict();
    upload(stream_, d_row_plastic_, row_pl);
    sweep_bytes_full_ = static_cast<double>(syn_local_) *
                        (dict ? 4.0 : (stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + 4.0);
}

void Engine::upload_dict() {
    if (dict_.empty()) {
        d_wdict_.release();
        return;
    }
    if (f64_) {
        upload(stream_, d_wdict_, dict_);
    } else {
        std::vector<float> f(dict_.begin(), dict_.end());
        upload(stream_, d_wdict_, f);
    }
}

double Engine::sparse_weight(const std::vector<uint8_t>& host_w, const std::vector<uint32_t>& meta, int64_t q) const {
    if (!dict_.empty()) return dict_[meta[q] >> 23];
    return f64_ ? reinterpret_cast<const double*>(host_w.data())[q]
                : static_cast<double>(reinterpret_cast<const float*>(host_w.data())[q]);
}

void Engine::build_generated() {
    const size_t esz = f64_ ? 8 : 4;
    slot_.clear();
    std::vector<uint8_t> row_pl(n_, 0);
    if (dense_) {
        pitch_ = round_up(std::max(nl_, 1), 32);
        const int64_t elems = static_cast<int64_t>(n_) * pitch_;
        d_w_.alloc(static_cast<size_t>(elems) * esz);
        if (has_delay_) d_delay_.alloc(static_cast<size_t>(elems));
        std::vector<uint8_t> kind(n_, kRowNone);
        any_mixed_ = false;
        if (er_.stdp) {
            for (int i = 0; i < n_; ++i) {
                const bool self_local = i >= first_ && i < first_ + nl_;
                if (er_.p >= 1.0) kind[i] = self_local ? kRowAllButSelf : kRowAll;
                else { kind[i] = kRowMixed; any_mixed_ = true; }
                row_pl[i] = 1;
            }
            if (nl_ == 0) std::fill(kind.begin(), kind.end(), kRowNone);
        }
        if (any_mixed_) d_mask_.alloc(static_cast<size_t>(n_) * (pitch_ / 32) * 4);
        launch_er_dense(er_, d_w_.p, f64_, has_delay_ ? d_delay_.as<uint8_t>() : nullptr,
                        any_mixed_ ? d_mask_.as<uint32_t>() : nullptr, first_, nl_, pitch_, stream_);
        stats_.kernel_launches += 1;
        upload(stream_, d_kind_, kind);
        if (er_.p >= 1.0) {
            const int64_t self_local = std::max(0, std::min(nl_, n_ - first_));
            syn_local_ = static_cast<int64_t>(n_) * nl_ - self_local;
        } else {
            syn_local_ = static_cast<int64_t>(er_.p * static_cast<double>(n_) * nl_);  // expectation
        }
        sweep_bytes_full_ = static_cast<double>(n_) * nl_ * ((stdp_on_ ? 2.0 : 1.0) * esz + (has_delay_ ? 1 : 0));
    } else {
        pb_ = sparse_pres_per_block();
        nblocks_ = (n_ + pb_ - 1) / pb_;
        const int64_t nseg = static_cast<int64_t>(nblocks_) * nl_;
        DevBuf d_counts;
        d_counts.alloc(static_cast<size_t>(nseg) * 8);
        launch_er_sparse_count(er_, first_, nl_, pb_, nblocks_, d_counts.as<int64_t>(), stream_);
        std::vector<int64_t> cnt(static_cast<size_t>(nseg));
        cuda_check(cudaMemcpyAsync(cnt.data(), d_counts.p, static_cast<size_t>(nseg) * 8, cudaMemcpyDeviceToHost, stream_), "counts D2H");
        cuda_check(cudaStreamSynchronize(stream_), "counts sync");
        std::vector<int64_t> off(static_cast<size_t>(nseg) + 1, 0);
        syn_local_ = 0;
        for (int64_t g = 0; g < nseg; ++g) {
            off[g + 1] = off[g] + round_up(cnt[g], 4);
            syn_local_ += cnt[g];
        }
        sparse_elems_ = off[nseg];
        upload(stream_, d_off_, off);
        d_meta_.alloc(static_cast<size_t>(sparse_elems_) * 4);
        // static nets use the weight dictionary {weight, 0.0 (padding)}: 4 B/synapse
        dict_.clear();
        if (!er_.stdp && !exact_) dict_ = {f64_ ? er_.weight_d : static_cast<double>(er_.weight_f), 0.0};
        const bool dict = !dict_.empty();
        d_w_.alloc(dict ? 16 : static_cast<size_t>(sparse_elems_) * esz);
        launch_er_sparse_fill(er_, first_, nl_, pb_, nblocks_, d_off_.as<int64_t>(), d_meta_.as<uint32_t>(),
                              dict ? nullptr : d_w_.p, f64_, stream_);
        upload_dict();
        stats_.kernel_launches += 2;
        if (er_.stdp) std::fill(row_pl.begin(), row_pl.end(), 1);
        sweep_bytes_full_ = static_cast<double>(syn_local_) * (dict ? 4.0 : (stdp_on_ ? 2.0 : 1.0) * esz + 4.0);
    }
    upload(stream_, d_row_plastic_, row_pl);
    if (er_.stdp && !stdp_on_)
        throw InvalidArgument("mat_init: plastic synapses were generated but no STDP config was set (sn_set_stdp)");
}

void Engine::plan_launches() {
    int sms = 148;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, opt_.device), "attr");
    const size_t esz = f64_ ? 8 : 4;
    persistent_ = opt_.persistent >= 0 && dense_ && !exact_ && opt_.world == 1 && nl_ > 0 &&
                  static_cast<double>(n_) * pitch_ * esz <= 64.0 * 1024 * 1024;  // L2-resident
    if (persistent_) {
        // 32-row chunks; split columns until the items fill the co-resident CTAs
        const int vec = dense_vec(f64_);
        const int resident = persistent_max_ctas(f64_, stdp_on_, has_delay_);
        rows_per_chunk_ = 32;
        nchunks_ = (n_ + 31) / 32;
        const int max_tiles = std::max(1, (nl_ + 32 * vec - 1) / (32 * vec));
        int ntiles = std::min(max_tiles, std::max(1, (resident + nchunks_ - 1) / nchunks_));
        ntiles = std::min(ntiles, std::max(1, (nl_ + dense_threads() * vec - 1) / (dense_threads() * vec) * 8));
        tile_w_ = static_cast<int32_t>(round_up((nl_ + ntiles - 1) / ntiles, vec));
        tile_w_ = std::min<int32_t>(std::max(tile_w_, vec), dense_threads() * vec);
        ntiles = (nl_ + tile_w_ - 1) / tile_w_;
        const bool tiny = static_cast<double>(n_) * pitch_ * esz <= 256.0 * 1024 &&
                          nl_ <= dense_threads() * vec;
        if (tiny) {  // one CTA: a single item avoids serial per-item round trips
            rows_per_chunk_ = static_cast<int32_t>(round_up(n_, 32));
            nchunks_ = 1;
            tile_w_ = static_cast<int32_t>(round_up(nl_, vec));
            ntiles = 1;
        }
        const int items = ntiles * nchunks_;
        persist_grid_ = tiny ? 1 : std::max(1, std::min(items, resident));
        if (const char* pc = std::getenv("SNB_PERSIST_CTAS"))  // A/B knob
            persist_grid_ = std::max(1, std::min(std::atoi(pc), resident));
        dense_grid_ = std::min(items, sms * 8);
        d_partial_.alloc(static_cast<size_t>(nchunks_) * std::max(nl_, 1) * 8);
        cuda_check(cudaMemsetAsync(d_partial_.p, 0, d_partial_.bytes, stream_), "memset");
        // column owners (one grid barrier per step) when the history is one word
        // and there are enough 32-post column groups to spread the sweep
        const char* pk = std::getenv("SNB_PERSIST_KERNEL");  // A/B knob: rows | cols
        cols_ = hw_ == 1 && !tiny && nl_ >= 64 && !(pk && std::string(pk) == "rows");
        if (pk && std::string(pk) == "cols" && hw_ == 1) cols_ = true;
        if (cols_) {  // 8-post column groups, all co-resident (wider groups lose to the row chunks)
            cols_ = false;
            for (int w : {8}) {
                const int groups = (nl_ + w - 1) / w;
                if (groups <= persistent_cols_max_ctas(f64_, stdp_on_, has_delay_, w)) {
                    cols_ = true;
                    col_width_ = w;
                    persist_grid_ = groups;
                    break;
                }
            }
        }
        // one thread-block cluster with distributed shared memory instead of a
        // grid barrier: static one-weight nets without plasticity (cfg2)
        cluster_ = false;
        double w0 = 0.0;
        if (!stdp_on_ && !tiny && dmax_ <= 31 && hw_ == 1 && !(pk && std::string(pk) != "cluster") &&
            uniform_weight(&w0) && w0 != 0.0) {
            int P = 0, D = 0;
            const int cs = cluster_plan(n_, nl_, f64_, dmax_, &P, &D);
            if (cs > 0) {
                cluster_ = true;
                cols_ = false;
                cl_cs_ = cs;
                cl_P_ = P;
                cl_D_ = D;
                cl_w0_ = w0;
                d_clcodes_.alloc(cluster_table_bytes(n_, P, D, cs));
                launch_cluster_table(dense_args(), nl_, P, D, cs, d_clcodes_.p, f64_, stream_);
                d_hist2_.alloc(static_cast<size_t>(2) * n_ * 8);
                cuda_check(cudaMemsetAsync(d_hist2_.p, 0, d_hist2_.bytes, stream_), "memset");
                persist_grid_ = cs;
            }
        }
        if (cols_) {
            d_hist2_.alloc(static_cast<size_t>(2) * n_ * 8);
            d_pot2_.alloc(static_cast<size_t>(2) * n_ * std::max(dp_, 1) * 8);  // fp64 traces
            d_act2_.alloc(static_cast<size_t>(3) * ((n_ + 31) / 32) * 4);
            for (DevBuf* b : {&d_hist2_, &d_pot2_, &d_act2_})
                cuda_check(cudaMemsetAsync(b->p, 0, b->bytes, stream_), "memset");
        }
    } else if (dense_) {
        const int vec = dense_vec(f64_);
        const int span = dense_threads() * vec;
        int ntiles = std::max(1, (nl_ + span - 1) / span);
        if (const char* nt = std::getenv("SNB_SWEEP_TILES")) ntiles = std::max(ntiles, std::atoi(nt));
        tile_w_ = static_cast<int32_t>(round_up((nl_ + ntiles - 1) / ntiles, vec));
        tile_w_ = std::max(tile_w_, vec);
        if (exact_) {
            nchunks_ = 1;
            rows_per_chunk_ = static_cast<int32_t>(round_up(n_, 32));
        } else {
            // ~`waves` items per co-resident CTA; either a one-wave grid claiming
            // items dynamically (SNB_SWEEP_SCHED=dynamic) or one CTA per item
            // scheduled by the hardware (default)
            const int resident = dense_stream_max_ctas(f64_, stdp_on_, has_delay_);
            const char* sched = std::getenv("SNB_SWEEP_SCHED");
            const char* wv = std::getenv("SNB_SWEEP_WAVES");
            dynamic_sched_ = sched && std::string(sched) == "dynamic";
            const double waves = wv ? std::atof(wv) : 4.0;
            int nch = std::max(1, static_cast<int>(std::lround(waves * resident / ntiles)));
            int rpc = std::max(32, (n_ + nch - 1) / nch);
            // 32-aligned chunks measured 2.5% faster than unaligned ones (tools/ab_sweep.sh)
            const char* al = std::getenv("SNB_SWEEP_ALIGN");
            rpc = static_cast<int>(round_up(rpc, al ? std::max(1, std::atoi(al)) : 32));
            if (const char* r = std::getenv("SNB_SWEEP_RPC")) rpc = std::atoi(r);
            nch = (n_ + rpc - 1) / rpc;
            rows_per_chunk_ = rpc;
            nchunks_ = nch;
            dense_grid_ = dynamic_sched_ ? std::min(ntiles * nchunks_, resident) : ntiles * nchunks_;
            // TMA-staged variant (fp32, unit delays): one CTA per SM claiming items
            const char* dk = std::getenv("SNB_DENSE_KERNEL");
            // default (tools/ab_tma.sh, cfg3: 1.284 ms vs 1.425 ms for k_dense_stream)
            // fp64 weights: 2.601 ms vs 2.990 ms (k_dense_stream) on a 32k fp64 STDP net; delays
            // 1-4 with STDP (delay bytes in the stages, pot^(d) staged per row): 1.746 vs 2.095 ms
            tma_ = !(dk && std::string(dk) == "stream");
            if (tma_ && has_delay_ && stdp_on_ && dp_ > dense_tma_max_dp()) tma_ = false;
            if (tma_ && has_delay_) {  // the delay bytes are bulk-copied: 16-byte multiples
                tile_w_ = static_cast<int32_t>(round_up(tile_w_, 16));
                ntiles = std::max(1, (nl_ + tile_w_ - 1) / tile_w_);
            }
            const int tma_rows = tma_ ? dense_tma_max_rows(tile_w_, f64_, has_delay_, stdp_on_) : 0;
            if (tma_rows < 64) tma_ = false;
            if (tma_) {
                const char* tw = std::getenv("SNB_TMA_WAVES");
                // items per SM per step: with the planner warp building the next
                // item's list in the background, finer items only shorten the
                // step's tail (cfg3 sweep: 14 -> 1.288 ms, 30 -> 1.271, 60 -> 1.270
                // but more partials for the neuron phase; fp64 32k 2.606 -> 2.538)
                const double tw_waves = tw ? std::atof(tw) : 30.0;
                int tn = std::max(1, static_cast<int>(std::lround(tw_waves * sms / ntiles)));
                int trpc = static_cast<int>(round_up(std::max(32, (n_ + tn - 1) / tn), 32));
                trpc = std::min(trpc, tma_rows);
                rows_per_chunk_ = trpc;
                nchunks_ = (n_ + trpc - 1) / trpc;
                dense_grid_ = std::min(sms, ntiles * nchunks_);
            }
        }
        const int items = ntiles * nchunks_;
        if (exact_) dense_grid_ = std::min(items, sms * 8);
        d_partial_.alloc(static_cast<size_t>(nchunks_) * std::max(nl_, 1) * 8);
        cuda_check(cudaMemsetAsync(d_partial_.p, 0, d_partial_.bytes, stream_), "memset");
    } else {
        const double avg = nl_ > 0 ? static_cast<double>(sparse_elems_) / (static_cast<double>(nblocks_) * nl_) : 0.0;
        sub_ = avg >= 256 ? 32 : avg >= 96 ? 16 : avg >= 40 ? 8 : 4;
        // dictionary lists are half as long in bytes; more posts per warp hide
        // more latency (cfg4, 160 entries/list: SUB 16 0.720 ms, 8 0.682, 4 0.652)
        if (!dict_.empty()) sub_ = avg >= 1024 ? 16 : avg >= 384 ? 8 : 4;
        // plastic lists with staged traces, ~30 synapses per (post, block): 2 lanes
        // x 4 chunks per post, 16 posts per warp in flight (sstdp1 0.376 vs 0.379 ms,
        // sstdp8 0.527 vs 0.550 at SUB 4)
        if (stdp_on_ && pot_staged_ && dict_.empty() && !exact_ && avg < 40) sub_ = 2;
        // one-weight lists (k_sparse_count): 8 lanes per post read whole 128-byte
        // lines (4 posts per warp-wide LDG.128); cfg4, 160 entries per list:
        // SUB 8 0.514 ms vs SUB 4 0.529 ms, 16 0.678
        if (dict_.size() == 2 && !stdp_on_) sub_ = avg >= 1024 ? 16 : avg >= 96 ? 8 : 4;
        // 16-bit segmented lists (k_sparse_count16): 4 lanes per post, 6 chunk loads each
        // (cfg4, ~180 entries per list: SUB 4 0.452 ms, 8 0.486, 2 0.568)
        if (dict_.size() == 2 && !stdp_on_ && !exact_ && hbits_ == 16 && pb_ == c16_block_pres() && c16_allowed())
            sub_ = avg >= 768 ? 8 : 4;
        if (const char* sv = std::getenv("SNB_SPARSE_SUB")) {  // A/B knob: lanes per post
            const int v = std::atoi(sv);
            if (v == 4 || v == 8 || v == 16 || v == 32 || (!dict_.empty() && v == 1) ||
                (v == 2 && (!dict_.empty() || (stdp_on_ && pot_staged_))))
                sub_ = v;
        }
        // default: SUB lanes per post (k_sparse_pull, 1.058 ms on cfg4); the flat
        // per-warp chunk stream (k_sparse_stream, 1.115 ms) stays selectable for
        // A/B runs with SNB_SPARSE_KERNEL=stream (tools/ab_sparse.sh)
        const char* sk = std::getenv("SNB_SPARSE_KERNEL");
        if (sk && std::string(sk) == "stream") sub_ = 0;
        // CTAs per SM the grid aims at.  16-bit count lists (cfg4): 12 at full
        // size (0.418 ms vs 0.431 at 8, 0.425 at 16; three waves of ~2,300 posts
        // per CTA), 4 for post partitions (an eighth of cfg4: 70.5 us vs 76.9 at
        // 8 -- every CTA stages a whole pre block, so fewer, fuller CTAs);
        // A/B knob SNB_SPARSE_CTAS_PER_SM (tools/ab_env.sh)
        const bool c16_plan = dict_.size() == 2 && !stdp_on_ && !exact_ && hbits_ == 16 &&
                              pb_ == c16_block_pres() && c16_allowed();
        const bool c8_plan = c16_plan && c16_bytes();  // byte image: one 1024-thread CTA per SM
        int per_sm = c8_plan ? 1 : c16_plan ? (nl_ >= 131072 ? 12 : 4) : 8;
        c16_threads_ = c16_plan ? c16_threads(nl_) : 256;
        const int warps = c16_threads_ / 32;  // per CTA
        if (c16_plan && !c8_plan) per_sm = std::max(1, per_sm * 8 / warps);  // same warps per SM for bigger CTAs
        if (const char* cp = std::getenv("SNB_SPARSE_CTAS_PER_SM")) per_sm = std::max(1, std::atoi(cp));
        const int target = sms * per_sm;
        int gx = std::max(1, target / std::max(1, nblocks_));
        const int unit = sub_ == 0 ? 8 : warps * (32 / sub_);
        posts_per_cta_ = static_cast<int32_t>(round_up((nl_ + gx - 1) / gx, unit));
        posts_per_cta_ = std::max(posts_per_cta_, unit);
        sparse_gx_ = std::max(1, (nl_ + posts_per_cta_ - 1) / posts_per_cta_);
        nchunks_ = nblocks_;
        d_partial_.alloc(static_cast<size_t>(nblocks_) * std::max(nl_, 1) * 8);
        cuda_check(cudaMemsetAsync(d_partial_.p, 0, d_partial_.bytes, stream_), "memset");
        // TMA-fed stream for static uniform-weight lists, opt-in (SNB_SPARSE_KERNEL=tma):
        // 1.27-2.7 ms on cfg4 against 0.56 ms for k_sparse_pull
        sparse_tma_ = !exact_ && !stdp_on_ && dict_.size() == 2 && nl_ > 0 && sk && std::string(sk) == "tma";
        if (sparse_tma_) sparse_tma_ = build_sparse_tma_plan(sms);
        // k_sparse_count reads lists in any order: deal them bank-aware
        const bool count_path = !exact_ && !stdp_on_ && dict_.size() == 2 && hbits_ != 64 && sub_ != 0 &&
                                !sparse_tma_ && nl_ > 0 && sparse_elems_ > 0;
        const char* bo = std::getenv("SNB_SPARSE_BANK_ORDER");  // A/B knob: 0 keeps pre order
        if (count_path && build_c16()) {
            bank_ordered_ = true;  // lists regrouped; every synapse carries dict_[0]
        } else if (count_path && !(bo && std::string(bo) == "0")) {
            size_t free_b = 0, total_b = 0;
            cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
            const size_t bytes = static_cast<size_t>(sparse_elems_) * 4;
            if (bytes + (256u << 20) < free_b) {
                DevBuf ordered;
                ordered.alloc(bytes);
                const char* bj = std::getenv("SNB_SPARSE_BANK_JOINT");  // A/B knob: 0 = per-list order
                const bool joint = !(bj && std::string(bj) == "0") &&
                                   launch_sparse_bank_joint(d_meta_.as<uint32_t>(), ordered.as<uint32_t>(),
                                                            d_off_.as<int64_t>(), nblocks_, nl_, sub_, hbits_, stream_);
                if (!joint) {
                    launch_sparse_bank_order(d_meta_.as<uint32_t>(), ordered.as<uint32_t>(), d_off_.as<int64_t>(),
                                             static_cast<int64_t>(nblocks_) * nl_, nl_, sub_, hbits_, stream_);
                    std::swap(d_meta_.p, ordered.p);
                    std::swap(d_meta_.bytes, ordered.bytes);
                }
                cuda_check(cudaStreamSynchronize(stream_), "bank order");
                bank_ordered_ = true;
            }
        }
    }
}

// One weight for every synapse (ER-generated nets, or host lists whose weights
// are all equal): the cluster loop counts delivering pres instead of summing.
bool Engine::uniform_weight(double* w0) const {
    if (generated_) {
        *w0 = f64_ ? er_.weight_d : static_cast<double>(er_.weight_f);
        return true;
    }
    if (weight_.empty()) return false;
    for (double w : weight_)
        if (w != weight_[0]) return false;
    *w0 = weight_[0];
    return true;
}

bool Engine::c16_allowed() {
    const char* e = std::getenv("SNB_SPARSE_COUNT16");  // A/B knob: 0 keeps the 32-bit lists
    return !(e && std::string(e) == "0");
}

// 16-bit segmented copy of the one-weight lists for k_sparse_count16 (layout
// in k_sparse.cu): per-segment counts on the device, chunk offsets and the
// list descriptors here, then the bank-scheduled fill.  False (the 32-bit count
// path stays) when the block layout does not match or a list needs more than
// 255 chunks of 8 entries.
bool Engine::build_c16() {
    if (!c16_allowed() || pb_ != c16_block_pres() || hbits_ != 16 || (sub_ != 2 && sub_ != 4 && sub_ != 8 && sub_ != 16))
        return false;
    const int64_t lists = static_cast<int64_t>(nblocks_) * nl_;
    DevBuf d_cnt;
    d_cnt.alloc(static_cast<size_t>(lists) * 8);
    launch_c16_count(d_meta_.as<uint32_t>(), d_off_.as<int64_t>(), lists, pb_, d_cnt.as<uint2>(), stream_);
    std::vector<uint32_t> cnt(static_cast<size_t>(lists) * 2);
    cuda_check(cudaMemcpyAsync(cnt.data(), d_cnt.p, cnt.size() * 4, cudaMemcpyDeviceToHost, stream_), "c16 counts D2H");
    cuda_check(cudaStreamSynchronize(stream_), "c16 counts");
    std::vector<uint32_t> desc(static_cast<size_t>(lists) * 2);
    uint64_t chunks = 0;
    // byte image (k_sparse_count8): the 32 / sub posts of a warp share one
    // row-major chunk stream; every descriptor carries the group's first chunk,
    // aligned to 128 bytes so the rows every post fills are 4 whole lines
    const bool grouped = c16_bytes();
    const int P = 32 / sub_;
    uint64_t group0 = 0, stored = 0;
    for (int64_t L = 0; L < lists; ++L) {
        if (grouped && (L % nl_) % P == 0) group0 = chunks = (chunks + 7) / 8 * 8;
        const uint32_t x = cnt[2 * L], y = cnt[2 * L + 1];
        const uint32_t n[4] = {x & 0xffffu, x >> 16, y & 0xffffu, y >> 16};
        uint32_t e[4], acc = 0;
        for (int s = 0; s < 4; ++s) {
            acc += (n[s] + 7) / 8;
            e[s] = acc;
        }
        if (acc > 255) return false;
        desc[2 * L] = static_cast<uint32_t>(grouped ? group0 : chunks);
        desc[2 * L + 1] = e[0] | (e[1] << 8) | (e[2] << 16) | (e[3] << 24);
        chunks += acc;
        stored += acc;
    }
    if (chunks >= (1ull << 32)) return false;
    size_t free_b = 0, total_b = 0;
    cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const size_t need = static_cast<size_t>(chunks) * 16 + static_cast<size_t>(sparse_elems_) * 4 + (256u << 20);
    if (need > free_b) return false;
    upload(stream_, d_c16desc_, desc);
    d_c16ent_.alloc(std::max<size_t>(static_cast<size_t>(chunks), 1) * 16);
    DevBuf tmp;
    tmp.alloc(std::max<size_t>(static_cast<size_t>(sparse_elems_), 1) * 4);
    if (!launch_c16_fill(d_meta_.as<uint32_t>(), tmp.as<uint32_t>(), d_off_.as<int64_t>(), d_c16desc_.as<uint2>(),
                         nblocks_, nl_, pb_, sub_, d_c16ent_.as<uint16_t>(), stream_)) {
        d_c16desc_.release();
        d_c16ent_.release();
        return false;
    }
    cuda_check(cudaStreamSynchronize(stream_), "c16 fill");
    if (const char* dump = std::getenv("SNB_C16_DUMP")) {  // debugging aid: descriptors + entries
        std::vector<uint16_t> ent(static_cast<size_t>(chunks) * 8);
        d2h(ent.data(), d_c16ent_.p, ent.size() * 2, "c16 dump");
        if (FILE* f = std::fopen(dump, "wb")) {
            const int64_t hdr[4] = {lists, static_cast<int64_t>(chunks), sub_, nl_};
            std::fwrite(hdr, 8, 4, f);
            std::fwrite(desc.data(), 4, desc.size(), f);
            std::fwrite(ent.data(), 2, ent.size(), f);
            std::fclose(f);
        }
    }
    c16_ = true;
    // bytes the sweep moves in this format: 2 B per stored entry (padding included),
    // the 8-byte descriptor and the 2-byte count of every (block, post) list
    sweep_bytes_full_ = static_cast<double>(stored) * 16.0 + static_cast<double>(lists) * 10.0;
    return true;
}

// Stage plan of k_sparse_tma: the (block, post) lists are cut into stages of
// whole posts (<= sparse_tma_stage_entries() entries, one pre block, at most
// sparse_tma_max_boundaries() posts); every CTA owns a contiguous run of
// stages inside one pre block, CTAs per block in proportion to its entries.  Returns false when
// a single list is longer than a stage (the pull kernel handles such nets).
bool Engine::build_sparse_tma_plan(int ctas) {
    const int64_t P = static_cast<int64_t>(nblocks_) * nl_;
    std::vector<int64_t> off(static_cast<size_t>(P) + 1);
    d2h(off.data(), d_off_.p, off.size() * 8, "offsets D2H");
    const int64_t Q = off[P];
    const int64_t E = sparse_tma_stage_entries();
    const int NB = sparse_tma_max_boundaries();
    for (int64_t k = 0; k < P; ++k)
        if (off[k + 1] - off[k] > E) return false;
    // CTAs per pre block in proportion to its entries (one block per CTA, so a
    // single history image), each block's posts split evenly by entries
    std::vector<std::pair<int64_t, int64_t>> ranges;
    {
        std::vector<int> per(static_cast<size_t>(nblocks_), 0);
        std::vector<double> want(static_cast<size_t>(nblocks_), 0.0);
        int given = 0;
        for (int b = 0; b < nblocks_; ++b) {
            const int64_t eb = off[static_cast<int64_t>(b + 1) * nl_] - off[static_cast<int64_t>(b) * nl_];
            want[b] = Q > 0 ? static_cast<double>(ctas) * static_cast<double>(eb) / static_cast<double>(Q) : 0.0;
            per[b] = eb > 0 ? std::max(1, static_cast<int>(want[b])) : 0;
            given += per[b];
        }
        while (given < ctas) {  // largest remainders first
            int best = -1;
            double gap = 0.0;
            for (int b = 0; b < nblocks_; ++b)
                if (per[b] > 0 && want[b] - per[b] > gap) { gap = want[b] - per[b]; best = b; }
            if (best < 0) break;
            ++per[best];
            ++given;
        }
        for (int b = 0; b < nblocks_; ++b) {
            const int64_t p0 = static_cast<int64_t>(b) * nl_, p1 = p0 + nl_;
            const int64_t q0 = off[p0], eb = off[p1] - q0;
            int64_t lo = p0;
            for (int c = 1; c <= per[b]; ++c) {
                int64_t hi = p1;
                if (c < per[b]) {
                    const int64_t target = q0 + eb * c / per[b];
                    hi = std::lower_bound(off.begin() + p0, off.begin() + p1, target) - off.begin();
                    hi = std::max(hi, lo);
                }
                if (hi > lo) ranges.emplace_back(lo, hi);
                lo = hi;
            }
        }
    }
    std::vector<SpStage> stages;
    std::vector<uint16_t> bnd;
    std::vector<int32_t> first, cblock;
    stages.reserve(static_cast<size_t>(Q / (E / 2) + ranges.size() + 16));
    bnd.reserve(static_cast<size_t>(P + 8 * (Q / (E / 2) + ranges.size())));
    for (const auto& [lo, hi] : ranges) {
        first.push_back(static_cast<int32_t>(stages.size()));
        cblock.push_back(static_cast<int32_t>(lo / nl_));
        for (int64_t k = lo; k < hi;) {
            const int64_t b = k / nl_;
            const int64_t q = off[k];
            int64_t j = k;
            while (j < hi && j / nl_ == b && off[j + 1] - q <= E && j - k < NB) ++j;
            SpStage st{};
            st.q = q;
            st.entries = static_cast<int32_t>(off[j] - q);
            st.k0 = static_cast<int32_t>(k + 1);
            st.nb = static_cast<int32_t>(j - k);
            st.block = static_cast<int32_t>(b);
            st.bnd_off = static_cast<int64_t>(bnd.size());
            for (int64_t i = k + 1; i <= j; ++i) bnd.push_back(static_cast<uint16_t>(off[i] - q));
            while (bnd.size() % 8) bnd.push_back(0);
            stages.push_back(st);
            k = j;
        }
    }
    first.push_back(static_cast<int32_t>(stages.size()));
    if (bnd.empty()) bnd.assign(8, 0);
    if (stages.empty()) stages.resize(1);
    upload(stream_, d_sp_stages_, stages);
    upload(stream_, d_sp_first_, first);
    upload(stream_, d_sp_block_, cblock);
    upload(stream_, d_sp_bnd_, bnd);
    sp_ctas_ = static_cast<int32_t>(cblock.size());
    return sp_ctas_ > 0;
}

}  // namespace snb
