// Host side of the B200 MAT engine, part 1: buffers, model building,
// validation with the reference's messages, sn_setup and the device state.
// (Layouts: engine_layout.cpp; step sequence: engine_run.cpp; multi-GPU
// exchange: engine_comm.cpp; results: engine_results.cpp.)
//
// Reference anchors:
//   validate_network / validate_stimulus / validate_stdp   proj/src/model.cpp:34-117
//   mat_init (SoA fill, weight build, stdp list)           proj/src/mat_engine.cpp:109-166
//   mat_run loop (stimulus, step, stdp, raster)            proj/src/mat_engine.cpp:252-287
#include "engine.hpp"

#include "engine_util.hpp"
#include "nccl_dl.hpp"

#include <algorithm>
#include <limits>
#include <cmath>
#include <cstring>
#include <numeric>
#include <sstream>
#include <thread>
#include <cstdlib>
#include <unordered_map>
#include <unordered_set>

namespace snb {

void cuda_check(cudaError_t err, const char* what) {
    if (err == cudaSuccess) return;
    if (err == cudaErrorMemoryAllocation)
        throw OutOfMemory(std::string("out of device memory in ") + what);
    throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(err));
}

void Engine::d2h(void* dst, const void* src, size_t bytes, const char* what) const {
    cuda_check(cudaStreamSynchronize(stream_), what);
    cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), what);
}

void DevBuf::alloc(size_t b) {
    release();
    if (b == 0) b = 16;
    cuda_check(cudaMalloc(&p, b), "cudaMalloc");
    bytes = b;
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}
void HostBuf::reserve(size_t b) {
    if (b <= bytes) return;
    release();
    b = std::max(b, 2 * bytes);  // geometric growth: pinned allocation is slow and synchronising
    cuda_check(cudaMallocHost(&p, b), "cudaMallocHost");
    bytes = b;
}
void HostBuf::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
}


// ---------------------------------------------------------------------------
Engine::Engine(const sn_options& opt) : opt_(opt) {
    if (opt_.world < 1) throw InvalidArgument("sn_engine_create: world must be >= 1");
    if (opt_.rank < 0 || opt_.rank >= opt_.world) throw InvalidArgument("sn_engine_create: rank out of range");
    if (opt_.storage < 0 || opt_.storage > 2) throw InvalidArgument("sn_engine_create: unknown storage");
    if (opt_.mode != SN_MODE_MAT && opt_.mode != SN_MODE_ABM) throw InvalidArgument("sn_engine_create: unknown mode");
    int count = 0;
    cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (opt_.device < 0 || opt_.device >= count)
        throw InvalidArgument("sn_engine_create: CUDA device " + std::to_string(opt_.device) +
                              " not present (" + std::to_string(count) + " visible)");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    f64_ = opt_.precision == SN_WEIGHTS_F64;
    exact_ = opt_.exact_order != 0;
    abm_ = opt_.mode == SN_MODE_ABM;
}

Engine::~Engine() {
    cudaSetDevice(opt_.device);
    if (stream_) cudaStreamSynchronize(stream_);
    delete comm_;
    for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    for (auto e : ev_pool_) cudaEventDestroy(e);
    for (auto& p : pending_) {
        (void)p;
    }
    if (stream_) cudaStreamDestroy(stream_);
}

// ---- agent-based mode ----------------------------------------------------------
// SimulationConfig::seed (model.hpp:80-85): keys the per-(agent, step) streams
// of the stochastic behaviours (abm_engine.cpp:163-164).
void Engine::set_seed(uint64_t seed) {
    require_not_setup("sn_set_seed");
    seed_ = seed;
}

// Behaviour of neurons [first, first + count) as the fire probability of
// StochasticLifBehavior (abm_engine.cpp:28-39); 1 = "lif".
void Engine::set_fire_probability(int64_t first, int64_t count, const double* p) {
    require_not_setup("sn_set_fire_probability");
    const int64_t n = static_cast<int64_t>(thr_.size());
    if (count < 0 || first < 0 || first + count > n)
        throw InvalidArgument("sn_set_fire_probability: neuron range [" + std::to_string(first) + ", " +
                              std::to_string(first + count) + ") outside the " + std::to_string(n) +
                              " neurons added");
    if (count > 0 && !p) throw InvalidArgument("sn_set_fire_probability: null array");
    for (int64_t i = 0; i < count; ++i)
        if (!(p[i] >= 0.0 && p[i] <= 1.0))  // abm_engine.cpp:30-32
            throw InvalidArgument("stochastic lif: fire probability must be in [0, 1]");
    if (fire_p_.size() < static_cast<size_t>(n)) fire_p_.resize(static_cast<size_t>(n), 1.0);
    std::copy(p, p + count, fire_p_.begin() + first);
}

uint64_t Engine::agent_stream_key(uint64_t seed, uint64_t agent) {
    // RandomStream(seed, 0x61626d2d6167656e, agent, step) keys (rng.hpp:19-24,
    // abm_engine.cpp:12); the final mix with the step happens on the device
    uint64_t k = host_mix64(seed + 0x9e3779b97f4a7c15ULL);
    k = host_mix64(k ^ 0x61626d2d6167656eULL);
    return host_mix64(k ^ agent);
}

void Engine::require_not_setup(const char* what) const {
    if (setup_done_) throw LogicError(std::string(what) + ": the network is fixed after sn_setup");
}
void Engine::require_setup(const char* what) const {
    if (!setup_done_) throw LogicError(std::string(what) + ": call sn_setup first");
}

void Engine::partition(int32_t n, int32_t rank, int32_t world, int32_t* first, int32_t* count) {
    // contiguous post ranges, each a multiple of 32 ids so spike words never straddle ranks
    const int64_t words = (static_cast<int64_t>(n) + 31) / 32;
    const int64_t per = (words + world - 1) / world * 32;
    const int64_t f = per * rank;
    const int64_t c = std::max<int64_t>(0, std::min<int64_t>(n - f, per));
    *first = static_cast<int32_t>(std::min<int64_t>(f, n));
    *count = static_cast<int32_t>(c);
}

// ---- model building --------------------------------------------------------
void Engine::add_neurons(int64_t count, const double* thr, const double* leak, const double* reset,
                         const int32_t* refr, const int32_t* axonal, int64_t* first_id) {
    require_not_setup("sn_add_neurons");
    if (count < 0) throw InvalidArgument("sn_add_neurons: count must be >= 0");
    if (count > 0 && (!thr || !leak || !reset || !refr))
        throw InvalidArgument("sn_add_neurons: null parameter array");
    if (generated_) throw LogicError("sn_add_neurons: network was generated with sn_generate_erdos_renyi");
    if (first_id) *first_id = static_cast<int64_t>(thr_.size());
    if (static_cast<int64_t>(thr_.size()) + count > INT32_MAX)
        throw InvalidArgument("sn_add_neurons: neuron ids must fit int32");
    thr_.insert(thr_.end(), thr, thr + count);
    leak_.insert(leak_.end(), leak, leak + count);
    reset_.insert(reset_.end(), reset, reset + count);
    refr_.insert(refr_.end(), refr, refr + count);
    if (axonal) axonal_.insert(axonal_.end(), axonal, axonal + count);
    else axonal_.insert(axonal_.end(), static_cast<size_t>(count), 0);
}

void Engine::add_synapses(int64_t count, const int32_t* pre, const int32_t* post, const double* w,
                          const int32_t* delay, const uint8_t* stdp) {
    require_not_setup("sn_add_synapses");
    if (count < 0) throw InvalidArgument("sn_add_synapses: count must be >= 0");
    if (count > 0 && (!pre || !post || !w)) throw InvalidArgument("sn_add_synapses: null parameter array");
    if (generated_) throw LogicError("sn_add_synapses: network was generated with sn_generate_erdos_renyi");
    pre_.insert(pre_.end(), pre, pre + count);
    post_.insert(post_.end(), post, post + count);
    weight_.insert(weight_.end(), w, w + count);
    if (delay) delay_.insert(delay_.end(), delay, delay + count);
    else delay_.insert(delay_.end(), static_cast<size_t>(count), 1);
    if (stdp) plastic_.insert(plastic_.end(), stdp, stdp + count);
    else plastic_.insert(plastic_.end(), static_cast<size_t>(count), 0);
}

void Engine::add_stimulus(int64_t count, const int32_t* step, const int32_t* neuron, const double* amp) {
    if (count < 0) throw InvalidArgument("sn_add_stimulus: count must be >= 0");
    if (count > 0 && (!step || !neuron || !amp)) throw InvalidArgument("sn_add_stimulus: null parameter array");
    const size_t base = st_step_.size();
    for (int64_t i = 0; i < count; ++i) {
        const std::string who = "stimulus[" + std::to_string(base + i) + "]";
        if (step[i] < 0)
            throw InvalidArgument(run_name() + ": " + who + ": step " + std::to_string(step[i]) + " is negative");
        if (!std::isfinite(amp[i])) throw InvalidArgument(run_name() + ": " + who + ": amplitude must be finite");
        if (setup_done_ && (neuron[i] < 0 || neuron[i] >= n_user_))
            throw InvalidArgument(run_name() + ": " + who + ": neuron id " + std::to_string(neuron[i]) +
                                  " out of range (" + std::to_string(n_user_) + " neurons)");
    }
    st_step_.insert(st_step_.end(), step, step + count);
    st_neuron_.insert(st_neuron_.end(), neuron, neuron + count);
    st_amp_.insert(st_amp_.end(), amp, amp + count);
    stim_dirty_ = true;
}

void Engine::clear_stimulus() {
    st_step_.clear();
    st_neuron_.clear();
    st_amp_.clear();
    stim_dirty_ = true;
}

void Engine::set_stdp(int32_t window, const double* ap, const double* am, double wmin, double wmax) {
    require_not_setup("sn_set_stdp");
    std::vector<std::string> bad;  // validate_stdp (model.cpp:104-117)
    if (window < 1) bad.push_back("stdp: window must be >= 1");
    if (window >= 1 && (!ap || !am)) throw InvalidArgument("sn_set_stdp: null kernel array");
    if (window >= 1) {
        for (int k = 0; k < window; ++k)
            if (!(ap[k] >= 0.0)) { bad.push_back("stdp: a_plus entries must be >= 0"); break; }
        for (int k = 0; k < window; ++k)
            if (!(am[k] >= 0.0)) { bad.push_back("stdp: a_minus entries must be >= 0"); break; }
    }
    if (!(wmin <= wmax)) bad.push_back("stdp: w_min must be <= w_max");
    throw_first("mat_init", bad);
    stdp_on_ = true;
    window_ = window;
    a_plus_.assign(ap, ap + window);
    a_minus_.assign(am, am + window);
    w_min_ = wmin;
    w_max_ = wmax;
}

void Engine::generate_er(int32_t n, double p, uint64_t seed, double weight, int32_t delay_max,
                         uint64_t delay_stream, int32_t by_syn, int32_t stdp) {
    require_not_setup("sn_generate_erdos_renyi");
    if (n < 1) throw InvalidArgument("erdos_renyi: n must be >= 1");           // netgen.cpp:20
    if (!(p >= 0.0 && p <= 1.0)) throw InvalidArgument("erdos_renyi: p must be in [0, 1]");
    if (!std::isfinite(weight)) throw InvalidArgument("erdos_renyi: weight must be finite");
    if (delay_max < 1) throw InvalidArgument("erdos_renyi: delay_max must be >= 1");
    if (by_syn && delay_max > 1 && p < 1.0)
        throw InvalidArgument("erdos_renyi: synapse-index keyed delays need p == 1");
    if (!pre_.empty()) throw LogicError("sn_generate_erdos_renyi: synapses were already added");
    generated_ = true;
    thr_.assign(n, 1.0);
    leak_.assign(n, 0.0);
    reset_.assign(n, 0.0);
    refr_.assign(n, 0);
    axonal_.assign(n, 0);
    er_.n = n;
    er_.p = p;
    er_.edge_key = stream_key(seed, 1);  // kEdgeStream (netgen.cpp:15)
    er_.delay_key = stream_key(seed, delay_stream);
    er_.delay_max = delay_max;
    er_.delay_by_synapse_index = by_syn;
    er_.weight_f = static_cast<float>(weight);
    er_.weight_d = weight;
    er_.stdp = stdp ? 1 : 0;
    er_delay_max_ = delay_max;
    if (n <= kTinyMaxNeurons) materialize_er();
}

// Small generated nets become ordinary synapse lists (host draws identical to
// the device generator and to netgen.cpp:36-51), so every list-based path --
// including the shared-memory step loop -- applies to them.
void Engine::materialize_er() {
    const int n = er_.n;
    auto u64_at = [](uint64_t key, uint64_t idx) { return host_mix64(key + idx * 0x9e3779b97f4a7c15ULL); };
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (i == j || !(er_.p > 0.0)) continue;
            const uint64_t pair = static_cast<uint64_t>(i) * static_cast<uint64_t>(n) + static_cast<uint64_t>(j);
            if (er_.p < 1.0 && static_cast<double>(u64_at(er_.edge_key, pair) >> 11) * 0x1.0p-53 >= er_.p) continue;
            int d = 1;
            if (er_.delay_max > 1) {
                const uint64_t key = er_.delay_by_synapse_index
                                         ? static_cast<uint64_t>(i) * static_cast<uint64_t>(n - 1) +
                                               static_cast<uint64_t>(j - (j > i ? 1 : 0))
                                         : pair;
                const unsigned __int128 prod = static_cast<unsigned __int128>(u64_at(er_.delay_key, key)) *
                                               static_cast<unsigned __int128>(er_.delay_max);
                d = 1 + static_cast<int>(static_cast<uint64_t>(prod >> 64));
            }
            pre_.push_back(i);
            post_.push_back(j);
            weight_.push_back(er_.weight_d);
            delay_.push_back(d);
            plastic_.push_back(static_cast<uint8_t>(er_.stdp));
        }
    generated_ = false;
}

void Engine::validate() const {
    std::vector<std::string> out;  // validate_network (model.cpp:34-84)
    const int n = static_cast<int>(thr_.size());
    for (int i = 0; i < n; ++i) {
        const std::string who = "neurons[" + std::to_string(i) + "]";
        if (!std::isfinite(thr_[i])) out.push_back(who + ": threshold must be finite");
        if (std::isnan(leak_[i]) || leak_[i] < 0.0)
            out.push_back(who + ": leak must be >= 0 or infinite (got " + fmt_double(leak_[i]) + ")");
        if (!std::isfinite(reset_[i])) out.push_back(who + ": reset must be finite");
        if (refr_[i] < 0)
            out.push_back(who + ": refractory_period must be >= 0 (got " + std::to_string(refr_[i]) + ")");
        if (axonal_[i] < 0)
            out.push_back(who + ": axonal_delay must be >= 0 (got " + std::to_string(axonal_[i]) + ")");
    }
    if (!generated_) {
        std::unordered_set<uint64_t> seen;
        seen.reserve(pre_.size());
        for (size_t s = 0; s < pre_.size(); ++s) {
            const std::string who = "synapses[" + std::to_string(s) + "]";
            const bool pre_ok = pre_[s] >= 0 && pre_[s] < n;
            const bool post_ok = post_[s] >= 0 && post_[s] < n;
            if (!pre_ok)
                out.push_back(who + ": pre id " + std::to_string(pre_[s]) + " out of range (" +
                              std::to_string(n) + " neurons)");
            if (!post_ok)
                out.push_back(who + ": post id " + std::to_string(post_[s]) + " out of range (" +
                              std::to_string(n) + " neurons)");
            if (!std::isfinite(weight_[s])) out.push_back(who + ": weight must be finite");
            if (delay_[s] < 1) out.push_back(who + ": delay must be >= 1 (got " + std::to_string(delay_[s]) + ")");
            if (pre_ok && post_ok) {
                const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(pre_[s])) << 32) |
                                     static_cast<uint32_t>(post_[s]);
                if (!seen.insert(key).second)
                    out.push_back(who + ": duplicate synapse (" + std::to_string(pre_[s]) + ", " +
                                  std::to_string(post_[s]) + ")");
            }
        }
    }
    if (abm_) {  // AbmWorld reports the first violation only (abm_engine.cpp:14-17, 79)
        if (!out.empty()) throw InvalidArgument("abm world: " + out.front());
    } else {
        throw_first("mat_init", out);
    }
    if (!abm_)
        for (size_t i = 0; i < fire_p_.size(); ++i)
            if (fire_p_[i] != 1.0)
                throw InvalidArgument("mat_init: homogeneous backend supports \"lif\" only; neuron " +
                                      std::to_string(i) + " has a stochastic behavior (fire probability " +
                                      fmt_double(fire_p_[i]) + ")");
    if (abm_ && stdp_on_) throw LogicError("abm world: the agent-based engine has no plasticity");
    for (size_t i = 0; i < st_neuron_.size(); ++i)
        if (st_neuron_[i] < 0 || st_neuron_[i] >= n)
            throw InvalidArgument(run_name() + ": stimulus[" + std::to_string(i) + "]: neuron id " +
                                  std::to_string(st_neuron_[i]) + " out of range (" + std::to_string(n) +
                                  " neurons)");
}

// ---- delay relays ---------------------------------------------------------------
// The sweeps read one 64-bit history word per pre, so effective delays (delay
// + axonal of the pre) up to 64 are native.  A longer synapse i -> j (d > 64;
// the reference accepts any delay, lowering.cpp:39-57) is rerouted through a
// chain of relay neurons of i: relay k fires exactly 64 k steps after i
// (threshold 0, infinite leak, reset 0, no refractory period, one weight-1
// input: u = 1 > 0 iff its upstream spiked 64 steps earlier), and the synapse
// leaves relay q = (d - 1) / 64 with delay d - 64 q in [1, 64].  Arrival times
// are unchanged, and so is STDP: the engine pairs the pre train shifted by
// d' - 1 through a synapse of delay d' (the lowered net's last proxy), and
// relay q's train shifted by d - 64 q - 1 is i's train shifted by d - 1.
// Relays live after the caller's neurons; their hops are appended after the
// caller's synapses, which keep their list order.  Single partition only.
void Engine::add_delay_relays() {
    const int n = static_cast<int>(thr_.size());
    const size_t m = pre_.size();
    std::vector<int32_t> chain(static_cast<size_t>(n), 0);
    bool any = false;
    for (size_t s = 0; s < m; ++s) {
        const int64_t d = static_cast<int64_t>(delay_[s]) + axonal_[pre_[s]];
        if (d <= kMaxNativeDelay) continue;
        if (axonal_[pre_[s]] >= kMaxNativeDelay)
            throw Unsupported("mat_init: neurons[" + std::to_string(pre_[s]) + "] has axonal_delay " +
                              std::to_string(axonal_[pre_[s]]) + "; axonal delays of 64 steps or more are unsupported");
        chain[pre_[s]] = std::max<int32_t>(chain[pre_[s]], static_cast<int32_t>((d - 1) / kMaxNativeDelay));
        any = true;
    }
    if (!any) return;
    if (opt_.world > 1)
        throw Unsupported("mat_init: delays over 64 steps are supported on single-partition engines only");
    pre_user_ = pre_;
    std::vector<int64_t> first_relay(static_cast<size_t>(n), -1);
    for (int i = 0; i < n; ++i) {
        if (!chain[i]) continue;
        first_relay[i] = static_cast<int64_t>(thr_.size());
        for (int k = 1; k <= chain[i]; ++k) {
            const int32_t r = static_cast<int32_t>(thr_.size());
            thr_.push_back(0.0);
            leak_.push_back(std::numeric_limits<double>::infinity());
            reset_.push_back(0.0);
            refr_.push_back(0);
            axonal_.push_back(0);
            if (!fire_p_.empty()) fire_p_.push_back(1.0);
            // hop into relay k: from i (its axonal delay counts) or from relay k - 1
            pre_.push_back(k == 1 ? i : r - 1);
            post_.push_back(r);
            weight_.push_back(1.0);
            delay_.push_back(k == 1 ? kMaxNativeDelay - axonal_[i] : kMaxNativeDelay);
            plastic_.push_back(0);
        }
    }
    if (thr_.size() > static_cast<size_t>(INT32_MAX)) throw InvalidArgument("mat_init: too many neurons with delay relays");
    for (size_t s = 0; s < m; ++s) {
        const int64_t d = static_cast<int64_t>(delay_[s]) + axonal_[pre_[s]];
        if (d <= kMaxNativeDelay) continue;
        const int64_t q = (d - 1) / kMaxNativeDelay;
        delay_[s] = static_cast<int32_t>(d - q * kMaxNativeDelay);
        pre_[s] = static_cast<int32_t>(first_relay[pre_[s]] + q - 1);
    }
    relays_ = true;
}

// Clears the relay neurons' bits of every raster row not yet stripped (ids
// >= n_user_; single partition, so local ids are global ids).
void Engine::strip_relays() {
    if (!relays_) return;
    for (RasterChunk& ch : raster_) {
        if (ch.stripped) continue;
        for (int r = 0; r < ch.rows; ++r) {
            uint32_t* row = ch.words.data() + static_cast<size_t>(r) * nl_words_;
            for (int w = n_user_ >> 5; w < nl_words_; ++w) {
                const int lo = n_user_ - w * 32;  // bits below lo are user neurons
                const uint32_t keep = lo >= 32 ? ~0u : lo <= 0 ? 0u : ((1u << lo) - 1u);
                relay_spikes_ += __builtin_popcount(row[w] & ~keep);
                row[w] &= keep;
            }
        }
        ch.stripped = true;
    }
}

// ---- setup -------------------------------------------------------------------
void Engine::setup() {
    NvtxRange nv("sn_setup");
    require_not_setup("sn_setup");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    validate();
    n_user_ = static_cast<int32_t>(thr_.size());
    if (thr_.empty()) {
        // mat_init / AbmWorld accept an empty network (mat_engine.cpp:109-166 has no
        // minimum size): every step is empty; no device state is needed
        n_ = nl_ = nl_words_ = 0;
        m_user_ = 0;
        setup_done_ = true;
        stats_.n_local = 0;
        return;
    }
    m_user_ = static_cast<int64_t>(pre_.size());
    if (!generated_) add_delay_relays();
    n_ = static_cast<int32_t>(thr_.size());
    if (!fire_p_.empty()) fire_p_.resize(static_cast<size_t>(n_), 1.0);
    any_stochastic_ = abm_ && std::any_of(fire_p_.begin(), fire_p_.end(), [](double p) { return p < 1.0; });
    partition(n_, opt_.rank, opt_.world, &first_, &nl_);
    {
        int32_t f0, c0;
        partition(n_, 0, opt_.world, &f0, &c0);
        part_ = static_cast<int32_t>(round_up(std::max(c0, 1), 32));  // words_ covers the whole bitmask
    }
    nl_words_ = (nl_ + 31) / 32;
    words_ = opt_.world * (part_ / 32);

    // effective delays (delay + axonal of the pre), spans
    dmax_ = 1;
    dp_ = 1;
    if (generated_) {
        dmax_ = er_delay_max_;
        if (er_.stdp) dp_ = er_delay_max_;
    } else {
        for (size_t s = 0; s < pre_.size(); ++s) {
            const int64_t d = static_cast<int64_t>(delay_[s]) + axonal_[pre_[s]];  // <= 64 after the relays
            dmax_ = std::max<int32_t>(dmax_, static_cast<int32_t>(d));
            if (stdp_on_ && plastic_[s]) dp_ = std::max<int32_t>(dp_, static_cast<int32_t>(d));
        }
    }
    has_delay_ = dmax_ > 1;
    hw_ = stdp_on_ ? static_cast<int32_t>((window_ + dp_ + 63) / 64) : 1;
    hw_ = std::max(hw_, 1);
    hbits_ = dmax_ == 1 ? 1 : dmax_ <= 16 ? 16 : dmax_ <= 32 ? 32 : 64;

    // storage choice (mat_engine.cpp:27-30 switches at n > 12000; here the
    // choice follows bytes per step instead)
    const int64_t m = generated_ ? -1 : static_cast<int64_t>(pre_.size());
    double density;
    if (generated_) density = er_.p;
    else density = n_ > 0 ? static_cast<double>(m) / (static_cast<double>(n_) * n_) : 0.0;
    const size_t esz = f64_ ? 8 : 4;
    const double dense_bytes = static_cast<double>(n_) * round_up(std::max(nl_, 1), 32) * esz;
    size_t free_b = 0, total_b = 0;
    cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    if (opt_.storage == SN_STORAGE_DENSE) dense_ = true;
    else if (opt_.storage == SN_STORAGE_SPARSE) dense_ = false;
    else dense_ = (density >= 0.1 || n_ <= 4096) && dense_bytes < 0.85 * static_cast<double>(free_b);

    tiny_ = !generated_ && opt_.world == 1 && opt_.persistent >= 0 && opt_.storage == SN_STORAGE_AUTO &&
            n_ <= kTinyMaxNeurons && build_tiny();
    if (tiny_) {
        dense_ = false;  // the shared-memory step loop owns the weights; no dense/sparse copy
    } else if (generated_) {
        build_generated();
    } else if (dense_) {
        build_dense_from_lists();
    } else {
        build_sparse_from_lists();
    }

    alloc_state();
    stim_dirty_ = true;
    build_stimulus_table();
    if (!tiny_) plan_launches();
    if (c16_) {  // folded-history buffers of partitioned runs (fold_hist())
        d_hist16_.alloc(static_cast<size_t>(2) * n_ * 2);
        cuda_check(cudaMemsetAsync(d_hist16_.p, 0, d_hist16_.bytes, stream_), "memset");
        d_step_copy_.alloc(8);
        cuda_check(cudaMemsetAsync(d_step_copy_.p, 0, 8, stream_), "memset");
    }
    if (opt_.stream_io) {  // pinned staging sized up front (1024 steps of spike words)
        h_raster_.reserve(static_cast<size_t>(1024) * std::max(nl_words_, 1) * 4);
        h_stage_.reserve(64 * 1024);
    }
    cuda_check(cudaStreamSynchronize(stream_), "setup sync");
    setup_done_ = true;
    stats_.synapses_local = syn_local_;
    stats_.dense = dense_ ? 1 : 0;
    stats_.n_local = relays_ ? n_user_ : nl_;
    stats_.first_local = first_;
    stats_.max_delay = dmax_;
}

void Engine::alloc_state() {
    std::vector<double> v(reset_.begin() + first_, reset_.begin() + first_ + nl_);
    upload(stream_, d_v_, v);  // membrane = reset (mat_engine.cpp:143)
    upload(stream_, d_thr_, std::vector<double>(thr_.begin() + first_, thr_.begin() + first_ + nl_));
    upload(stream_, d_leak_, std::vector<double>(leak_.begin() + first_, leak_.begin() + first_ + nl_));
    upload(stream_, d_reset_, std::vector<double>(reset_.begin() + first_, reset_.begin() + first_ + nl_));
    upload(stream_, d_refr_, std::vector<int32_t>(refr_.begin() + first_, refr_.begin() + first_ + nl_));
    d_cnt_.alloc(static_cast<size_t>(std::max(nl_, 1)) * 4);
    cuda_check(cudaMemsetAsync(d_cnt_.p, 0, d_cnt_.bytes, stream_), "memset");
    const size_t wbytes = static_cast<size_t>(std::max(words_, (n_ + 31) / 32)) * 4;
    d_bits_.alloc(wbytes);
    d_active_.alloc(wbytes);
    cuda_check(cudaMemsetAsync(d_bits_.p, 0, wbytes, stream_), "memset");
    cuda_check(cudaMemsetAsync(d_active_.p, 0, wbytes, stream_), "memset");
    if (opt_.world > 1) {  // p2p exchange buffers: step t lands in buffer t & 1
        d_xbits_.alloc(2 * wbytes);
        cuda_check(cudaMemsetAsync(d_xbits_.p, 0, 2 * wbytes, stream_), "memset");
    }
    d_hist_.alloc(static_cast<size_t>(hw_) * n_ * 8);
    cuda_check(cudaMemsetAsync(d_hist_.p, 0, d_hist_.bytes, stream_), "memset");
    d_hist_lo_.alloc(static_cast<size_t>(n_) * 4);
    cuda_check(cudaMemsetAsync(d_hist_lo_.p, 0, d_hist_lo_.bytes, stream_), "memset");
    const size_t np = static_cast<size_t>(n_) * (stdp_on_ ? dp_ : 1);
    d_pot64_.alloc(np * 8);
    d_dep64_.alloc(static_cast<size_t>(n_) * 8);
    for (DevBuf* b : {&d_pot64_, &d_dep64_})
        cuda_check(cudaMemsetAsync(b->p, 0, b->bytes, stream_), "memset");
    if (stdp_on_) {
        upload(stream_, d_ap_, a_plus_);
        upload(stream_, d_am_, a_minus_);
    } else {
        d_ap_.alloc(8);
        d_am_.alloc(8);
    }
    d_step_.alloc(8);
    d_work_.alloc(8);
    d_flags_.alloc(static_cast<size_t>(opt_.world) * 4);
    d_done_.alloc(8);
    d_err_.alloc(8);
    for (DevBuf* b : {&d_flags_, &d_done_, &d_err_})
        cuda_check(cudaMemsetAsync(b->p, 0, b->bytes, stream_), "memset");
    cuda_check(cudaMemsetAsync(d_work_.p, 0, 8, stream_), "memset");
    d_spikes_.alloc(16);
    cuda_check(cudaMemsetAsync(d_step_.p, 0, 8, stream_), "memset");
    cuda_check(cudaMemsetAsync(d_spikes_.p, 0, 16, stream_), "memset");
    d_uexact_.alloc(static_cast<size_t>(std::max(nl_, 1)) * 8);
    launch_prologue(d_uexact_.as<double>(), d_v_.as<double>(), d_leak_.as<double>(), d_reset_.as<double>(), nl_, abm_,
                    stream_);
    if (any_stochastic_) {  // per-neuron fire probabilities and agent stream keys of this partition
        std::vector<double> fp(fire_p_.begin() + first_, fire_p_.begin() + first_ + nl_);
        std::vector<uint64_t> key(static_cast<size_t>(nl_));
        for (int j = 0; j < nl_; ++j) key[j] = agent_stream_key(seed_, static_cast<uint64_t>(first_ + j));
        upload(stream_, d_firep_, fp);
        upload(stream_, d_akey_, key);
    }
}

void Engine::build_stimulus_table() {
    if (!stim_dirty_) return;
    // stable by step; per step sum amplitudes per neuron in list order from 0.0
    // (mat_engine.cpp:258-275), keep local neurons, neuron ascending
    std::vector<size_t> ord(st_step_.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return st_step_[a] < st_step_[b]; });
    int32_t steps = 0;
    for (int32_t s : st_step_) steps = std::max(steps, s + 1);
    hs_off_.assign(static_cast<size_t>(steps) + 1, 0);
    hs_neuron_.clear();
    hs_amp_.clear();
    size_t k = 0;
    for (int32_t t = 0; t < steps; ++t) {
        std::vector<std::pair<int32_t, double>> acc;  // neuron -> sum, first-appearance order
        std::vector<int32_t> seen_idx;
        while (k < ord.size() && st_step_[ord[k]] == t) {
            const size_t e = ord[k++];
            const int32_t j = st_neuron_[e];
            if (j < first_ || j >= first_ + nl_) continue;
            bool found = false;
            for (auto& pr : acc)
                if (pr.first == j) { pr.second += st_amp_[e]; found = true; break; }
            if (!found) acc.emplace_back(j, 0.0 + st_amp_[e]);
        }
        std::sort(acc.begin(), acc.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (auto& pr : acc) {
            hs_neuron_.push_back(pr.first);
            hs_amp_.push_back(pr.second);
        }
        hs_off_[t + 1] = static_cast<int64_t>(hs_neuron_.size());
    }
    if (!opt_.stream_io) {
        upload(stream_, d_st_off_, hs_off_);
        upload(stream_, d_st_neuron_, hs_neuron_);
        upload(stream_, d_st_amp_, hs_amp_);
        st_steps_dev_ = steps;
    }
    stim_dirty_ = false;
}

}  // namespace snb
