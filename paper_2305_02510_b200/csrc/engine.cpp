// Host side of the B200 MAT engine: validation with the reference's messages,
// device layout construction, the per-step launch sequence, results.
//
// Reference anchors:
//   validate_network / validate_stimulus / validate_stdp   proj/src/model.cpp:34-117
//   mat_init (SoA fill, weight build, stdp list)           proj/src/mat_engine.cpp:109-166
//   mat_run loop (stimulus, step, stdp, raster)            proj/src/mat_engine.cpp:252-287
#include "engine.hpp"

#include "nccl_dl.hpp"

#include <algorithm>
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

namespace {

std::string fmt_double(double v) {  // model.cpp:26-30
    std::ostringstream os;
    os << v;
    return os.str();
}

void throw_first(const char* where, const std::vector<std::string>& v) {  // mat_engine.cpp:15-21
    if (v.empty()) return;
    std::string msg = std::string(where) + ": " + v.front();
    if (v.size() > 1) msg += " (+" + std::to_string(v.size() - 1) + " more)";
    throw InvalidArgument(msg);
}

template <typename T>
void upload(DevBuf& d, const std::vector<T>& h) {
    d.alloc(h.size() * sizeof(T));
    if (!h.empty()) cuda_check(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

uint64_t host_mix64(uint64_t z) {  // rng.hpp:8-12
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

}  // namespace

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
        if (setup_done_ && (neuron[i] < 0 || neuron[i] >= n_))
            throw InvalidArgument(run_name() + ": " + who + ": neuron id " + std::to_string(neuron[i]) +
                                  " out of range (" + std::to_string(n_) + " neurons)");
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
    upload(d_toff_, off);
    upload(d_meta_, meta);
    upload(d_tpidx_, pidx);
    if (f64_) upload(d_w_, wd);
    else upload(d_w_, wf);
    syn_local_ = static_cast<int64_t>(pre_.size());
    sweep_bytes_full_ = static_cast<double>(pre_.size()) * ((stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + 4.0);
    return true;
}

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
    a.spike_count = d_spikes_.as<unsigned long long>();
    a.d_step = d_step_.as<int32_t>();
    a.abm = abm_ ? 1 : 0;
    a.fire_p = any_stochastic_ ? d_firep_.as<double>() : nullptr;
    a.agent_key = any_stochastic_ ? d_akey_.as<uint64_t>() : nullptr;
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

// ---- setup -------------------------------------------------------------------
void Engine::setup() {
    require_not_setup("sn_setup");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    validate();
    n_ = static_cast<int32_t>(thr_.size());
    if (n_ < 1) throw InvalidArgument(std::string(abm_ ? "abm world" : "mat_init") + ": the network has no neurons");
    if (!fire_p_.empty()) fire_p_.resize(static_cast<size_t>(n_), 1.0);
    any_stochastic_ = abm_ && std::any_of(fire_p_.begin(), fire_p_.end(), [](double p) { return p < 1.0; });
    partition(n_, opt_.rank, opt_.world, &first_, &nl_);
    {
        int32_t f0, c0;
        partition(n_, 0, opt_.world, &f0, &c0);
        part_ = std::max(c0, 32);
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
            const int64_t d = static_cast<int64_t>(delay_[s]) + axonal_[pre_[s]];
            if (d > 64)
                throw Unsupported("mat_init: synapses[" + std::to_string(s) + "] has effective delay " +
                                  std::to_string(d) + "; this engine supports delays up to 64 steps");
            dmax_ = std::max<int32_t>(dmax_, static_cast<int32_t>(d));
            if (stdp_on_ && plastic_[s]) dp_ = std::max<int32_t>(dp_, static_cast<int32_t>(d));
        }
    }
    has_delay_ = dmax_ > 1;
    hw_ = stdp_on_ ? static_cast<int32_t>((window_ + dp_ + 63) / 64) : 1;
    hw_ = std::max(hw_, 1);
    if (hw_ > 8)
        throw Unsupported("mat_init: STDP window + delay span exceeds the 512-step history of this engine");
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
    if (opt_.stream_io) {  // pinned staging sized up front (1024 steps of spike words)
        h_raster_.reserve(static_cast<size_t>(1024) * std::max(nl_words_, 1) * 4);
        h_stage_.reserve(64 * 1024);
    }
    cuda_check(cudaStreamSynchronize(stream_), "setup sync");
    setup_done_ = true;
    stats_.synapses_local = syn_local_;
    stats_.dense = dense_ ? 1 : 0;
    stats_.n_local = nl_;
    stats_.first_local = first_;
    stats_.max_delay = dmax_;
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
    if (f64_) upload(d_w_, wd);
    else upload(d_w_, wf);
    if (has_delay_) upload(d_delay_, dl);
    if (any_mixed_) {
        std::vector<uint32_t> mask(static_cast<size_t>(n_) * (pitch_ / 32), 0u);
        for (size_t s = 0; s < pre_.size(); ++s) {
            if (slot_[s] < 0 || !plastic_[s]) continue;
            const int64_t off = slot_[s];
            const int64_t row = off / pitch_, c = off % pitch_;
            mask[row * (pitch_ / 32) + c / 32] |= 1u << (c % 32);
        }
        upload(d_mask_, mask);
    }
    upload(d_kind_, kind);
    upload(d_row_plastic_, row_pl);
    sweep_bytes_full_ = static_cast<double>(n_) * nl_ * ((stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + (has_delay_ ? 1 : 0));
}

void Engine::build_sparse_from_lists() {
    pb_ = sparse_block_pres(hbits_);
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
    upload(d_off_, off);
    upload(d_meta_, meta);
    if (dict) d_w_.alloc(16);
    else if (f64_) upload(d_w_, wd);
    else upload(d_w_, wf);
    upload_dict();
    upload(d_row_plastic_, row_pl);
    sweep_bytes_full_ = static_cast<double>(syn_local_) *
                        (dict ? 4.0 : (stdp_on_ ? 2.0 : 1.0) * (f64_ ? 8 : 4) + 4.0);
}

void Engine::upload_dict() {
    if (dict_.empty()) {
        d_wdict_.release();
        return;
    }
    if (f64_) {
        upload(d_wdict_, dict_);
    } else {
        std::vector<float> f(dict_.begin(), dict_.end());
        upload(d_wdict_, f);
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
        upload(d_kind_, kind);
        if (er_.p >= 1.0) {
            const int64_t self_local = std::max(0, std::min(nl_, n_ - first_));
            syn_local_ = static_cast<int64_t>(n_) * nl_ - self_local;
        } else {
            syn_local_ = static_cast<int64_t>(er_.p * static_cast<double>(n_) * nl_);  // expectation
        }
        sweep_bytes_full_ = static_cast<double>(n_) * nl_ * ((stdp_on_ ? 2.0 : 1.0) * esz + (has_delay_ ? 1 : 0));
    } else {
        pb_ = sparse_block_pres(hbits_);
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
        upload(d_off_, off);
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
    upload(d_row_plastic_, row_pl);
    if (er_.stdp && !stdp_on_)
        throw InvalidArgument("mat_init: plastic synapses were generated but no STDP config was set (sn_set_stdp)");
}

void Engine::alloc_state() {
    std::vector<double> v(reset_.begin() + first_, reset_.begin() + first_ + nl_);
    upload(d_v_, v);  // membrane = reset (mat_engine.cpp:143)
    upload(d_thr_, std::vector<double>(thr_.begin() + first_, thr_.begin() + first_ + nl_));
    upload(d_leak_, std::vector<double>(leak_.begin() + first_, leak_.begin() + first_ + nl_));
    upload(d_reset_, std::vector<double>(reset_.begin() + first_, reset_.begin() + first_ + nl_));
    upload(d_refr_, std::vector<int32_t>(refr_.begin() + first_, refr_.begin() + first_ + nl_));
    d_cnt_.alloc(static_cast<size_t>(std::max(nl_, 1)) * 4);
    cuda_check(cudaMemsetAsync(d_cnt_.p, 0, d_cnt_.bytes, stream_), "memset");
    const size_t wbytes = static_cast<size_t>(std::max(words_, (n_ + 31) / 32)) * 4;
    d_bits_.alloc(wbytes);
    d_active_.alloc(wbytes);
    cuda_check(cudaMemsetAsync(d_bits_.p, 0, wbytes, stream_), "memset");
    cuda_check(cudaMemsetAsync(d_active_.p, 0, wbytes, stream_), "memset");
    d_hist_.alloc(static_cast<size_t>(hw_) * n_ * 8);
    cuda_check(cudaMemsetAsync(d_hist_.p, 0, d_hist_.bytes, stream_), "memset");
    d_hist_lo_.alloc(static_cast<size_t>(n_) * 4);
    cuda_check(cudaMemsetAsync(d_hist_lo_.p, 0, d_hist_lo_.bytes, stream_), "memset");
    const size_t np = static_cast<size_t>(n_) * (stdp_on_ ? dp_ : 1);
    d_pot64_.alloc(np * 8);
    d_pot32_.alloc(np * 4);
    d_dep64_.alloc(static_cast<size_t>(n_) * 8);
    d_dep32_.alloc(static_cast<size_t>(n_) * 4);
    for (DevBuf* b : {&d_pot64_, &d_pot32_, &d_dep64_, &d_dep32_})
        cuda_check(cudaMemsetAsync(b->p, 0, b->bytes, stream_), "memset");
    if (stdp_on_) {
        upload(d_ap_, a_plus_);
        upload(d_am_, a_minus_);
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
        upload(d_firep_, fp);
        upload(d_akey_, key);
    }
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
        if (cols_) {
            const size_t esz2 = f64_ ? 8 : 4;
            d_hist2_.alloc(static_cast<size_t>(2) * n_ * 8);
            d_pot2_.alloc(static_cast<size_t>(2) * n_ * std::max(dp_, 1) * esz2);
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
            tma_ = !f64_ && !has_delay_ && !(dk && std::string(dk) == "stream");
            if (tma_) {
                const char* tw = std::getenv("SNB_TMA_WAVES");
                const double tw_waves = tw ? std::atof(tw) : 14.0;
                int tn = std::max(1, static_cast<int>(std::lround(tw_waves * sms / ntiles)));
                int trpc = static_cast<int>(round_up(std::max(32, (n_ + tn - 1) / tn), 32));
                trpc = std::min(trpc, dense_tma_max_rows());
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
        // one-weight lists (k_sparse_count): 8 lanes per post read whole 128-byte
        // lines (4 posts per warp-wide LDG.128); cfg4, 160 entries per list:
        // SUB 8 0.514 ms vs SUB 4 0.529 ms, 16 0.678
        if (dict_.size() == 2 && !stdp_on_) sub_ = avg >= 1024 ? 16 : avg >= 96 ? 8 : 4;
        if (const char* sv = std::getenv("SNB_SPARSE_SUB")) {  // A/B knob: lanes per post
            const int v = std::atoi(sv);
            if (v == 4 || v == 8 || v == 16 || v == 32 || (!dict_.empty() && (v == 1 || v == 2))) sub_ = v;
        }
        // default: SUB lanes per post (k_sparse_pull, 1.058 ms on cfg4); the flat
        // per-warp chunk stream (k_sparse_stream, 1.115 ms) stays selectable for
        // A/B runs with SNB_SPARSE_KERNEL=stream (tools/ab_sparse.sh)
        const char* sk = std::getenv("SNB_SPARSE_KERNEL");
        if (sk && std::string(sk) == "stream") sub_ = 0;
        const int target = sms * 8;
        int gx = std::max(1, target / std::max(1, nblocks_));
        const int unit = sub_ == 0 ? 8 : 8 * (32 / sub_);
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
        if (count_path && !(bo && std::string(bo) == "0")) {
            size_t free_b = 0, total_b = 0;
            cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
            const size_t bytes = static_cast<size_t>(sparse_elems_) * 4;
            if (bytes + (256u << 20) < free_b) {
                DevBuf ordered;
                ordered.alloc(bytes);
                launch_sparse_bank_order(d_meta_.as<uint32_t>(), ordered.as<uint32_t>(), d_off_.as<int64_t>(),
                                         static_cast<int64_t>(nblocks_) * nl_, nl_, sub_, hbits_, stream_);
                cuda_check(cudaStreamSynchronize(stream_), "bank order");
                std::swap(d_meta_.p, ordered.p);
                std::swap(d_meta_.bytes, ordered.bytes);
                bank_ordered_ = true;
            }
        }
    }
}

// Stage plan of k_sparse_tma: the (block, post) lists are cut into stages of
// whole posts (<= sparse_tma_stage_entries() entries, one pre block, at most
// sparse_tma_max_boundaries() posts); every CTA owns a contiguous run of
// stages inside one pre block, CTAs per block in proportion to its entries.  Returns false when
// a single list is longer than a stage (the pull kernel handles such nets).
bool Engine::build_sparse_tma_plan(int ctas) {
    const int64_t P = static_cast<int64_t>(nblocks_) * nl_;
    std::vector<int64_t> off(static_cast<size_t>(P) + 1);
    cuda_check(cudaMemcpy(off.data(), d_off_.p, off.size() * 8, cudaMemcpyDeviceToHost), "offsets D2H");
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
    upload(d_sp_stages_, stages);
    upload(d_sp_first_, first);
    upload(d_sp_block_, cblock);
    upload(d_sp_bnd_, bnd);
    sp_ctas_ = static_cast<int32_t>(cblock.size());
    return sp_ctas_ > 0;
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
        upload(d_st_off_, hs_off_);
        upload(d_st_neuron_, hs_neuron_);
        upload(d_st_amp_, hs_amp_);
        st_steps_dev_ = steps;
    }
    stim_dirty_ = false;
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
    a.nchunks = nchunks_;
    a.u_exact = d_uexact_.as<double>();
    a.st_off = st_off;
    a.st_neuron = st_neuron;
    a.st_amp = st_amp;
    a.st_steps = st_steps;
    a.st_base = st_base;
    a.d_step = d_step_.as<int32_t>();
    a.work = (dense_ && !exact_) ? d_work_.as<int32_t>() : nullptr;
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
    h.pot32 = d_pot32_.as<float>();
    h.dep64 = d_dep64_.as<double>();
    h.dep32 = d_dep32_.as<float>();
    h.row_plastic = d_row_plastic_.as<uint8_t>();
    h.active = d_active_.as<uint32_t>();
    h.d_step = d_step_.as<int32_t>();
    h.hist_lo = (!dense_ && (hbits_ == 16 || hbits_ == 32)) ? d_hist_lo_.as<uint32_t>() : nullptr;
    h.active_count = d_spikes_.as<unsigned long long>() + 1;
    if (p2p_) {
        h.flags = d_flags_.as<int32_t>();
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
    a.pot = f64_ ? static_cast<const void*>(d_pot64_.p) : static_cast<const void*>(d_pot32_.p);
    a.dep = f64_ ? static_cast<const void*>(d_dep64_.p) : static_cast<const void*>(d_dep32_.p);
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
    return a;
}

void Engine::launch_sweep_only() {
    if (dense_) {
        DenseArgs a = dense_args();
        if (tma_) launch_dense_tma(a, stdp_on_, dense_grid_, stream_);
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
        a.pot = f64_ ? static_cast<const void*>(d_pot64_.p) : static_cast<const void*>(d_pot32_.p);
        a.dep = f64_ ? static_cast<const void*>(d_dep64_.p) : static_cast<const void*>(d_dep32_.p);
        a.dp = stdp_on_ ? dp_ : 1;
        a.w_min = w_min_;
        a.w_max = w_max_;
        a.posts_per_cta = posts_per_cta_;
        a.wdict = dict_.empty() ? nullptr : d_wdict_.p;
        a.dict_size = static_cast<int32_t>(dict_.size());
        a.partial = d_partial_.as<double>();
        a.v = d_v_.as<double>();
        a.leak = d_leak_.as<double>();
        a.reset = d_reset_.as<double>();
        a.u_exact = d_uexact_.as<double>();
        a.d_step = d_step_.as<int32_t>();
        a.abm = abm_ ? 1 : 0;
        if (nl_ == 0) {
            launch_step_bump(a.d_step, stream_);
        } else if (sparse_tma_) {
            SpStagePlan plan{d_sp_stages_.as<SpStage>(), d_sp_first_.as<int32_t>(), d_sp_block_.as<int32_t>(),
                             d_sp_bnd_.as<uint16_t>()};
            launch_sparse_tma(a, plan, sp_ctas_, f64_, hbits_, stream_);
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
    const bool fused = opt_.world == 1;
    const HistArgs h = hist_args();
    cudaEvent_t e0{}, e1{}, e2{}, e3{};
    if (prof) { e0 = get_event(); cuda_check(cudaEventRecord(e0, stream_), "rec"); }
    launch_neuron(na, exact_, fused, h, stream_);
    stats_.kernel_launches += 1;
    if (prof) { e1 = get_event(); cuda_check(cudaEventRecord(e1, stream_), "rec"); pending_.push_back({e0, e1, 0, 0.0}); }
    if (!fused && exchange) {
        if (prof) { e0 = get_event(); cuda_check(cudaEventRecord(e0, stream_), "rec"); }
        if (comm_ && !p2p_) comm_->all_gather_inplace(d_bits_.as<uint32_t>(), static_cast<size_t>(part_ / 32), stream_);
        launch_hist(h, stream_);
        stats_.kernel_launches += 1;
        if (prof) { e1 = get_event(); cuda_check(cudaEventRecord(e1, stream_), "rec"); pending_.push_back({e0, e1, 2, 0.0}); }
    }
    if (prof) { e2 = get_event(); cuda_check(cudaEventRecord(e2, stream_), "rec"); }
    launch_sweep();
    if (prof) { e3 = get_event(); cuda_check(cudaEventRecord(e3, stream_), "rec"); pending_.push_back({e2, e3, 1, 0.0}); }
}

// The step loop as CUDA graphs of up to 64 steps (kernels read the step from
// d_step, so one graph serves every chunk of a simulate call).  With
// profiling, per-kernel CUDA events are captured into the graph (event record
// nodes) and read after each replay, so the timed loop keeps graph launch
// costs while reporting per-kernel device time.  Returns the summed device
// time of the chunks.
double Engine::run_graph_chunks(const NeuronArgs& na, int steps) {
    const int chunk = std::min(steps, 64);
    const bool prof = opt_.profile != 0;
    const bool fused = opt_.world == 1;
    const int per = 6;
    std::vector<cudaEvent_t> ev(prof ? static_cast<size_t>(chunk) * per : 0);
    for (auto& e : ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    const HistArgs h = hist_args();
    auto capture = [&](int k) {
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
                launch_hist(h, stream_);
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
    cudaGraphExec_t full = capture(chunk);
    cudaGraphExec_t tail = (steps % chunk) ? capture(steps % chunk) : nullptr;
    const int per_step_kernels = fused ? 2 : 3;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans;
    double total = 0.0;
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
    require_setup("sn_simulate");
    if (steps < 1) throw InvalidArgument(run_name() + ": steps must be >= 1");
    if (opt_.world > 1 && !comm_ && !p2p_)
        throw LogicError("sn_simulate: partitioned engine needs sn_comm_init or sn_p2p_open "
                         "(or use sn_step_local/sn_step_finish)");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
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
            if (cols_) {
                ColArgs ca{};
                ca.hist2 = d_hist2_.as<uint64_t>();
                ca.pot2 = d_pot2_.p;
                ca.act3 = d_act2_.as<uint32_t>();
                ca.row_plastic = d_row_plastic_.as<uint8_t>();
                ca.a_plus = d_ap_.as<double>();
                ca.a_minus = d_am_.as<double>();
                ca.window = window_;
                ca.dmax = dmax_;
                // activity and raster words are OR-ed by 8-post groups: start from zero
                cuda_check(cudaMemsetAsync(d_act2_.p, 0, d_act2_.bytes, stream_), "memset");
                if (raster && nl_words_ > 0)
                    cuda_check(cudaMemsetAsync(raster, 0, static_cast<size_t>(steps) * nl_words_ * 4, stream_), "memset");
                launch_persistent_cols(na, dense_args(), ca, f64_, stdp_on_, has_delay_, col_width_, persist_grid_,
                                       steps, stream_);
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
        } else if (opt_.use_graphs) {
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
        if (cnt) cuda_check(cudaMemcpy(trace_.data() + old, d_trace_.p, cnt * 8, cudaMemcpyDeviceToHost), "trace D2H");
        trace_rows_ += steps;
    }
    t_ += steps;
    stats_.steps_done = t_;
    events_valid_ = false;
}

void Engine::synchronize() { cuda_check(cudaStreamSynchronize(stream_), "sn_synchronize"); }

// ---- host-driven exchange (partition emulation / custom transports) ---------
void Engine::step_local() {
    require_setup("sn_step_local");
    if (tiny_) throw LogicError("sn_step_local: single-partition engines run through sn_simulate");
    host_exchange_ = true;
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
    cuda_check(cudaMemcpy(out, d_bits_.p, static_cast<size_t>(words) * 4, cudaMemcpyDeviceToHost), "bits D2H");
}

void Engine::put_spike_words(int32_t first_word, const uint32_t* w, int64_t count) {
    require_setup("sn_put_spike_words");
    if (first_word < 0 || first_word + count > words_) throw InvalidArgument("sn_put_spike_words: range outside the bitmask");
    cuda_check(cudaMemcpy(d_bits_.as<uint32_t>() + first_word, w, static_cast<size_t>(count) * 4, cudaMemcpyHostToDevice), "bits H2D");
}

void Engine::step_finish() {
    require_setup("sn_step_finish");
    if (tiny_) throw LogicError("sn_step_finish: single-partition engines run through sn_simulate");
    if (opt_.world > 1) {
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
        if (nl_) cuda_check(cudaMemcpy(trace_.data() + old, d_trace_.p, static_cast<size_t>(nl_) * 8, cudaMemcpyDeviceToHost), "trace D2H");
        trace_rows_ += 1;
    }
    t_ += 1;
    stats_.steps_done = t_;
    events_valid_ = false;
}

void Engine::comm_init(const uint8_t* id, int32_t rank, int32_t world) {
    if (world != opt_.world || rank != opt_.rank)
        throw InvalidArgument("sn_comm_init: rank/world differ from the engine options");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    delete comm_;
    comm_ = nullptr;
    if (world > 1) comm_ = new NcclComm(id, rank, world);
}

// ---- peer-to-peer exchange ---------------------------------------------------
// Each rank exports (cudaIpcGetMemHandle) its full spike bitmask and its
// flag array; after opening every peer's pair, the neuron kernel stores its
// spike words straight into all peers' bitmasks over NVLink and releases
// flag[rank] = t + 1 in each of them; k_hist acquires all flags before
// reading the bitmask.  No NCCL call remains on the step path.
void Engine::p2p_get_handles(uint8_t* out, int64_t cap) {
    require_setup("sn_p2p_get_handles");
    if (cap < 2 * kIpcHandleBytes) throw InvalidArgument("sn_p2p_get_handles: buffer smaller than 128 bytes");
    cudaIpcMemHandle_t hb, hf;
    cuda_check(cudaIpcGetMemHandle(&hb, d_bits_.p), "cudaIpcGetMemHandle(bits)");
    cuda_check(cudaIpcGetMemHandle(&hf, d_flags_.p), "cudaIpcGetMemHandle(flags)");
    std::memcpy(out, &hb, kIpcHandleBytes);
    std::memcpy(out + kIpcHandleBytes, &hf, kIpcHandleBytes);
}

void Engine::set_peer_tables(const std::vector<uint32_t*>& bits, const std::vector<int32_t*>& flags) {
    d_peer_bits_.alloc(bits.size() * sizeof(uint32_t*));
    d_peer_flags_.alloc(flags.size() * sizeof(int32_t*));
    cuda_check(cudaMemcpy(d_peer_bits_.p, bits.data(), bits.size() * sizeof(uint32_t*), cudaMemcpyHostToDevice), "peer table");
    cuda_check(cudaMemcpy(d_peer_flags_.p, flags.data(), flags.size() * sizeof(int32_t*), cudaMemcpyHostToDevice), "peer table");
    p2p_ = true;
}

void Engine::p2p_open(const uint8_t* all, int32_t world) {
    require_setup("sn_p2p_open");
    if (world != opt_.world) throw InvalidArgument("sn_p2p_open: world differs from the engine options");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    std::vector<uint32_t*> bits(world);
    std::vector<int32_t*> flags(world);
    for (int q = 0; q < world; ++q) {
        if (q == opt_.rank) {
            bits[q] = d_bits_.as<uint32_t>();
            flags[q] = d_flags_.as<int32_t>();
            continue;
        }
        cudaIpcMemHandle_t hb, hf;
        std::memcpy(&hb, all + static_cast<size_t>(q) * 2 * kIpcHandleBytes, kIpcHandleBytes);
        std::memcpy(&hf, all + static_cast<size_t>(q) * 2 * kIpcHandleBytes + kIpcHandleBytes, kIpcHandleBytes);
        void* pb = nullptr;
        void* pf = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&pb, hb, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(bits)");
        ipc_opened_.push_back(pb);
        cuda_check(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(flags)");
        ipc_opened_.push_back(pf);
        bits[q] = static_cast<uint32_t*>(pb);
        flags[q] = static_cast<int32_t*>(pf);
    }
    set_peer_tables(bits, flags);
}

void Engine::p2p_connect_local(Engine* const* engines, int32_t world) {
    std::vector<uint32_t*> bits(world);
    std::vector<int32_t*> flags(world);
    for (int q = 0; q < world; ++q) {
        Engine* e = engines[q];
        if (!e || !e->setup_done_) throw LogicError("sn_p2p_connect_local: every engine must be set up");
        if (e->opt_.world != world || e->opt_.rank != q)
            throw InvalidArgument("sn_p2p_connect_local: engines must be ranks 0..world-1 in order");
        if (e->opt_.device != engines[0]->opt_.device)
            throw InvalidArgument("sn_p2p_connect_local: engines must share one device (use sn_p2p_open across GPUs)");
        bits[q] = e->d_bits_.as<uint32_t>();
        flags[q] = e->d_flags_.as<int32_t>();
    }
    for (int q = 0; q < world; ++q) {
        cuda_check(cudaSetDevice(engines[q]->opt_.device), "cudaSetDevice");
        engines[q]->set_peer_tables(bits, flags);
    }
}

void Engine::check_exchange_error() {
    if (!p2p_) return;
    int32_t err = 0;
    cuda_check(cudaMemcpy(&err, d_err_.p, 4, cudaMemcpyDeviceToHost), "exchange error D2H");
    if (err) throw NcclError("peer-to-peer spike exchange timed out (a peer rank stopped publishing)");
}

// ---- results -------------------------------------------------------------------
// Bitmask raster -> (step, neuron) events, ascending: per-row popcounts, a
// prefix sum, then rows decoded in parallel straight into the two arrays.
void Engine::decode_raster() {
    if (events_valid_) return;
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
    raster_.clear();
    dec_rows_.clear();
    dec_start_.clear();
    events_valid_ = true;
}

void Engine::get_membrane(double* out, int64_t count) {
    require_setup("sn_get_membrane");
    if (count < nl_) throw InvalidArgument("sn_get_membrane: buffer smaller than the local neuron count");
    if (nl_) cuda_check(cudaMemcpy(out, d_v_.p, static_cast<size_t>(nl_) * 8, cudaMemcpyDeviceToHost), "membrane D2H");
}

int64_t Engine::trace_rows() { return trace_rows_; }

void Engine::get_trace(double* out, int64_t count) {
    if (count < static_cast<int64_t>(trace_.size())) throw InvalidArgument("sn_get_membrane_trace: buffer too small");
    std::memcpy(out, trace_.data(), trace_.size() * 8);
}

void Engine::get_synapse_weights(double* out, int64_t count) {
    require_setup("sn_get_synapse_weights");
    if (generated_) throw Unsupported("sn_get_synapse_weights: generated networks have no synapse list; use sn_get_weight_matrix");
    if (count < static_cast<int64_t>(pre_.size())) throw InvalidArgument("sn_get_synapse_weights: buffer too small");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    const size_t esz = f64_ ? 8 : 4;
    std::vector<uint8_t> host(d_w_.bytes);
    cuda_check(cudaMemcpy(host.data(), d_w_.p, d_w_.bytes, cudaMemcpyDeviceToHost), "weights D2H");
    std::vector<uint32_t> meta;
    if (!dense_ && !dict_.empty()) {
        meta.resize(static_cast<size_t>(sparse_elems_));
        if (!meta.empty()) cuda_check(cudaMemcpy(meta.data(), d_meta_.p, meta.size() * 4, cudaMemcpyDeviceToHost), "meta D2H");
    }
    for (size_t s = 0; s < pre_.size(); ++s) {
        if (slot_[s] < 0) { out[s] = 0.0; continue; }
        if (bank_ordered_) { out[s] = dict_[0]; continue; }  // lists reordered; one weight
        if (!meta.empty()) out[s] = dict_[meta[slot_[s]] >> 23];
        else if (esz == 8) out[s] = reinterpret_cast<const double*>(host.data())[slot_[s]];
        else out[s] = static_cast<double>(reinterpret_cast<const float*>(host.data())[slot_[s]]);
    }
}

void Engine::get_weight_matrix(double* out, int64_t count) {
    require_setup("sn_get_weight_matrix");
    if (count < static_cast<int64_t>(n_) * nl_) throw InvalidArgument("sn_get_weight_matrix: buffer too small");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    std::fill(out, out + static_cast<int64_t>(n_) * nl_, 0.0);
    const size_t esz = f64_ ? 8 : 4;
    std::vector<uint8_t> host(d_w_.bytes);
    cuda_check(cudaMemcpy(host.data(), d_w_.p, d_w_.bytes, cudaMemcpyDeviceToHost), "weights D2H");
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
        cuda_check(cudaMemcpy(off.data(), d_off_.p, off.size() * 8, cudaMemcpyDeviceToHost), "off D2H");
        if (!meta.empty()) cuda_check(cudaMemcpy(meta.data(), d_meta_.p, meta.size() * 4, cudaMemcpyDeviceToHost), "meta D2H");
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
    if (setup_done_) {
        unsigned long long c[2] = {0, 0};
        cuda_check(cudaMemcpy(c, d_spikes_.p, 16, cudaMemcpyDeviceToHost), "stats D2H");
        stats_.spike_count = static_cast<int64_t>(c[0]);
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
            stats_.sweep_kernel = persistent_ ? (cols_ ? SN_SWEEP_PERSISTENT_COLS : SN_SWEEP_PERSISTENT)
                                  : exact_    ? SN_SWEEP_DENSE_EXACT
                                  : tma_      ? SN_SWEEP_DENSE_TMA
                                              : SN_SWEEP_DENSE_STREAM;
            stats_.sweep_ctas = persistent_ ? persist_grid_ : dense_grid_;
        } else {
            stats_.sweep_kernel = exact_ ? SN_SWEEP_SPARSE_EXACT
                                  : sparse_tma_ ? SN_SWEEP_SPARSE_TMA
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
    if (setup_done_) cuda_check(cudaMemset(d_spikes_.as<unsigned long long>() + 1, 0, 8), "reset");
}

}  // namespace snb
