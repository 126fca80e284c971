// Multi-GPU spike exchange: NCCL communicator setup and the peer-to-peer
// protocol (IPC-mapped bitmasks and step flags) fused into k_neuron / k_hist.
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

void Engine::comm_init(const uint8_t* id, int32_t rank, int32_t world) {
    if (world != opt_.world || rank != opt_.rank)
        throw InvalidArgument("sn_comm_init: rank/world differ from the engine options");
    cuda_check(cudaSetDevice(opt_.device), "cudaSetDevice");
    if (world == 1 && (tiny_ || persistent_))
        throw LogicError("sn_comm_init: this single-partition engine runs whole simulate calls in one kernel "
                         "(create it with persistent = 0 and a dense or sparse storage)");
    if (world == 1 && t_ > 0)  // switches a 1-rank engine to the partitioned step sequence
        throw LogicError("sn_comm_init: a single-partition engine joins a communicator before its first step");
    delete comm_;
    comm_ = nullptr;
    // world 1: a one-rank communicator switches the engine to the partitioned
    // step sequence (k_neuron -> in-graph ncclAllGather -> k_hist -> sweep),
    // the exact launch sequence of every rank of an N-GPU run
    comm_ = new NcclComm(id, rank, world);
}

// ---- peer-to-peer exchange ---------------------------------------------------
// Each rank exports (cudaIpcGetMemHandle) its exchange bitmask (two
// step-parity buffers) and its flag array; after opening every peer's pair,
// the neuron kernel stores its spike words of step t straight into buffer
// t & 1 of every rank over NVLink and releases flag[rank] = t + 1 in each of
// them; k_hist acquires all flags before reading buffer t & 1 into the local
// bitmask.  Double buffering is what makes free-running ranks safe: a rank
// can be at most one step ahead of its slowest peer (its k_hist(t + 1) waits
// for every flag t + 2), so its step t + 2 stores never hit a buffer a peer
// is still reading for step t.  No NCCL call remains on the step path.
void Engine::p2p_get_handles(uint8_t* out, int64_t cap) {
    require_setup("sn_p2p_get_handles");
    if (cap < 2 * kIpcHandleBytes) throw InvalidArgument("sn_p2p_get_handles: buffer smaller than 128 bytes");
    cudaIpcMemHandle_t hb, hf;
    cuda_check(cudaIpcGetMemHandle(&hb, d_xbits_.p), "cudaIpcGetMemHandle(bits)");
    cuda_check(cudaIpcGetMemHandle(&hf, d_flags_.p), "cudaIpcGetMemHandle(flags)");
    std::memcpy(out, &hb, kIpcHandleBytes);
    std::memcpy(out + kIpcHandleBytes, &hf, kIpcHandleBytes);
}

void Engine::set_peer_tables(const std::vector<uint32_t*>& bits, const std::vector<int32_t*>& flags) {
    if (c16_ && t_ > 0)  // the p2p exchange keeps k_hist; the folded history would be lost
        throw LogicError("sn_p2p_open: connect the peer-to-peer exchange before the first step");
    d_peer_bits_.alloc(bits.size() * sizeof(uint32_t*));
    d_peer_flags_.alloc(flags.size() * sizeof(int32_t*));
    h2d_sync(stream_, d_peer_bits_.p, bits.data(), bits.size() * sizeof(uint32_t*), "peer table");
    h2d_sync(stream_, d_peer_flags_.p, flags.data(), flags.size() * sizeof(int32_t*), "peer table");
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
            bits[q] = d_xbits_.as<uint32_t>();
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
        bits[q] = e->d_xbits_.as<uint32_t>();
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
    d2h(&err, d_err_.p, 4, "exchange error D2H");
    if (err) throw NcclError("peer-to-peer spike exchange timed out (a peer rank stopped publishing)");
}

}  // namespace snb
