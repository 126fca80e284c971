#pragma once

#include "engine.hpp"

#include <nccl.h>

namespace snb {

void nccl_unique_id(uint8_t* out);

struct NcclComm {
    NcclComm(const uint8_t* id, int rank, int world);
    ~NcclComm();
    NcclComm(const NcclComm&) = delete;
    NcclComm& operator=(const NcclComm&) = delete;
    void all_gather_inplace(uint32_t* buf, size_t words_per_rank, cudaStream_t s);
    int rank_ = 0, world_ = 1;
    ncclComm_t comm_ = nullptr;
};

}  // namespace snb
