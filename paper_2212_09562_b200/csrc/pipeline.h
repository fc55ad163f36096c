// Host orchestration of the device construction pipeline.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/recsplit.h"

namespace rs {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct BuildParams {
    uint64_t n;
    uint32_t leaf, bucket;
    bool rf;
    uint64_t g;
    int device;
    uint32_t shards;  // virtual shards (>= 1)
};

struct BuildOutput {
    std::vector<uint8_t> bytes;
    std::vector<uint64_t> values;  // only when requested
    recsplit_stats stats{};
};

// d_keys: device pointer (n keys) on params.device; work ordered on st.
void build_on_device(const uint64_t* d_keys, const BuildParams& p, cudaStream_t st, bool want_values,
                     BuildOutput& out);

// Kernel-level entry points for parity tests (host arrays).
void search_leaves_host(const uint64_t* lo, const uint8_t* isb, const uint32_t* off, uint32_t n_nodes, bool rf,
                        uint64_t* out);
void search_splits_host(const uint64_t* lo, const uint32_t* off, uint32_t n_nodes, uint32_t leaf, uint64_t* out);

}  // namespace rs
