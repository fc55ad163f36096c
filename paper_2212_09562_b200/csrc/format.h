// Serialized-MPHF reader shared by the host and device queries.
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "tables.h"

namespace rs {

struct EFView {
    uint32_t L;
    uint64_t nlow, nup;
    const uint8_t* low;
    const uint8_t* up;
};

struct Parsed {
    uint32_t leaf;
    bool rf;
    bool strings;  // built from string keys (header flags bit 1, R16)
    uint64_t g, n, B, D, dC, beta;
    int64_t dR;
    EFView ec, ep;
    const uint8_t* data;
    std::vector<uint64_t> C, P;  // decoded index (B + 1 entries each)
    uint64_t smax = 1;
    std::shared_ptr<const Tables> T;
};

// Returns 0 or RECSPLIT_E_FORMAT with a message in *err.
int parse_mphf(const uint8_t* blob, size_t size, Parsed& M, std::string* err);

}  // namespace rs
