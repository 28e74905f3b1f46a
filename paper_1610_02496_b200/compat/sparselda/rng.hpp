// Counter-based draws of the reference API (rng.hpp:12-83) on the host: Philox4x32-10 keyed by
// (seed_lo, seed_hi) over the counter (kind, element_lo, element_hi, block).  The device kernels
// use the same generator (csrc/common.cuh); this copy serves host callers (sample_token,
// vanilla_sample) and is pinned to the Random123 known-answer vectors in tests/test_oracle.py.
#pragma once

#include <array>
#include <cstdint>

namespace sparselda {

namespace philox {

inline constexpr std::uint32_t kW32A = 0x9E3779B9u, kW32B = 0xBB67AE85u;    // Weyl key bumps
inline constexpr std::uint32_t kM4x32A = 0xD2511F53u, kM4x32B = 0xCD9E8D57u;  // round multipliers

inline std::array<std::uint32_t, 4> block(std::array<std::uint32_t, 4> c, std::array<std::uint32_t, 2> k) {
    for (int r = 0; r < 10; ++r) {
        const std::uint64_t p0 = std::uint64_t{kM4x32A} * c[0];
        const std::uint64_t p1 = std::uint64_t{kM4x32B} * c[2];
        c = {static_cast<std::uint32_t>(p1 >> 32) ^ c[1] ^ k[0], static_cast<std::uint32_t>(p1),
             static_cast<std::uint32_t>(p0 >> 32) ^ c[3] ^ k[1], static_cast<std::uint32_t>(p0)};
        k[0] += kW32A;
        k[1] += kW32B;
    }
    return c;
}

}  // namespace philox

// Reserved stream kinds (training iterations use their iteration number).
inline constexpr std::uint32_t kInitAssignStream = 0xFFFFFFFFu;
inline constexpr std::uint32_t kHeldoutInitStream = 0xFFFD0000u;
inline constexpr std::uint32_t kHeldoutSweepBase = 0xFFFE0000u;

// Uniform doubles in [0, 1) from the stream (seed, kind, element): Philox block b yields
// (o1:o0) first, then (o3:o2), each as its top 53 bits times 2^-53.
class RngStream {
public:
    RngStream(std::uint64_t seed, std::uint32_t kind, std::uint64_t element)
        : key_{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32)},
          kind_(kind), element_(element) {}

    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

    std::uint64_t next_u64() {
        if (left_ == 0) {
            const auto o = philox::block({kind_, static_cast<std::uint32_t>(element_),
                                          static_cast<std::uint32_t>(element_ >> 32), blk_++},
                                         key_);
            pair_[0] = (std::uint64_t{o[1]} << 32) | o[0];
            pair_[1] = (std::uint64_t{o[3]} << 32) | o[2];
            left_ = 2;
        }
        return pair_[2 - left_--];
    }

private:
    std::array<std::uint32_t, 2> key_;
    std::uint32_t kind_;
    std::uint64_t element_;
    std::uint32_t blk_ = 0;
    std::uint64_t pair_[2] = {0, 0};
    int left_ = 0;
};

}  // namespace sparselda
