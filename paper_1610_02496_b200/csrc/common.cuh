// common.cuh -- device primitives shared by the ESCA kernels (sm_100a).
//
// Bit-exactness contract (SURVEY.md §7 "Hard parts" 1): every float op on the
// sampling / phi / tree path uses an explicit round-to-nearest intrinsic
// (__fadd_rn, __fmul_rn, __fdiv_rn, __dadd_rn, __dmul_rn, __ddiv_rn) so that
// no FMA contraction or re-association can change a bit relative to the
// reference's sequential SSE arithmetic; the library is additionally built
// with -fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace slda {

constexpr uint32_t kInvalidTopic = 0xFFFFFFFFu;     // types.hpp:17
constexpr uint32_t kInitAssignStream = 0xFFFFFFFFu; // rng.hpp:43
constexpr uint32_t kHeldoutInitStream = 0xFFFD0000u;
constexpr uint32_t kHeldoutSweepBase = 0xFFFE0000u;

// K is padded to a multiple of kBlock.  The device search is lower_bound over
// the row's inclusive prefix L4 (acceptance.cpp:140-200 proves WaryTree::sample
// equal to it for every W).
constexpr uint32_t kBlock = 32;
// Leaf width of the device descent: L8[j] = L4[8j+7] is staged in shared memory and
// the final 8 prefixes are one 32-byte sector.
constexpr uint32_t kLeaf = 8;

// Philox4x32-10, rng.hpp:14-37.  Counter (kind, elem_lo, elem_hi, block),
// key (seed_lo, seed_hi) -- rng.hpp:51-54.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// The first two next_double() draws of RngStream(seed, kind, element)
// (rng.hpp:57-76) narrowed to f32 exactly as sample_token does
// (sampler.hpp:190-191): f32(f64(m) * 2^-53) == f32(m) * 2^-53 for m < 2^53,
// because scaling by a power of two commutes with round-to-nearest here.
__device__ __forceinline__ void draw2_f32(uint64_t seed, uint32_t kind, uint64_t element,
                                          float& u0, float& u1) {
    const uint4 o = philox4x32_10(
        make_uint4(kind, static_cast<uint32_t>(element), static_cast<uint32_t>(element >> 32), 0u),
        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const uint64_t b1 = (static_cast<uint64_t>(o.y) << 32) | o.x;
    const uint64_t b0 = (static_cast<uint64_t>(o.w) << 32) | o.z;
    u0 = __fmul_rn(__ull2float_rn(b1 >> 11), 0x1p-53f);
    u1 = __fmul_rn(__ull2float_rn(b0 >> 11), 0x1p-53f);
}

// uniform_topic (trainer.cpp:217-221, corpus.cpp:91-94): topic = u32(u0 * K) in f64.
__device__ __forceinline__ uint32_t uniform_topic(uint64_t seed, uint32_t kind, uint64_t element,
                                                  uint32_t K) {
    const uint4 o = philox4x32_10(
        make_uint4(kind, static_cast<uint32_t>(element), static_cast<uint32_t>(element >> 32), 0u),
        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const uint64_t b1 = (static_cast<uint64_t>(o.y) << 32) | o.x;
    const double u = __dmul_rn(__ull2double_rn(b1 >> 11), 0x1p-53);
    const uint32_t t = __double2uint_rz(__dmul_rn(u, static_cast<double>(K)));
    return t < K ? t : K - 1;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Grid size for a grid-stride kernel over n items: at most `cap` CTAs (default 32 per SM).
inline uint32_t grid_for(uint64_t n, uint32_t threads, uint32_t cap = 148u * 32u) {
    const uint64_t g = (n + threads - 1) / threads;
    return static_cast<uint32_t>(g == 0 ? 1 : (g > cap ? cap : g));
}

}  // namespace slda
