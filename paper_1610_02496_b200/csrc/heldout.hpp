// heldout.hpp -- device held-out log-likelihood (eval.cpp:49-133).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace slda {

struct HeldoutArgs {
    const uint64_t* est_off;   // D+1, estimation tokens (even positions, eval.cpp:14-28)
    const uint32_t* est_word;
    const uint64_t* evl_off;   // D+1, evaluation tokens (odd positions)
    const uint32_t* evl_word;
    const float* bhat;
    const float* l8;
    const float* q;
    const double* row_mass;    // filled by launch_heldout
    double* ll_out;            // per evaluation token log(mass / denom)
    uint64_t seed;
    double alpha;
    uint32_t burn_in, K, K_pad, l8_stride, n_l8;
    uint32_t cap;              // power of two >= the longest estimation half
};

cudaError_t launch_heldout(const HeldoutArgs& a, uint32_t num_docs, uint32_t V, uint32_t K,
                           uint32_t K_pad, double* row_mass, cudaStream_t s);

}  // namespace slda
