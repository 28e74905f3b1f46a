// host.cpp -- host-only parts of the C-ABI: document sharding and the M-step word-row
// slices.  No device code.  (The synthetic corpus generator is corpus_gen.cpp.)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/saberlda.h"

void slda_set_error_internal(const std::string& msg);  // engine.cu

extern "C" {

int slda_shard_bounds(uint32_t num_docs, uint64_t num_tokens, const uint32_t* doc_lengths_in,
                      uint32_t num_shards, uint32_t* bounds) {
    // chunk_boundaries (corpus.cpp:103-121): each range grows until its load
    // strictly exceeds the per-range share of the remaining tokens, leaving
    // at least one document for every later range.
    if (!bounds) return SLDA_ERR_VALIDATION;
    if (num_docs == 0) {
        if (num_shards != 1) {
            slda_set_error_internal("empty corpus admits exactly one shard");
            return SLDA_ERR_VALIDATION;
        }
        bounds[0] = bounds[1] = 0;
        return SLDA_OK;
    }
    if (num_shards < 1 || num_shards > num_docs || !doc_lengths_in) {
        slda_set_error_internal("num_shards must be in [1, D]");
        return SLDA_ERR_VALIDATION;
    }
    bounds[0] = 0;
    uint64_t remaining = num_tokens;
    uint32_t doc = 0;
    for (uint32_t c = 0; c < num_shards; ++c) {
        const uint64_t left = num_shards - c;
        const uint64_t basis = remaining;
        uint64_t taken = 0;
        do {
            taken += doc_lengths_in[doc];
            ++doc;
        } while (static_cast<uint64_t>(num_docs - doc) > left - 1 && taken * left <= basis);
        remaining -= taken;
        bounds[c + 1] = doc;
    }
    bounds[num_shards] = num_docs;
    return SLDA_OK;
}

int slda_word_slice(uint32_t vocab_size, uint32_t world, uint32_t rank, uint32_t* row_begin,
                    uint32_t* row_end, uint32_t* padded_rows) {
    if (world == 0 || rank >= world || !row_begin || !row_end) {
        slda_set_error_internal("rank must be < world and world >= 1");
        return SLDA_ERR_VALIDATION;
    }
    const uint64_t padded = (static_cast<uint64_t>(vocab_size) + world - 1) / world * world;
    const uint64_t rows = padded / world;
    *row_begin = static_cast<uint32_t>(std::min<uint64_t>(vocab_size, rank * rows));
    *row_end = static_cast<uint32_t>(std::min<uint64_t>(vocab_size, (rank + 1) * rows));
    if (padded_rows) *padded_rows = static_cast<uint32_t>(padded);
    return SLDA_OK;
}

}  // extern "C"
