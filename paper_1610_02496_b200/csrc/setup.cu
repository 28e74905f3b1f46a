// setup.cu -- K1/K2: the device-side init_state (PDOW layout, schedule, initial topics,
// recount) and the assignments read-back, on sm_100a.
//
// Reference paths are relative to /root/reference/proj.  See DESIGN.md §3.
#include "common.cuh"
#include "kernels.hpp"

namespace slda {

// ============================================================================
// K1/K2 setup -- build_chunks (corpus.cpp:125-198), build_schedule (:200-210),
// init_assignments (corpus.cpp:87-96), count_chunk_into (trainer.cpp:223-235).
// ============================================================================

__global__ void deinterleave_kernel(const uint32_t* __restrict__ aos, uint64_t T, uint32_t doc_begin,
                                    uint32_t* doc_local, uint32_t* word, uint32_t* topic) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        doc_local[i] = aos[3 * i] - doc_begin;
        word[i] = aos[3 * i + 1];
        if (topic) topic[i] = aos[3 * i + 2];
    }
}

cudaError_t launch_deinterleave(const uint32_t* aos, uint64_t T, uint32_t doc_begin,
                                uint32_t* doc_local, uint32_t* word, uint32_t* topic,
                                cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    deinterleave_kernel<<<grid_for(T, 256), 256, 0, s>>>(aos, T, doc_begin, doc_local, word, topic);
    return cudaGetLastError();
}

__global__ void check_sorted_kernel(const uint32_t* doc_local, uint64_t T, uint32_t* flag) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x + 1; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (doc_local[i] < doc_local[i - 1]) *flag = 1u;
    }
}

cudaError_t launch_check_sorted(const uint32_t* doc_local, uint64_t T, uint32_t* unsorted_flag,
                                cudaStream_t s) {
    if (T < 2) return cudaSuccess;
    check_sorted_kernel<<<grid_for(T, 256), 256, 0, s>>>(doc_local, T, unsorted_flag);
    return cudaGetLastError();
}

__global__ void doc_hist_kernel(const uint32_t* doc_local, uint64_t T, uint32_t* counts) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        atomicAdd(counts + doc_local[i], 1u);
}

cudaError_t launch_doc_hist(const uint32_t* doc_local, uint64_t T, uint32_t* counts, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    doc_hist_kernel<<<grid_for(T, 256), 256, 0, s>>>(doc_local, T, counts);
    return cudaGetLastError();
}

__global__ void iota_kernel(uint32_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint32_t>(i);
}

cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n);
    return cudaGetLastError();
}

__global__ void invert_perm_kernel(const uint32_t* input_of_slot, uint64_t T, uint32_t* slot_of_input) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        slot_of_input[input_of_slot[j]] = static_cast<uint32_t>(j);
}

cudaError_t launch_invert_perm(const uint32_t* input_of_slot, uint64_t T, uint32_t* slot_of_input,
                               cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    invert_perm_kernel<<<grid_for(T, 256), 256, 0, s>>>(input_of_slot, T, slot_of_input);
    return cudaGetLastError();
}

// Execution-order sort key, laid out in slot order so that equal keys keep slot
// (== corpus) order under the stable radix sort:
//   word | (lmax - len_doc) | doc_local
// i.e. the reference's (word, doc, token_id) order (corpus.cpp:157-167) refined by
// descending document length inside each word segment, so the lanes of a sampler
// warp walk C_dk rows of similar length.  lbits == 0 gives the canonical order.
__global__ void make_keys_kernel(const uint32_t* word, const uint32_t* doc_local,
                                 const uint32_t* input_of_slot, const uint32_t* doc_len, uint64_t T,
                                 KeyLayout kl, unsigned long long* keys, uint32_t* vals) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = input_of_slot ? input_of_slot[j] : j;
        const uint32_t d = doc_local[i];
        const unsigned long long lk = kl.lbits ? static_cast<unsigned long long>(kl.lmax - doc_len[d]) : 0ull;
        keys[j] = (static_cast<unsigned long long>(word[i]) << (kl.dbits + kl.lbits)) | (lk << kl.dbits) | d;
        vals[j] = static_cast<uint32_t>(j);
    }
}

cudaError_t launch_make_keys(const uint32_t* word, const uint32_t* doc_local, const uint32_t* input_of_slot,
                             const uint32_t* doc_len, uint64_t T, KeyLayout kl, unsigned long long* keys,
                             uint32_t* vals, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    make_keys_kernel<<<grid_for(T, 256), 256, 0, s>>>(word, doc_local, input_of_slot, doc_len, T, kl, keys, vals);
    return cudaGetLastError();
}

// tok = {C_dk row offset (quads), slot}; flags mark word-segment starts.
__global__ void make_tok_kernel(const unsigned long long* keys, const uint32_t* slots, const uint32_t* row4,
                                uint64_t T, KeyLayout kl, uint2* tok, uint32_t* seg_flag) {
    const unsigned long long dmask = (1ull << kl.dbits) - 1ull;
    const uint32_t ws = kl.dbits + kl.lbits;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long k = keys[i];
        tok[i] = make_uint2(row4[k & dmask], slots[i]);
        seg_flag[i] = (i == 0 || (keys[i - 1] >> ws) != (k >> ws)) ? 1u : 0u;
    }
}

cudaError_t launch_make_tok(const unsigned long long* keys, const uint32_t* slots, const uint32_t* row4,
                            uint64_t T, KeyLayout kl, uint2* tok, uint32_t* seg_flag, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    make_tok_kernel<<<grid_for(T, 256), 256, 0, s>>>(keys, slots, row4, T, kl, tok, seg_flag);
    return cudaGetLastError();
}

__global__ void emit_segments_kernel(const unsigned long long* keys, const uint32_t* seg_flag,
                                     const uint32_t* seg_index, uint64_t T, uint32_t wshift,
                                     uint32_t* seg_word, uint32_t* seg_off) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (seg_flag[i]) {
            const uint32_t s = seg_index[i];
            seg_word[s] = static_cast<uint32_t>(keys[i] >> wshift);
            seg_off[s] = static_cast<uint32_t>(i);
        }
    }
}

cudaError_t launch_emit_segments(const unsigned long long* keys, const uint32_t* seg_flag,
                                 const uint32_t* seg_index, uint64_t T, uint32_t wshift,
                                 uint32_t* seg_word, uint32_t* seg_off, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    emit_segments_kernel<<<grid_for(T, 256), 256, 0, s>>>(keys, seg_flag, seg_index, T, wshift, seg_word,
                                                         seg_off);
    return cudaGetLastError();
}

// build_schedule sort key: (length desc, word asc) -- corpus.cpp:201-205.
__global__ void segment_lengths_kernel(const uint32_t* seg_off, uint32_t nseg, uint64_t T,
                                       uint32_t* seg_len, unsigned long long* sched_keys,
                                       uint32_t* sched_vals, const uint32_t* seg_word,
                                       uint32_t* unit_count) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const uint64_t end = s + 1 < nseg ? seg_off[s + 1] : T;
    const uint32_t len = static_cast<uint32_t>(end - seg_off[s]);
    seg_len[s] = len;
    sched_keys[s] = (static_cast<unsigned long long>(0xFFFFFFFFu - len) << 32) | seg_word[s];
    sched_vals[s] = s;
    if (unit_count) unit_count[s] = (len + kUnitMaxTokens - 1) / kUnitMaxTokens;
}

cudaError_t launch_segment_lengths(const uint32_t* seg_off, uint32_t nseg, uint64_t T,
                                   uint32_t* seg_len, unsigned long long* sched_keys,
                                   uint32_t* sched_vals, const uint32_t* seg_word,
                                   uint32_t* unit_count, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    segment_lengths_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(seg_off, nseg, T, seg_len, sched_keys,
                                                             sched_vals, seg_word, unit_count);
    return cudaGetLastError();
}

// unit_count here is indexed by schedule position (permuted by the caller).
__global__ void emit_units_kernel(const uint32_t* schedule, const uint32_t* seg_word,
                                  const uint32_t* seg_off, const uint32_t* seg_len,
                                  const uint32_t* unit_start, uint32_t nseg, Unit* units) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nseg) return;
    const uint32_t s = schedule[p];
    const uint32_t len = seg_len[s];
    uint32_t u = unit_start[p];
    for (uint32_t o = 0; o < len; o += kUnitMaxTokens, ++u) {
        const uint32_t l = len - o < kUnitMaxTokens ? len - o : kUnitMaxTokens;
        units[u] = Unit{seg_word[s], seg_off[s] + o, l, 0u};
    }
}

cudaError_t launch_emit_units(const uint32_t* schedule, const uint32_t* seg_word,
                              const uint32_t* seg_off, const uint32_t* seg_len,
                              const uint32_t* unit_start, uint32_t nseg, Unit* units,
                              cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    emit_units_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(schedule, seg_word, seg_off, seg_len,
                                                        unit_start, nseg, units);
    return cudaGetLastError();
}

// C_dk row capacity in uint4 units: header + nnz_d entries with nnz_d <= len_d
// (test_counts.cpp:149-150), rounded up to 32 entries (one 128-byte line).
__global__ void row_quads_kernel(const uint32_t* doc_start, uint32_t D, uint32_t* quads) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    // Rounded up to a whole 128-byte line: every row starts line-aligned, so each 4-sector
    // group the sampler loads is exactly one L1 line (scripts/mb_pattern.cu: a third fewer
    // L1TEX wavefronts per loaded byte than 32-byte-aligned rows).
    quads[d] = ((((doc_start[d + 1] - doc_start[d] + 8u) >> 3) << 1) + 7u) & ~7u;
}

cudaError_t launch_row_quads(const uint32_t* doc_start, uint32_t D, uint32_t* quads, cudaStream_t s) {
    if (D == 0) return cudaSuccess;
    row_quads_kernel<<<(D + 255) / 256, 256, 0, s>>>(doc_start, D, quads);
    return cudaGetLastError();
}

// flags[d] = lo < length(d) <= hi
__global__ void long_flags_kernel(const uint32_t* doc_start, uint32_t D, uint32_t lo, uint32_t hi, uint32_t* flags) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    const uint32_t n = doc_start[d + 1] - doc_start[d];
    flags[d] = n > lo && n <= hi ? 1u : 0u;
}

cudaError_t launch_long_flags(const uint32_t* doc_start, uint32_t D, uint32_t lo, uint32_t hi, uint32_t* flags,
                              cudaStream_t s) {
    if (D == 0) return cudaSuccess;
    long_flags_kernel<<<(D + 255) / 256, 256, 0, s>>>(doc_start, D, lo, hi, flags);
    return cudaGetLastError();
}

__global__ void init_topics_kernel(uint64_t T, const uint64_t* ids, uint64_t id_base, uint64_t seed,
                                   uint32_t K, uint16_t* z) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t id = ids ? ids[j] : id_base + j;
        z[j] = static_cast<uint16_t>(uniform_topic(seed, kInitAssignStream, id, K));
    }
}

cudaError_t launch_init_topics(uint64_t T, const uint64_t* ids, uint64_t id_base, uint64_t seed,
                               uint32_t K, uint16_t* z, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    init_topics_kernel<<<grid_for(T, 256), 256, 0, s>>>(T, ids, id_base, seed, K, z);
    return cudaGetLastError();
}

__global__ void given_topics_kernel(const uint32_t* topic_in, const uint32_t* input_of_slot, uint64_t T,
                                    uint16_t* z) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        z[j] = static_cast<uint16_t>(topic_in[input_of_slot ? input_of_slot[j] : j]);
}

cudaError_t launch_given_topics(const uint32_t* topic_in, const uint32_t* input_of_slot, uint64_t T,
                                uint16_t* z, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    given_topics_kernel<<<grid_for(T, 256), 256, 0, s>>>(topic_in, input_of_slot, T, z);
    return cudaGetLastError();
}

__global__ void ids_by_slot_kernel(const uint64_t* ids_in, const uint32_t* input_of_slot, uint64_t T,
                                   uint64_t id_base, uint64_t* ids_out) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = input_of_slot ? input_of_slot[j] : j;
        ids_out[j] = ids_in ? ids_in[i] : id_base + i;
    }
}

cudaError_t launch_ids_by_slot(const uint64_t* ids_in, const uint32_t* input_of_slot, uint64_t T,
                               uint64_t id_base, uint64_t* ids_out, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    ids_by_slot_kernel<<<grid_for(T, 256), 256, 0, s>>>(ids_in, input_of_slot, T, id_base, ids_out);
    return cudaGetLastError();
}

// count_chunk_into (trainer.cpp:223-235) in word order.  With freshly drawn topics
// (init_assignments) the topic is recomputed from the token id -- the same Philox draw as
// init_topics_kernel -- instead of gathered from z by slot (a random 2-byte read per token).
__global__ void __launch_bounds__(256) recount_kernel(const uint2* tok, const Unit* units,
                                                      const uint16_t* z, uint32_t* B, uint32_t K_pad,
                                                      RecountDraw draw) {
    const Unit u = units[blockIdx.x];
    uint32_t* brow = B + static_cast<size_t>(u.word) * K_pad;
    for (uint32_t i = threadIdx.x; i < u.length; i += blockDim.x) {
        const uint32_t slot = tok[u.offset + i].y;
        uint32_t topic;
        if (draw.K) {
            const uint64_t id = draw.ids ? draw.ids[slot] : draw.id_base + slot;
            topic = uniform_topic(draw.seed, kInitAssignStream, id, draw.K);
        } else {
            topic = z[slot];
        }
        atomicAdd(brow + topic, 1u);
    }
}

cudaError_t launch_recount(const uint2* tok, const Unit* units, uint32_t n_units, const uint16_t* z,
                           uint32_t* B, uint32_t K_pad, RecountDraw draw, cudaStream_t s) {
    if (n_units == 0) return cudaSuccess;
    recount_kernel<<<n_units, 256, 0, s>>>(tok, units, z, B, K_pad, draw);
    return cudaGetLastError();
}

__global__ void validate_kernel(const uint32_t* __restrict__ aos, uint64_t T, uint32_t doc_begin,
                                uint32_t doc_end, uint32_t V, uint32_t K, ValidateOut* out) {
    // Per-thread minima, then one atomic per warp and quantity (a corpus of sentinel topics
    // would otherwise serialise T atomics on one address).
    unsigned long long bad_doc = ~0ull, bad_word = ~0ull, first_invalid = ~0ull, first_big = ~0ull;
    uint32_t unsorted = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t d = aos[3 * i], w = aos[3 * i + 1], t = aos[3 * i + 2];
        if ((d < doc_begin || d >= doc_end) && bad_doc == ~0ull) bad_doc = i;
        if (w >= V && bad_word == ~0ull) bad_word = i;
        if (t == kInvalidTopic) first_invalid = min(first_invalid, static_cast<unsigned long long>(i));
        else if (t >= K) first_big = min(first_big, static_cast<unsigned long long>(i));
        if (i > 0 && aos[3 * (i - 1)] > d) unsorted = 1u;
    }
    for (int o = 16; o > 0; o >>= 1) {
        bad_doc = min(bad_doc, __shfl_xor_sync(0xffffffffu, bad_doc, o));
        bad_word = min(bad_word, __shfl_xor_sync(0xffffffffu, bad_word, o));
        first_invalid = min(first_invalid, __shfl_xor_sync(0xffffffffu, first_invalid, o));
        first_big = min(first_big, __shfl_xor_sync(0xffffffffu, first_big, o));
        unsorted |= __shfl_xor_sync(0xffffffffu, unsorted, o);
    }
    if (lane_id() == 0) {
        if (bad_doc != ~0ull) atomicMin(&out->bad_doc, bad_doc);
        if (bad_word != ~0ull) atomicMin(&out->bad_word, bad_word);
        if (first_invalid != ~0ull) atomicMin(&out->first_invalid, first_invalid);
        if (first_big != ~0ull) atomicMin(&out->first_big, first_big);
        if (unsorted) out->unsorted = 1u;
    }
}

cudaError_t launch_validate(const uint32_t* aos, uint64_t T, uint32_t doc_begin, uint32_t doc_end,
                            uint32_t V, uint32_t K, ValidateOut* out, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    validate_kernel<<<grid_for(T, 256), 256, 0, s>>>(aos, T, doc_begin, doc_end, V, K, out);
    return cudaGetLastError();
}

__global__ void sched_counts_kernel(const uint32_t* schedule, const uint32_t* seg_len, uint32_t nseg,
                                    uint32_t* counts) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nseg) return;
    counts[p] = (seg_len[schedule[p]] + kUnitMaxTokens - 1) / kUnitMaxTokens;
}

cudaError_t launch_sched_counts(const uint32_t* schedule, const uint32_t* seg_len, uint32_t nseg,
                                uint32_t* counts, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    sched_counts_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(schedule, seg_len, nseg, counts);
    return cudaGetLastError();
}


// gather_assignments (trainer.cpp:203-213): slot-ordered u16 topics -> corpus-order u32.
// input_of_slot == null: doc-sorted corpus, slot == corpus position (a widening copy).
__global__ void assignments_kernel(const uint16_t* z, const uint32_t* input_of_slot, uint64_t T, uint32_t* out) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[input_of_slot ? input_of_slot[j] : j] = z[j];
}

cudaError_t launch_assignments(const uint16_t* z, const uint32_t* input_of_slot, uint64_t T, uint32_t* out,
                               cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    assignments_kernel<<<grid_for(T, 256), 256, 0, s>>>(z, input_of_slot, T, out);
    return cudaGetLastError();
}

}  // namespace slda
