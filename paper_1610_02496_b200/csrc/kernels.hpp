// kernels.hpp -- host launchers for the ESCA device kernels (sampler.cu, ssc.cu, mstep.cu, setup.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace slda {

// Sampler work unit: one (word, token range) slice of a PDOW word segment.
// Heavy words are split into several units (PAPER.md:621-636 heavy-first).
struct Unit {
    uint32_t word, offset, length, pad;
};

constexpr uint32_t kUnitMaxTokens = 8192;  // sampler: max tokens per unit (one CTA)
constexpr uint32_t kSscWarpCap = 512;      // SSC: docs up to this length take the warp path
constexpr uint32_t kSscMidCap = 2048;      // SSC: longer ones up to this take the medium warp pass

struct SamplerArgs {
    const uint2* tok;       // execution order: {C_dk row offset in uint4 units, slot}
    const Unit* units;      // heavy-first
    const uint32_t* A;      // C_dk rows: [nnz-1 | entries topic | count << tbits | zero pad to 8]
    const float* bhat;      // V_pad x K_pad
    const float* l8;        // V_pad x l8_stride (L4 block maxima)
    const float* q;         // V_pad
    const uint64_t* ids;    // RNG element id per slot, or null -> id_base + slot
    uint16_t* z;            // new topic per slot
    uint32_t* B;            // V_pad x K_pad, zeroed by the caller
    uint64_t seed, id_base;
    uint32_t stream_kind;   // iteration number (trainer.cpp:423)
    uint32_t K, K_pad, l8_stride, n_l8, tbits;
    unsigned long long* row_entries;  // optional: sum of nnz over tokens (roofline)
    int shape;              // launch shape (sampler_shape_from_name); -1 = default by K
    uint32_t vanilla;       // SamplerKind::kVanilla: the O(K) dense-row draw (sampler.hpp:222-236)
    float alpha;            // f32(alpha), the vanilla draw's smoothing (trainer.cpp:283)
    // z staging (resident engines): the new topic of execution position i goes to
    // zx[zx_pos ? zx_pos[i] : i] instead of z[slot] -- coalesced stores; launch_zmove then
    // brings the topics to z by slot (zmove.cu).  Null: z[slot] directly (streaming chunks).
    uint16_t* zx;
    const uint32_t* zx_pos;
    uint32_t async_next;    // prefetching quad kernels: the next round's first line by cp.async into shared
                            // memory a round ahead (default; SLDA_ASYNC_NEXT=0: in registers, a group ahead)
};

// Sampler launch shapes (sampler.cu launch_sampler); -1 = by phi row size.
enum { kShapeRound = 0, kShapeQuad512 = 1, kShapeQuad256 = 2, kShapeGlobal = 3, kShapeVanilla = 4 };
int sampler_shape_from_name(const char* name);
// The kernel launch_sampler runs for these arguments (a.shape: forced shape or -1).
int sampler_shape(const SamplerArgs& a);

cudaError_t launch_sampler(const SamplerArgs& a, uint32_t n_units, cudaStream_t s);

// ---- z transpose (zmove.cu): execution order -> slot order in three coalesced passes ---------
constexpr uint32_t kZChunkLog2 = 14;  // permute chunk: 16384 entries (32 KB of topics in smem)
constexpr uint32_t kZTileLog2 = 14;   // final tile: 16384 slots
// Per chunk of 16384 positions: out[zbase[run] + k] = src[chunk base + (zsk[k] & 16383)] for every
// sorted position k of the chunk, run = zsk[k] >> 14 (a run's destinations are consecutive): each
// CTA stages a chunk of src in shared memory and stores it in runs.
cudaError_t launch_zpermute(const uint16_t* src, const uint32_t* zsk, const uint32_t* zbase, uint32_t R, uint64_t T,
                            uint16_t* out, cudaStream_t s);
// z[tile base + loc[m]] = zf[m] per 16384-slot tile, through shared memory.
cudaError_t launch_ztile(const uint16_t* zf, const uint16_t* loc, uint64_t T, uint16_t* z, cudaStream_t s);
// Setup of the static tables (two levels): per-(key, chunk) counts into a flat array in
// destination order (its exclusive scan gives each run's first destination), then the stable
// per-chunk ranking that writes zsk (source index | run << 14), the chunk's run table (zbase: R
// u32) and slot_of (level 1) or the tile-local slots (level 2).
size_t zlayout_flat_size(uint64_t T, uint32_t shift, uint32_t level);
uint32_t zlayout_keys(uint64_t T, uint32_t shift, uint32_t level);  // R: runs per chunk
cudaError_t launch_zlayout_count(const uint2* tok, const uint32_t* slot_of, uint64_t T, uint32_t shift,
                                 uint32_t level, uint32_t* cnt, size_t flat, cudaStream_t s);
cudaError_t launch_zlayout_emit(const uint2* tok, const uint32_t* slot_of, uint64_t T, uint32_t shift, uint32_t level,
                                const uint32_t* off, uint32_t* zsk, uint32_t* zbase, uint32_t* slot_of_out,
                                uint16_t* loc_out, cudaStream_t s);

struct SscArgs {
    const uint16_t* z;          // topics by slot (doc-grouped)
    const uint32_t* doc_start;  // D+1 slot offsets
    uint32_t D;
    const uint32_t* row4;       // per doc: row offset in uint4 units
    uint32_t* A;
    uint32_t tbits, K_pad;
    const uint32_t* long_docs;  // docs longer than kSscWarpCap: the n_huge > kSscMidCap first
    uint32_t n_long, n_huge;
    uint32_t* hist_scratch;     // n_long_ctas x K_pad (global fallback for large K)
    unsigned long long* nnz_total;
};

cudaError_t launch_ssc(const SscArgs& a, cudaStream_t s);

cudaError_t launch_colsum(const uint32_t* B, uint32_t row_begin, uint32_t row_end, uint32_t K_pad,
                          unsigned long long* colsum, cudaStream_t s);
// C_k as the histogram of the topics (engines holding all of C_wk's tokens); zhist_fits:
// the K_pad bins fit shared memory.
bool zhist_fits(uint32_t K_pad);
cudaError_t launch_zhist(const uint16_t* z, uint64_t T, uint32_t K_pad, unsigned long long* colsum, cudaStream_t s);
// denom: 2*K_pad doubles -- denom_k, then RN(1/denom_k) (read by the phi kernel).
cudaError_t launch_denom(const unsigned long long* colsum, uint32_t K, uint32_t K_pad, uint32_t V,
                         double beta, double* denom, float* zv, cudaStream_t s);
// Peer-memory exchange (engine.cu m_step_peer): up to kMaxPeers ranks, C_wk exchanged as
// sparse per-row entries (topic | count << 16) with a {offset, n} index per row.
constexpr uint32_t kMaxPeers = 8;
struct SparseRows {
    const uint2* info;        // per row: {entry offset, entry count}, indexed by row - base
    const uint32_t* entries;
    uint32_t base;
};
struct PeerSparse {
    SparseRows src[kMaxPeers];
    uint32_t n;
};
cudaError_t launch_phi(const uint32_t* B, const double* denom, const float* zv, float* bhat,
                       float* l8, float* q, uint32_t row_begin, uint32_t row_end,
                       uint32_t K, uint32_t K_pad, uint32_t l8_stride, double beta, float falpha,
                       cudaStream_t s);
// L4 (the inclusive f32 prefix of every phi row) materialised for the getter.
cudaError_t launch_l4(const float* bhat, uint32_t rows, uint32_t K_pad, float* l4, cudaStream_t s);
cudaError_t launch_peer_barrier(unsigned long long* counter, unsigned long long target, cudaStream_t s);
cudaError_t launch_sparsify(const uint32_t* B, uint32_t row_lo, uint32_t row_hi, uint32_t K_pad, uint2* info,
                            uint32_t* entries, uint32_t* cursor, uint32_t cap, uint32_t* overflow, cudaStream_t s);
cudaError_t launch_gather_add(const PeerSparse& ps, uint32_t row_lo, uint32_t row_hi, uint32_t skip_lo,
                              uint32_t skip_hi, uint32_t per_slice, uint32_t* B, uint32_t K_pad,
                              unsigned long long* bytes, cudaStream_t s);

// Setup kernels.
cudaError_t launch_deinterleave(const uint32_t* aos, uint64_t T, uint32_t doc_begin,
                                uint32_t* doc_local, uint32_t* word, uint32_t* topic,
                                cudaStream_t s);
cudaError_t launch_check_sorted(const uint32_t* doc_local, uint64_t T, uint32_t* unsorted_flag,
                                cudaStream_t s);
cudaError_t launch_doc_hist(const uint32_t* doc_local, uint64_t T, uint32_t* counts,
                            cudaStream_t s);
cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t s);
cudaError_t launch_invert_perm(const uint32_t* input_of_slot, uint64_t T, uint32_t* slot_of_input,
                               cudaStream_t s);
struct KeyLayout {
    uint32_t dbits, lbits, lmax;  // doc bits, length bits (0 = canonical order), max length
};
cudaError_t launch_make_keys(const uint32_t* word, const uint32_t* doc_local, const uint32_t* input_of_slot,
                             const uint32_t* doc_len, uint64_t T, KeyLayout kl, unsigned long long* keys,
                             uint32_t* vals, cudaStream_t s);
cudaError_t launch_make_tok(const unsigned long long* keys, const uint32_t* slots, const uint32_t* row4,
                            uint64_t T, KeyLayout kl, uint2* tok, uint32_t* seg_flag, cudaStream_t s);
cudaError_t launch_emit_segments(const unsigned long long* keys, const uint32_t* seg_flag,
                                 const uint32_t* seg_index, uint64_t T, uint32_t wshift,
                                 uint32_t* seg_word, uint32_t* seg_off, cudaStream_t s);
cudaError_t launch_segment_lengths(const uint32_t* seg_off, uint32_t nseg, uint64_t T,
                                   uint32_t* seg_len, unsigned long long* sched_keys,
                                   uint32_t* sched_vals, const uint32_t* seg_word,
                                   uint32_t* unit_count, cudaStream_t s);
cudaError_t launch_emit_units(const uint32_t* schedule, const uint32_t* seg_word,
                              const uint32_t* seg_off, const uint32_t* seg_len,
                              const uint32_t* unit_start, uint32_t nseg, Unit* units,
                              cudaStream_t s);
cudaError_t launch_row_quads(const uint32_t* doc_start, uint32_t D, uint32_t* quads,
                             cudaStream_t s);
cudaError_t launch_long_flags(const uint32_t* doc_start, uint32_t D, uint32_t lo, uint32_t hi, uint32_t* flags,
                              cudaStream_t s);
cudaError_t launch_init_topics(uint64_t T, const uint64_t* ids, uint64_t id_base, uint64_t seed,
                               uint32_t K, uint16_t* z, cudaStream_t s);
cudaError_t launch_given_topics(const uint32_t* topic_in, const uint32_t* input_of_slot,
                                uint64_t T, uint16_t* z, cudaStream_t s);
cudaError_t launch_ids_by_slot(const uint64_t* ids_in, const uint32_t* input_of_slot, uint64_t T,
                               uint64_t id_base, uint64_t* ids_out, cudaStream_t s);
// Range checks + the reference's topic rule (trainer.cpp:369-378): records the first
// token index with an invalid topic and the first with topic >= K.
struct ValidateOut {
    unsigned long long first_invalid, first_big, bad_doc, bad_word;
    uint32_t unsorted;
};
cudaError_t launch_validate(const uint32_t* aos, uint64_t T, uint32_t doc_begin, uint32_t doc_end,
                            uint32_t V, uint32_t K, ValidateOut* out, cudaStream_t s);
cudaError_t launch_sched_counts(const uint32_t* schedule, const uint32_t* seg_len, uint32_t nseg,
                                uint32_t* counts, cudaStream_t s);
// gather_assignments: u16 topics by slot -> u32 topics in corpus order.
cudaError_t launch_assignments(const uint16_t* z, const uint32_t* input_of_slot, uint64_t T, uint32_t* out,
                               cudaStream_t s);
// K != 0: the topics are init_assignments draws (recomputed from the token ids, not read from z).
struct RecountDraw {
    uint64_t seed, id_base;
    const uint64_t* ids;
    uint32_t K;
};
cudaError_t launch_recount(const uint2* tok, const Unit* units, uint32_t n_units,
                           const uint16_t* z, uint32_t* B, uint32_t K_pad, RecountDraw draw, cudaStream_t s);

}  // namespace slda
