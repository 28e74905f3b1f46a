// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI over the UNMODIFIED reference (`/root/reference/proj`), compiled
// together with the reference's own src/*.cpp by oracle/Makefile into
// oracle/_ref/libsparselda_ref.so.  Used (1) to pin the C oracle
// (tests/golden/make_golden.py), and (2) as bench.py's reference arm /
// cpu_baseline (kind "reference").  Nothing here is product code and no
// reference source is copied: this file only calls the reference API
// (trainer.hpp:172-182, eval.hpp:40-41, corpus.hpp:49-57).
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "sparselda/corpus.hpp"
#include "sparselda/counts.hpp"
#include "sparselda/eval.hpp"
#include "sparselda/rng.hpp"
#include "sparselda/sampler.hpp"
#include "sparselda/trainer.hpp"

using namespace sparselda;

namespace {
thread_local std::string g_error;

Corpus make_corpus(uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens) {
    Corpus c;
    c.num_docs = D;
    c.vocab_size = V;
    c.num_tokens = T;
    c.tokens.resize(T);
    std::memcpy(c.tokens.data(), tokens, sizeof(Token) * T);
    c.doc_lengths.assign(D, 0);
    c.word_freqs.assign(V, 0);
    for (const Token& t : c.tokens) {
        c.doc_lengths[t.doc] += 1;
        c.word_freqs[t.word] += 1;
    }
    return c;
}

struct RefModel {
    Corpus corpus;
    TrainConfig cfg;
    ModelState state;
    IterationStats last;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

void ref_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const auto o = philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = o[i];
}

void ref_uniform2(uint64_t seed, uint32_t kind, uint64_t element, double* u0, double* u1) {
    RngStream s(seed, kind, element);
    *u0 = s.next_double();
    *u1 = s.next_double();
}

// workers: 0 = hardware concurrency; chunks: 0 = auto (budget 2^40 -> 1);
// sampler: 0 SamplerKind::kSparse, 1 SamplerKind::kVanilla (trainer.hpp:18).
void* ref_init_sampler(uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens, uint32_t K,
                       double alpha, double beta, uint64_t seed, uint32_t num_chunks, uint32_t workers,
                       uint32_t sampler) {
    try {
        auto* m = new RefModel;
        m->corpus = make_corpus(D, V, T, tokens);
        m->cfg.num_topics = K;
        m->cfg.alpha = alpha;
        m->cfg.beta = beta;
        m->cfg.seed = seed;
        m->cfg.num_chunks = num_chunks;
        m->cfg.num_workers = workers;
        m->cfg.memory_budget = 1ull << 40;  // never spill
        m->cfg.tree_branch = K > 32768 ? 41 : 32;
        m->cfg.sampler = sampler ? SamplerKind::kVanilla : SamplerKind::kSparse;
        m->cfg = m->cfg.resolved(m->corpus);
        m->state = init_state(m->corpus, m->cfg);
        return m;
    } catch (const std::exception& e) {
        g_error = e.what();
        return nullptr;
    }
}

void* ref_init(uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens, uint32_t K,
               double alpha, double beta, uint64_t seed, uint32_t num_chunks, uint32_t workers) {
    return ref_init_sampler(D, V, T, tokens, K, alpha, beta, seed, num_chunks, workers, 0);
}

void ref_free(void* h) { delete static_cast<RefModel*>(h); }

int ref_iterate(void* h, double* elapsed_s, double* mean_doc_topics) {
    auto* m = static_cast<RefModel*>(h);
    try {
        m->last = run_iteration(m->state, m->cfg);
        if (elapsed_s) *elapsed_s = m->last.elapsed_s;
        if (mean_doc_topics) *mean_doc_topics = m->last.mean_doc_topics;
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

uint32_t ref_num_workers(void* h) { return static_cast<RefModel*>(h)->cfg.num_workers; }
uint32_t ref_num_chunks(void* h) { return static_cast<RefModel*>(h)->cfg.num_chunks; }
double ref_alpha(void* h) { return static_cast<RefModel*>(h)->state.alpha; }

void ref_get_word_topic(void* h, uint32_t* out) {
    auto& s = static_cast<RefModel*>(h)->state;
    for (uint32_t v = 0; v < s.vocab_size; ++v) {
        const auto row = s.word_topic.row(v);
        std::memcpy(out + static_cast<size_t>(v) * s.num_topics, row.data(), 4 * row.size());
    }
}

void ref_get_word_topic_prob(void* h, float* out) {
    auto& s = static_cast<RefModel*>(h)->state;
    for (uint32_t v = 0; v < s.vocab_size; ++v) {
        const auto row = s.word_topic_prob.row(v);
        std::memcpy(out + static_cast<size_t>(v) * s.num_topics, row.data(), 4 * row.size());
    }
}

// Real (un-padded) L4 prefix of every word's tree, sampler.hpp:119.
void ref_get_l4(void* h, float* out) {
    auto& s = static_cast<RefModel*>(h)->state;
    for (uint32_t v = 0; v < s.vocab_size; ++v) {
        const auto p = s.trees[v].prefix();
        std::memcpy(out + static_cast<size_t>(v) * s.num_topics, p.data(), 4 * p.size());
    }
}

void ref_get_tree_mass(void* h, float* out) {
    auto& s = static_cast<RefModel*>(h)->state;
    std::memcpy(out, s.tree_mass.data(), 4 * s.tree_mass.size());
}

void ref_get_assignments(void* h, uint32_t* out) {
    auto& s = static_cast<RefModel*>(h)->state;
    const auto a = s.gather_assignments();
    std::memcpy(out, a.data(), 4 * a.size());
}

// Doc-topic rows concatenated over chunks in doc order.
uint64_t ref_doc_topic_nnz(void* h) {
    auto& s = static_cast<RefModel*>(h)->state;
    uint64_t nnz = 0;
    for (size_t c = 0; c < s.chunks.size(); ++c) {
        const ChunkSlot& slot = s.chunks.acquire(c);
        nnz += slot.doc_topic_dense.empty() ? slot.doc_topic.nnz() : slot.doc_topic_dense.nnz();
    }
    return nnz;
}

void ref_get_doc_topic(void* h, uint64_t* row_offsets, uint32_t* topics, uint32_t* counts) {
    auto& s = static_cast<RefModel*>(h)->state;
    uint64_t pos = 0;
    uint32_t row = 0;
    row_offsets[0] = 0;
    for (size_t c = 0; c < s.chunks.size(); ++c) {
        const ChunkSlot& slot = s.chunks.acquire(c);
        if (!slot.doc_topic_dense.empty()) {  // vanilla mode: the dense rows' nonzero cells
            for (uint32_t d = 0; d < slot.doc_topic_dense.num_rows(); ++d) {
                const auto r = slot.doc_topic_dense.row(d);
                for (uint32_t k = 0; k < r.size(); ++k) {
                    if (!r[k]) continue;
                    topics[pos] = k;
                    counts[pos] = r[k];
                    ++pos;
                }
                row_offsets[++row] = pos;
            }
            continue;
        }
        for (uint32_t d = 0; d < slot.doc_topic.num_rows(); ++d) {
            const auto r = slot.doc_topic.row(d);
            for (size_t i = 0; i < r.size(); ++i) {
                topics[pos] = r.topics[i];
                counts[pos] = r.counts[i];
                ++pos;
            }
            row_offsets[++row] = pos;
        }
    }
}

// PDOW of chunk c (corpus.cpp:125-198) with its schedule order applied
// (init_state calls build_schedule, trainer.cpp:389).
uint32_t ref_chunk_size(void* h, uint32_t c) {
    return static_cast<RefModel*>(h)->state.chunks.acquire(c).chunk.size();
}
uint32_t ref_chunk_segments(void* h, uint32_t c) {
    return static_cast<uint32_t>(
        static_cast<RefModel*>(h)->state.chunks.acquire(c).chunk.word_segments.size());
}
void ref_get_chunk(void* h, uint32_t c, uint32_t* doc_range, uint32_t* sorted_doc,
                   uint32_t* sorted_word, uint32_t* token_ids, uint32_t* shuffle_ptrs,
                   uint32_t* doc_offsets, uint32_t* seg_word, uint32_t* seg_offset,
                   uint32_t* seg_length) {
    const Chunk& ch = static_cast<RefModel*>(h)->state.chunks.acquire(c).chunk;
    doc_range[0] = ch.doc_begin;
    doc_range[1] = ch.doc_end;
    for (uint32_t i = 0; i < ch.size(); ++i) {
        sorted_doc[i] = ch.tokens[i].doc;
        sorted_word[i] = ch.tokens[i].word;
        token_ids[i] = ch.token_ids[i];
        shuffle_ptrs[i] = ch.shuffle_ptrs[i];
    }
    std::memcpy(doc_offsets, ch.doc_offsets.data(), 4 * ch.doc_offsets.size());
    for (size_t s = 0; s < ch.word_segments.size(); ++s) {
        seg_word[s] = ch.word_segments[s].word;
        seg_offset[s] = ch.word_segments[s].offset;
        seg_length[s] = ch.word_segments[s].length;
    }
}

int ref_heldout_ll(void* h, uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens,
                   uint32_t burn_in, uint32_t workers, uint64_t seed, double* per_token_ll,
                   uint64_t* tokens_evaluated) {
    try {
        auto* m = static_cast<RefModel*>(h);
        const Corpus held = make_corpus(D, V, T, tokens);
        const HeldoutSet set = HeldoutSet::from_corpus(held);
        const EvalReport r = heldout_ll(m->state, set, burn_in, workers, seed);
        *per_token_ll = r.per_token_ll;
        *tokens_evaluated = r.tokens_evaluated;
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// save_checkpoint (trainer.cpp:469-478) of the reference model: the byte format the device
// checkpoint must reproduce (acceptance criterion 7, acceptance.cpp:389-421).
int ref_save_checkpoint(void* h, const char* path) {
    try {
        save_checkpoint(path, static_cast<RefModel*>(h)->state);
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// load_docword (corpus.cpp:30-68) over a text buffer: the token count (tokens copied up to
// cap, T x 3 uint32), or -1 with the reference's message in ref_last_error().
int64_t ref_load_docword(const char* text, uint64_t n, uint32_t* tokens, uint64_t cap) {
    try {
        std::istringstream in(std::string(text, n));
        const Corpus c = load_docword(in);
        const uint64_t m = c.tokens.size() < cap ? c.tokens.size() : cap;
        if (tokens && m) std::memcpy(tokens, c.tokens.data(), sizeof(Token) * m);
        return static_cast<int64_t>(c.tokens.size());
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// Building blocks exposed for known-answer tests.
uint32_t ref_segmented_count(const uint32_t* seg, uint32_t n, uint32_t* topics, uint32_t* counts) {
    const SparseTopicRow r = segmented_count(std::span<const TopicId>(seg, n));
    for (size_t i = 0; i < r.size(); ++i) {
        topics[i] = r.topics[i];
        counts[i] = r.counts[i];
    }
    return static_cast<uint32_t>(r.size());
}

int ref_preprocess(uint32_t V, uint32_t K, const uint32_t* b, double beta, float* out) {
    try {
        WordTopicMatrix m(V, K);
        for (uint32_t v = 0; v < V; ++v)
            for (uint32_t k = 0; k < K; ++k) m.cell(v, k) = b[static_cast<size_t>(v) * K + k];
        const WordTopicProb p = preprocess(m, beta, 1);
        for (uint32_t v = 0; v < V; ++v) {
            const auto row = p.row(v);
            std::memcpy(out + static_cast<size_t>(v) * K, row.data(), 4 * K);
        }
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

// sample_token<float> with the reference's own tree (sampler.hpp:183-204).
uint32_t ref_sample_token(uint32_t nnz, const uint32_t* topics, const uint32_t* counts,
                          const float* bhat_row, uint32_t K, float alpha, uint64_t seed,
                          uint32_t kind, uint64_t element) {
    const auto built = build_tree<float>(std::span<const float>(bhat_row, K), alpha,
                                         K > 32768 ? 41 : 32);
    std::vector<float> scratch;
    RngStream rng(seed, kind, element);
    SparseTopicRowView view{{topics, nnz}, {counts, nnz}};
    return sample_token<float>(view, std::span<const float>(bhat_row, K), built.q, built.tree,
                               rng, scratch);
}

}  // extern "C"
