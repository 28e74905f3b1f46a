// Corpus and chunk types of the reference API (corpus.hpp:12-72).  The Corpus and its loaders
// are sparselda_b200's (multi-threaded UCI ingest, identical tokens and error messages);
// build_chunks derives the PDOW layout from the engine's device build (slda_get_pdow).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <string>
#include <utility>
#include <vector>

#include "sparselda/types.hpp"

namespace sparselda {

// A distinct type (not an alias) so that unqualified calls such as init_state(corpus, cfg)
// resolve to this namespace's overloads rather than ambiguously also to sparselda_b200's.
struct Corpus : sparselda_b200::Corpus {
    Corpus() = default;
    Corpus(sparselda_b200::Corpus&& c) : sparselda_b200::Corpus(std::move(c)) {}
    Corpus(const sparselda_b200::Corpus& c) : sparselda_b200::Corpus(c) {}
};

Corpus load_uci(std::istream& docword, std::istream& vocab);
Corpus load_docword(std::istream& docword);
void init_assignments(Corpus& corpus, std::uint32_t num_topics, std::uint64_t seed);

struct WordSegment {  // one word's run inside a chunk's word-major order
    WordId word;
    std::uint32_t offset;
    std::uint32_t length;
};

// A contiguous document range in PDOW (word-major) order, with the permutation back to the
// document-grouped order.
struct Chunk {
    DocId doc_begin = 0;
    DocId doc_end = 0;
    std::vector<Token> tokens;
    std::vector<std::uint32_t> token_ids;
    std::vector<WordSegment> word_segments;
    std::vector<std::uint32_t> shuffle_ptrs;
    std::vector<std::uint32_t> doc_offsets;

    std::uint32_t doc_count() const { return doc_end - doc_begin; }
    std::uint32_t size() const { return static_cast<std::uint32_t>(tokens.size()); }
};

std::vector<Chunk> build_chunks(const Corpus& corpus, std::uint32_t num_chunks);
std::vector<WordId> build_schedule(Chunk& chunk);
std::uint32_t auto_num_chunks(const Corpus& corpus, std::uint32_t num_topics, std::uint64_t budget_bytes);

}  // namespace sparselda
