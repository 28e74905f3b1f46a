// sparselda_b200.hpp -- the reference's C++ API (`sparselda::`, proj/include/sparselda/*.hpp)
// re-declared over the B200 engine's C-ABI (include/saberlda.h).
//
// Same names, argument meaning and error behaviour as the reference so a caller
// switches with `namespace sparselda = sparselda_b200;`.  Differences: the
// model state lives in HBM, so ModelState exposes its matrices through
// copying getters instead of public members; num_workers / memory_budget /
// spill_dir are accepted and validated but have no effect (results never
// depended on them: acceptance.cpp:389-445); num_chunks > 1 with a corpus state
// above device_budget streams the chunks through the GPU (out-of-core).
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
#include <iosfwd>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "saberlda.h"

namespace sparselda_b200 {

inline constexpr const char* kVersion = "0.1.0";

using DocId = std::uint32_t;
using WordId = std::uint32_t;
using TopicId = std::uint32_t;
inline constexpr TopicId kInvalidTopic = 0xFFFFFFFFu;  // types.hpp:17

struct Token {  // types.hpp:21-25 (same layout: the C-ABI takes it as-is)
    DocId doc;
    WordId word;
    TopicId topic;
};
static_assert(sizeof(Token) == 12, "Token must match sparselda::Token");

struct ValidationError : std::runtime_error {  // types.hpp:28-30
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {  // types.hpp:33-35
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {  // CUDA / NCCL failure
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

// Throws the exception matching a C-ABI status code.
void check(int status);

// ---------------------------------------------------------------- corpus --
struct Corpus {  // corpus.hpp:12-20
    std::uint32_t num_docs = 0;
    std::uint32_t vocab_size = 0;
    std::uint64_t num_tokens = 0;
    std::vector<Token> tokens;
    std::vector<std::uint32_t> doc_lengths;
    std::vector<std::uint64_t> word_freqs;
    std::vector<std::string> vocab;

    void finalize();  // recompute num_tokens, doc_lengths, word_freqs
};

Corpus load_uci(std::istream& docword, std::istream& vocab);        // corpus.hpp:49
Corpus load_docword(std::istream& docword);                          // corpus.hpp:53
// The same over an in-memory (or mapped) docword file; parses with all host threads.
Corpus load_docword_buffer(const char* data, std::size_t size);
// load_uci over files (the docword file memory-mapped); IoError when either cannot be opened.
Corpus load_uci_files(const std::string& docword_path, const std::string& vocab_path);
void load_vocab(Corpus& corpus, std::istream& vocab);
void init_assignments(Corpus& corpus, std::uint32_t num_topics, std::uint64_t seed);  // :57
// Synthetic corpora; family 0 = G, 1 = U.
Corpus generate_corpus(const slda_gen_params& params);

// ---------------------------------------------------------------- config --
enum class SamplerKind { kSparse, kVanilla };

struct TrainConfig {  // trainer.hpp:20-36
    std::uint32_t num_topics = 0;
    double alpha = 0.0;
    double beta = 0.01;
    std::uint32_t iterations = 100;
    std::uint32_t num_chunks = 0;
    unsigned num_workers = 0;
    std::uint64_t seed = 0;
    std::uint64_t memory_budget = 1ull << 30;
    std::uint32_t eval_every = 0;
    SamplerKind sampler = SamplerKind::kSparse;
    std::uint32_t tree_branch = 32;
    std::string spill_dir;
    int device = -1;  // CUDA ordinal (-1: current)
    // Device memory the corpus state may use (0: the free memory).  With num_chunks > 1 and a
    // larger state the engine streams its chunks through the GPU (slda_config.device_budget).
    std::uint64_t device_budget = 0;

    TrainConfig resolved(const Corpus& corpus) const;  // trainer.cpp:15-35
};

struct IterationStats {  // trainer.hpp:38-44
    std::uint32_t iteration = 0;
    std::uint64_t tokens = 0;
    double elapsed_s = 0.0;
    double mtokens_per_s = 0.0;
    double mean_doc_topics = 0.0;
    double device_ms = 0.0;
};

struct MetricsEntry {
    IterationStats stats;
    std::optional<double> heldout_ll;
};
std::string format_metrics_line(const MetricsEntry& entry);  // trainer.cpp:37-47
using MetricsSink = std::function<void(const MetricsEntry&)>;

// One document's sorted (topic, count) pairs (counts.hpp:14-24).
struct SparseTopicRow {
    std::vector<TopicId> topics;
    std::vector<std::uint32_t> counts;
    std::size_t size() const { return topics.size(); }
};

// CSR C_dk over the model's documents (counts.hpp:33-80).
struct DocTopicMatrix {
    std::vector<std::uint64_t> row_offsets;
    std::vector<TopicId> topics;
    std::vector<std::uint32_t> counts;
    std::uint32_t num_rows() const {
        return row_offsets.empty() ? 0 : static_cast<std::uint32_t>(row_offsets.size() - 1);
    }
    std::uint64_t nnz() const { return topics.size(); }
};

// The single-chunk PDOW layout (corpus.hpp:33-43) of the engine's shard.
struct ChunkLayout {
    DocId doc_begin = 0, doc_end = 0;
    std::vector<DocId> sorted_doc;
    std::vector<WordId> sorted_word;
    std::vector<std::uint64_t> token_ids;
    std::vector<std::uint32_t> shuffle_ptrs, doc_offsets;
    std::vector<WordId> seg_word;             // ascending word
    std::vector<std::uint32_t> seg_offset, seg_length;
    std::vector<std::uint32_t> schedule;      // heavy-first segment indices (build_schedule)
};

// ---------------------------------------------------------------- model --
class ModelState {  // trainer.hpp:149-166
public:
    ModelState() = default;
    ModelState(ModelState&&) noexcept = default;
    ModelState& operator=(ModelState&&) noexcept = default;

    std::uint32_t num_docs = 0;
    std::uint32_t vocab_size = 0;
    std::uint64_t num_tokens = 0;
    std::uint32_t num_topics = 0;
    double alpha = 0.0;
    double beta = 0.0;
    std::uint64_t seed = 0;
    std::uint32_t iteration = 0;
    SamplerKind sampler = SamplerKind::kSparse;  // TrainConfig::sampler at init (trainer.hpp:30)

    // B, B-hat, Q, L4 (V x K row-major / V) copied from the device.
    std::vector<std::uint32_t> word_topic() const;
    std::vector<float> word_topic_prob() const;
    std::vector<float> tree_mass() const;
    std::vector<float> tree_prefix() const;
    std::vector<TopicId> gather_assignments() const;  // trainer.cpp:203-213
    DocTopicMatrix doc_topic() const;
    ChunkLayout chunk_layout() const;
    slda_kernel_times kernel_times() const;
    slda_info info() const;
    bool has_chunks() const { return has_chunks_; }

    slda_engine* engine() const { return engine_.get(); }

private:
    struct Deleter {
        void operator()(slda_engine* e) const { slda_destroy(e); }
    };
    std::unique_ptr<slda_engine, Deleter> engine_;
    bool has_chunks_ = false;

    friend ModelState init_state(const Corpus&, const TrainConfig&);
    friend ModelState init_shard(const Corpus&, const TrainConfig&, std::uint32_t, std::uint32_t);
    friend ModelState init_view(const slda_corpus_view&, const TrainConfig&, std::uint32_t, std::uint32_t,
                                std::uint32_t);
    friend ModelState model_from_counts(std::uint32_t, std::uint32_t, const std::vector<std::uint32_t>&,
                                        std::uint64_t, std::uint32_t, double, double, std::uint64_t, int);
    friend IterationStats run_iteration(ModelState&, const TrainConfig&);
};

ModelState init_state(const Corpus& corpus, const TrainConfig& cfg);          // trainer.hpp:172
// Document shard `rank` of `world` (one process per GPU, peer-memory exchange over NVLink): the shard
// is the rank-th contiguous document range of the chunk_boundaries rule
// (corpus.cpp:103-121).  Collective over all ranks.
std::vector<std::uint32_t> shard_bounds(const Corpus& corpus, std::uint32_t world);
ModelState init_shard(const Corpus& corpus, const TrainConfig& cfg, std::uint32_t rank,
                      std::uint32_t world);
// Engine over a borrowed corpus view (already sharded by the caller); the config is
// validated as TrainConfig::resolved would for a corpus of view.num_docs documents.
ModelState init_view(const slda_corpus_view& view, const TrainConfig& cfg, std::uint32_t rank,
                     std::uint32_t world, std::uint32_t init_mode);
IterationStats run_iteration(ModelState& state, const TrainConfig& cfg);      // trainer.hpp:177
using HeldoutProbe = std::function<double(ModelState&)>;
ModelState train(const Corpus& corpus, const TrainConfig& cfg, const MetricsSink& sink = {},
                 const HeldoutProbe& heldout_probe = {});                    // trainer.hpp:181-182
ModelState model_from_counts(std::uint32_t vocab_size, std::uint32_t num_topics,
                             const std::vector<std::uint32_t>& word_topic, std::uint64_t num_tokens,
                             std::uint32_t iteration, double alpha, double beta, std::uint64_t seed,
                             int device = -1);

// ---------------------------------------------------------------- eval --
struct EvalReport {  // eval.hpp:31-35
    double per_token_ll = 0.0;
    std::uint64_t tokens_evaluated = 0;
    std::uint32_t iteration = 0;
};
std::string format_eval_line(const EvalReport& report);
// heldout_ll (eval.hpp:40-41) on device; the corpus is split by HeldoutSet::from_corpus.
EvalReport heldout_ll(ModelState& model, const Corpus& heldout, std::uint32_t burn_in = 20,
                      unsigned workers = 1, std::uint64_t seed = 0);
double throughput_mtokens(std::uint64_t tokens, double elapsed_s);
std::vector<std::vector<std::pair<WordId, float>>> top_words(const ModelState& model, std::uint32_t n);
// "topic k: word:prob ..." per topic (eval.cpp:163-181); vocab entries empty or missing print the id.
void print_topics(std::ostream& out, const ModelState& model, const std::vector<std::string>& vocab,
                  std::uint32_t n);

// ------------------------------------------------------ building blocks --
SparseTopicRow segmented_count(std::span<const TopicId> segment);  // counts.cpp:65-94
std::size_t prefix_search(std::span<const double> prefix, double x);  // sampler.hpp:18-41
class WaryTree {  // sampler.hpp:50-134 (double, as the Python binding)
public:
    explicit WaryTree(std::span<const double> weights, std::uint32_t branch = 32);
    std::uint32_t sample(double x) const;
    double total() const { return total_; }
    std::uint32_t size() const { return size_; }
    std::uint32_t branch() const { return branch_; }
    const std::vector<double>& level2() const { return top_; }
    const std::vector<double>& level3() const { return mid_; }
    const std::vector<double>& level4() const { return bottom_; }

private:
    std::uint32_t branch_ = 32, size_ = 0;
    double total_ = 0;
    std::vector<double> top_, mid_, bottom_;
};

// ---------------------------------------------------------- checkpoints --
struct Checkpoint {  // trainer.hpp:184-195
    std::uint32_t num_docs = 0, vocab_size = 0;
    std::uint64_t num_tokens = 0;
    std::uint32_t num_topics = 0, iteration = 0;
    double alpha = 0.0, beta = 0.0;
    std::uint64_t seed = 0;
    std::vector<TopicId> assignments;
    std::vector<std::uint32_t> word_topic;  // V x K
};
void save_checkpoint(const std::filesystem::path& path, const ModelState& state);  // trainer.cpp:469-478
Checkpoint load_checkpoint(const std::filesystem::path& path);                     // trainer.cpp:480-512
ModelState model_from_checkpoint(const Checkpoint& ckpt, unsigned workers = 0);    // trainer.cpp:514-532
// Resume training bit-identically: corpus topics from the checkpoint and the RNG
// stream continuing at ckpt.iteration (the reference restarts at 0).
ModelState resume_from_checkpoint(const Corpus& corpus, const Checkpoint& ckpt, const TrainConfig& cfg);

}  // namespace sparselda_b200
