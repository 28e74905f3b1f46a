// Trainer API of the reference (trainer.hpp:18-202) over the B200 engine.  init_state builds the
// device engine (PDOW, topic init, C_dk, C_wk, phi, trees on the GPU); run_iteration is one
// device iteration.  ModelState keeps the reference's public members, but they are mirrors of
// device state: word_topic / word_topic_prob / tree_mass / trees fetch from HBM on first use
// after an iteration, and chunks.acquire(c) materialises chunk c's PDOW slice and its C_dk rows
// from the engine.  The reference's chunk count only changes how the state is presented (the
// engine holds every document resident), so results never depend on it (acceptance.cpp:426-445).
#pragma once

#include <atomic>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "sparselda/corpus.hpp"
#include "sparselda/counts.hpp"
#include "sparselda/sampler.hpp"
#include "sparselda/types.hpp"

namespace sparselda {

using sparselda_b200::SamplerKind;

// A distinct type for the same reason as Corpus.  resolved() is the reference's rule
// (trainer.cpp:15-35): num_chunks = auto_num_chunks(memory_budget) when 0.
struct TrainConfig : sparselda_b200::TrainConfig {
    TrainConfig resolved(const Corpus& corpus) const;
};
using sparselda_b200::IterationStats;
using sparselda_b200::MetricsEntry;
using sparselda_b200::MetricsSink;
using sparselda_b200::format_metrics_line;

// Dense per-document counts (the vanilla baseline's layout).
class DenseDocTopic {
public:
    void rebuild(const Chunk& chunk, std::uint32_t num_topics);
    std::span<const std::uint32_t> row(std::uint32_t local_doc) const {
        return {cells_.data() + static_cast<std::size_t>(local_doc) * K_, K_};
    }
    std::uint32_t num_rows() const { return rows_; }
    std::uint32_t num_topics() const { return K_; }
    std::uint64_t nnz() const { return nnz_; }
    bool empty() const { return cells_.empty(); }
    const std::vector<std::uint32_t>& cells() const { return cells_; }
    std::vector<std::uint32_t>& raw_cells() { return cells_; }
    void set_shape(std::uint32_t rows, std::uint32_t num_topics, std::uint64_t nnz) {
        rows_ = rows;
        K_ = num_topics;
        nnz_ = nnz;
    }

private:
    std::uint32_t rows_ = 0, K_ = 0;
    std::uint64_t nnz_ = 0;
    std::vector<std::uint32_t> cells_;
};

struct ChunkSlot {
    Chunk chunk;
    DocTopicMatrix doc_topic;
    DenseDocTopic doc_topic_dense;  // vanilla models only
};

struct ModelState;
struct Checkpoint;

// Chunks of a model: the reference's chunk_boundaries split of the documents (or, standalone,
// resident slots).  acquire(c) fills slot c from the engine when the model moved on since it
// was last filled; release is a no-op (nothing spills: the device holds the state).
class ChunkStore {
public:
    ChunkStore() = default;
    ChunkStore(const ChunkStore&) = delete;
    ChunkStore& operator=(const ChunkStore&) = delete;
    ChunkStore(ChunkStore&&) noexcept = default;
    ChunkStore& operator=(ChunkStore&&) noexcept = default;

    static ChunkStore make_resident(std::vector<ChunkSlot> slots);
    static ChunkStore make_file_backed(std::vector<ChunkSlot> slots, const std::filesystem::path& dir);

    std::size_t size() const { return slots_.size(); }
    bool file_backed() const { return false; }
    ChunkSlot& acquire(std::size_t index);
    void release(std::size_t index);

private:
    friend struct ModelState;
    friend ModelState init_state(const Corpus&, const TrainConfig&);
    struct Source;  // engine-backed slots (compat.cpp)
    std::vector<ChunkSlot> slots_;
    std::vector<std::uint64_t> filled_;  // link epoch each slot was filled at (0: never)
    std::shared_ptr<Source> src_;
};

struct WorkUnit {
    std::uint32_t chunk;
    std::uint32_t segment;
};

class WorkQueue {  // dynamic claiming of units (trainer.hpp:133-147); host-side utility
public:
    explicit WorkQueue(std::vector<WorkUnit> units) : units_(std::move(units)) {}
    std::optional<WorkUnit> claim() {
        const std::size_t i = next_.fetch_add(1, std::memory_order_relaxed);
        return i < units_.size() ? std::optional<WorkUnit>(units_[i]) : std::nullopt;
    }
    std::size_t size() const { return units_.size(); }

private:
    std::vector<WorkUnit> units_;
    std::atomic<std::size_t> next_{0};
};

// Per-word W-ary trees of the model, built on the host from the device's phi rows when indexed
// (the device samples from its own L4/L8 levels; these are for host callers).
class TreeSet {
public:
    const WaryTree<float>& operator[](WordId v) const;
    std::size_t size() const;
    bool empty() const { return size() == 0; }

private:
    friend struct ModelState;
    const ModelState* model_ = nullptr;
    mutable std::vector<WaryTree<float>> trees_;
    mutable std::vector<std::uint64_t> built_;
};

// Q_v per word (tree_mass), mirrored from the device.
class MassVector {
public:
    float operator[](WordId v) const { return get()[v]; }
    std::size_t size() const { return get().size(); }
    const float* data() const { return get().data(); }
    auto begin() const { return get().begin(); }
    auto end() const { return get().end(); }
    const std::vector<float>& get() const;

private:
    friend struct ModelState;
    detail::Mirror<float> m_;
    std::uint32_t V_ = 0;
};

struct ModelState {
    ModelState();
    ModelState(ModelState&& o) noexcept;
    ModelState& operator=(ModelState&& o) noexcept;
    ModelState(const ModelState&) = delete;
    ModelState& operator=(const ModelState&) = delete;

    std::uint32_t num_docs = 0;
    std::uint32_t vocab_size = 0;
    std::uint64_t num_tokens = 0;
    std::uint32_t num_topics = 0;
    double alpha = 0.0;
    double beta = 0.0;
    std::uint64_t seed = 0;
    std::uint32_t iteration = 0;

    WordTopicMatrix word_topic;
    WordTopicProb word_topic_prob;
    MassVector tree_mass;
    TreeSet trees;
    ChunkStore chunks;

    std::vector<TopicId> gather_assignments();

    // The device model underneath (kernel times, info, the native API).
    sparselda_b200::ModelState& device() { return dev_; }
    const sparselda_b200::ModelState& device() const { return dev_; }
    // Binds the mirrors to dev_'s engine; called whenever dev_ is (re)placed.
    void attach();
    // Marks every mirror stale (after an iteration).
    void advance();
    std::uint64_t link_epoch() const { return link_->epoch; }
    std::uint32_t tree_branch() const { return branch_; }

private:
    friend ModelState init_state(const Corpus&, const TrainConfig&);
    friend IterationStats run_iteration(ModelState&, const TrainConfig&);
    friend void save_checkpoint(const std::filesystem::path&, ModelState&);
    friend ModelState model_from_checkpoint(const Checkpoint&, unsigned);
    sparselda_b200::ModelState dev_;
    std::unique_ptr<detail::EngineLink> link_;
    std::uint32_t branch_ = 32;  // TrainConfig::tree_branch of the host trees
};

ModelState init_state(const Corpus& corpus, const TrainConfig& cfg);
IterationStats run_iteration(ModelState& state, const TrainConfig& cfg);

using HeldoutProbe = std::function<double(ModelState&)>;
ModelState train(const Corpus& corpus, const TrainConfig& cfg, const MetricsSink& sink = {},
                 const HeldoutProbe& heldout_probe = {});

struct Checkpoint {
    std::uint32_t num_docs = 0;
    std::uint32_t vocab_size = 0;
    std::uint64_t num_tokens = 0;
    std::uint32_t num_topics = 0;
    std::uint32_t iteration = 0;
    double alpha = 0.0;
    double beta = 0.0;
    std::uint64_t seed = 0;
    std::vector<TopicId> assignments;
    WordTopicMatrix word_topic;
};

void save_checkpoint(const std::filesystem::path& path, ModelState& state);
Checkpoint load_checkpoint(const std::filesystem::path& path);
ModelState model_from_checkpoint(const Checkpoint& ckpt, unsigned workers = 0);

}  // namespace sparselda
