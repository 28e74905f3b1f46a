// compat.cpp -- the source-compatible `sparselda` API (paper_1610_02496_b200/compat/sparselda/)
// over the B200 engine.  Training, phi, trees and held-out scoring run on the device through
// sparselda_b200 / the C-ABI; this file only adapts shapes: the model's public members become
// mirrors of device buffers, chunks are presentation slices of the engine's resident state.
// Reference paths are relative to /root/reference/proj.
#include <algorithm>
#include <cstdio>
#include <istream>
#include <numeric>
#include <ostream>
#include <sstream>

#include "sparselda/counts.hpp"
#include "sparselda/eval.hpp"
#include "sparselda/trainer.hpp"

namespace sparselda {

namespace b2 = sparselda_b200;

// ------------------------------------------------------------------ counts --

std::uint64_t DocTopicMatrix::total() const {
    return std::accumulate(counts_.begin(), counts_.end(), std::uint64_t{0});
}
void DocTopicMatrix::start_rows(std::uint32_t rows) {
    offsets_.assign(1, 0);
    offsets_.reserve(static_cast<std::size_t>(rows) + 1);
    topics_.clear();
    counts_.clear();
}
void DocTopicMatrix::append_row(const SparseTopicRow& r) {
    topics_.insert(topics_.end(), r.topics.begin(), r.topics.end());
    counts_.insert(counts_.end(), r.counts.begin(), r.counts.end());
    offsets_.push_back(topics_.size());
}
void DocTopicMatrix::adopt(std::vector<std::uint64_t> ro, std::vector<TopicId> t, std::vector<std::uint32_t> c) {
    if (ro.empty() || ro.back() != t.size() || t.size() != c.size()) throw ValidationError("inconsistent CSR arrays");
    offsets_ = std::move(ro);
    topics_ = std::move(t);
    counts_ = std::move(c);
}

const std::vector<std::uint32_t>& WordTopicMatrix::data() const {
    return m_.get([this](slda_engine* e, std::vector<std::uint32_t>& out) {
        out.resize(static_cast<std::size_t>(V_) * K_);
        b2::check(slda_get_word_topic(e, out.data()));
    });
}
void WordTopicMatrix::bind(const detail::EngineLink* link, std::uint32_t V, std::uint32_t K) {
    V_ = V;
    K_ = K;
    m_.link = link;
    m_.seen = 0;
    m_.cells.clear();
}
void WordTopicMatrix::atomic_add(WordId v, TopicId k, std::uint32_t amount) { cell(v, k) += amount; }
std::uint64_t WordTopicMatrix::total() const {
    const auto& c = data();
    return std::accumulate(c.begin(), c.end(), std::uint64_t{0});
}
std::uint64_t WordTopicMatrix::row_total(WordId v) const {
    const auto r = row(v);
    return std::accumulate(r.begin(), r.end(), std::uint64_t{0});
}

const std::vector<float>& WordTopicProb::data() const {
    return m_.get([this](slda_engine* e, std::vector<float>& out) {
        out.resize(static_cast<std::size_t>(V_) * K_);
        b2::check(slda_get_word_topic_prob(e, out.data()));
    });
}
void WordTopicProb::bind(const detail::EngineLink* link, std::uint32_t V, std::uint32_t K, double beta) {
    V_ = V;
    K_ = K;
    beta_ = beta;
    m_.link = link;
    m_.seen = 0;
    m_.cells.clear();
}

void segmented_count(std::span<const TopicId> segment, SparseTopicRow& out, std::vector<TopicId>& scratch);

// preprocess (counts.cpp:37-63) on the device: a counts-only engine runs the colsum + phi kernels.
WordTopicProb preprocess(const WordTopicMatrix& b, double beta, unsigned) {
    const std::uint32_t V = b.num_words(), K = b.num_topics();
    WordTopicProb out(V, K, beta);
    if (V == 0 || K == 0) return out;
    const b2::ModelState m = b2::model_from_counts(V, K, b.data(), b.total(), 0, 50.0 / K, beta, 0);
    const std::vector<float> phi = m.word_topic_prob();
    for (WordId v = 0; v < V; ++v) std::copy_n(phi.data() + static_cast<std::size_t>(v) * K, K, out.mutable_row(v).data());
    return out;
}

SparseTopicRow segmented_count(std::span<const TopicId> segment) {
    SparseTopicRow r;
    std::vector<TopicId> scratch;
    segmented_count(segment, r, scratch);
    return r;
}

void segmented_count(std::span<const TopicId> segment, SparseTopicRow& out, std::vector<TopicId>& scratch) {
    scratch.assign(segment.begin(), segment.end());
    std::sort(scratch.begin(), scratch.end());
    out.clear();
    for (std::size_t i = 0; i < scratch.size();) {
        std::size_t j = i + 1;
        while (j < scratch.size() && scratch[j] == scratch[i]) ++j;
        out.topics.push_back(scratch[i]);
        out.counts.push_back(static_cast<std::uint32_t>(j - i));
        i = j;
    }
}

// rebuild_doc_topic (counts.cpp:103-125) on a host chunk: doc-grouped topics, one count per doc.
DocTopicMatrix rebuild_doc_topic(const Chunk& chunk) {
    std::vector<TopicId> grouped(chunk.size());
    for (std::uint32_t i = 0; i < chunk.size(); ++i) {
        if (chunk.tokens[i].topic == kInvalidTopic) throw ValidationError("uninitialized topic assignment in chunk");
        grouped[chunk.shuffle_ptrs[i]] = chunk.tokens[i].topic;
    }
    DocTopicMatrix a;
    a.start_rows(chunk.doc_count());
    SparseTopicRow row;
    std::vector<TopicId> scratch;
    for (std::uint32_t d = 0; d < chunk.doc_count(); ++d) {
        const std::uint32_t b = chunk.doc_offsets[d], e = chunk.doc_offsets[d + 1];
        segmented_count({grouped.data() + b, e - b}, row, scratch);
        a.append_row(row);
    }
    return a;
}

void accumulate_word_topic(WordTopicMatrix& b, WordId word, const SparseTopicRow& tc) {
    if (word >= b.num_words()) throw ValidationError("word id out of range");
    for (std::size_t i = 0; i < tc.size(); ++i) b.atomic_add(word, tc.topics[i], tc.counts[i]);
}
void reset_word_topic(WordTopicMatrix& b) {
    for (WordId v = 0; v < b.num_words(); ++v)
        for (TopicId k = 0; k < b.num_topics(); ++k) b.cell(v, k) = 0;
}

// Text dump of C_wk (counts.cpp:140-176): "V K T iteration", then "v k count" per non-zero.
void dump_word_topic(std::ostream& out, const WordTopicMatrix& b, std::uint64_t num_tokens, std::uint32_t iteration) {
    out << b.num_words() << ' ' << b.num_topics() << ' ' << num_tokens << ' ' << iteration << '\n';
    const std::vector<std::uint32_t>& c = b.data();
    for (std::size_t i = 0; i < c.size(); ++i)
        if (c[i]) out << i / b.num_topics() << ' ' << i % b.num_topics() << ' ' << c[i] << '\n';
}

WordTopicMatrix parse_word_topic(std::istream& in, std::uint64_t& num_tokens, std::uint32_t& iteration) {
    std::string line;
    if (!std::getline(in, line)) throw ValidationError("word-topic dump: missing header");
    std::uint32_t V = 0, K = 0;
    if (!(std::istringstream(line) >> V >> K >> num_tokens >> iteration))
        throw ValidationError("word-topic dump: malformed header");
    WordTopicMatrix b(V, K);
    std::uint64_t sum = 0;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::uint64_t v = 0, k = 0, c = 0;
        if (!(std::istringstream(line) >> v >> k >> c) || v >= V || k >= K)
            throw ValidationError("word-topic dump: malformed entry \"" + line + "\"");
        b.cell(static_cast<WordId>(v), static_cast<TopicId>(k)) = static_cast<std::uint32_t>(c);
        sum += c;
    }
    if (sum != num_tokens) throw ValidationError("word-topic dump: stored counts do not sum to T");
    return b;
}

// ------------------------------------------------------------------ corpus --

Corpus load_uci(std::istream& docword, std::istream& vocab) { return b2::load_uci(docword, vocab); }
Corpus load_docword(std::istream& docword) { return b2::load_docword(docword); }
void init_assignments(Corpus& corpus, std::uint32_t num_topics, std::uint64_t seed) {
    b2::init_assignments(corpus, num_topics, seed);
}

namespace {

std::vector<std::uint32_t> doc_bounds(const Corpus& corpus, std::uint32_t n) {
    std::vector<std::uint32_t> b(static_cast<std::size_t>(n) + 1, 0);
    b2::check(slda_shard_bounds(corpus.num_docs, corpus.tokens.size(), corpus.doc_lengths.data(), n, b.data()));
    return b;
}

// Chunk [b, e) of a whole-corpus PDOW layout: the (word, doc, id) order restricted to the range
// is that chunk's own PDOW order (corpus.cpp:155-167); segments, offsets and the word-major ->
// doc-grouped pointers follow from it (corpus.cpp:175-195).
Chunk slice_chunk(const b2::ChunkLayout& L, const std::vector<TopicId>& topics, DocId b, DocId e) {
    Chunk c;
    c.doc_begin = b;
    c.doc_end = e;
    for (std::size_t i = 0; i < L.sorted_doc.size(); ++i) {
        const DocId d = L.sorted_doc[i];
        if (d < b || d >= e) continue;
        const std::uint64_t id = L.token_ids[i];
        c.tokens.push_back(Token{d, L.sorted_word[i], topics.empty() ? kInvalidTopic : topics[id]});
        c.token_ids.push_back(static_cast<std::uint32_t>(id));
    }
    for (std::uint32_t i = 0; i < c.size();) {
        std::uint32_t j = i;
        while (j < c.size() && c.tokens[j].word == c.tokens[i].word) ++j;
        c.word_segments.push_back(WordSegment{c.tokens[i].word, i, j - i});
        i = j;
    }
    c.doc_offsets.assign(static_cast<std::size_t>(e - b) + 1, 0);
    for (const Token& t : c.tokens) ++c.doc_offsets[t.doc - b + 1];
    std::partial_sum(c.doc_offsets.begin(), c.doc_offsets.end(), c.doc_offsets.begin());
    std::vector<std::uint32_t> next(c.doc_offsets.begin(), c.doc_offsets.end() - 1);
    c.shuffle_ptrs.resize(c.size());
    for (std::uint32_t i = 0; i < c.size(); ++i) c.shuffle_ptrs[i] = next[c.tokens[i].doc - b]++;
    return c;
}

}  // namespace

// build_chunks (corpus.cpp:124-198): the engine builds the PDOW layout on the device (a K=1
// engine over the corpus), and each chunk is its document range's slice of it.
std::vector<Chunk> build_chunks(const Corpus& corpus, std::uint32_t num_chunks) {
    if (corpus.num_docs == 0) {
        if (num_chunks != 1) throw ValidationError("empty corpus admits exactly one chunk");
        return {Chunk{}};
    }
    if (num_chunks < 1 || num_chunks > corpus.num_docs)
        throw ValidationError("num_chunks must be in [1, D=" + std::to_string(corpus.num_docs) + "]");
    Corpus probe = corpus;
    for (Token& t : probe.tokens) t.topic = 0;
    b2::TrainConfig cfg;
    cfg.num_topics = 1;
    const b2::ModelState m = b2::init_state(probe, cfg);
    const b2::ChunkLayout L = m.chunk_layout();
    std::vector<TopicId> topics(corpus.tokens.size());
    for (std::size_t t = 0; t < topics.size(); ++t) topics[t] = corpus.tokens[t].topic;
    const std::vector<std::uint32_t> b = doc_bounds(corpus, num_chunks);
    std::vector<Chunk> out;
    for (std::uint32_t c = 0; c < num_chunks; ++c) out.push_back(slice_chunk(L, topics, b[c], b[c + 1]));
    return out;
}

// build_schedule (corpus.cpp:200-210): longest segment first, ties by word.
std::vector<WordId> build_schedule(Chunk& chunk) {
    std::stable_sort(chunk.word_segments.begin(), chunk.word_segments.end(), [](const WordSegment& x, const WordSegment& y) {
        return x.length != y.length ? x.length > y.length : x.word < y.word;
    });
    std::vector<WordId> order;
    for (const WordSegment& s : chunk.word_segments) order.push_back(s.word);
    return order;
}

// auto_num_chunks (corpus.cpp:212-253): fewest chunks whose largest one -- tokens (12 B) +
// ids and pointers (8 B) per token, 8 B per row entry bound min(len, K) -- fits the budget.
std::uint32_t auto_num_chunks(const Corpus& corpus, std::uint32_t num_topics, std::uint64_t budget_bytes) {
    if (corpus.num_docs <= 1) return 1;
    auto worst = [&](std::uint32_t n) {
        const std::vector<std::uint32_t> b = doc_bounds(corpus, n);
        std::uint64_t w = 0;
        for (std::uint32_t c = 0; c < n; ++c) {
            std::uint64_t cost = 0;
            for (DocId d = b[c]; d < b[c + 1]; ++d)
                cost += std::uint64_t{corpus.doc_lengths[d]} * 20 + 8 * std::min<std::uint64_t>(corpus.doc_lengths[d], num_topics);
            w = std::max(w, cost);
        }
        return w;
    };
    std::uint32_t lo = 1, hi = corpus.num_docs;
    if (worst(lo) <= budget_bytes) return lo;
    while (lo < hi) {
        const std::uint32_t mid = lo + (hi - lo) / 2;
        if (worst(mid) <= budget_bytes) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// ----------------------------------------------------------------- trainer --

void DenseDocTopic::rebuild(const Chunk& chunk, std::uint32_t num_topics) {
    rows_ = chunk.doc_count();
    K_ = num_topics;
    nnz_ = 0;
    cells_.assign(static_cast<std::size_t>(rows_) * K_, 0u);
    for (const Token& t : chunk.tokens) {
        if (t.topic == kInvalidTopic) throw ValidationError("uninitialized topic assignment in chunk");
        if (cells_[static_cast<std::size_t>(t.doc - chunk.doc_begin) * K_ + t.topic]++ == 0) ++nnz_;
    }
}

// Engine-backed chunk slots: the chunk bounds, the engine's PDOW layout (static), and per
// model epoch its C_dk rows and assignments.
struct ChunkStore::Source {
    const detail::EngineLink* link = nullptr;
    std::vector<std::uint32_t> bounds;
    std::uint32_t K = 0;
    bool vanilla = false;
    bool have_layout = false;
    b2::ChunkLayout layout;
    std::uint64_t seen = 0;
    b2::DocTopicMatrix rows;
    std::vector<TopicId> topics;
    const b2::ModelState* dev = nullptr;
};

ChunkStore ChunkStore::make_resident(std::vector<ChunkSlot> slots) {
    ChunkStore s;
    s.slots_ = std::move(slots);
    s.filled_.assign(s.slots_.size(), 0);
    return s;
}
// Nothing spills: every slot stays resident (the engine keeps the model in HBM).
ChunkStore ChunkStore::make_file_backed(std::vector<ChunkSlot> slots, const std::filesystem::path&) {
    return make_resident(std::move(slots));
}

ChunkSlot& ChunkStore::acquire(std::size_t index) {
    if (index >= slots_.size()) throw ValidationError("chunk index out of range");
    ChunkSlot& slot = slots_[index];
    if (!src_ || !src_->link->engine || filled_[index] == src_->link->epoch) return slot;
    Source& s = *src_;
    if (!s.have_layout) {
        s.layout = s.dev->chunk_layout();
        s.have_layout = true;
    }
    if (s.seen != s.link->epoch) {
        s.rows = s.dev->doc_topic();
        s.topics = s.dev->gather_assignments();
        s.seen = s.link->epoch;
    }
    const DocId b = s.bounds[index], e = s.bounds[index + 1];
    slot.chunk = slice_chunk(s.layout, s.topics, b, e);
    const std::uint64_t o0 = s.rows.row_offsets[b], o1 = s.rows.row_offsets[e];
    std::vector<std::uint64_t> ro(s.rows.row_offsets.begin() + b, s.rows.row_offsets.begin() + e + 1);
    for (std::uint64_t& o : ro) o -= o0;
    slot.doc_topic.adopt(std::move(ro), {s.rows.topics.begin() + o0, s.rows.topics.begin() + o1},
                         {s.rows.counts.begin() + o0, s.rows.counts.begin() + o1});
    if (s.vanilla) slot.doc_topic_dense.rebuild(slot.chunk, s.K);
    filled_[index] = s.link->epoch;
    return slot;
}
void ChunkStore::release(std::size_t) {}

const WaryTree<float>& TreeSet::operator[](WordId v) const {
    const std::size_t n = size();
    if (v >= n) throw ValidationError("word id out of range");
    if (trees_.size() != n) {
        trees_.assign(n, WaryTree<float>{});
        built_.assign(n, 0);
    }
    const std::uint64_t epoch = model_->link_epoch();
    if (built_[v] != epoch) {
        trees_[v].build(model_->word_topic_prob.row(v), model_->tree_branch());
        built_[v] = epoch;
    }
    return trees_[v];
}
std::size_t TreeSet::size() const { return model_ ? model_->vocab_size : trees_.size(); }

const std::vector<float>& MassVector::get() const {
    return m_.get([this](slda_engine* e, std::vector<float>& out) {
        out.resize(V_);
        b2::check(slda_get_tree_mass(e, out.data()));
    });
}

ModelState::ModelState() : link_(std::make_unique<detail::EngineLink>()) { attach(); }

ModelState::ModelState(ModelState&& o) noexcept { *this = std::move(o); }

ModelState& ModelState::operator=(ModelState&& o) noexcept {
    num_docs = o.num_docs;
    vocab_size = o.vocab_size;
    num_tokens = o.num_tokens;
    num_topics = o.num_topics;
    alpha = o.alpha;
    beta = o.beta;
    seed = o.seed;
    iteration = o.iteration;
    word_topic = std::move(o.word_topic);
    word_topic_prob = std::move(o.word_topic_prob);
    tree_mass = std::move(o.tree_mass);
    trees = std::move(o.trees);
    chunks = std::move(o.chunks);
    dev_ = std::move(o.dev_);
    link_ = std::move(o.link_);
    branch_ = o.branch_;
    trees.model_ = this;
    if (chunks.src_) chunks.src_->dev = &dev_;
    return *this;
}

void ModelState::attach() {
    link_->engine = dev_.engine();
    ++link_->epoch;
    if (link_->engine) {
        word_topic.bind(link_.get(), vocab_size, num_topics);
        word_topic_prob.bind(link_.get(), vocab_size, num_topics, beta);
        tree_mass.m_.link = link_.get();
        tree_mass.m_.seen = 0;
        tree_mass.V_ = vocab_size;
        trees.model_ = this;
    }
}

void ModelState::advance() { ++link_->epoch; }

std::vector<TopicId> ModelState::gather_assignments() {
    if (!dev_.engine() || !dev_.has_chunks()) return {};
    return dev_.gather_assignments();
}

namespace {
void copy_header(ModelState& s, const b2::ModelState& d) {
    s.num_docs = d.num_docs;
    s.vocab_size = d.vocab_size;
    s.num_tokens = d.num_tokens;
    s.num_topics = d.num_topics;
    s.alpha = d.alpha;
    s.beta = d.beta;
    s.seed = d.seed;
    s.iteration = d.iteration;
}
}  // namespace

TrainConfig TrainConfig::resolved(const Corpus& corpus) const {
    TrainConfig out;
    static_cast<b2::TrainConfig&>(out) = b2::TrainConfig::resolved(corpus);
    if (num_chunks == 0) {
        out.num_chunks = auto_num_chunks(corpus, out.num_topics, out.memory_budget);
        if (corpus.num_docs > 0 && out.num_chunks > corpus.num_docs) throw ValidationError("num_chunks exceeds document count");
    }
    return out;
}

// init_state (trainer.cpp:354-417): the device engine; chunks are the reference's split of the
// documents for resolved num_chunks (auto_num_chunks from memory_budget when 0).
ModelState init_state(const Corpus& corpus, const TrainConfig& raw) {
    const TrainConfig cfg = raw.resolved(corpus);
    const std::uint32_t n_chunks = corpus.num_docs == 0 ? 1 : cfg.num_chunks;
    ModelState s;
    s.dev_ = b2::init_state(corpus, cfg);
    copy_header(s, s.dev_);
    s.branch_ = cfg.tree_branch;
    s.attach();
    auto src = std::make_shared<ChunkStore::Source>();
    src->link = s.link_.get();
    src->dev = &s.dev_;
    src->K = cfg.num_topics;
    src->vanilla = cfg.sampler == SamplerKind::kVanilla;
    src->bounds = corpus.num_docs ? doc_bounds(corpus, n_chunks) : std::vector<std::uint32_t>{0, 0};
    s.chunks.slots_.assign(n_chunks, ChunkSlot{});
    s.chunks.filled_.assign(n_chunks, 0);
    for (std::uint32_t c = 0; c < n_chunks; ++c) {
        s.chunks.slots_[c].chunk.doc_begin = src->bounds[c];
        s.chunks.slots_[c].chunk.doc_end = src->bounds[c + 1];
    }
    s.chunks.src_ = std::move(src);
    return s;
}

IterationStats run_iteration(ModelState& state, const TrainConfig& cfg) {
    const IterationStats st = b2::run_iteration(state.dev_, cfg);
    state.iteration = st.iteration;
    state.advance();
    return st;
}

ModelState train(const Corpus& corpus, const TrainConfig& raw, const MetricsSink& sink, const HeldoutProbe& probe) {
    const TrainConfig cfg = raw.resolved(corpus);
    ModelState state = sparselda::init_state(corpus, cfg);
    for (std::uint32_t i = 0; i < cfg.iterations; ++i) {  // trainer.cpp:451-464
        MetricsEntry entry;
        entry.stats = run_iteration(state, cfg);
        if (probe && cfg.eval_every > 0 && entry.stats.iteration % cfg.eval_every == 0) entry.heldout_ll = probe(state);
        if (sink) sink(entry);
    }
    return state;
}

void save_checkpoint(const std::filesystem::path& path, ModelState& state) { b2::save_checkpoint(path, state.dev_); }

Checkpoint load_checkpoint(const std::filesystem::path& path) {
    const b2::Checkpoint c = b2::load_checkpoint(path);
    Checkpoint out;
    out.num_docs = c.num_docs;
    out.vocab_size = c.vocab_size;
    out.num_tokens = c.num_tokens;
    out.num_topics = c.num_topics;
    out.iteration = c.iteration;
    out.alpha = c.alpha;
    out.beta = c.beta;
    out.seed = c.seed;
    out.assignments = c.assignments;
    out.word_topic = WordTopicMatrix(c.vocab_size, c.num_topics);
    for (WordId v = 0; v < c.vocab_size; ++v)
        for (TopicId k = 0; k < c.num_topics; ++k)
            out.word_topic.cell(v, k) = c.word_topic[static_cast<std::size_t>(v) * c.num_topics + k];
    return out;
}

// model_from_checkpoint (trainer.cpp:514-532): phi and the trees from the counts, on the device.
ModelState model_from_checkpoint(const Checkpoint& ck, unsigned) {
    ModelState s;
    s.dev_ = b2::model_from_counts(ck.vocab_size, ck.num_topics, ck.word_topic.data(), ck.num_tokens, ck.iteration,
                                   ck.alpha, ck.beta, ck.seed);
    copy_header(s, s.dev_);
    s.num_docs = ck.num_docs;
    s.branch_ = ck.num_topics > 32768 ? 41 : 32;
    s.attach();
    return s;
}

// ------------------------------------------------------------------- eval --

HeldoutSet HeldoutSet::from_corpus(const Corpus& corpus) {  // eval.cpp:14-28
    HeldoutSet h;
    h.vocab_size = corpus.vocab_size;
    h.docs.resize(corpus.num_docs);
    std::vector<std::uint32_t> pos(corpus.num_docs, 0);
    for (const Token& t : corpus.tokens)
        (pos[t.doc]++ % 2 ? h.docs[t.doc].evaluation : h.docs[t.doc].estimation).push_back(t.word);
    return h;
}
std::uint64_t HeldoutSet::estimation_tokens() const {
    std::uint64_t n = 0;
    for (const Doc& d : docs) n += d.estimation.size();
    return n;
}
std::uint64_t HeldoutSet::evaluation_tokens() const {
    std::uint64_t n = 0;
    for (const Doc& d : docs) n += d.evaluation.size();
    return n;
}

// heldout_ll (eval.cpp:49-133) on the device.  The engine takes the held-out corpus and splits
// it by from_corpus's alternation, so the set is re-interleaved into that corpus (the split of
// the result is the set itself).
EvalReport heldout_ll(ModelState& model, const HeldoutSet& h, std::uint32_t burn_in, unsigned workers,
                      std::uint64_t seed) {
    if (h.docs.empty()) throw ValidationError("held-out set is empty");
    if (h.vocab_size != model.vocab_size) throw ValidationError("held-out vocabulary size does not match model");
    if (h.evaluation_tokens() == 0) throw ValidationError("held-out set has no evaluation tokens");
    Corpus c;
    c.num_docs = static_cast<std::uint32_t>(h.docs.size());
    c.vocab_size = h.vocab_size;
    for (DocId d = 0; d < c.num_docs; ++d) {
        const HeldoutSet::Doc& doc = h.docs[d];
        const std::size_t ne = doc.estimation.size(), nv = doc.evaluation.size();
        if (!(ne == nv || ne == nv + 1))
            throw ValidationError("held-out document halves must alternate as HeldoutSet::from_corpus splits them");
        for (std::size_t j = 0; j < ne + nv; ++j)
            c.tokens.push_back(Token{d, j % 2 ? doc.evaluation[j / 2] : doc.estimation[j / 2], kInvalidTopic});
    }
    c.finalize();
    return b2::heldout_ll(model.device(), c, burn_in, workers, seed);
}

double throughput_mtokens(const IterationStats& s) { return throughput_mtokens(s.tokens, s.elapsed_s); }

// top_words (eval.cpp:139-158): n most probable words per topic, ties by word id.
std::vector<std::vector<std::pair<WordId, float>>> top_words(const WordTopicProb& bhat, std::uint32_t n) {
    if (n > bhat.num_words()) throw ValidationError("top_words n exceeds vocabulary size");
    std::vector<std::vector<std::pair<WordId, float>>> out(bhat.num_topics());
    std::vector<std::pair<WordId, float>> col(bhat.num_words());
    for (TopicId k = 0; k < bhat.num_topics(); ++k) {
        for (WordId v = 0; v < bhat.num_words(); ++v) col[v] = {v, bhat.at(v, k)};
        std::partial_sort(col.begin(), col.begin() + n, col.end(),
                          [](const auto& a, const auto& b) { return a.second != b.second ? a.second > b.second : a.first < b.first; });
        out[k].assign(col.begin(), col.begin() + n);
    }
    return out;
}

void print_topics(std::ostream& out, const WordTopicProb& bhat, const std::vector<std::string>& vocab, std::uint32_t n) {
    const auto ranked = top_words(bhat, n);
    for (TopicId k = 0; k < ranked.size(); ++k) {
        out << "topic " << k << ':';
        for (const auto& [w, p] : ranked[k]) {
            char num[48];
            std::snprintf(num, sizeof(num), "%.6f", p);
            out << ' ';
            if (w < vocab.size() && !vocab[w].empty()) out << vocab[w]; else out << w;
            out << ':' << num;
        }
        out << '\n';
    }
}

}  // namespace sparselda
