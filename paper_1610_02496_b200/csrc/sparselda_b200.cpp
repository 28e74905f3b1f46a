// sparselda_b200.cpp -- host C++ API over the C-ABI.  See sparselda_b200.hpp.
// Reference paths are relative to /root/reference/proj.
#include "sparselda_b200.hpp"

#include <algorithm>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cstring>
#include <iterator>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iomanip>
#include <istream>
#include <limits>
#include <sstream>
#include <thread>

namespace sparselda_b200 {

void check(int status) {
    if (status == SLDA_OK) return;
    const std::string msg = slda_last_error();
    if (status == SLDA_ERR_VALIDATION) throw ValidationError(msg);
    if (status == SLDA_ERR_IO) throw IoError(msg);
    throw DeviceError(msg);
}

// ---------------------------------------------------------------- corpus --

void Corpus::finalize() {
    num_tokens = tokens.size();
    doc_lengths.assign(num_docs, 0);
    word_freqs.assign(vocab_size, 0);
    for (const Token& t : tokens) {
        doc_lengths[t.doc] += 1;
        word_freqs[t.word] += 1;
    }
}

namespace {

[[noreturn]] void parse_fail(std::uint64_t line, const std::string& what) {
    throw ValidationError("docword line " + std::to_string(line) + ": " + what);
}

std::uint64_t header_value(std::istream& in, std::uint64_t line, const char* name) {
    std::string text;
    if (!std::getline(in, text)) parse_fail(line, std::string("missing ") + name + " header line");
    std::istringstream f(text);
    long long v = -1;
    if (!(f >> v) || v < 0) parse_fail(line, std::string("malformed ") + name + " header");
    std::string extra;
    if (f >> extra) parse_fail(line, std::string("trailing data after ") + name + " header");
    return static_cast<std::uint64_t>(v);
}

}  // namespace

// UCI bag-of-words (corpus.cpp:30-68): D, V, NNZ then "docID wordID count", 1-based.
//
// The reference reads the entries line by line on one thread (the ingest bottleneck at
// PubMed/ClueWeb scale).  Here the NNZ entry lines are split into byte
// ranges at line boundaries and parsed by all host threads; tokens are then expanded in file
// order into one allocation.  Accepted input, token order and every error (message and line
// number -- the first failing line in file order wins) are the reference's: lines the fast
// integer scanner does not accept outright are re-parsed with the reference's stream
// semantics (`>>` into long long, trailing-data check).
namespace {

struct EntryLine {
    bool ok;
    long long d, w, n;
};

bool ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// Three non-negative decimal fields (<= 18 digits) separated and surrounded by whitespace;
// false for anything else (signs, overflow, trailing data, missing fields), which then takes
// the stream path.
bool scan_entry(const char* p, const char* e, long long* v) {
    for (int f = 0; f < 3; ++f) {
        while (p < e && ws(*p)) ++p;
        const char* q = p;
        long long x = 0;
        while (p < e && *p >= '0' && *p <= '9' && p - q < 18) x = x * 10 + (*p++ - '0');
        if (p == q || (p < e && !ws(*p))) return false;
        v[f] = x;
    }
    while (p < e && ws(*p)) ++p;
    return p == e;
}

// The reference's per-line semantics (corpus.cpp:45-58); returns an error message or "".
std::string parse_entry_stream(const std::string& text, long long* v) {
    std::istringstream f(text);
    if (!(f >> v[0] >> v[1] >> v[2])) return "malformed entry, expected \"docID wordID count\"";
    std::string extra;
    if (f >> extra) return "trailing data after entry";
    return "";
}

struct Chunk {
    const char* begin;
    const char* end;          // exclusive; ends after a '\n' or at the buffer end
    std::uint64_t first_line; // file line number of the chunk's first line
    std::vector<std::uint32_t> d, w;
    std::vector<std::uint64_t> n;
    std::uint64_t tokens = 0;
    std::uint64_t err_line = 0;  // 0 = none
    std::string err;
};

}  // namespace

Corpus load_docword_buffer(const char* data, std::size_t size) {
    Corpus c;
    const char* p = data;
    const char* const end = data + size;
    // Header lines through the reference's own stream semantics.
    auto next_line = [&](std::string& out) -> bool {  // std::getline over the buffer
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
        const char* le = nl ? nl : end;
        out.assign(p, le);
        p = nl ? nl + 1 : end;
        return true;
    };
    std::uint64_t hdr[3];
    const char* names[3] = {"D", "V", "NNZ"};
    for (int i = 0; i < 3; ++i) {
        std::string text;
        if (!next_line(text)) parse_fail(static_cast<std::uint64_t>(i) + 1, std::string("missing ") + names[i] + " header line");
        std::istringstream hs(text + "\n");
        hdr[i] = header_value(hs, static_cast<std::uint64_t>(i) + 1, names[i]);
    }
    const std::uint64_t D = hdr[0], V = hdr[1], nnz = hdr[2];
    if (D > 0xFFFFFFFFull || V > 0xFFFFFFFFull) parse_fail(1, "dimension exceeds 32-bit id space");
    c.num_docs = static_cast<std::uint32_t>(D);
    c.vocab_size = static_cast<std::uint32_t>(V);
    c.doc_lengths.assign(c.num_docs, 0);
    c.word_freqs.assign(c.vocab_size, 0);

    // Byte ranges at line starts, one or more per thread.
    const std::size_t body = static_cast<std::size_t>(end - p);
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt == 0 ? 1 : (nt > 64 ? 64 : nt);
    if (body < (1u << 20)) nt = 1;
    std::vector<Chunk> chunks;
    {
        const char* b = p;
        for (unsigned i = 0; i < nt && b < end; ++i) {
            const char* e = i + 1 == nt ? end : p + body / nt * (i + 1);
            if (e < b) e = b;
            if (e < end) {
                const char* nl = static_cast<const char*>(std::memchr(e, '\n', static_cast<std::size_t>(end - e)));
                e = nl ? nl + 1 : end;
            }
            Chunk ch;
            ch.begin = b;
            ch.end = e;
            chunks.push_back(std::move(ch));
            b = e;
        }
    }
    // Pass 1: lines per chunk (a line is '\n'-terminated, or the non-empty remainder at EOF).
    std::vector<std::uint64_t> lines(chunks.size(), 0);
    auto run = [&](auto&& fn) {
        std::vector<std::thread> th;
        for (std::size_t i = 1; i < chunks.size(); ++i) th.emplace_back(fn, i);
        if (!chunks.empty()) fn(0);
        for (auto& t : th) t.join();
    };
    run([&](std::size_t i) {
        std::uint64_t n = 0;
        for (const char* q = chunks[i].begin; q < chunks[i].end;) {
            const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<std::size_t>(chunks[i].end - q)));
            ++n;
            q = nl ? nl + 1 : chunks[i].end;
        }
        lines[i] = n;
    });
    // Keep exactly the first nnz lines (the reference reads no further).
    std::uint64_t seen = 0, line0 = 4;
    std::size_t used = 0;
    for (; used < chunks.size() && seen < nnz; ++used) {
        chunks[used].first_line = line0 + seen;
        if (seen + lines[used] > nnz) {  // cut inside this chunk after (nnz - seen) lines
            const char* q = chunks[used].begin;
            for (std::uint64_t k = 0; k < nnz - seen; ++k) {
                const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<std::size_t>(chunks[used].end - q)));
                q = nl ? nl + 1 : chunks[used].end;
            }
            chunks[used].end = q;
            lines[used] = nnz - seen;
        }
        seen += lines[used];
    }
    chunks.resize(used);
    const std::uint64_t eof_line = seen < nnz ? line0 + seen : 0;  // first missing entry line

    // Pass 2: parse.
    run([&](std::size_t i) {
        Chunk& ch = chunks[i];
        std::uint64_t line = ch.first_line;
        std::string text;
        for (const char* q = ch.begin; q < ch.end; ++line) {
            const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<std::size_t>(ch.end - q)));
            const char* le = nl ? nl : ch.end;
            long long v[3];
            std::string err;
            if (!scan_entry(q, le, v)) {
                text.assign(q, le);
                err = parse_entry_stream(text, v);
            }
            q = nl ? nl + 1 : ch.end;
            if (err.empty()) {
                if (v[0] < 1 || static_cast<std::uint64_t>(v[0]) > D) err = "docID out of range [1, D]";
                else if (v[1] < 1 || static_cast<std::uint64_t>(v[1]) > V) err = "wordID out of range [1, V]";
                else if (v[2] < 1) err = "count must be >= 1";
            }
            if (!err.empty()) {
                ch.err_line = line;
                ch.err = err;
                return;
            }
            ch.d.push_back(static_cast<std::uint32_t>(v[0] - 1));
            ch.w.push_back(static_cast<std::uint32_t>(v[1] - 1));
            ch.n.push_back(static_cast<std::uint64_t>(v[2]));
            ch.tokens += static_cast<std::uint64_t>(v[2]);
        }
    });
    for (const Chunk& ch : chunks)
        if (ch.err_line) parse_fail(ch.err_line, ch.err);  // chunks are in file order
    if (eof_line) parse_fail(eof_line, "unexpected end of file, expected entry");

    // Pass 3: expand tokens in file order; per-document / per-word totals.
    std::vector<std::uint64_t> off(chunks.size() + 1, 0);
    for (std::size_t i = 0; i < chunks.size(); ++i) off[i + 1] = off[i] + chunks[i].tokens;
    c.tokens.resize(off.back());
    run([&](std::size_t i) {
        const Chunk& ch = chunks[i];
        Token* t = c.tokens.data() + off[i];
        for (std::size_t k = 0; k < ch.d.size(); ++k) {
            const Token tok{ch.d[k], ch.w[k], kInvalidTopic};
            std::fill(t, t + ch.n[k], tok);
            t += ch.n[k];
            __atomic_fetch_add(&c.doc_lengths[ch.d[k]], static_cast<std::uint32_t>(ch.n[k]), __ATOMIC_RELAXED);
            __atomic_fetch_add(&c.word_freqs[ch.w[k]], ch.n[k], __ATOMIC_RELAXED);
        }
    });
    c.num_tokens = c.tokens.size();
    return c;
}

Corpus load_docword(std::istream& in) {
    std::ostringstream ss;
    ss << in.rdbuf();
    const std::string buf = ss.str();
    return load_docword_buffer(buf.data(), buf.size());
}

Corpus load_uci_files(const std::string& docword_path, const std::string& vocab_path) {
    const int fd = ::open(docword_path.c_str(), O_RDONLY);
    if (fd < 0) throw IoError("cannot open docword file " + docword_path);
    struct stat st {};
    if (::fstat(fd, &st) != 0) {
        ::close(fd);
        throw IoError("cannot stat docword file " + docword_path);
    }
    const std::size_t size = static_cast<std::size_t>(st.st_size);
    void* map = size ? ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0) : nullptr;
    ::close(fd);
    if (size && map == MAP_FAILED) throw IoError("cannot map docword file " + docword_path);
    std::ifstream vocab(vocab_path);
    if (!vocab) {
        if (size) ::munmap(map, size);
        throw IoError("cannot open vocab file " + vocab_path);
    }
    Corpus c;
    try {
        c = load_docword_buffer(static_cast<const char*>(map), size);
    } catch (...) {
        if (size) ::munmap(map, size);
        throw;
    }
    if (size) ::munmap(map, size);
    load_vocab(c, vocab);
    return c;
}

void load_vocab(Corpus& c, std::istream& vocab) {
    c.vocab.reserve(c.vocab_size);
    std::string term;
    std::uint64_t line = 0;
    while (std::getline(vocab, term)) {
        ++line;
        if (!term.empty() && term.back() == '\r') term.pop_back();
        if (line > c.vocab_size)
            throw ValidationError("vocab line " + std::to_string(line) + ": more than V=" +
                                  std::to_string(c.vocab_size) + " entries");
        c.vocab.push_back(term);
    }
    if (line != c.vocab_size)
        throw ValidationError("vocab line " + std::to_string(line) + ": expected V=" +
                              std::to_string(c.vocab_size) + " entries, got " + std::to_string(line));
}

Corpus load_uci(std::istream& docword, std::istream& vocab) {
    Corpus c = load_docword(docword);
    load_vocab(c, vocab);
    return c;
}

namespace {
// RngStream(seed, kind, element).next_double() (rng.hpp:49-83), first draw only.
double first_uniform(std::uint64_t seed, std::uint32_t kind, std::uint64_t element) {
    std::uint32_t c0 = kind, c1 = static_cast<std::uint32_t>(element),
                  c2 = static_cast<std::uint32_t>(element >> 32), c3 = 0;
    std::uint32_t k0 = static_cast<std::uint32_t>(seed), k1 = static_cast<std::uint32_t>(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * c0;
        const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * c2;
        const std::uint32_t n0 = static_cast<std::uint32_t>(p1 >> 32) ^ c1 ^ k0;
        const std::uint32_t n2 = static_cast<std::uint32_t>(p0 >> 32) ^ c3 ^ k1;
        c1 = static_cast<std::uint32_t>(p1);
        c3 = static_cast<std::uint32_t>(p0);
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    const std::uint64_t bits = (static_cast<std::uint64_t>(c1) << 32) | c0;
    return static_cast<double>(bits >> 11) * 0x1.0p-53;
}
}  // namespace

// init_assignments (corpus.cpp:87-96) -- corpus preparation on the host, as the
// reference's Corpus method; training itself draws on device (trainer.cpp:383-388).
void init_assignments(Corpus& corpus, std::uint32_t num_topics, std::uint64_t seed) {
    if (num_topics == 0) throw ValidationError("number of topics must be >= 1");
    for (std::uint64_t t = 0; t < corpus.tokens.size(); ++t) {
        auto topic = static_cast<TopicId>(first_uniform(seed, 0xFFFFFFFFu, t) * num_topics);
        corpus.tokens[t].topic = topic < num_topics ? topic : num_topics - 1;
    }
}

Corpus generate_corpus(const slda_gen_params& params) {
    std::uint64_t T = 0;
    check(slda_generate_corpus_size(&params, &T));
    Corpus c;
    c.num_docs = params.num_docs;
    c.vocab_size = params.vocab_size;
    c.tokens.resize(T);
    check(slda_generate_corpus(&params, reinterpret_cast<std::uint32_t*>(c.tokens.data()), T));
    c.finalize();
    return c;
}

// ---------------------------------------------------------------- config --

TrainConfig TrainConfig::resolved(const Corpus& corpus) const {
    TrainConfig out = *this;
    if (out.num_topics == 0) throw ValidationError("number of topics must be >= 1");
    if (out.alpha <= 0.0) out.alpha = 50.0 / out.num_topics;
    if (out.beta <= 0.0) throw ValidationError("beta must be > 0");
    if (out.tree_branch < 2) throw ValidationError("tree branch must be >= 2");
    const std::uint64_t cap = static_cast<std::uint64_t>(out.tree_branch) * out.tree_branch * out.tree_branch;
    if (out.num_topics > cap)
        throw ValidationError("K=" + std::to_string(out.num_topics) + " exceeds tree capacity W^3=" +
                              std::to_string(cap));
    if (out.num_chunks == 0) out.num_chunks = 1;  // one resident shard per GPU
    if (corpus.num_docs > 0 && out.num_chunks > corpus.num_docs)
        throw ValidationError("num_chunks exceeds document count");
    if (out.num_workers == 0) {
        const unsigned hw = std::thread::hardware_concurrency();
        out.num_workers = hw ? hw : 1;
    }
    return out;
}

std::string format_metrics_line(const MetricsEntry& entry) {
    char buf[160];
    if (entry.heldout_ll.has_value()) {
        std::snprintf(buf, sizeof(buf), "%u %.6f %.6f %.6f", entry.stats.iteration, entry.stats.elapsed_s,
                      entry.stats.mtokens_per_s, *entry.heldout_ll);
    } else {
        std::snprintf(buf, sizeof(buf), "%u %.6f %.6f", entry.stats.iteration, entry.stats.elapsed_s,
                      entry.stats.mtokens_per_s);
    }
    return buf;
}

// ---------------------------------------------------------------- model --

std::vector<std::uint32_t> ModelState::word_topic() const {
    std::vector<std::uint32_t> out(static_cast<std::size_t>(vocab_size) * num_topics);
    check(slda_get_word_topic(engine_.get(), out.data()));
    return out;
}
std::vector<float> ModelState::word_topic_prob() const {
    std::vector<float> out(static_cast<std::size_t>(vocab_size) * num_topics);
    check(slda_get_word_topic_prob(engine_.get(), out.data()));
    return out;
}
std::vector<float> ModelState::tree_mass() const {
    std::vector<float> out(vocab_size);
    check(slda_get_tree_mass(engine_.get(), out.data()));
    return out;
}
std::vector<float> ModelState::tree_prefix() const {
    std::vector<float> out(static_cast<std::size_t>(vocab_size) * num_topics);
    check(slda_get_tree_prefix(engine_.get(), out.data()));
    return out;
}
std::vector<TopicId> ModelState::gather_assignments() const {
    if (!has_chunks_) throw ValidationError("model carries no chunks (loaded from a checkpoint)");
    std::vector<TopicId> out(num_tokens);
    check(slda_get_assignments(engine_.get(), out.data()));
    return out;
}
DocTopicMatrix ModelState::doc_topic() const {
    DocTopicMatrix m;
    std::uint64_t nnz = 0;
    check(slda_get_doc_topic_nnz(engine_.get(), &nnz));
    const slda_info in = info();
    m.row_offsets.resize(static_cast<std::size_t>(in.doc_end - in.doc_begin) + 1);
    m.topics.resize(nnz);
    m.counts.resize(nnz);
    check(slda_get_doc_topic(engine_.get(), m.row_offsets.data(), m.topics.data(), m.counts.data()));
    return m;
}
ChunkLayout ModelState::chunk_layout() const {
    const slda_info in = info();
    ChunkLayout c;
    c.doc_begin = in.doc_begin;
    c.doc_end = in.doc_end;
    const std::size_t T = in.num_tokens, S = in.num_segments;
    c.sorted_doc.resize(T);
    c.sorted_word.resize(T);
    c.token_ids.resize(T);
    c.shuffle_ptrs.resize(T);
    c.doc_offsets.resize(static_cast<std::size_t>(in.doc_end - in.doc_begin) + 1);
    c.seg_word.resize(S);
    c.seg_offset.resize(S);
    c.seg_length.resize(S);
    c.schedule.resize(S);
    check(slda_get_pdow(engine_.get(), c.sorted_doc.data(), c.sorted_word.data(), c.token_ids.data(),
                        c.shuffle_ptrs.data(), c.doc_offsets.data(), c.seg_word.data(), c.seg_offset.data(),
                        c.seg_length.data(), c.schedule.data()));
    return c;
}
slda_kernel_times ModelState::kernel_times() const {
    slda_kernel_times t{};
    check(slda_get_kernel_times(engine_.get(), &t));
    return t;
}
slda_info ModelState::info() const {
    slda_info in{};
    check(slda_get_info(engine_.get(), &in));
    return in;
}

ModelState init_state(const Corpus& corpus, const TrainConfig& raw_cfg) {
    const TrainConfig cfg = raw_cfg.resolved(corpus);
    slda_corpus_view view{};
    view.num_docs = corpus.num_docs;
    view.vocab_size = corpus.vocab_size;
    view.num_tokens = corpus.tokens.size();
    view.tokens = reinterpret_cast<const std::uint32_t*>(corpus.tokens.data());
    view.doc_begin = 0;
    view.doc_end = corpus.num_docs;
    view.token_id_base = 0;
    slda_config c{};
    c.num_topics = cfg.num_topics;
    c.alpha = cfg.alpha;
    c.beta = cfg.beta;
    c.seed = cfg.seed;
    c.tree_branch = cfg.tree_branch;
    c.sampler = cfg.sampler == SamplerKind::kVanilla ? SLDA_SAMPLER_VANILLA : SLDA_SAMPLER_SPARSE;
    c.num_chunks = cfg.num_chunks;
    c.device_budget = cfg.device_budget;
    c.init_mode = SLDA_INIT_AUTO;
    c.device = cfg.device;
    c.rank = 0;
    c.world_size = 1;
    slda_engine* e = nullptr;
    check(slda_create(&view, &c, &e));
    ModelState s;
    s.engine_.reset(e);
    s.has_chunks_ = true;
    s.num_docs = corpus.num_docs;
    s.vocab_size = corpus.vocab_size;
    s.num_tokens = corpus.tokens.size();
    s.num_topics = cfg.num_topics;
    s.alpha = cfg.alpha;
    s.beta = cfg.beta;
    s.seed = cfg.seed;
    s.sampler = cfg.sampler;
    s.iteration = 0;
    return s;
}

std::vector<std::uint32_t> shard_bounds(const Corpus& corpus, std::uint32_t world) {
    std::vector<std::uint32_t> b(static_cast<std::size_t>(world) + 1, 0);
    check(slda_shard_bounds(corpus.num_docs, corpus.tokens.size(), corpus.doc_lengths.data(), world, b.data()));
    return b;
}

ModelState init_shard(const Corpus& corpus, const TrainConfig& raw_cfg, std::uint32_t rank,
                      std::uint32_t world) {
    const TrainConfig cfg = raw_cfg.resolved(corpus);
    if (rank >= world) throw ValidationError("rank must be < world");
    // The reference's corpus-wide topic rule (trainer.cpp:369-378), decided once for all shards.
    std::uint32_t mode = SLDA_INIT_GIVEN;
    for (const Token& t : corpus.tokens) {
        if (t.topic == kInvalidTopic) {
            mode = SLDA_INIT_DRAW;
            break;
        }
        if (t.topic >= cfg.num_topics) throw ValidationError("token topic exceeds configured K");
    }
    const std::vector<std::uint32_t> bounds = shard_bounds(corpus, world);
    const DocId b = bounds[rank], e = bounds[rank + 1];
    // Tokens of the shard in corpus order, with their corpus positions as RNG ids.
    std::vector<Token> toks;
    std::vector<std::uint64_t> ids;
    bool contiguous = true;
    std::uint64_t first = 0;
    for (std::uint64_t t = 0; t < corpus.tokens.size(); ++t) {
        const DocId d = corpus.tokens[t].doc;
        if (d < b || d >= e) continue;
        if (toks.empty()) first = t;
        else if (ids.back() + 1 != t) contiguous = false;
        toks.push_back(corpus.tokens[t]);
        ids.push_back(t);
    }
    slda_corpus_view view{};
    view.num_docs = corpus.num_docs;
    view.vocab_size = corpus.vocab_size;
    view.num_tokens = toks.size();
    view.tokens = reinterpret_cast<const std::uint32_t*>(toks.data());
    view.doc_begin = b;
    view.doc_end = e;
    view.token_id_base = first;
    view.token_ids = contiguous ? nullptr : ids.data();
    slda_config c{};
    c.num_topics = cfg.num_topics;
    c.alpha = cfg.alpha;
    c.beta = cfg.beta;
    c.seed = cfg.seed;
    c.tree_branch = cfg.tree_branch;
    c.sampler = cfg.sampler == SamplerKind::kVanilla ? SLDA_SAMPLER_VANILLA : SLDA_SAMPLER_SPARSE;
    c.num_chunks = cfg.num_chunks;
    c.device_budget = cfg.device_budget;
    c.init_mode = mode;
    c.device = cfg.device;
    c.rank = rank;
    c.world_size = world;
    slda_engine* eng = nullptr;
    check(slda_create(&view, &c, &eng));
    ModelState s;
    s.engine_.reset(eng);
    s.has_chunks_ = true;
    s.num_docs = e - b;
    s.vocab_size = corpus.vocab_size;
    s.num_tokens = toks.size();
    s.num_topics = cfg.num_topics;
    s.alpha = cfg.alpha;
    s.beta = cfg.beta;
    s.seed = cfg.seed;
    s.sampler = cfg.sampler;
    return s;
}

ModelState init_view(const slda_corpus_view& view, const TrainConfig& raw_cfg, std::uint32_t rank,
                     std::uint32_t world, std::uint32_t init_mode) {
    Corpus shape;
    shape.num_docs = view.num_docs;
    const TrainConfig cfg = raw_cfg.resolved(shape);
    slda_config c{};
    c.num_topics = cfg.num_topics;
    c.alpha = cfg.alpha;
    c.beta = cfg.beta;
    c.seed = cfg.seed;
    c.tree_branch = cfg.tree_branch;
    c.sampler = cfg.sampler == SamplerKind::kVanilla ? SLDA_SAMPLER_VANILLA : SLDA_SAMPLER_SPARSE;
    c.num_chunks = cfg.num_chunks;
    c.device_budget = cfg.device_budget;
    c.init_mode = init_mode;
    c.device = cfg.device;
    c.rank = rank;
    c.world_size = world;
    slda_engine* eng = nullptr;
    check(slda_create(&view, &c, &eng));
    ModelState s;
    s.engine_.reset(eng);
    s.has_chunks_ = true;
    s.num_docs = view.doc_end - view.doc_begin;
    s.vocab_size = view.vocab_size;
    s.num_tokens = view.num_tokens;
    s.num_topics = cfg.num_topics;
    s.alpha = cfg.alpha;
    s.beta = cfg.beta;
    s.seed = cfg.seed;
    s.sampler = cfg.sampler;
    return s;
}

IterationStats run_iteration(ModelState& state, const TrainConfig& cfg) {
    if (!state.engine_) throw ValidationError("model has no engine");
    // The reference keeps dense or sparse doc-topic rows per the init-time kind
    // (trainer.cpp:391-397); switching kinds between iterations is not a supported state.
    if (cfg.sampler != state.sampler) throw ValidationError("sampler kind differs from the one the model was initialised with");
    if (!state.has_chunks_) throw ValidationError("model carries no chunks (loaded from a checkpoint)");
    slda_iteration_stats st{};
    check(slda_iterate(state.engine_.get(), &st));
    state.iteration = st.iteration;
    IterationStats out;
    out.iteration = st.iteration;
    out.tokens = st.tokens;
    out.elapsed_s = st.elapsed_s;
    out.mtokens_per_s = st.mtokens_per_s;
    out.mean_doc_topics = st.mean_doc_topics;
    out.device_ms = st.device_ms;
    return out;
}

ModelState train(const Corpus& corpus, const TrainConfig& raw_cfg, const MetricsSink& sink,
                 const HeldoutProbe& probe) {
    const TrainConfig cfg = raw_cfg.resolved(corpus);
    ModelState state = init_state(corpus, cfg);
    for (std::uint32_t i = 0; i < cfg.iterations; ++i) {  // trainer.cpp:451-464
        MetricsEntry entry;
        entry.stats = run_iteration(state, cfg);
        if (probe && cfg.eval_every > 0 && entry.stats.iteration % cfg.eval_every == 0)
            entry.heldout_ll = probe(state);
        if (sink) sink(entry);
    }
    return state;
}

ModelState model_from_counts(std::uint32_t vocab_size, std::uint32_t num_topics,
                             const std::vector<std::uint32_t>& word_topic, std::uint64_t num_tokens,
                             std::uint32_t iteration, double alpha, double beta, std::uint64_t seed, int device) {
    if (word_topic.size() != static_cast<std::size_t>(vocab_size) * num_topics)
        throw ValidationError("word_topic must be V x K");
    slda_config c{};
    c.num_topics = num_topics;
    c.alpha = alpha;
    c.beta = beta;
    c.seed = seed;
    c.tree_branch = num_topics > 32768 ? 41 : 32;
    c.device = device;
    c.world_size = 1;
    slda_engine* e = nullptr;
    check(slda_create_from_counts(vocab_size, word_topic.data(), num_tokens, iteration, &c, &e));
    ModelState s;
    s.engine_.reset(e);
    s.has_chunks_ = false;
    s.vocab_size = vocab_size;
    s.num_tokens = num_tokens;
    s.num_topics = num_topics;
    s.alpha = alpha;
    s.beta = beta;
    s.seed = seed;
    s.iteration = iteration;
    return s;
}

// ---------------------------------------------------------------- eval --

std::string format_eval_line(const EvalReport& r) {  // eval.cpp:42-47
    char buf[96];
    std::snprintf(buf, sizeof(buf), "%u %.6f %llu", r.iteration, r.per_token_ll,
                  static_cast<unsigned long long>(r.tokens_evaluated));
    return buf;
}

EvalReport heldout_ll(ModelState& model, const Corpus& heldout, std::uint32_t burn_in, unsigned,
                      std::uint64_t seed) {
    EvalReport r;
    check(slda_heldout_ll(model.engine(), heldout.num_docs, heldout.vocab_size, heldout.tokens.size(),
                          reinterpret_cast<const std::uint32_t*>(heldout.tokens.data()), burn_in, seed,
                          &r.per_token_ll, &r.tokens_evaluated));
    r.iteration = model.iteration;
    return r;
}

double throughput_mtokens(std::uint64_t tokens, double elapsed_s) {
    if (elapsed_s <= 0.0) throw ValidationError("throughput requires positive elapsed time");
    return static_cast<double>(tokens) / elapsed_s / 1e6;
}

// top_words (eval.cpp:139-158): per topic, n most probable words, ties by id.
std::vector<std::vector<std::pair<WordId, float>>> top_words(const ModelState& model, std::uint32_t n) {
    if (n > model.vocab_size) throw ValidationError("top_words n exceeds vocabulary size");
    const std::vector<float> bhat = model.word_topic_prob();
    const std::uint32_t V = model.vocab_size, K = model.num_topics;
    std::vector<std::vector<std::pair<WordId, float>>> out(K);
    std::vector<std::pair<WordId, float>> column(V);
    for (TopicId k = 0; k < K; ++k) {
        for (WordId v = 0; v < V; ++v) column[v] = {v, bhat[static_cast<std::size_t>(v) * K + k]};
        std::partial_sort(column.begin(), column.begin() + n, column.end(), [](const auto& a, const auto& b) {
            if (a.second != b.second) return a.second > b.second;
            return a.first < b.first;
        });
        out[k].assign(column.begin(), column.begin() + n);
    }
    return out;
}

void print_topics(std::ostream& out, const ModelState& model, const std::vector<std::string>& vocab,
                  std::uint32_t n) {
    const auto ranked = top_words(model, n);
    for (TopicId k = 0; k < ranked.size(); ++k) {
        out << "topic " << k << ':';
        for (const auto& [word, prob] : ranked[k]) {
            char p[48];
            std::snprintf(p, sizeof(p), "%.6f", prob);
            out << ' ' << (word < vocab.size() && !vocab[word].empty() ? vocab[word] : std::to_string(word)) << ':' << p;
        }
        out << '\n';
    }
}

// ------------------------------------------------------ building blocks --

SparseTopicRow segmented_count(std::span<const TopicId> segment) {
    std::vector<TopicId> s(segment.begin(), segment.end());
    std::sort(s.begin(), s.end());
    SparseTopicRow r;
    for (std::size_t i = 0; i < s.size(); ++i) {
        if (i == 0 || s[i] != s[i - 1]) {
            r.topics.push_back(s[i]);
            r.counts.push_back(1);
        } else {
            ++r.counts.back();
        }
    }
    return r;
}

std::size_t prefix_search(std::span<const double> prefix, double x) {
    if (prefix.empty()) throw ValidationError("prefix_search on empty sequence");
    const double last = prefix.back();
    if (x > last) {
        const double slack = 16.0 * std::numeric_limits<double>::epsilon() * (last > 1.0 ? last : 1.0);
        if (x > last + slack)
            throw ValidationError("prefix_search target " + std::to_string(x) + " beyond prefix total " +
                                  std::to_string(last));
        return prefix.size() - 1;
    }
    return static_cast<std::size_t>(std::lower_bound(prefix.begin(), prefix.end(), x) - prefix.begin());
}

WaryTree::WaryTree(std::span<const double> w, std::uint32_t branch) {
    if (branch < 2) throw ValidationError("tree branching factor must be >= 2");
    const std::uint64_t capacity = static_cast<std::uint64_t>(branch) * branch * branch;
    if (w.size() > capacity)
        throw ValidationError("tree capacity exceeded: K=" + std::to_string(w.size()) +
                              " > W^3=" + std::to_string(capacity));
    if (w.empty()) throw ValidationError("tree requires at least one weight");
    branch_ = branch;
    size_ = static_cast<std::uint32_t>(w.size());
    auto padded = [&](std::uint32_t n) { return (n + branch_ - 1) / branch_ * branch_; };
    bottom_.assign(padded(size_), 0.0);
    double run = 0;
    for (std::uint32_t i = 0; i < size_; ++i) bottom_[i] = (run += w[i]);
    total_ = run;
    std::fill(bottom_.begin() + size_, bottom_.end(), total_);
    const std::uint32_t n3r = static_cast<std::uint32_t>(bottom_.size()) / branch_;
    mid_.assign(padded(n3r), total_);
    for (std::uint32_t i = 0; i < n3r; ++i) mid_[i] = bottom_[(i + 1) * branch_ - 1];
    const std::uint32_t n2r = static_cast<std::uint32_t>(mid_.size()) / branch_;
    top_.assign(branch_, total_);
    for (std::uint32_t i = 0; i < n2r; ++i) top_[i] = mid_[(i + 1) * branch_ - 1];
}

std::uint32_t WaryTree::sample(double x) const {
    if (!(x <= total_)) x = total_;
    auto first = [&](const double* b) {
        for (std::uint32_t i = 0; i < branch_; ++i)
            if (b[i] >= x) return i;
        return branch_ - 1;
    };
    const std::uint32_t i2 = first(top_.data());
    const std::uint32_t i3 = i2 * branch_ + first(mid_.data() + i2 * branch_);
    const std::uint32_t i4 = i3 * branch_ + first(bottom_.data() + i3 * branch_);
    return i4 < size_ ? i4 : size_ - 1;
}

// ---------------------------------------------------------- checkpoints --

// Text format of save_checkpoint (trainer.cpp:469-478) + dump_word_topic (counts.cpp:140-150).
void save_checkpoint(const std::filesystem::path& path, const ModelState& state) {
    // A document shard holds only its own documents' assignments (and word_topic() is a
    // collective), so its file would carry the global C_wk with the shard's T: refuse it.
    if (state.engine() && state.info().world_size > 1)
        throw ValidationError("save_checkpoint: model is one document shard of a multi-GPU run (world_size > 1)");
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw IoError("cannot write checkpoint " + path.string());
    out << "sparselda-checkpoint 1 " << state.num_docs << ' ' << state.vocab_size << ' ' << state.num_tokens
        << ' ' << state.num_topics << ' ' << state.iteration << ' ' << std::setprecision(17) << state.alpha
        << ' ' << state.beta << ' ' << state.seed << '\n';
    for (const TopicId t : state.gather_assignments()) out << t << '\n';
    const std::vector<std::uint32_t> b = state.word_topic();
    out << state.vocab_size << ' ' << state.num_topics << ' ' << state.num_tokens << ' ' << state.iteration << '\n';
    for (WordId v = 0; v < state.vocab_size; ++v)
        for (TopicId k = 0; k < state.num_topics; ++k) {
            const std::uint32_t c = b[static_cast<std::size_t>(v) * state.num_topics + k];
            if (c) out << v << ' ' << k << ' ' << c << '\n';
        }
    if (!out) throw IoError("short write to checkpoint " + path.string());
}

Checkpoint load_checkpoint(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot read checkpoint " + path.string());
    std::string magic;
    std::uint32_t version = 0;
    Checkpoint ck;
    in >> magic >> version;
    if (magic != "sparselda-checkpoint" || version != 1)
        throw ValidationError("unrecognized checkpoint header in " + path.string());
    in >> ck.num_docs >> ck.vocab_size >> ck.num_tokens >> ck.num_topics >> ck.iteration >> ck.alpha >> ck.beta >>
        ck.seed;
    if (!in) throw ValidationError("malformed checkpoint header in " + path.string());
    ck.assignments.resize(ck.num_tokens);
    for (std::uint64_t t = 0; t < ck.num_tokens; ++t) {
        if (!(in >> ck.assignments[t])) throw ValidationError("checkpoint truncated in assignments");
        if (ck.assignments[t] >= ck.num_topics) throw ValidationError("checkpoint assignment out of range");
    }
    in.ignore(1, '\n');
    // parse_word_topic (counts.cpp:152-176)
    std::string text;
    if (!std::getline(in, text)) throw ValidationError("word-topic dump: missing header");
    std::istringstream header(text);
    std::uint32_t V = 0, K = 0, it = 0;
    std::uint64_t T = 0;
    if (!(header >> V >> K >> T >> it)) throw ValidationError("word-topic dump: malformed header");
    ck.word_topic.assign(static_cast<std::size_t>(V) * K, 0);
    std::uint64_t stored = 0;
    while (std::getline(in, text)) {
        if (text.empty()) continue;
        std::istringstream f(text);
        std::uint64_t v = 0, k = 0, c = 0;
        if (!(f >> v >> k >> c) || v >= V || k >= K)
            throw ValidationError("word-topic dump: malformed entry \"" + text + "\"");
        ck.word_topic[v * K + k] = static_cast<std::uint32_t>(c);
        stored += c;
    }
    if (stored != T) throw ValidationError("word-topic dump: stored counts do not sum to T");
    if (T != ck.num_tokens || it != ck.iteration || V != ck.vocab_size || K != ck.num_topics)
        throw ValidationError("checkpoint sections disagree in " + path.string());
    return ck;
}

ModelState model_from_checkpoint(const Checkpoint& ck, unsigned) {
    ModelState s = model_from_counts(ck.vocab_size, ck.num_topics, ck.word_topic, ck.num_tokens, ck.iteration,
                                     ck.alpha, ck.beta, ck.seed);
    s.num_docs = ck.num_docs;
    return s;
}

ModelState resume_from_checkpoint(const Corpus& corpus, const Checkpoint& ck, const TrainConfig& cfg_in) {
    if (corpus.tokens.size() != ck.num_tokens || corpus.num_docs != ck.num_docs ||
        corpus.vocab_size != ck.vocab_size)
        throw ValidationError("checkpoint does not match the corpus");
    Corpus c = corpus;
    for (std::uint64_t t = 0; t < ck.num_tokens; ++t) c.tokens[t].topic = ck.assignments[t];
    TrainConfig cfg = cfg_in;
    cfg.num_topics = ck.num_topics;
    cfg.alpha = ck.alpha;
    cfg.beta = ck.beta;
    cfg.seed = ck.seed;
    ModelState s = init_state(c, cfg);
    check(slda_set_iteration(s.engine(), ck.iteration));
    s.iteration = ck.iteration;
    return s;
}

}  // namespace sparselda_b200
